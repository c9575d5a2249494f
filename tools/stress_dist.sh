# multi-lane distributed stress on one GPU (two ranks as processes); usage:
#   bash tools/stress_dist.sh  -> lines "lanes=L ... : rank r ok True"
cd "$(dirname "$0")/.."
run() {  # lanes n lw depth copies spread
  T=$(python -c "import secrets; print(secrets.token_hex(4))")
  for r in 0 1; do
    DGKR_STRESS_LW=$3 DGKR_STRESS_DEPTH=$4 DGKR_STRESS_COPIES=$5 DGKR_STRESS_SPREAD=$6 \
      timeout 600 python tools/dist_shm_worker.py $r 2 $T $1 $2 /tmp/p.bin > gpurun_out/w$r.log 2>&1 &
  done
  wait
  echo "lanes=$1 n=$2 lw=$3 depth=$4 copies=$5 spread=$6:"; grep -m3 "fault\|failed" gpurun_out/w0.log | cut -c1-200; tail -1 gpurun_out/w0.log | cut -c1-200; grep -m3 "fault\|failed" gpurun_out/w1.log | cut -c1-200; tail -1 gpurun_out/w1.log | cut -c1-200
}
for i in 1 2; do run ${L:-8} 16 ${LW:-16} ${D:-4} 64 1; done
run 16 32 16 24 64 1
run 8 16 12 24 64 1
run 8 16 16 24 64 0
