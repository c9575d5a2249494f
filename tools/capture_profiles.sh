#!/usr/bin/env bash
# Evidence for profiles/ (run on the GPU box from the repo root, one GPU):
#   1. the official bench line (no profiler attached),
#   2. the launch list of one C2 proof (ncu, gpu__time_duration only),
#   3. --set full captures of the first three k_round launches (scan / fold
#      natural / fold bit-reversed at T = 2^22) and of the bookkeeping kernels,
#      exported as raw CSV (the .ncu-rep stays on the box; gpurun_out <= 64 MiB).
# Each ncu pass runs only after the same command exited 0 without ncu.
# The ncu passes run with the sum-check tail launch off (DGKR_TAIL_PAIRS=0):
# ncu serialises launches, so the host cannot answer the tail kernel's
# mailbox while it runs and every tail launch would hand back after its
# timeout; the small rounds then appear as k_round_small launches.
set -u
OUT=${OUT:-gpurun_out/prof}
mkdir -p "$OUT"
timeout 900 python bench.py --steps 3 --warmup 3 > "$OUT/bench.json" 2> "$OUT/bench.err" || echo "bench rc=$?"
timeout 300 python tools/profile_step.py c2 1 > "$OUT/step.log" 2>&1 || { echo "profile_step failed"; exit 1; }
DGKR_TAIL_PAIRS=0 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file "$OUT/launches.csv" python tools/profile_step.py c2 1 > "$OUT/ncu_launch.log" 2>&1 || echo "launch list rc=$?"
DGKR_TAIL_PAIRS=0 timeout 1800 ncu --set full --import-source on --clock-control none -k regex:k_round -c 3 \
    -o /tmp/round_full -f python tools/profile_step.py c2 1 > "$OUT/ncu_round.log" 2>&1 || echo "round capture rc=$?"
ncu -i /tmp/round_full.ncu-rep --page raw --csv > "$OUT/round_raw.csv" 2>/dev/null
ncu -i /tmp/round_full.ncu-rep --page details --csv > "$OUT/round_details.csv" 2>/dev/null
DGKR_TAIL_PAIRS=0 timeout 1800 ncu --set full --clock-control none -k regex:"k_bookkeep|k_split_eq_expand" -c 4 \
    -o /tmp/bk_full -f python tools/profile_step.py c2 1 > "$OUT/ncu_bk.log" 2>&1 || echo "bookkeep capture rc=$?"
ncu -i /tmp/bk_full.ncu-rep --page raw --csv > "$OUT/bk_raw.csv" 2>/dev/null
gzip -f "$OUT"/*.csv
ls -la "$OUT"
