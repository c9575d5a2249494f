#!/usr/bin/env bash
# Protocol check of bench.py's multi-rank arm with every rank on ONE GPU
# (this pool's boxes have one): torchrun world N, gloo for the torch plumbing,
# shared-memory lanes for the per-round exchange. Not a scaling number -- the
# ranks share one device. Writes profiles-style JSON lines to $OUT.
set -u
OUT=${OUT:-gpurun_out}
for N in ${WORLDS:-2 4 8}; do
  DGKR_DEVICE=0 DGKR_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node "$N" \
    --master-addr 127.0.0.1 --master-port $((29600 + N)) bench.py --gpus "$N" --lanes ${LANES:-4} --steps 2 --warmup 1 \
    > "$OUT/dist_world${N}_shared_gpu.json" 2> "$OUT/dist_world${N}_shared_gpu.err"
  echo "world $N rc=$?"
done
