#!/usr/bin/env bash
# compute-sanitizer over small instances of every kernel family (one GPU):
#   memcheck  -- out-of-bounds / misaligned device accesses, leaks
#   racecheck -- shared-memory hazards (block reductions, NTT / Merkle / round
#                kernels that stage in shared memory, the TMA-staged rounds)
#   synccheck -- barrier misuse
# Each tool runs the smoke proof and a -k selection of the GPU parity tests.
set -u
OUT=${OUT:-gpurun_out/sanitize}
mkdir -p "$OUT"
SEL="test_product_sum_matches_oracle and 5-3 or test_gkr_matches_oracle or test_pcs or test_distpc_matches_oracle or test_pairsum"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 20 \
    python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/${tool}_smoke.txt" 2>&1
  echo "$tool smoke rc=$?"
  timeout 2400 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 20 \
    python -m pytest tests/test_gpu_parity.py -q -x -k "$SEL" > "$OUT/${tool}_parity.txt" 2>&1
  echo "$tool parity rc=$?"
done
DGKR_TMA_MIN_PAIRS=256 timeout 2400 compute-sanitizer --tool racecheck --error-exitcode 99 --print-limit 20 \
  python -m pytest tests/test_gpu_round_tma.py -q -x -k "equals_register_round and 21888 and 9-4" > "$OUT/racecheck_tma.txt" 2>&1
echo "racecheck tma rc=$?"
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 99 --print-limit 20 \
  python -m pytest tests/test_gpu_fri.py tests/test_gpu_beacon.py -q -x > "$OUT/memcheck_fri_beacon.txt" 2>&1
echo "memcheck fri/beacon rc=$?"
for f in "$OUT"/*.txt; do echo "== $f"; grep -E "ERROR SUMMARY|passed|failed|error" "$f" | tail -3; done
