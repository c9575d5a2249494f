#!/usr/bin/env bash
# ncu evidence for the commitment-side kernels:
# NTT (shared-memory stages + radix-4 global passes), FRI fold, column
# digests + Merkle levels, beacon path verification. Each program first runs
# without ncu; one GPU; --set full on a few launches each. Run from the repo root.
set -u
OUT=${OUT:-gpurun_out/aux}
REP=${REP:-/tmp/aux_rep}  # .ncu-rep files stay off gpurun_out (<= 64 MiB comes back)
mkdir -p "$OUT" "$REP"
NCU="ncu --set full --import-source on --clock-control none -f"
timeout 300 python tools/profile_fri.py 24 > "$OUT/fri_plain.log" 2>&1 || { echo "profile_fri failed"; exit 1; }
timeout 900 $NCU -k regex:"k_ntt_local|k_ntt_stage2|k_fri_fold" -c 5 -o "$REP/ntt" python tools/profile_fri.py 24 > "$OUT/ncu_ntt.log" 2>&1 || echo "ntt capture rc=$?"
timeout 300 python tools/bench_pcs.py 24 24 0 > "$OUT/pcs_plain.json" 2>&1 || echo "bench_pcs rc=$?"
timeout 900 $NCU -k regex:"k_column_digest|k_merkle_level" -c 3 -o "$REP/merkle" python tools/bench_pcs.py 24 24 0 > "$OUT/ncu_merkle.log" 2>&1 || echo "merkle capture rc=$?"
timeout 300 python tools/bench_beacon.py 1048576 > "$OUT/beacon_plain.json" 2>&1 || echo "bench_beacon rc=$?"
timeout 900 $NCU -k regex:"k_beacon_verify" -c 1 -o "$REP/beacon" python tools/bench_beacon.py 1048576 > "$OUT/ncu_beacon.log" 2>&1 || echo "beacon capture rc=$?"
for r in ntt merkle beacon; do
  [ -f "$REP/$r.ncu-rep" ] && ncu -i "$REP/$r.ncu-rep" --page raw --csv > "$OUT/${r}_raw.csv" 2>/dev/null && gzip -f "$OUT/${r}_raw.csv"
done
ls -la "$OUT"
