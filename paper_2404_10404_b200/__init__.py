"""B200 (sm_100a) prover for the Sisu distributed-GKR hot path (arXiv 2404.10404).

The product is the CUDA library ``libdgkr_b200.so`` behind the C ABI in
``include/dgkr_b200.h``; this package is its Python mirror of the reference
API (``/root/reference/proj/include/dgkr``). See DESIGN.md.
"""
from .prover import (BN254_P, GOLDILOCKS_P, Circuit, Context, Field, Transcript, dist_sumcheck, distpc,
                     Comm, gkr_prove, gkr_verify, gkr_input_claims, gkr_prove_batch, gkr_prove_dist, gkr_prove_dist_emulated, gkr_prove_stream, load_inputs_lane, pcs_commit, ntt, rs_encode, fri_prove, fri_prove_dist, fri_prove_dist_emulated, pcs_open, prove_layer_sum, prove_product_sum, sha256,
                     distinct_ah, pairwise_distinct_check, chain_update, bitchange_experiment, bitchange_csv,
                     beacon_root, beacon_prove, beacon_verify, set_tuning, get_tuning)

__all__ = ["BN254_P", "GOLDILOCKS_P", "Circuit", "Context", "Field", "Transcript", "dist_sumcheck", "distpc",
           "Comm", "gkr_prove", "gkr_verify", "gkr_input_claims", "gkr_prove_batch", "gkr_prove_dist", "gkr_prove_dist_emulated", "gkr_prove_stream", "load_inputs_lane", "pcs_commit", "ntt", "rs_encode", "fri_prove", "fri_prove_dist", "fri_prove_dist_emulated", "pcs_open", "prove_layer_sum", "prove_product_sum", "sha256",
           "distinct_ah", "pairwise_distinct_check", "chain_update", "bitchange_experiment", "bitchange_csv",
           "beacon_root", "beacon_prove", "beacon_verify", "set_tuning", "get_tuning"]
