"""ORACLE TEST INFRASTRUCTURE — CPU checker for the GPU prover.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this package. The product path (paper_2404_10404_b200) never
does; it fails loudly when its CUDA extension is missing.
"""
