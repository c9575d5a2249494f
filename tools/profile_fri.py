"""One fri_prove at a codeword size (for ncu launch lists). Not a bench.
usage: python tools/profile_fri.py [log2 codeword]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2404_10404_b200 as P  # noqa: E402
from paper_2404_10404_b200 import workloads as W  # noqa: E402

e = int(sys.argv[1]) if len(sys.argv) > 1 else 26
ctx = P.Context(0)
f = P.Field.bn254()
co = W.random_inputs(f.p, 1 << (e - 1), e).tobytes()
P.fri_prove(ctx, f, co, 1, 4, 32, P.Transcript(f, "fri"))
