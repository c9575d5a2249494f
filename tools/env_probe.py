"""Prints the injection-related environment a profiler/sanitizer gives the
process (run under ncu / compute-sanitizer on the GPU box)."""
import os

import torch  # noqa: F401  (a CUDA context, so injection happens)

torch.zeros(1, device="cuda")
print("ENV", {k: v for k, v in os.environ.items() if "INJECT" in k or "PRELOAD" in k or "NSIGHT" in k or "NV_TPS" in k or k.startswith("NV_COMPUTE")})
