"""Synthetic workloads of BASELINE.json / SURVEY.md §8(d), as flat circuits.

* ``layered_circuit``: uniform-width layered circuit — every gate is one
  fan-in-2 nested gate reading the previous layer at uniformly random
  indices, add/mul 50/50 (C1: 2^12 x 16 layers; C2 sub-circuit: 2^16 x 24).
* ``replicate``: the data-parallel (Sisu) view — n identical copies, copy c
  at gate offset c * width in every layer (wires never cross copies), which is
  what ``dgkr_circuit_create(..., n_copies)`` proves without materialising it.
* ``random_inputs``: canonical field elements as a uint8 array (rejection
  sampling on masked bytes, the scheme of random_element, field.hpp:225-239).
"""
from __future__ import annotations

from typing import Tuple

import numpy as np

Flat = Tuple[np.ndarray, np.ndarray, np.ndarray, np.ndarray]


def layered_circuit(seed: int, log_width: int, depth: int, mul_percent: int = 50,
                    input_log: int | None = None) -> Tuple[int, Flat]:
    """Returns (input_size, (layer_gate_start, gate_nested_start, nested, min_padded))."""
    rng = np.random.default_rng(seed)
    w = 1 << log_width
    in_size = 1 << (log_width if input_log is None else input_log)
    sizes = [in_size] + [w] * depth
    nested = np.zeros((depth * w, 5), dtype=np.uint32)
    for li in range(1, depth + 1):
        blk = nested[(li - 1) * w: li * w]
        blk[:, 0] = (rng.integers(0, 100, size=w) < mul_percent).astype(np.uint32)
        blk[:, 1] = li - 1
        blk[:, 2] = rng.integers(0, sizes[li - 1], size=w, dtype=np.uint32)
        blk[:, 3] = li - 1
        blk[:, 4] = rng.integers(0, sizes[li - 1], size=w, dtype=np.uint32)
    lgs = np.arange(depth + 1, dtype=np.uint64) * w
    gns = np.arange(depth * w + 1, dtype=np.uint64)
    minp = np.ones(depth + 1, dtype=np.uint64)
    return in_size, (lgs, gns, nested, minp)


def replicate(input_size: int, flat: Flat, n: int) -> Tuple[int, Flat]:
    """Full circuit of n data-parallel copies (requires power-of-two layer
    sizes, like dgkr_circuit_create with n_copies)."""
    lgs, gns, nested, minp = flat
    depth = len(lgs) - 1
    sizes = [input_size] + [int(lgs[i + 1] - lgs[i]) for i in range(depth)]
    out_nested = []
    out_gns = [0]
    for li in range(1, depth + 1):
        g0, g1 = int(lgs[li - 1]), int(lgs[li])
        k0, k1 = int(gns[g0]), int(gns[g1])
        blk = nested[k0:k1]
        counts = np.diff(gns[g0:g1 + 1].astype(np.int64))
        for c in range(n):
            e = blk.copy()
            e[:, 2] += np.array([sizes[x] for x in e[:, 1]], dtype=np.uint32) * c
            e[:, 4] += np.array([sizes[x] for x in e[:, 3]], dtype=np.uint32) * c
            out_nested.append(e)
            out_gns.extend((out_gns[-1] + np.cumsum(counts)).tolist())
    new_lgs = lgs.astype(np.uint64) * n
    return input_size * n, (new_lgs, np.array(out_gns, dtype=np.uint64),
                            np.concatenate(out_nested) if out_nested else np.zeros((0, 5), np.uint32),
                            np.ones(depth + 1, dtype=np.uint64))


def random_inputs(p: int, n: int, seed: int) -> np.ndarray:
    """n canonical elements (little-endian, width ceil(bits/8)) as uint8[n*w]."""
    bits = p.bit_length()
    w = (bits + 7) // 8
    top = bits - 8 * (w - 1)
    mask = 0xFF if top >= 8 else (1 << top) - 1
    rng = np.random.default_rng(seed)
    out = np.empty((n, w), dtype=np.uint8)
    filled = 0
    pb = np.frombuffer(p.to_bytes(w, "little"), dtype=np.uint8)
    while filled < n:
        need = n - filled
        cand = rng.integers(0, 256, size=(need + need // 2 + 16, w), dtype=np.uint8)
        cand[:, -1] &= mask
        # lexicographic compare from the most significant byte: cand < p
        lt = np.zeros(len(cand), dtype=bool)
        eq = np.ones(len(cand), dtype=bool)
        for b in range(w - 1, -1, -1):
            lt |= eq & (cand[:, b] < pb[b])
            eq &= cand[:, b] == pb[b]
        ok = cand[lt][:need]
        out[filled:filled + len(ok)] = ok
        filled += len(ok)
    return out.reshape(-1)
