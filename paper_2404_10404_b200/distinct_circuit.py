"""Pairwise-distinct check as a data-parallel GKR circuit (BASELINE.json
config C4, "permutation/grand-product"). The
reference checks distinctness natively (distinct.hpp:53-68: AH(A) = AH(A*)
plus a strict-ascent scan of the claimed sort A*); this is the circuit form,
whose construction has no reference (unpinned), proved by the GPU GKR prover.

Copy c of the sub-circuit takes k items a_{ck..ck+k-1} of A and k+1 items
s_{ck..ck+k} of the claimed ascending list A* (consecutive copies overlap by
one item), a public challenge r, 32-bit witnesses of every gap
s_{i+1} - s_i - 1 and public random-linear-combination coefficients. Its four
outputs:

  PA_c = prod_i (r - a_i),   PB_c = prod_i (r - s_i)        (product trees)
  RC_c = sum_t R_t c_t       over booleanity of the gap bits and the gap
                             recomposition sum_j 2^j d_ij - (s_{i+1}-s_i-1)
  0

A accepts as pairwise distinct iff prod_c PA_c = prod_c PB_c (A* is a
permutation of A, Schwartz-Zippel over r) and every RC_c = 0 (A* strictly
ascends: every gap is a 32-bit number >= 0). Padding appends the same
strictly ascending dummies above max(A) to both lists. r and R are drawn by
the caller after committing to the inputs (Fiat-Shamir).
"""
from __future__ import annotations

import hashlib
from typing import List, Sequence, Tuple

import numpy as np

from .workloads import Flat

GAP_BITS = 32


class _Layout:
    def __init__(self, k: int):
        self.k = k
        n = 0

        def alloc(m):
            nonlocal n
            r = list(range(n, n + m))
            n += m
            return r

        self.zero, self.one, self.m1, self.r = alloc(4)
        self.pow = alloc(GAP_BITS)
        self.a = alloc(k)
        self.s = alloc(k + 1)
        self.gap = [alloc(GAP_BITS) for _ in range(k)]
        self.n_constraints = k * GAP_BITS + k
        self.rlc = alloc(self.n_constraints)
        self.n = n


def _flat(layers: List[List[list]]) -> Tuple[np.ndarray, np.ndarray, np.ndarray, np.ndarray]:
    lgs, gns, rows = [0], [0], []
    for layer in layers:
        for g in layer:
            rows.extend(g)
            gns.append(gns[-1] + len(g))
        lgs.append(lgs[-1] + len(layer))
    return (np.array(lgs, np.uint64), np.array(gns, np.uint64), np.array(rows, np.uint32).reshape(-1, 5),
            np.ones(len(layers) + 1, np.uint64))


def build_distinct_circuit(k: int = 64) -> Tuple[int, Flat, _Layout]:
    """-> (input_size, flat sub-circuit, layout) for k items per copy (k a power of two >= 2)"""
    if k < 2 or k & (k - 1):
        raise ValueError("k must be a power of two >= 2")
    L = _Layout(k)
    z, one, m1, r = L.zero, L.one, L.m1, L.r
    # L1: (r - a_i), (r - s_i) for i < k; gaps s_{i+1} - s_i - 1; booleanity of gap bits
    L1 = []
    for i in range(k):
        L1.append([(0, 0, r, 0, z), (1, 0, m1, 0, L.a[i])])
    for i in range(k):
        L1.append([(0, 0, r, 0, z), (1, 0, m1, 0, L.s[i])])
    gap0 = len(L1)
    for i in range(k):
        L1.append([(0, 0, L.s[i + 1], 0, z), (1, 0, m1, 0, L.s[i]), (1, 0, m1, 0, one)])
    bool0 = len(L1)
    for i in range(k):
        for j in range(GAP_BITS):
            b = L.gap[i][j]
            L1.append([(1, 0, b, 0, b), (1, 0, b, 0, m1)])
    layers = [L1]
    # L2: first product level of both lists + gap recomposition constraints
    L2 = [[(1, 1, 2 * i, 1, 2 * i + 1)] for i in range(k // 2)]
    L2 += [[(1, 1, k + 2 * i, 1, k + 2 * i + 1)] for i in range(k // 2)]
    rec0 = len(L2)
    for i in range(k):
        L2.append([(1, 0, L.pow[j], 0, L.gap[i][j]) for j in range(GAP_BITS)] + [(1, 0, m1, 1, gap0 + i)])
    layers.append(L2)
    # product tree levels: each layer keeps [A products | B products]
    width = k // 2
    while width > 1:
        prev = len(layers)
        layers.append([[(1, prev, 2 * i, prev, 2 * i + 1)] for i in range(width // 2)]
                      + [[(1, prev, width + 2 * i, prev, width + 2 * i + 1)] for i in range(width // 2)])
        width //= 2
    # output layer: PA, PB, RC, 0
    top = len(layers)
    cons = [(1, 0, L.rlc[t], 1, bool0 + t) for t in range(k * GAP_BITS)]
    cons += [(1, 0, L.rlc[k * GAP_BITS + i], 2, rec0 + i) for i in range(k)]
    layers.append([[(0, top, 0, 0, z)], [(0, top, 1, 0, z)], cons, [(0, 0, z, 0, z)]])
    for layer in layers:  # power-of-two widths (data-parallel precondition)
        n = 1
        while n < len(layer):
            n *= 2
        layer.extend([[(0, 0, z, 0, z)]] * (n - len(layer)))
    insz = 1
    while insz < L.n:
        insz *= 2
    return insz, _flat(layers), L


def derive_challenges(p: int, seed: bytes, n_rlc: int) -> Tuple[int, List[int]]:
    """(r, R_0..R_{n-1}) from a seed (e.g. a transcript challenge over the
    input commitment)"""
    def h(i):
        return int.from_bytes(hashlib.sha256(seed + i.to_bytes(8, "little")).digest(), "little") % p
    return h(0), [h(1 + t) for t in range(n_rlc)]


def distinct_witness(p: int, layout: _Layout, input_size: int, items: Sequence[int], sorted_items: Sequence[int],
                     r: int, rlc: Sequence[int]) -> Tuple[np.ndarray, int]:
    """input layers (copy-major canonical bytes) and the copy count. A gap that
    is negative or >= 2^32 is written truncated to 32 bits, so the circuit's
    RC output exposes it."""
    k = layout.k
    n = len(items)
    if len(sorted_items) != n:
        raise ValueError("lists differ in length")
    copies = 1
    while copies * k < n:
        copies *= 2
    hi = max(list(items) + list(sorted_items) + [0]) + 1
    pad = [hi + j for j in range(copies * k - n + 1)]
    a = list(items) + pad[:-1]
    s = list(sorted_items) + pad
    w = (p.bit_length() + 7) // 8
    vals = np.zeros((copies, input_size), dtype=object)
    vals[:] = 0
    vals[:, layout.one] = 1
    vals[:, layout.m1] = p - 1
    vals[:, layout.r] = r % p
    for j in range(GAP_BITS):
        vals[:, layout.pow[j]] = 1 << j
    for t, v in enumerate(rlc):
        vals[:, layout.rlc[t]] = v % p
    for c in range(copies):
        for i in range(k):
            vals[c, layout.a[i]] = a[c * k + i] % p
        for i in range(k + 1):
            vals[c, layout.s[i]] = s[c * k + i] % p
        for i in range(k):
            gap = (s[c * k + i + 1] - s[c * k + i] - 1) & ((1 << GAP_BITS) - 1)
            for j in range(GAP_BITS):
                vals[c, layout.gap[i][j]] = (gap >> j) & 1
    raw = b"".join(int(v).to_bytes(w, "little") for v in vals.reshape(-1))
    return np.frombuffer(raw, dtype=np.uint8).copy(), copies


def accept(p: int, outputs: Sequence[int], copies: int) -> bool:
    """verifier's final check on the claimed outputs (4 per copy)"""
    pa = pb = 1
    for c in range(copies):
        o = outputs[4 * c: 4 * c + 4]
        if o[2] != 0 or o[3] != 0:
            return False
        pa = pa * o[0] % p
        pb = pb * o[1] % p
    return pa == pb
