"""SHA-256 inside a data-parallel GKR circuit (the
in-circuit form of config C3; the reference has only native SHA-256,
sha256.hpp, and the Merkle paths of beacon.hpp:151-174).

One copy of the sub-circuit checks ONE SHA-256 compression
``H_out = compress(H_in, block)`` (FIPS 180-4 §6.2.2). Sequential dependencies
are broken by witness bits in the input layer (the Virgo/Sisu setting: the
input layer is committed, e.g. with ``pcs_commit``): every round's new ``a``
and ``e`` words, the message schedule ``W_16..W_63``, the digest, and the
carry quotients of every mod-2^32 addition. All 64 rounds then constrain in
parallel, so the circuit has depth 4 whatever the number of rounds:

  L1  pairwise bit products  x*y          (XOR3 / Maj / Ch operands)
  L2  triple products        (x*y)*z
  L3  bit functions          XOR3 = x+y+z-2(xy+xz+yz)+4xyz, XOR2, Ch = ef+g-eg,
                             Maj = ab+ac+bc-2abc  (accumulation gates, constant
                             coefficients taken from constant input wires)
  L4  constraints (outputs)  booleanity b*b - b, and per addition
                             sum_i 2^i out_i + 2^32 q - sum_terms - K = 0

The proof's claimed outputs are all zero iff the witness is a correct
compression. Gates are the reference's fan-in-2 add/mul nested gates
(circuit.hpp:20-41) only; constants (0, 1, -1, -2, 4, +-2^i) are input
wires. ``sha256_witness`` builds the input layer for a batch of compressions
(vectorised over copies); replicate with ``n_copies`` for the data-parallel
proof (copy index = high variables, as the Sisu layout).
"""
from __future__ import annotations

from typing import Dict, List, NamedTuple, Optional, Tuple

import numpy as np

from .workloads import Flat

K256 = np.array([
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
    0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
    0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
    0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
    0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
    0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
    0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2],
    dtype=np.uint64)
IV = np.array([0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a, 0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19],
              dtype=np.uint64)
NPOW = 36  # constant powers 2^0 .. 2^35


class _Layout:
    """input-layer indices of one copy"""

    def __init__(self):
        self.n = 0
        self.const: Dict[str, int] = {}
        self.pow: List[int] = []
        self.npow: List[int] = []
        self.words: Dict[Tuple[str, int], List[int]] = {}  # (name, t) -> 32 bit wires (LSB first)
        self.qbits: Dict[Tuple[str, int], List[int]] = {}  # carry quotient bits
        self.bits: List[int] = []  # every wire that must be boolean
        self.rlc: List[int] = []   # random-linear-combination coefficients (rlc circuits)

    def alloc(self, k: int) -> List[int]:
        r = list(range(self.n, self.n + k))
        self.n += k
        return r

    def word(self, name: str, t: int) -> List[int]:
        w = self.alloc(32)
        self.words[(name, t)] = w
        self.bits.extend(w)
        return w

    def q(self, name: str, t: int, nb: int) -> List[int]:
        w = self.alloc(nb)
        self.qbits[(name, t)] = w
        self.bits.extend(w)
        return w


def _layout() -> _Layout:
    L = _Layout()
    for name in ("zero", "one", "m1", "neg2", "four"):
        L.const[name] = L.alloc(1)[0]
    L.pow = L.alloc(NPOW)
    L.npow = L.alloc(NPOW)
    for i in range(8):
        L.word("hin", i)
    for t in range(64):
        L.word("w", t)
    for t in range(16, 64):
        L.q("w", t, 2)          # 4 terms -> quotient < 4
    for t in range(1, 65):
        L.word("a", t)
        L.word("e", t)
        L.q("a", t, 3)          # 7 terms (+K) -> quotient < 8
        L.q("e", t, 3)          # 6 terms (+K) -> quotient < 8
    for i in range(8):
        L.word("hout", i)
        L.q("hout", i, 1)       # 2 terms -> quotient < 2
    return L


class _Builder:
    """layers 1..4 of gates; a gate = list of (is_mul, la, ga, lb, gb)"""

    def __init__(self, L: _Layout):
        self.L = L
        self.layers: List[List[list]] = [[], [], [], []]
        self.memo: Dict[tuple, Tuple[int, int]] = {}

    def gate(self, layer: int, nested: list, key=None) -> Tuple[int, int]:
        if key is not None and key in self.memo:
            return self.memo[key]
        self.layers[layer - 1].append(nested)
        ref = (layer, len(self.layers[layer - 1]) - 1)
        if key is not None:
            self.memo[key] = ref
        return ref

    def prod2(self, x: int, y: int) -> Tuple[int, int]:
        x, y = min(x, y), max(x, y)
        return self.gate(1, [(1, 0, x, 0, y)], ("p2", x, y))

    def prod3(self, x: int, y: int, z: int) -> Tuple[int, int]:
        x, y, z = sorted((x, y, z))
        l, g = self.prod2(x, y)
        return self.gate(2, [(1, l, g, 0, z)], ("p3", x, y, z))

    def c(self, name: str) -> int:
        return self.L.const[name]

    def xor(self, xs: List[int]) -> Tuple[int, int]:
        """XOR of 2 or 3 input bits as an L3 value"""
        zero, neg2, four = self.c("zero"), self.c("neg2"), self.c("four")
        if len(xs) == 2:
            x, y = xs
            pl, pg = self.prod2(x, y)
            return self.gate(3, [(0, 0, x, 0, y), (1, 0, neg2, pl, pg)], ("x2", *sorted(xs)))
        x, y, z = xs
        nested = [(0, 0, x, 0, y), (0, 0, z, 0, zero)]
        for u, v in ((x, y), (x, z), (y, z)):
            pl, pg = self.prod2(u, v)
            nested.append((1, 0, neg2, pl, pg))
        tl, tg = self.prod3(x, y, z)
        nested.append((1, 0, four, tl, tg))
        return self.gate(3, nested, ("x3", *sorted(xs)))

    def ch(self, e: int, f: int, g: int) -> Tuple[int, int]:
        m1, zero = self.c("m1"), self.c("zero")
        efl, efg = self.prod2(e, f)
        egl, egg = self.prod2(e, g)
        one = self.c("one")
        # ef + g - eg  (= ef*1 + g + (-1)*eg)
        return self.gate(3, [(1, efl, efg, 0, one), (0, 0, g, 0, zero), (1, 0, m1, egl, egg)], ("ch", e, f, g))

    def maj(self, a: int, b: int, c: int) -> Tuple[int, int]:
        one, neg2 = self.c("one"), self.c("neg2")
        nested = []
        for u, v in ((a, b), (a, c), (b, c)):
            pl, pg = self.prod2(u, v)
            nested.append((1, pl, pg, 0, one))
        tl, tg = self.prod3(a, b, c)
        nested.append((1, 0, neg2, tl, tg))
        return self.gate(3, nested, ("maj", a, b, c))


def _rotr(w: List[int], n: int) -> List[int]:
    """bit i of ROTR^n(x) = bit (i + n) mod 32 of x"""
    return [w[(i + n) % 32] for i in range(32)]


def _big_sigma(B: _Builder, w: List[int], r: Tuple[int, int, int]) -> List[Tuple[int, int]]:
    a, b, c = _rotr(w, r[0]), _rotr(w, r[1]), _rotr(w, r[2])
    return [B.xor([a[i], b[i], c[i]]) for i in range(32)]


def _small_sigma(B: _Builder, w: List[int], r1: int, r2: int, s: int) -> List[Tuple[int, int]]:
    a, b = _rotr(w, r1), _rotr(w, r2)
    out = []
    for i in range(32):
        if i + s < 32:
            out.append(B.xor([a[i], b[i], w[i + s]]))
        else:
            out.append(B.xor([a[i], b[i]]))
    return out


def build_compression_circuit(rlc: bool = False) -> Tuple[int, Flat, _Layout]:
    """-> (input_size (power of two), flat circuit, input layout) of one compression.

    rlc=False: the output layer is the constraint vector (8,192 padded outputs
    per copy, every one absorbed by the reference transcript).
    rlc=True: one more layer folds the constraints of a copy into ONE output
    sum_i R_i c_i, with the coefficients R_i public inputs (layout.rlc). In the
    committed-witness setting the caller draws them by Fiat-Shamir after
    committing the witness (e.g. from a transcript over pcs_commit's root);
    a non-zero constraint then survives with probability >= 1 - n/p."""
    L = _layout()
    B = _Builder(L)
    pw, npw, one = L.pow, L.npow, L.const["one"]
    W = {t: L.words[("w", t)] for t in range(64)}

    def A(t):
        return L.words[("a", t)] if t >= 1 else L.words[("hin", -t)]

    def E(t):
        return L.words[("e", t)] if t >= 1 else L.words[("hin", 4 - t)]

    constraints: List[list] = []

    def plus_bits(bits: List[int], sign: int) -> list:  # +-sum_i 2^i bit_i (L0 bits)
        cs = pw if sign > 0 else npw
        return [(1, 0, cs[i], 0, bits[i]) for i in range(32)]

    def plus_vals(vals: List[Tuple[int, int]], sign: int) -> list:  # +-sum_i 2^i v_i (L3 values)
        cs = pw if sign > 0 else npw
        return [(1, 0, cs[i], vals[i][0], vals[i][1]) for i in range(32)]

    def plus_q(qb: List[int]) -> list:  # + 2^32 * (q0 + 2 q1 + ...)
        return [(1, 0, pw[32 + j], 0, qb[j]) for j in range(len(qb))]

    def minus_const(k: int) -> list:
        return [(1, 0, npw[i], 0, one) for i in range(32) if (k >> i) & 1]

    # message schedule W_t = s1(W_{t-2}) + W_{t-7} + s0(W_{t-15}) + W_{t-16}, t = 16..63
    for t in range(16, 64):
        s1 = _small_sigma(B, W[t - 2], 17, 19, 10)
        s0 = _small_sigma(B, W[t - 15], 7, 18, 3)
        constraints.append(plus_bits(W[t], 1) + plus_q(L.qbits[("w", t)]) + plus_vals(s1, -1)
                           + plus_bits(W[t - 7], -1) + plus_vals(s0, -1) + plus_bits(W[t - 16], -1))
    # rounds
    for t in range(64):
        a, b, c, d = A(t), A(t - 1), A(t - 2), A(t - 3)
        e, f, g, h = E(t), E(t - 1), E(t - 2), E(t - 3)
        S1 = _big_sigma(B, e, (6, 11, 25))
        ch = [B.ch(e[i], f[i], g[i]) for i in range(32)]
        S0 = _big_sigma(B, a, (2, 13, 22))
        mj = [B.maj(a[i], b[i], c[i]) for i in range(32)]
        T1 = plus_bits(h, -1) + plus_vals(S1, -1) + plus_vals(ch, -1) + minus_const(int(K256[t])) + plus_bits(W[t], -1)
        # E[t+1] = d + T1 ; A[t+1] = T1 + T2
        constraints.append(plus_bits(E(t + 1), 1) + plus_q(L.qbits[("e", t + 1)]) + plus_bits(d, -1) + T1)
        constraints.append(plus_bits(A(t + 1), 1) + plus_q(L.qbits[("a", t + 1)]) + T1 + plus_vals(S0, -1)
                           + plus_vals(mj, -1))
    # digest: H_out_i = H_in_i + state_i
    final = [A(64), A(63), A(62), A(61), E(64), E(63), E(62), E(61)]
    for i in range(8):
        constraints.append(plus_bits(L.words[("hout", i)], 1) + plus_q(L.qbits[("hout", i)])
                           + plus_bits(L.words[("hin", i)], -1) + plus_bits(final[i], -1))
    # booleanity b*b + b*(-1)
    m1 = L.const["m1"]
    for bw in L.bits:
        constraints.append([(1, 0, bw, 0, bw), (1, 0, bw, 0, m1)])
    B.layers[3] = constraints
    L.rlc = []
    if rlc:
        L.rlc = L.alloc(len(constraints))
        B.layers.append([[(1, 0, L.rlc[i], 4, i) for i in range(len(constraints))]])
    # pad every layer to a power of two with zero gates (data-parallel precondition)
    zero = L.const["zero"]
    input_size = 1
    while input_size < L.n:
        input_size *= 2
    for layer in B.layers:
        n = 1
        while n < len(layer):
            n *= 2
        layer.extend([[(0, 0, zero, 0, zero)]] * (n - len(layer)))
    lgs, gns, rows = [0], [0], []
    for layer in B.layers:
        for g in layer:
            rows.extend(g)
            gns.append(gns[-1] + len(g))
        lgs.append(lgs[-1] + len(layer))
    flat = (np.array(lgs, np.uint64), np.array(gns, np.uint64), np.array(rows, np.uint32).reshape(-1, 5),
            np.ones(len(B.layers) + 1, np.uint64))
    return input_size, flat, L


def _u32(x):
    return np.asarray(x, dtype=np.uint64) & 0xFFFFFFFF


def _rotr_v(x, n):
    return ((x >> n) | (x << (32 - n))) & 0xFFFFFFFF


def compress_trace(h_in: np.ndarray, block: np.ndarray):
    """vectorised FIPS 180-4 compression over N instances: h_in (N, 8),
    block (N, 16) big-endian message words -> dict of every witness word"""
    h_in, block = _u32(h_in), _u32(block)
    N = h_in.shape[0]
    W = np.zeros((N, 64), np.uint64)
    qw = np.zeros((N, 64), np.uint64)
    W[:, :16] = block
    for t in range(16, 64):
        x2, x15 = W[:, t - 2], W[:, t - 15]
        s1 = _rotr_v(x2, 17) ^ _rotr_v(x2, 19) ^ (x2 >> 10)
        s0 = _rotr_v(x15, 7) ^ _rotr_v(x15, 18) ^ (x15 >> 3)
        tot = s1 + W[:, t - 7] + s0 + W[:, t - 16]
        W[:, t], qw[:, t] = tot & 0xFFFFFFFF, tot >> 32
    A = {-k: h_in[:, k] for k in range(4)}
    E = {-k: h_in[:, 4 + k] for k in range(4)}
    qa, qe = {}, {}
    for t in range(64):
        a, b, c, d = A[t], A[t - 1], A[t - 2], A[t - 3]
        e, f, g, h = E[t], E[t - 1], E[t - 2], E[t - 3]
        S1 = _rotr_v(e, 6) ^ _rotr_v(e, 11) ^ _rotr_v(e, 25)
        ch = (e & f) ^ (~e & 0xFFFFFFFF & g)
        S0 = _rotr_v(a, 2) ^ _rotr_v(a, 13) ^ _rotr_v(a, 22)
        mj = (a & b) ^ (a & c) ^ (b & c)
        t1 = h + S1 + ch + K256[t] + W[:, t]
        ne = d + t1
        na = t1 + S0 + mj
        E[t + 1], qe[t + 1] = ne & 0xFFFFFFFF, ne >> 32
        A[t + 1], qa[t + 1] = na & 0xFFFFFFFF, na >> 32
    final = [A[64], A[63], A[62], A[61], E[64], E[63], E[62], E[61]]
    hout = np.stack([(h_in[:, i] + final[i]) & 0xFFFFFFFF for i in range(8)], axis=1)
    qh = np.stack([(h_in[:, i] + final[i]) >> 32 for i in range(8)], axis=1)
    return {"W": W, "qw": qw, "A": A, "E": E, "qa": qa, "qe": qe, "hout": hout, "qh": qh}


def rlc_coefficients(p: int, seed: bytes, n: int) -> List[int]:
    """n coefficients R_i = SHA256(seed || LE64 i) mod p (seed: e.g. a
    transcript challenge drawn after the witness commitment)"""
    import hashlib
    return [int.from_bytes(hashlib.sha256(seed + i.to_bytes(8, "little")).digest(), "little") % p for i in range(n)]


def sha256_witness(p: int, layout: _Layout, input_size: int, h_in: np.ndarray,
                   block: np.ndarray, rlc: Optional[List[int]] = None) -> Tuple[np.ndarray, np.ndarray]:
    """input layers (N copies x input_size field elements, canonical bytes,
    copy-major, uint8[N * input_size * w]) for the compression circuit, and
    the digests (N, 8). rlc: the R_i of an rlc=True circuit (shared by all
    copies)."""
    tr = compress_trace(h_in, block)
    N = tr["W"].shape[0]
    w = (p.bit_length() + 7) // 8
    base = np.zeros((input_size, w), dtype=np.uint8)
    Lc = layout.const

    def put_const(i, v):
        base[i] = np.frombuffer(int(v % p).to_bytes(w, "little"), dtype=np.uint8)

    for name, v in (("zero", 0), ("one", 1), ("m1", -1), ("neg2", -2), ("four", 4)):
        put_const(Lc[name], v)
    for i in range(NPOW):
        put_const(layout.pow[i], 1 << i)
        put_const(layout.npow[i], -(1 << i))
    if layout.rlc:
        if rlc is None or len(rlc) != len(layout.rlc):
            raise ValueError("this circuit needs len(layout.rlc) coefficients")
        for idx, v in zip(layout.rlc, rlc):
            put_const(idx, v)
    out = np.broadcast_to(base, (N, input_size, w)).copy()
    cols: List[np.ndarray] = []   # bit wire indices
    bits: List[np.ndarray] = []   # (N, nb) bit values, LSB first

    def put_bits(idx, val, nb):
        cols.append(np.asarray(idx[:nb], np.int64))
        bits.append(((val[:, None] >> np.arange(nb, dtype=np.uint64)) & 1).astype(np.uint8))

    h = _u32(h_in)
    for i in range(8):
        put_bits(layout.words[("hin", i)], h[:, i], 32)
        put_bits(layout.words[("hout", i)], tr["hout"][:, i], 32)
        put_bits(layout.qbits[("hout", i)], tr["qh"][:, i], 1)
    for t in range(64):
        put_bits(layout.words[("w", t)], tr["W"][:, t], 32)
    for t in range(16, 64):
        put_bits(layout.qbits[("w", t)], tr["qw"][:, t], 2)
    for t in range(1, 65):
        put_bits(layout.words[("a", t)], tr["A"][t], 32)
        put_bits(layout.words[("e", t)], tr["E"][t], 32)
        put_bits(layout.qbits[("a", t)], tr["qa"][t], 3)
        put_bits(layout.qbits[("e", t)], tr["qe"][t], 3)
    # one scatter of every bit wire (low byte; the other bytes stay zero)
    out[:, np.concatenate(cols), 0] = np.concatenate(bits, axis=1)
    return out.reshape(-1), tr["hout"]


def merkle_path_compressions(leaf_msg: bytes, siblings, index: int):
    """(h_in, block) pairs of every SHA-256 compression verifying one Merkle
    path of 64-byte nodes (beacon.hpp:151-174 without the zero-cache tail):
    SHA256(64-byte message) = compress(compress(IV, msg), padding block)."""
    pad = np.zeros(16, np.uint64)
    pad[0], pad[15] = 0x80000000, 512
    h_in, blocks = [], []

    def hash64(msg: bytes) -> np.ndarray:
        b = digest_words(msg)
        tr = compress_trace(IV[None, :], b[None, :])
        h_in.extend([IV, tr["hout"][0]])
        blocks.extend([b, pad])
        tr2 = compress_trace(tr["hout"], pad[None, :])
        return tr2["hout"][0]

    def to_bytes(words) -> bytes:
        return b"".join(int(x).to_bytes(4, "big") for x in words)

    h = to_bytes(hash64(leaf_msg))
    node = index
    for s in siblings:
        h = to_bytes(hash64(s + h if node & 1 else h + s))
        node >>= 1
    return np.array(h_in, np.uint64), np.array(blocks, np.uint64), h


def digest_words(data: bytes) -> np.ndarray:
    return np.frombuffer(data, dtype=">u4").astype(np.uint64)


class RlcProof(NamedTuple):
    root: bytes          # witness commitment (input layer, R_i slots zero)
    proof: bytes         # GkrProof bytes on the continued transcript
    digests: np.ndarray  # (m, 8) output chaining values
    inputs: np.ndarray   # the input layer with the R_i filled in


def _witness_root(ctx, field, inputs: np.ndarray) -> bytes:
    """pcs_commit (pcs.hpp:105-113) of the input layer as one row, zero-padded
    to a power-of-two column count (merkle.hpp:16-19 needs one)"""
    from . import prover as P
    w = field.width
    cols = len(inputs) // w
    padded = 1 << max(0, (cols - 1).bit_length())
    row = inputs if padded == cols else np.concatenate([inputs, np.zeros((padded - cols) * w, np.uint8)])
    return P.pcs_commit(ctx, field, [row])


def _rlc_seed(tr, root: bytes) -> bytes:
    tr.absorb_bytes(root)
    return tr.field.encode([tr.challenge()])


def prove_compressions_rlc(ctx, field, h_in: np.ndarray, blocks: np.ndarray, label: str = "sha.rlc",
                           built=None):
    """Committed-witness proof of a batch of compressions with the rlc=True
    circuit (one claimed output per compression):

      1. the input layer with every R_i slot zero is committed (pcs_commit);
      2. the transcript absorbs the root and draws one challenge c;
      3. R_i = rlc_coefficients(p, bytes(c), n) fill the R_i slots;
      4. gkr_prove on the same transcript.

    The R_i are fixed only after the witness is, so a wrong witness leaves
    sum_i R_i c_i non-zero except with probability ~n/p. The number of
    compressions is padded to a power of two with compress(IV, 0) copies.
    built: an optional (input_size, flat, layout, Circuit) from a previous
    call with the same copy count. Returns (RlcProof, built); RlcProof.inputs
    is the witness the verifier below checks against."""
    from . import prover as P
    m = len(h_in)
    copies = 1 << max(0, (m - 1).bit_length())
    if copies != m:
        h_in = np.concatenate([h_in, np.tile(IV, (copies - m, 1))])
        blocks = np.concatenate([blocks, np.zeros((copies - m, 16), np.uint64)])
    if built is None:
        insz, flat, L = build_compression_circuit(rlc=True)
        built = (insz, flat, L, P.Circuit(ctx, insz, *flat, n_copies=copies))
    insz, flat, L, dc = built
    p = field.p
    inputs, hout = sha256_witness(p, L, insz, h_in, blocks, rlc=[0] * len(L.rlc))
    root = _witness_root(ctx, field, inputs)
    tr = P.Transcript(field, label, [copies])
    coeffs = rlc_coefficients(p, _rlc_seed(tr, root), len(L.rlc))
    _put_rlc(field, L, insz, copies, inputs, coeffs)
    proof = P.gkr_prove(ctx, dc, inputs, tr)
    return RlcProof(root, proof, hout[:m], inputs), built


def _put_rlc(field, L, insz, copies, inputs, coeffs) -> None:
    w = field.width
    view = inputs.reshape(copies, insz, w)
    enc = np.frombuffer(field.encode(coeffs), np.uint8).reshape(len(coeffs), w)
    view[:, L.rlc, :] = enc[None, :, :]


def verify_compressions_rlc(ctx, field, built, inputs: np.ndarray, root: bytes, proof: bytes,
                            label: str = "sha.rlc") -> bool:
    """Verifier of prove_compressions_rlc given the witness (the setting of
    gkr_verify with inputs, gkr.hpp:314-325): the root matches the input layer
    with the R_i slots zeroed, the R_i in the input layer are the ones the
    transcript draws after absorbing the root, every claimed output is zero,
    and the GKR proof verifies on the continued transcript."""
    from . import prover as P
    insz, _, L, dc = built
    w = field.width
    copies = len(inputs) // (insz * w)
    zeroed = inputs.copy()
    _put_rlc(field, L, insz, copies, zeroed, [0] * len(L.rlc))
    if _witness_root(ctx, field, zeroed) != root:
        return False
    tr = P.Transcript(field, label, [copies])
    coeffs = rlc_coefficients(field.p, _rlc_seed(tr, root), len(L.rlc))
    want = zeroed.copy()
    _put_rlc(field, L, insz, copies, want, coeffs)
    if not np.array_equal(want, inputs):
        return False
    n = int.from_bytes(proof[:4], "little")
    if any(proof[4:4 + n * w]):
        return False
    return P.gkr_verify(dc, proof, tr, inputs=inputs)
