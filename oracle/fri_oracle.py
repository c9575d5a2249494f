"""ORACLE TEST INFRASTRUCTURE — Reed-Solomon / NTT / FRI restatement.

PARITY UNPINNED: the reference has no NTT, RS encoding or FRI (it replaced
Virgo's VPD/low-degree test with the Merkle column commitment of pcs.hpp;
SPEC.md:8, :369). This module restates OUR
specification (include/dgkr_b200.h) so the GPU implementation
is checked against an independent restatement plus algebraic properties
(NTT∘iNTT = id, folds of RS codewords are RS codewords, an honest-prover /
tampered-proof verifier). Transcript and SHA-256 are the reference's
(transcript.hpp, via dgkr_oracle).
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

from .dgkr_oracle import Field, MerkleTree, Transcript, sha256


def two_adic(fld: Field) -> Tuple[int, int, int]:
    """(s, w, g): p-1 = 2^s t, g = smallest quadratic non-residue, w = g^t."""
    p = fld.p
    t, s = p - 1, 0
    while t % 2 == 0:
        t //= 2
        s += 1
    for z in range(2, 1000):
        if pow(z, (p - 1) // 2, p) == p - 1:
            return s, pow(z, t, p), z
    raise ValueError("no non-residue found")


def root_of_unity(fld: Field, log_n: int) -> int:
    s, w, _ = two_adic(fld)
    if log_n > s:
        raise ValueError("domain too large")
    return pow(w, 1 << (s - log_n), fld.p)


def ntt(fld: Field, a: Sequence[int], inverse: bool = False) -> List[int]:
    """out[i] = sum_j a[j] w^(ij) (naive O(N^2) for small N; the spec)."""
    p = fld.p
    n = len(a)
    log_n = n.bit_length() - 1
    w = root_of_unity(fld, log_n)
    if inverse:
        w = pow(w, p - 2, p)
    out = [sum(a[j] * pow(w, i * j, p) for j in range(n)) % p for i in range(n)]
    if inverse:
        ninv = pow(n, p - 2, p)
        out = [x * ninv % p for x in out]
    return out


def ntt_fast(fld: Field, a: Sequence[int], inverse: bool = False) -> List[int]:
    """Same as ntt() via recursive radix-2 (for moderate N)."""
    p = fld.p
    n = len(a)
    w = root_of_unity(fld, n.bit_length() - 1)
    if inverse:
        w = pow(w, p - 2, p)

    def rec(v, w):
        m = len(v)
        if m == 1:
            return list(v)
        e, o = rec(v[0::2], w * w % p), rec(v[1::2], w * w % p)
        out = [0] * m
        x = 1
        for i in range(m // 2):
            t = x * o[i] % p
            out[i] = (e[i] + t) % p
            out[i + m // 2] = (e[i] - t) % p
            x = x * w % p
        return out

    out = rec(list(a), w)
    if inverse:
        ninv = pow(n, p - 2, p)
        out = [x * ninv % p for x in out]
    return out


def rs_encode(fld: Field, coeffs: Sequence[int], blowup_log: int) -> List[int]:
    """f(g w_N^i) for i < N = len(coeffs) << blowup_log."""
    p = fld.p
    _, _, g = two_adic(fld)
    n = len(coeffs)
    N = n << blowup_log
    scaled = [c * pow(g, j, p) % p for j, c in enumerate(coeffs)] + [0] * (N - n)
    return ntt_fast(fld, scaled)


def fri_fold(fld: Field, f: Sequence[int], beta: int, layer: int, log_n0: int) -> List[int]:
    p = fld.p
    _, _, g = two_adic(fld)
    w = root_of_unity(fld, log_n0)
    h = len(f) // 2
    inv2 = pow(2, p - 2, p)
    out = []
    for i in range(h):
        x = pow(g, 1 << layer, p) * pow(w, (1 << layer) * i, p) % p
        xinv = pow(x, p - 2, p)
        f0, f1 = f[i], f[i + h]
        out.append(((f0 + f1) + beta * xinv % p * (f0 - f1)) * inv2 % p)
    return out


def _leaves(fld: Field, f: Sequence[int]) -> List[bytes]:
    return [sha256(fld.to_bytes(x)) for x in f]


def fri_prove(fld: Field, coeffs: Sequence[int], blowup_log: int, final_log: int, queries: int,
              tr: Transcript) -> bytes:
    """dgkr_fri_prove restated (proof layout in include/dgkr_b200.h)."""
    n = len(coeffs)
    log_n0 = n.bit_length() - 1 + blowup_log
    L = log_n0 - final_log
    layers = [rs_encode(fld, coeffs, blowup_log)]
    trees, roots = [], []
    for l in range(L):
        t = MerkleTree(_leaves(fld, layers[l]))
        trees.append(t)
        roots.append(t.root)
        tr.absorb_bytes(t.root)
        beta = tr.challenge()
        layers.append(fri_fold(fld, layers[l], beta, l, log_n0))
    for x in layers[L]:
        tr.absorb(x)
    H = (1 << log_n0) // 2
    qi: List[int] = []
    if L > 0:
        if queries >= H:
            qi = list(range(H))
        else:
            seen = set()
            while len(qi) < queries:
                j = tr.challenge_index(H)
                if j not in seen:
                    seen.add(j)
                    qi.append(j)
    out = L.to_bytes(4, "little") + b"".join(roots) + len(layers[L]).to_bytes(4, "little")
    out += fld.elems_to_bytes(layers[L]) + len(qi).to_bytes(4, "little")
    for i in qi:
        out += i.to_bytes(4, "little")
        for l in range(L):
            hl = len(layers[l]) // 2
            il = i % hl
            out += fld.to_bytes(layers[l][il]) + fld.to_bytes(layers[l][il + hl])
            out += b"".join(trees[l].path(il)) + b"".join(trees[l].path(il + hl))
    return out


def fri_verify(fld: Field, proof: bytes, n: int, blowup_log: int, final_log: int, queries: int,
               tr: Transcript) -> bool:
    """Verifier for the spec: Merkle paths, fold consistency along each query,
    the final layer is a codeword of degree < n >> L."""
    p = fld.p
    w_ = fld.width
    _, _, g = two_adic(fld)
    log_n0 = n.bit_length() - 1 + blowup_log
    L = log_n0 - final_log
    w = root_of_unity(fld, log_n0)
    pos = 0

    def take(k):
        nonlocal pos
        b = proof[pos:pos + k]
        if len(b) != k:
            raise ValueError("truncated")
        pos += k
        return b

    try:
        if int.from_bytes(take(4), "little") != L:
            return False
        roots = [take(32) for _ in range(L)]
        betas = []
        for l in range(L):
            tr.absorb_bytes(roots[l])
            betas.append(tr.challenge())
        nf = int.from_bytes(take(4), "little")
        if nf != 1 << final_log:
            return False
        final = fld.elems_from_bytes(take(nf * w_))
        if any(x >= p for x in final):
            return False
        for x in final:
            tr.absorb(x)
        # low degree of the final layer: its coefficients above n >> L vanish
        coeffs = ntt_fast(fld, final, inverse=True)  # on coset g^(2^L)<w'>: f(g' w'^i)
        gL = pow(g, 1 << L, p)
        coeffs = [c * pow(gL, p - 1 - j, p) % p for j, c in enumerate(coeffs)]
        deg_bound = max(n >> L, 1)
        if any(coeffs[deg_bound:]):
            return False
        H = (1 << log_n0) // 2
        Q = int.from_bytes(take(4), "little")
        want_q = H if queries >= H else queries
        if L > 0 and Q != want_q:
            return False
        expect = []
        if L > 0:
            if queries >= H:
                expect = list(range(H))
            else:
                seen = set()
                while len(expect) < queries:
                    j = tr.challenge_index(H)
                    if j not in seen:
                        seen.add(j)
                        expect.append(j)
        for k in range(Q):
            i = int.from_bytes(take(4), "little")
            if i != expect[k]:
                return False
            carry = None
            for l in range(L):
                Nl = (1 << log_n0) >> l
                hl = Nl // 2
                il = i % hl
                f0 = fld.from_bytes(take(w_))
                f1 = fld.from_bytes(take(w_))
                depth = Nl.bit_length() - 1
                p0 = [take(32) for _ in range(depth)]
                p1 = [take(32) for _ in range(depth)]
                if not MerkleTree.verify_path(roots[l], sha256(fld.to_bytes(f0)), il, p0):
                    return False
                if not MerkleTree.verify_path(roots[l], sha256(fld.to_bytes(f1)), il + hl, p1):
                    return False
                if carry is not None:
                    prev_pos, val = carry
                    if (f0 if prev_pos == il else f1) != val:
                        return False
                x = pow(g, 1 << l, p) * pow(w, (1 << l) * il, p) % p
                folded = ((f0 + f1) + betas[l] * pow(x, p - 2, p) % p * (f0 - f1)) * pow(2, p - 2, p) % p
                # f_{l+1}[il]: at layer l+1 it is the opened value at il (= i mod h_{l+1} or that + h_{l+1})
                carry = (il, folded)
            if L > 0 and final[carry[0]] != carry[1]:
                return False
        return pos == len(proof)
    except ValueError:
        return False


# --- distributed FRI (dgkr_fri_prove_dist; include/dgkr_b200.h) ---

def _draw_queries(tr: Transcript, H: int, queries: int, L: int) -> List[int]:
    if L == 0:
        return []
    if queries >= H:
        return list(range(H))
    qi: List[int] = []
    seen = set()
    while len(qi) < queries:
        j = tr.challenge_index(H)
        if j not in seen:
            seen.add(j)
            qi.append(j)
    return qi


def fri_prove_dist(fld: Field, chunks: Sequence[Sequence[int]], blowup_log: int, final_log: int, queries: int,
                   tr: Transcript) -> List[bytes]:
    """Rank r folds chunks[r]; one shared transcript: per layer all ranks'
    roots in rank order, then every rank's final layer in rank order, then the
    shared query positions. Returns one proof per rank."""
    world = len(chunks)
    n = len(chunks[0])
    log_n0 = n.bit_length() - 1 + blowup_log
    L = log_n0 - final_log
    layers = [[rs_encode(fld, c, blowup_log)] for c in chunks]
    trees: List[List[MerkleTree]] = [[] for _ in range(world)]
    roots: List[List[bytes]] = []
    for l in range(L):
        rl = []
        for r in range(world):
            t = MerkleTree(_leaves(fld, layers[r][l]))
            trees[r].append(t)
            rl.append(t.root)
        roots.append(rl)
        for x in rl:
            tr.absorb_bytes(x)
        beta = tr.challenge()
        for r in range(world):
            layers[r].append(fri_fold(fld, layers[r][l], beta, l, log_n0))
    for r in range(world):
        for x in layers[r][L]:
            tr.absorb(x)
    qi = _draw_queries(tr, (1 << log_n0) // 2, queries, L)
    nf = len(layers[0][L])
    head = L.to_bytes(4, "little") + b"".join(b"".join(rl) for rl in roots) + nf.to_bytes(4, "little")
    head += b"".join(fld.elems_to_bytes(layers[r][L]) for r in range(world)) + len(qi).to_bytes(4, "little")
    out = []
    for r in range(world):
        pr = world.to_bytes(4, "little") + r.to_bytes(4, "little") + head
        for i in qi:
            pr += i.to_bytes(4, "little")
            for l in range(L):
                hl = len(layers[r][l]) // 2
                il = i % hl
                pr += fld.to_bytes(layers[r][l][il]) + fld.to_bytes(layers[r][l][il + hl])
                pr += b"".join(trees[r][l].path(il)) + b"".join(trees[r][l].path(il + hl))
        out.append(pr)
    return out


def fri_verify_dist(fld: Field, proofs: Sequence[bytes], n: int, blowup_log: int, final_log: int, queries: int,
                    tr: Transcript) -> bool:
    """Accept iff the `world` per-rank proofs agree on every rank's roots and
    final layer, each final layer has degree < n >> L, and each rank's query
    openings verify against its own roots with the shared betas."""
    p = fld.p
    w_ = fld.width
    world = len(proofs)
    _, _, g = two_adic(fld)
    log_n0 = n.bit_length() - 1 + blowup_log
    L = log_n0 - final_log
    w = root_of_unity(fld, log_n0)
    nf = 1 << final_log
    head_len = 4 + L * world * 32 + 4 + world * nf * w_ + 4
    if world < 1 or any(len(pr) < 8 + head_len for pr in proofs):
        return False
    heads = [pr[8:8 + head_len] for pr in proofs]
    if any(h != heads[0] for h in heads):
        return False
    for r, pr in enumerate(proofs):
        if int.from_bytes(pr[0:4], "little") != world or int.from_bytes(pr[4:8], "little") != r:
            return False
    h = heads[0]
    if int.from_bytes(h[0:4], "little") != L:
        return False
    pos = 4
    roots = []
    for _ in range(L):
        roots.append([h[pos + 32 * r: pos + 32 * r + 32] for r in range(world)])
        pos += 32 * world
    if int.from_bytes(h[pos:pos + 4], "little") != nf:
        return False
    pos += 4
    finals = []
    for _ in range(world):
        finals.append(fld.elems_from_bytes(h[pos:pos + nf * w_]))
        pos += nf * w_
    Q = int.from_bytes(h[pos:pos + 4], "little")
    betas = []
    for l in range(L):
        for x in roots[l]:
            tr.absorb_bytes(x)
        betas.append(tr.challenge())
    gL = pow(g, 1 << L, p)
    deg_bound = max(n >> L, 1)
    for fin in finals:
        if any(x >= p for x in fin):
            return False
        coeffs = ntt_fast(fld, fin, inverse=True)
        coeffs = [c * pow(gL, p - 1 - j, p) % p for j, c in enumerate(coeffs)]
        if any(coeffs[deg_bound:]):
            return False
    for fin in finals:
        for x in fin:
            tr.absorb(x)
    H = (1 << log_n0) // 2
    expect = _draw_queries(tr, H, queries, L)
    if Q != len(expect):
        return False
    inv2 = pow(2, p - 2, p)
    for r, pr in enumerate(proofs):
        pos = 8 + head_len

        def take(k):
            nonlocal pos
            b = pr[pos:pos + k]
            if len(b) != k:
                raise ValueError("truncated")
            pos += k
            return b

        try:
            for k in range(Q):
                if int.from_bytes(take(4), "little") != expect[k]:
                    return False
                i = expect[k]
                carry = None
                for l in range(L):
                    Nl = (1 << log_n0) >> l
                    hl = Nl // 2
                    il = i % hl
                    f0 = fld.from_bytes(take(w_))
                    f1 = fld.from_bytes(take(w_))
                    depth = Nl.bit_length() - 1
                    p0 = [take(32) for _ in range(depth)]
                    p1 = [take(32) for _ in range(depth)]
                    if not MerkleTree.verify_path(roots[l][r], sha256(fld.to_bytes(f0)), il, p0):
                        return False
                    if not MerkleTree.verify_path(roots[l][r], sha256(fld.to_bytes(f1)), il + hl, p1):
                        return False
                    if carry is not None and (f0 if carry[0] == il else f1) != carry[1]:
                        return False
                    x = pow(g, 1 << l, p) * pow(w, (1 << l) * il, p) % p
                    carry = (il, ((f0 + f1) + betas[l] * pow(x, p - 2, p) % p * (f0 - f1)) * inv2 % p)
                if L > 0 and finals[r][carry[0]] != carry[1]:
                    return False
        except ValueError:
            return False
        if pos != len(pr):
            return False
    return True
