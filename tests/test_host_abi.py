"""CPU: the C-ABI library loads, exports every symbol include/dgkr_b200.h
declares, and its host-side pieces (SHA-256, transcript, field encoding)
match the oracle. No GPU compute is called here."""
import hashlib
import os

import numpy as np
import pytest

import paper_2404_10404_b200 as P
from oracle import dgkr_oracle as O
from paper_2404_10404_b200 import workloads as W
from paper_2404_10404_b200._lib import InvalidArgument, header_symbols, lib


def test_library_exports_every_header_symbol():
    syms = header_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib(), s)]
    assert not missing, missing


def test_abi_version():
    assert lib().dgkr_abi_version() == 3


@pytest.mark.parametrize("n", [0, 1, 3, 55, 56, 63, 64, 65, 119, 120, 1000])
def test_sha256_kats(n):
    data = bytes((i * 7 + 3) & 0xFF for i in range(n))
    assert P.sha256(data) == hashlib.sha256(data).digest()


def test_sha256_fips_vectors():
    assert P.sha256(b"").hex() == "e3b0c44298fc1c149afbf4c8996fb92427ae41e4649b934ca495991b7852b855"
    assert P.sha256(b"abc").hex() == "ba7816bf8f01cfea414140de5dae2223b00361a396177a9cb410ff61f20015ad"


@pytest.mark.parametrize("p", [O.BN254_P, 97, O.GOLDILOCKS_P])
def test_field_widths(p):
    f = P.Field(p)
    of = O.Field(p)
    assert f.width == of.width and f.bits == of.bits


def test_field_rejects_unsupported_moduli():
    with pytest.raises(P._lib.DgkrError):
        P.Field(2**256 + 297)  # 257 bits: wider than the 256-bit limbs
    with pytest.raises(P._lib.DgkrError):
        P.Field(1 << 20)  # even


@pytest.mark.parametrize("p", [2**255 - 19, 2**256 - 2**32 - 977])
def test_wide_moduli_host_field_matches_oracle(p):
    """255- and 256-bit primes (the reference accepts any prime, field.hpp:26-40):
    the host field's carry-aware add and 257-bit Montgomery reduction drive the
    transcript exactly like the oracle"""
    rng = np.random.default_rng(p % 1009)
    f, of = P.Field(p), O.Field(p)
    assert (f.width, f.bits) == (of.width, of.bits)
    t, ot = P.Transcript(f, "wide", [3]), O.Transcript("wide", of, [3])
    el = [p - 1, p - 2, 0, 1] + O.random_elements(of, 12, rng)
    t.absorb_elems(el)
    for e in el:
        ot.absorb(e)
    for _ in range(20):
        assert t.challenge() == ot.challenge()
    assert t.state == ot.state


@pytest.mark.parametrize("p", [O.BN254_P, 97, O.GOLDILOCKS_P])
def test_transcript_matches_oracle(p):
    rng = np.random.default_rng(p % 1000)
    f, of = P.Field(p), O.Field(p)
    t, ot = P.Transcript(f, "lbl", [7, 9]), O.Transcript("lbl", of, [7, 9])
    el = O.random_elements(of, 17, rng)
    t.absorb_elems(el)
    for e in el:
        ot.absorb(e)
    t.absorb_bytes(b"\x01" * 32)
    ot.absorb_bytes(b"\x01" * 32)
    for _ in range(25):
        assert t.challenge() == ot.challenge()
    for b in (1, 7, 1000, 2**63 + 5):
        assert t.challenge_index(b) == ot.challenge_index(b)
    assert t.state == ot.state and t.draws == ot.draws


def test_transcript_rejects_noncanonical():
    f = P.Field(97)
    t = P.Transcript(f, "x")
    with pytest.raises(InvalidArgument):
        t.absorb_elems(bytes([97]))


def test_random_inputs_canonical():
    for p in (O.BN254_P, 97, O.GOLDILOCKS_P):
        of = O.Field(p)
        x = W.random_inputs(p, 500, 1)
        vals = of.elems_from_bytes(x.tobytes())
        assert len(vals) == 500 and all(v < p for v in vals)


def test_replicate_matches_definition():
    insz, flat = W.layered_circuit(3, 3, 2)
    full_in, full = W.replicate(insz, flat, 4)
    c = O.Circuit.from_flat(full_in, *full)
    sub = O.Circuit.from_flat(insz, *flat)
    vals = list(range(1, full_in + 1))
    out = c.evaluate(vals, 97)[-1]
    for k in range(4):
        sv = sub.evaluate(vals[k * insz:(k + 1) * insz], 97)[-1]
        assert out[k * 8:(k + 1) * 8] == sv


@pytest.mark.parametrize("k,n,threads", [(1, 5, 1), (2, 100, 1), (3, 33, 1), (4, 64, 1), (7, 17, 1),
                                         (5, 70000, 5), (9, 40000, 9), (3, 1, 3)])
def test_absorb_multi_equals_separate_chains(k, n, threads):
    """k transcripts absorbing k element streams interleaved (multi-buffer
    SHA-NI), and through the stream's combining absorb scheduler with one
    thread per transcript (chunk hand-offs at 2^15), equal k separate absorbs."""
    import ctypes as C

    from paper_2404_10404_b200._lib import Transcript_t, check

    f = P.Field.bn254()
    data = [W.random_inputs(f.p, n, 50 + j) for j in range(k)]
    want = []
    for j in range(k):
        t = P.Transcript(f, "multi", [j])
        t.absorb_elems(data[j].tobytes())
        want.append(t.state)
    ts = [Transcript_t() for _ in range(k)]
    for j in range(k):
        ts[j] = P.Transcript(f, "multi", [j]).t
    tptr = (C.POINTER(Transcript_t) * k)(*[C.pointer(t) for t in ts])
    eptr = (C.c_void_p * k)(*[d.ctypes.data for d in data])
    check(lib().dgkr_transcript_absorb_elems_multi(f.handle, tptr, C.c_size_t(k), eptr, C.c_size_t(n),
                                                   C.c_int(threads)))
    assert [bytes(t.state) for t in ts] == want


@pytest.mark.parametrize("knob,default", [("small_round_pairs", 256), ("tma_min_pairs", 0), ("fuse_round1", 0),
                                          ("absorb_chains", 1), ("tail_pairs", 256), ("tail_timeout_us", 20000),
                                          ("spin_yield", 0)])
def test_tuning_knobs_roundtrip(knob, default):
    """Launch knobs are process-wide host state (no GPU involved): defaults,
    set/get round trip, and the reference-style error for unknown names."""
    for env in ("DGKR_SMALL_PAIRS", "DGKR_TMA_MIN_PAIRS", "DGKR_FUSE_ROUND1", "DGKR_ABSORB_CHAINS",
                "DGKR_TAIL_PAIRS", "DGKR_SPIN_YIELD"):
        if env in os.environ:
            pytest.skip(f"{env} overrides the default")
    old = P.get_tuning(knob)
    assert old == default
    try:
        P.set_tuning(knob, 3 if knob == "absorb_chains" else 7)
        assert P.get_tuning(knob) == (3 if knob == "absorb_chains" else 7)
    finally:
        P.set_tuning(knob, old)
    with pytest.raises(InvalidArgument):
        P.set_tuning(knob + "_typo", 1)
