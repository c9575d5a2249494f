"""Python mirror of the reference prover API over the C ABI
(``include/dgkr_b200.h``). Names and argument meaning follow
``/root/reference/proj/include/dgkr`` so the parity tests read like the
reference's own tests; every prover call runs on the GPU through
``libdgkr_b200.so`` (no CPU fallback).

Field elements are passed either as Python ints (converted to canonical
little-endian bytes) or as ready canonical byte buffers (``bytes`` /
``numpy.uint8`` arrays), which is what the benchmark uses.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence, Tuple, Union

import numpy as np

from ._lib import InvalidArgument, Profile_t, Transcript_t, check, lib

BN254_P = 21888242871839275222246405745257275088548364400416034343698204186575808495617
GOLDILOCKS_P = 18446744069414584321

Elems = Union[bytes, bytearray, memoryview, np.ndarray, Sequence[int]]


def _buf(b) -> C.c_void_p:
    if isinstance(b, np.ndarray):
        return b.ctypes.data_as(C.c_void_p)
    return C.cast(C.c_char_p(bytes(b)), C.c_void_p)


class Field:
    """FieldConfig (field.hpp:23-80)."""

    def __init__(self, modulus: int):
        self.p = int(modulus)
        mb = self.p.to_bytes(max(1, (self.p.bit_length() + 7) // 8), "little")
        h = C.c_void_p()
        check(lib().dgkr_field_create(C.c_char_p(mb), C.c_size_t(len(mb)), C.byref(h)))
        self._h = h
        self.width = int(lib().dgkr_field_width(h))
        self.bits = int(lib().dgkr_field_bits(h))

    @staticmethod
    def bn254() -> "Field":
        return Field(BN254_P)

    @staticmethod
    def goldilocks() -> "Field":
        return Field(GOLDILOCKS_P)

    def __del__(self):
        try:
            if self._h:
                lib().dgkr_field_destroy(self._h)
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def encode(self, vals: Elems) -> bytes:
        """canonical LE bytes (field.hpp:159-167) of a sequence of ints, or
        pass-through of ready byte buffers"""
        if isinstance(vals, (bytes, bytearray, memoryview)):
            return bytes(vals)
        if isinstance(vals, np.ndarray):
            return vals.astype(np.uint8, copy=False).tobytes()
        w = self.width
        return b"".join(int(v).to_bytes(w, "little") for v in vals)

    def decode(self, b: bytes) -> List[int]:
        w = self.width
        return [int.from_bytes(b[i:i + w], "little") for i in range(0, len(b), w)]


def set_tuning(name: str, value: int) -> None:
    """Process-wide launch tuning (dgkr_set_tuning): "small_round_pairs",
    "tma_min_pairs" (0 disables the TMA-staged round kernel). Proof bytes never
    depend on it."""
    check(lib().dgkr_set_tuning(name.encode(), C.c_uint64(value)))


def get_tuning(name: str) -> int:
    v = C.c_uint64()
    check(lib().dgkr_get_tuning(name.encode(), C.byref(v)))
    return v.value


class Transcript:
    """dgkr::Transcript (transcript.hpp:17-130); host-side SHA-256 chain."""

    def __init__(self, field: Field, label: str, pre: Sequence[int] = ()):
        self.field = field
        self.t = Transcript_t()
        check(lib().dgkr_transcript_init(field.handle, label.encode(), C.byref(self.t)))
        for v in pre:
            self.absorb_u64(v)

    def absorb_bytes(self, data: bytes) -> None:
        check(lib().dgkr_transcript_absorb_bytes(self.field.handle, C.byref(self.t), C.c_char_p(bytes(data)),
                                                 C.c_size_t(len(data))))

    def absorb(self, v: int) -> None:
        b = self.field.encode([v])
        check(lib().dgkr_transcript_absorb_elems(self.field.handle, C.byref(self.t), C.c_char_p(b), C.c_size_t(1)))

    def absorb_elems(self, vals: Elems) -> None:
        b = self.field.encode(vals)
        check(lib().dgkr_transcript_absorb_elems(self.field.handle, C.byref(self.t), C.c_char_p(b),
                                                 C.c_size_t(len(b) // self.field.width)))

    def absorb_u64(self, v: int) -> None:
        check(lib().dgkr_transcript_absorb_u64(self.field.handle, C.byref(self.t), C.c_uint64(v)))

    def challenge(self) -> int:
        out = C.create_string_buffer(self.field.width)
        check(lib().dgkr_transcript_challenge(self.field.handle, C.byref(self.t), out))
        return int.from_bytes(out.raw, "little")

    def challenge_index(self, bound: int) -> int:
        out = C.c_uint64()
        check(lib().dgkr_transcript_challenge_index(self.field.handle, C.byref(self.t), C.c_uint64(bound),
                                                    C.byref(out)))
        return out.value

    @property
    def state(self) -> bytes:
        return bytes(self.t.state)

    @property
    def draws(self) -> int:
        return int(self.t.draws)


def sha256(data: bytes) -> bytes:
    out = C.create_string_buffer(32)
    check(lib().dgkr_sha256(C.c_char_p(bytes(data)), C.c_size_t(len(data)), out))
    return out.raw


class Context:
    """One CUDA device + stream + workspaces (dgkr_ctx)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib().dgkr_ctx_create(C.c_int(device), C.byref(h)))
        self._h = h
        self.device = device

    def __del__(self):
        try:
            if self._h:
                lib().dgkr_ctx_destroy(self._h)
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def set_profile(self, on: bool) -> None:
        check(lib().dgkr_ctx_set_profile(self._h, C.c_int(1 if on else 0)))

    def profile(self) -> dict:
        p = Profile_t()
        check(lib().dgkr_ctx_get_profile(self._h, C.byref(p)))
        return p.as_dict()

    def device_info(self) -> Tuple[int, int, int]:
        a, b, c = C.c_int(), C.c_int(), C.c_int()
        check(lib().dgkr_ctx_device_info(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value


def _out(cap: int):
    return C.create_string_buffer(max(1, cap)), C.c_size_t()


def prove_product_sum(ctx: Context, pairs: Sequence[Tuple[Elems, Elems]], tr: Transcript) -> bytes:
    """prove_product_sum (sumcheck.hpp:226-241) -> SumcheckProof::to_bytes."""
    f = tr.field
    tabs = [f.encode(x) for pair in pairs for x in pair]
    n = len(tabs[0]) // f.width if tabs else 0
    vars_ = max(0, n.bit_length() - 1)
    if tabs and any(len(t) != len(tabs[0]) for t in tabs):
        from ._lib import InvalidArgument

        raise InvalidArgument(1, "mixed table sizes in product sum")
    if n & (n - 1):
        from ._lib import InvalidArgument

        raise InvalidArgument(1, "table size must be 2^num_vars")
    data = b"".join(tabs)
    cap = 64 + (vars_ + 2) * 4 * f.width + 2 * len(pairs) * f.width + 64
    out, ln = _out(cap)
    check(lib().dgkr_prove_product_sum(ctx.handle, f.handle, C.c_size_t(len(pairs)), C.c_size_t(vars_),
                                       C.c_char_p(data), C.byref(tr.t), out, C.c_size_t(cap), C.byref(ln)))
    return out.raw[: ln.value]


def prove_layer_sum(ctx: Context, side_vars: int, slot_tables: Sequence[Elems], wires, claimed: int,
                    tr: Transcript):
    """prove_layer_sum (sumcheck.hpp:342-448). wires: objects with is_mul,
    weight, x_slot, y_slot, x_index, y_index. Returns (proof bytes, x_point,
    y_point)."""
    f = tr.field
    meta = np.array([(int(w.is_mul), w.x_slot, w.y_slot) for w in wires], dtype=np.uint32).reshape(-1, 3)
    idx = np.array([(w.x_index, w.y_index) for w in wires], dtype=np.uint64).reshape(-1, 2)
    weights = f.encode([w.weight for w in wires])
    tables = b"".join(f.encode(t) for t in slot_tables)
    cap = 64 + (2 * side_vars + 2) * 4 * f.width + 2 * len(slot_tables) * f.width + 64
    out, ln = _out(cap)
    xp = C.create_string_buffer(max(1, side_vars * f.width))
    yp = C.create_string_buffer(max(1, side_vars * f.width))
    check(lib().dgkr_prove_layer_sum(ctx.handle, f.handle, C.c_size_t(side_vars), C.c_size_t(len(slot_tables)),
                                     C.c_char_p(tables), C.c_size_t(len(wires)), _buf(meta), _buf(idx),
                                     C.c_char_p(weights), C.c_char_p(f.encode([claimed])), C.byref(tr.t), out,
                                     C.c_size_t(cap), C.byref(ln), xp, yp))
    return out.raw[: ln.value], f.decode(xp.raw[: side_vars * f.width]), f.decode(yp.raw[: side_vars * f.width])


class Circuit:
    """Device-resident GeneralCircuit (circuit.hpp:63) in the flat layout of
    include/dgkr_b200.h; n_copies > 1 replicates it data-parallel (Sisu)."""

    def __init__(self, ctx: Context, input_size: int, layer_gate_start, gate_nested_start, nested,
                 min_padded=None, n_copies: int = 1):
        self.ctx = ctx
        self.input_size = int(input_size)
        self.n_copies = int(n_copies)
        lgs = np.ascontiguousarray(layer_gate_start, dtype=np.uint64)
        gns = np.ascontiguousarray(gate_nested_start, dtype=np.uint64)
        nst = np.ascontiguousarray(nested, dtype=np.uint32).reshape(-1, 5)
        self.depth = len(lgs) - 1
        mp = None if min_padded is None else np.ascontiguousarray(min_padded, dtype=np.uint64)
        h = C.c_void_p()
        check(lib().dgkr_circuit_create(ctx.handle, C.c_uint32(self.input_size), C.c_uint32(self.depth), _buf(lgs),
                                        _buf(gns), _buf(nst) if len(nst) else C.c_void_p(None),
                                        _buf(mp) if mp is not None else C.c_void_p(None),
                                        C.c_uint32(self.n_copies), C.byref(h)))
        self._h = h
        self.n_gates = int(lgs[-1]) * self.n_copies
        self.output_size = int(lib().dgkr_circuit_output_size(h))

    def save(self, path: str) -> None:
        """binary CSR circuit file (dgkr_circuit_save; layout in include/dgkr_b200.h)"""
        check(lib().dgkr_circuit_save(self._h, str(path).encode()))

    @staticmethod
    def load(ctx: Context, path: str, n_copies: int = 0) -> "Circuit":
        """dgkr_circuit_load: a binary CSR circuit file (n_copies = 0: the file's)"""
        import struct
        with open(path, "rb") as fh:
            head = fh.read(40)
        if len(head) < 40 or head[:8] != b"DGKRCSR1":
            raise InvalidArgument(1, f"{path}: not a DGKRCSR1 circuit file")
        insz, depth, ncp, _, n_gates, _ = struct.unpack("<4I2Q", head[8:40])
        self = Circuit.__new__(Circuit)
        self.ctx = ctx
        self.input_size, self.depth = int(insz), int(depth)
        self.n_copies = int(n_copies or ncp)
        h = C.c_void_p()
        check(lib().dgkr_circuit_load(ctx.handle, str(path).encode(), C.c_uint32(n_copies), C.byref(h)))
        self._h = h
        self.n_gates = int(n_gates) * self.n_copies
        self.output_size = int(lib().dgkr_circuit_output_size(h))
        return self

    @staticmethod
    def from_oracle(ctx: Context, c, n_copies: int = 1) -> "Circuit":
        lgs, gns, nested, minp = c.to_flat()
        return Circuit(ctx, c.input_size, lgs, gns, nested, minp, n_copies)

    def __del__(self):
        try:
            if self._h:
                lib().dgkr_circuit_destroy(self._h)
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def evaluate(self, field: Field, inputs: Elems) -> bytes:
        """padded output layer, canonical bytes (circuit.hpp:164-193)"""
        data = field.encode(inputs)
        cap = self.output_size * field.width
        out, ln = _out(cap)
        check(lib().dgkr_circuit_evaluate(self.ctx.handle, self._h, field.handle, _buf(np.frombuffer(data, np.uint8)),
                                          out, C.c_size_t(cap), C.byref(ln)))
        return out.raw[: ln.value]

    def proof_bound(self, field: Field) -> int:
        return int(lib().dgkr_gkr_proof_bound(self._h, field.handle))


def gkr_prove(ctx: Context, circuit: Circuit, inputs: Elems, tr: Transcript, out_buf=None) -> bytes:
    """gkr_prove (gkr.hpp:182-244) -> GkrProof bytes (layout in dgkr_b200.h)."""
    f = tr.field
    data = inputs if isinstance(inputs, np.ndarray) else np.frombuffer(f.encode(inputs), np.uint8)
    cap = circuit.proof_bound(f)
    if out_buf is None or len(out_buf) < cap:
        out_buf = C.create_string_buffer(cap)
    ln = C.c_size_t()
    check(lib().dgkr_gkr_prove(ctx.handle, circuit.handle, f.handle, _buf(data), C.byref(tr.t), out_buf,
                               C.c_size_t(cap), C.byref(ln)))
    return out_buf.raw[: ln.value]


def gkr_verify(circuit: Circuit, proof: bytes, tr: Transcript, outputs: Optional[Elems] = None,
               inputs: Optional[Elems] = None) -> bool:
    """gkr_verify (gkr.hpp:253-311) on the host; with `inputs`, also
    check_input_claims (:314-325). `outputs`: the claimed output statement."""
    f = tr.field
    ob = f.encode(outputs) if outputs is not None else None
    ib = None
    if inputs is not None:
        ib = inputs.tobytes() if isinstance(inputs, np.ndarray) else f.encode(inputs)
    acc = C.c_int()
    check(lib().dgkr_gkr_verify(circuit.handle, f.handle, C.c_char_p(ob) if ob is not None else None,
                                C.c_size_t(len(ob) // f.width if ob is not None else 0),
                                C.c_char_p(ib) if ib is not None else None, C.c_char_p(bytes(proof)),
                                C.c_size_t(len(proof)), C.byref(tr.t), C.byref(acc)))
    return bool(acc.value)


def gkr_input_claims(circuit: Circuit, proof: bytes, tr: Transcript):
    """(accept, claims) with claims = [([(point, weight), ...], value)] of the
    input layer (dgkr_gkr_input_claims)"""
    f = tr.field
    w = f.width
    cap = 4096 + 8 * len(proof)
    out, ln = _out(cap)
    acc = C.c_int()
    check(lib().dgkr_gkr_input_claims(circuit.handle, f.handle, C.c_char_p(bytes(proof)), C.c_size_t(len(proof)),
                                      C.byref(tr.t), C.byref(acc), out, C.c_size_t(cap), C.byref(ln)))
    raw = out.raw[: ln.value]
    pos = 0

    def u32():
        nonlocal pos
        v = int.from_bytes(raw[pos:pos + 4], "little")
        pos += 4
        return v

    def elem():
        nonlocal pos
        v = int.from_bytes(raw[pos:pos + w], "little")
        pos += w
        return v

    claims = []
    for _ in range(u32()):
        terms = []
        for _ in range(u32()):
            nv = u32()
            point = [elem() for _ in range(nv)]
            terms.append((point, elem()))
        claims.append((terms, elem()))
    return bool(acc.value), claims


def gkr_prove_batch(ctx: Context, circuit: Circuit, inputs: Optional[Sequence[Elems]], trs: Sequence[Transcript],
                    out_bufs=None) -> List[bytes]:
    """n independent gkr_prove calls run concurrently (one lane = stream +
    workspace + host thread per proof); inputs=None proves the inputs loaded
    per lane with load_inputs_lane. Transcripts are advanced in place."""
    n = len(trs)
    f = trs[0].field
    cap = circuit.proof_bound(f)
    if out_bufs is None:
        out_bufs = [np.empty(cap, dtype=np.uint8) for _ in range(n)]
    keep = []
    in_ptrs = None
    if inputs is not None:
        arrs = [x if isinstance(x, np.ndarray) else np.frombuffer(f.encode(x), np.uint8) for x in inputs]
        keep.extend(arrs)
        in_ptrs = (C.c_void_p * n)(*[a.ctypes.data for a in arrs])
    tarr = (Transcript_t * n)()
    for i, t in enumerate(trs):
        tarr[i] = t.t
    outs = (C.c_void_p * n)(*[b.ctypes.data for b in out_bufs])
    caps = (C.c_size_t * n)(*[len(b) for b in out_bufs])
    lens = (C.c_size_t * n)()
    check(lib().dgkr_gkr_prove_batch(ctx.handle, circuit.handle, f.handle, C.c_size_t(n), in_ptrs, tarr, outs, caps,
                                     lens))
    for i, t in enumerate(trs):
        t.t = tarr[i]
    return [out_bufs[i][: lens[i]].tobytes() for i in range(n)]


def ntt(ctx: Context, field: Field, data: Elems, inverse: bool = False) -> List[int]:
    """dgkr_ntt: natural-order NTT of 2^k elements (inverse: w^-1, 1/N)."""
    b = field.encode(data)
    n = len(b) // field.width
    out = C.create_string_buffer(len(b))
    check(lib().dgkr_ntt(ctx.handle, field.handle, C.c_char_p(b), C.c_uint(n.bit_length() - 1),
                         C.c_int(1 if inverse else 0), out))
    return field.decode(out.raw)


def rs_encode(ctx: Context, field: Field, coeffs: Elems, blowup_log: int) -> List[int]:
    """dgkr_rs_encode: f(g w_N^i), N = n << blowup_log."""
    b = field.encode(coeffs)
    n = len(b) // field.width
    out = C.create_string_buffer((n << blowup_log) * field.width)
    check(lib().dgkr_rs_encode(ctx.handle, field.handle, C.c_char_p(b), C.c_size_t(n), C.c_uint(blowup_log), out))
    return field.decode(out.raw)


def fri_prove(ctx: Context, field: Field, coeffs: Elems, blowup_log: int, final_log: int, queries: int,
              tr: Transcript) -> bytes:
    """dgkr_fri_prove (proof layout in include/dgkr_b200.h)."""
    b = field.encode(coeffs)
    n = len(b) // field.width
    log_n0 = n.bit_length() - 1 + blowup_log
    L = max(log_n0 - final_log, 0)
    H = (1 << log_n0) // 2
    q = min(queries, H) if L else 0
    cap = 64 + L * 32 + (1 << final_log) * field.width + q * (4 + L * (2 * field.width + 2 * 32 * log_n0))
    out = C.create_string_buffer(cap)
    ln = C.c_size_t()
    check(lib().dgkr_fri_prove(ctx.handle, field.handle, C.c_char_p(b), C.c_size_t(n), C.c_uint(blowup_log),
                               C.c_uint(final_log), C.c_size_t(queries), C.byref(tr.t), out, C.c_size_t(cap),
                               C.byref(ln)))
    return out.raw[: ln.value]


def _fri_cap(field: Field, n: int, blowup_log: int, final_log: int, queries: int, world: int) -> int:
    log_n0 = n.bit_length() - 1 + blowup_log
    L = max(log_n0 - final_log, 0)
    H = (1 << log_n0) // 2
    q = min(queries, H) if L else 0
    return (64 + world * (L * 32 + (1 << final_log) * field.width)
            + q * (4 + L * (2 * field.width + 2 * 32 * log_n0)))


def fri_prove_dist(ctx: Context, comm: "Comm", field: Field, coeffs: Elems, blowup_log: int, final_log: int,
                   queries: int, tr: Transcript) -> bytes:
    """dgkr_fri_prove_dist: this rank's chunk of a distributed FRI (proof
    layout in include/dgkr_b200.h); every rank calls it collectively."""
    b = field.encode(coeffs)
    n = len(b) // field.width
    cap = _fri_cap(field, n, blowup_log, final_log, queries, comm.world)
    out = C.create_string_buffer(cap)
    ln = C.c_size_t()
    check(lib().dgkr_fri_prove_dist(ctx.handle, comm.handle, field.handle, C.c_char_p(b), C.c_size_t(n),
                                    C.c_uint(blowup_log), C.c_uint(final_log), C.c_size_t(queries), C.byref(tr.t),
                                    out, C.c_size_t(cap), C.byref(ln)))
    return out.raw[: ln.value]


def fri_prove_dist_emulated(ctx: Context, field: Field, chunks: Sequence[Elems], blowup_log: int, final_log: int,
                            queries: int, tr: Transcript) -> List[bytes]:
    """dgkr_fri_prove_dist_emulated: len(chunks) ranks as threads on lanes of
    one device; returns one proof per rank (tr ends in the shared state)."""
    world = len(chunks)
    bs = [field.encode(c) for c in chunks]
    if len({len(x) for x in bs}) != 1:
        raise ValueError("all ranks need chunks of the same size")
    n = len(bs[0]) // field.width
    cap = _fri_cap(field, n, blowup_log, final_log, queries, world)
    outs = [C.create_string_buffer(cap) for _ in range(world)]
    ptrs = (C.c_void_p * world)(*[C.cast(o, C.c_void_p) for o in outs])
    caps = (C.c_size_t * world)(*([cap] * world))
    lens = (C.c_size_t * world)()
    ins = (C.c_char_p * world)(*bs)
    check(lib().dgkr_fri_prove_dist_emulated(ctx.handle, field.handle, C.c_int(world), ins,
                                             C.c_size_t(n), C.c_uint(blowup_log), C.c_uint(final_log),
                                             C.c_size_t(queries), C.byref(tr.t), ptrs, caps, lens))
    return [outs[r].raw[: lens[r]] for r in range(world)]


def gkr_prove_stream(ctx: Context, circuit: Circuit, n: int, lanes: int, field: Field, label: str = "stream",
                     inputs: Optional[Sequence[Elems]] = None, out_bufs=None):
    """n proofs over `lanes` lanes as a work queue (dgkr_gkr_prove_stream).
    inputs=None: proof i runs on lane i mod lanes and proves the inputs loaded
    there (static assignment; host inputs use a work queue). Returns
    (proofs, transcripts, per-lane profile dicts)."""
    from ._lib import Profile_t

    cap = circuit.proof_bound(field)
    if out_bufs is None:
        out_bufs = [np.empty(cap, dtype=np.uint8) for _ in range(n)]
    keep = []
    in_ptrs = None
    if inputs is not None:
        arrs = [x if isinstance(x, np.ndarray) else np.frombuffer(field.encode(x), np.uint8) for x in inputs]
        keep.extend(arrs)
        in_ptrs = (C.c_void_p * n)(*[a.ctypes.data for a in arrs])
    tarr = (Transcript_t * n)()
    for i in range(n):
        tarr[i] = Transcript(field, label).t
    outs = (C.c_void_p * n)(*[out_bufs[i].ctypes.data for i in range(n)])
    caps = (C.c_size_t * n)(*[len(out_bufs[i]) for i in range(n)])
    lens = (C.c_size_t * n)()
    nl = min(n, lanes)
    profs = (Profile_t * nl)()
    check(lib().dgkr_gkr_prove_stream(ctx.handle, circuit.handle, field.handle, C.c_size_t(n), C.c_size_t(lanes),
                                      in_ptrs, tarr, outs, caps, lens, profs))
    return ([out_bufs[i][: lens[i]] for i in range(n)], [bytes(tarr[i].state) for i in range(n)],
            [profs[i].as_dict() for i in range(nl)])


def gkr_prove_dist_emulated(ctx: Context, circuit: Circuit, world: int, inputs_all: Elems, tr: Transcript) -> bytes:
    """The multi-GPU data-parallel prover with `world` ranks emulated as host
    threads on one GPU (circuit = one rank's share, n_copies = total/world).
    Returns the proof, which every rank must have produced identically."""
    f = tr.field
    data = inputs_all if isinstance(inputs_all, np.ndarray) else np.frombuffer(f.encode(inputs_all), np.uint8)
    cap = circuit.proof_bound(f) + (world - 1) * circuit.output_size * f.width + 4096 * world
    out = np.empty(cap, dtype=np.uint8)
    ln = C.c_size_t()
    check(lib().dgkr_gkr_prove_dist_emulated(ctx.handle, circuit.handle, f.handle, C.c_int(world), _buf(data),
                                             C.byref(tr.t), _buf(out), C.c_size_t(cap), C.byref(ln)))
    return out[: ln.value].tobytes()


class Comm:
    """NCCL communicator for one rank (dgkr_comm); uid from nccl_unique_id()."""

    def __init__(self, ctx: Context, uid: bytes, rank: int, world: int):
        h = C.c_void_p()
        check(lib().dgkr_comm_create_nccl(ctx.handle, C.c_char_p(bytes(uid)), C.c_int(rank), C.c_int(world),
                                          C.byref(h)))
        self._h = h
        self.rank, self.world = rank, world

    @staticmethod
    def nccl_unique_id() -> bytes:
        out = C.create_string_buffer(128)
        check(lib().dgkr_comm_nccl_unique_id(out))
        return out.raw

    @property
    def handle(self):
        return self._h

    def __del__(self):
        try:
            if self._h:
                lib().dgkr_comm_destroy(self._h)
        except Exception:
            pass


def gkr_prove_dist(ctx: Context, comm: Comm, circuit: Circuit, inputs: Optional[Elems], tr: Transcript,
                   out_buf=None) -> bytes:
    """One rank of the multi-GPU prover (inputs = this rank's share, or None
    for inputs loaded with load_inputs_lane(..., lane=0, ...))."""
    f = tr.field
    cap = circuit.proof_bound(f) + (comm.world - 1) * circuit.output_size * f.width + 4096 * comm.world
    if out_buf is None or len(out_buf) < cap:
        out_buf = np.empty(cap, dtype=np.uint8)
    data = None if inputs is None else (inputs if isinstance(inputs, np.ndarray) else
                                        np.frombuffer(f.encode(inputs), np.uint8))
    ln = C.c_size_t()
    check(lib().dgkr_gkr_prove_dist(ctx.handle, comm.handle, circuit.handle, f.handle,
                                    _buf(data) if data is not None else C.c_void_p(None), C.byref(tr.t),
                                    _buf(out_buf), C.c_size_t(cap), C.byref(ln)))
    return out_buf[: ln.value].tobytes()


def load_inputs_lane(ctx: Context, circuit: Circuit, field: Field, lane: int, inputs: Elems) -> None:
    data = inputs if isinstance(inputs, np.ndarray) else np.frombuffer(field.encode(inputs), np.uint8)
    check(lib().dgkr_circuit_load_inputs_lane(ctx.handle, circuit.handle, field.handle, C.c_int(lane), _buf(data)))


def pcs_commit(ctx: Context, field: Field, rows: Sequence[Elems]) -> bytes:
    """pcs::commit (pcs.hpp:105-113) -> 32-byte root"""
    if not rows:
        raise InvalidArgument(1, "matrix needs at least one row")  # pcs.hpp:35-37
    r0 = rows[0]
    if all(isinstance(r, np.ndarray) and r.dtype == np.uint8 for r in rows):
        # byte rows: one contiguous buffer without the bytes round trip
        sizes = {r.size for r in rows}
        if len(sizes) != 1 or r0.size % field.width:
            raise InvalidArgument(1, "ragged evaluation matrix")  # pcs.hpp:38-43
        data = np.ascontiguousarray(r0 if len(rows) == 1 else np.concatenate([r.reshape(-1) for r in rows]))
        cols = r0.size // field.width
    else:
        enc = [field.encode(r) for r in rows]
        if len({len(e) for e in enc}) != 1 or len(enc[0]) % field.width:
            raise InvalidArgument(1, "ragged evaluation matrix")
        data = np.frombuffer(b"".join(enc), np.uint8)
        cols = len(enc[0]) // field.width
    root = C.create_string_buffer(32)
    check(lib().dgkr_pcs_commit(ctx.handle, field.handle, C.c_size_t(len(rows)), C.c_size_t(cols),
                                _buf(data), root))
    return root.raw


def pcs_open(ctx: Context, field: Field, rows: Sequence[Elems], r: Sequence[int], tr: Transcript,
             spot_checks: int = 32) -> bytes:
    """pcs::open (pcs.hpp:212-254) -> Opening::to_bytes"""
    enc = [field.encode(x) for x in rows]
    if not enc or len({len(e) for e in enc}) != 1 or len(enc[0]) % field.width:
        raise InvalidArgument(1, "ragged evaluation matrix")
    data = b"".join(enc)
    M = len(rows)
    cols = len(enc[0]) // field.width
    depth = max(0, (cols - 1).bit_length())
    cap = 64 + (len(r) + 2 + M + cols) * field.width + min(spot_checks, cols) * (4 + M * field.width + 32 * depth) + 64
    out = np.empty(cap, dtype=np.uint8)  # not zero-filled: the opening overwrites what it returns
    ln = C.c_size_t()
    check(lib().dgkr_pcs_open(ctx.handle, field.handle, C.c_size_t(M), C.c_size_t(cols), C.c_char_p(data),
                              C.c_char_p(field.encode(r)), C.c_size_t(len(r)), C.c_size_t(spot_checks),
                              C.byref(tr.t), out.ctypes.data_as(C.c_void_p), C.c_size_t(cap), C.byref(ln)))
    return out[: ln.value].tobytes()


def dist_sumcheck(ctx: Context, n_workers: int, pairs, tr: Transcript):
    """shard_pairs + dist_sumcheck (cluster.hpp:190-320) -> (proof bytes,
    TrafficStats json)"""
    f = tr.field
    tabs = [f.encode(x) for pair in pairs for x in pair]
    n = len(tabs[0]) // f.width
    vars_ = max(0, n.bit_length() - 1)
    cap = 64 + (vars_ + 2) * 4 * f.width + 2 * len(pairs) * f.width + 64
    out, ln = _out(cap)
    js = C.create_string_buffer(4096)
    check(lib().dgkr_dist_sumcheck(ctx.handle, f.handle, C.c_size_t(n_workers), C.c_size_t(len(pairs)),
                                   C.c_size_t(vars_), C.c_char_p(b"".join(tabs)), C.byref(tr.t), out, C.c_size_t(cap),
                                   C.byref(ln), js, C.c_size_t(4096)))
    return out.raw[: ln.value], js.value.decode()


def dist_sumcheck_emulated(ctx: Context, world: int, pairs, tr: Transcript) -> bytes:
    """dist_sumcheck on `world` ranks (host threads on lanes of one GPU, each
    holding its shard_pairs slice, cluster.hpp:190-217) exchanging round sums
    through a communicator (dgkr_dist_sumcheck_emulated) -> proof bytes"""
    f = tr.field
    tabs = [f.encode(x) for pair in pairs for x in pair]
    n = len(tabs[0]) // f.width
    vars_ = max(0, n.bit_length() - 1)
    cap = 64 + (vars_ + 2) * 4 * f.width + 2 * len(pairs) * f.width + 64
    out, ln = _out(cap)
    check(lib().dgkr_dist_sumcheck_emulated(ctx.handle, f.handle, C.c_int(world), C.c_size_t(len(pairs)),
                                            C.c_size_t(vars_), C.c_char_p(b"".join(tabs)), C.byref(tr.t), out,
                                            C.c_size_t(cap), C.byref(ln)))
    return out.raw[: ln.value]


def distpc(ctx, field: Field, rows: Sequence[Elems], r: Sequence[int], spot_checks: int = 32,
           n_clusters: int = 0):
    """DistPc::commit + open (cluster.hpp:336-412) -> (roots, cluster opening
    bytes, combined value, TrafficStats json). ctx: a Context, or a list of
    Contexts (one per device) the clusters are spread over (dgkr_distpc_multi)."""
    N = len(rows)
    data = b"".join(field.encode(x) for x in rows)
    cols = len(field.encode(rows[0])) // field.width
    row_vars = max(0, cols.bit_length() - 1)
    roots = C.create_string_buffer(32 * N)
    nr = C.c_size_t()
    cap = N * (64 + (len(r) + 2 + N + cols) * field.width + min(spot_checks, cols) * (4 + N * field.width + 32 * 64)) + 1024
    out, ln = _out(cap)
    comb = C.create_string_buffer(field.width)
    js = C.create_string_buffer(8192)
    ctxs = list(ctx) if isinstance(ctx, (list, tuple)) else [ctx]
    handles = (C.c_void_p * len(ctxs))(*[c.handle.value for c in ctxs])
    check(lib().dgkr_distpc_multi(handles, C.c_size_t(len(ctxs)), field.handle, C.c_size_t(N), C.c_size_t(n_clusters),
                                  C.c_size_t(row_vars), C.c_char_p(data), C.c_char_p(field.encode(r)),
                                  C.c_size_t(len(r)), C.c_size_t(spot_checks), roots, C.byref(nr), out, C.c_size_t(cap),
                                  C.byref(ln), comb, js, C.c_size_t(8192)))
    raw = out.raw[: ln.value]
    ops = []
    pos = 0
    while pos < len(raw):
        n = int.from_bytes(raw[pos:pos + 4], "little")
        ops.append(raw[pos + 4:pos + 4 + n])
        pos += 4 + n
    return ([roots.raw[32 * i:32 * (i + 1)] for i in range(nr.value)], ops, int.from_bytes(comb.raw, "little"),
            js.value.decode())


# ---------------------------------------------------------------------------
# distinct.hpp (config C4): associative array hash over validator indexes
# ---------------------------------------------------------------------------
def distinct_ah(ctx: Context, field: Field, items: Elems) -> int:
    """distinct::ah (distinct.hpp:37-44): sum_i F(e_i), F = 3 rounds of (r + e + 2^32-1)^3"""
    b = field.encode(items)
    out = C.create_string_buffer(field.width)
    check(lib().dgkr_distinct_ah(ctx.handle, field.handle, C.c_char_p(b), C.c_size_t(len(b) // field.width), out))
    return int.from_bytes(out.raw, "little")


def pairwise_distinct_check(ctx: Context, field: Field, a: Elems, a_sorted: Elems) -> bool:
    """distinct::pairwise_distinct_check (distinct.hpp:53-68)"""
    ba, bs = field.encode(a), field.encode(a_sorted)
    ok = C.c_int()
    check(lib().dgkr_distinct_check(ctx.handle, field.handle, C.c_char_p(ba), C.c_size_t(len(ba) // field.width),
                                    C.c_char_p(bs), C.c_size_t(len(bs) // field.width), C.byref(ok)))
    return bool(ok.value)


def chain_update(ctx: Context, field: Field, h: int, n_max: int, items: Elems) -> int:
    """distinct::chain_update (distinct.hpp:82-92): h + AH(items); OutOfRange if an item > n_max"""
    b = field.encode(items)
    out = C.create_string_buffer(field.width)
    check(lib().dgkr_distinct_chain_update(ctx.handle, field.handle, C.c_char_p(field.encode([h])),
                                           C.c_uint64(n_max), C.c_char_p(b), C.c_size_t(len(b) // field.width), out))
    return int.from_bytes(out.raw, "little")


def bitchange_experiment(ctx: Context, field: Field, count: int) -> Tuple[List[int], List[float]]:
    """distinct::bitchange_experiment (distinct.hpp:112-145): per-bit set counts
    and probabilities of canonical F(x+1) - F(x), x = 1..count"""
    bits = field.bits
    counts = (C.c_uint64 * max(bits, 1))()
    check(lib().dgkr_distinct_bitchange(ctx.handle, field.handle, C.c_size_t(count), counts))
    cs = list(counts[:bits])
    return cs, [c / count for c in cs]


def bitchange_csv(probabilities: Sequence[float]) -> str:
    """BitChangeResult::to_csv (distinct.hpp:98-106)"""
    return "index,bit_change\n" + "".join(f"{i},{p:g}\n" for i, p in enumerate(probabilities))


# ---------------------------------------------------------------------------
# beacon.hpp (config C3): validator tree root, membership paths, batched verify
# ---------------------------------------------------------------------------
def _u64_arr(vals) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(vals, dtype=np.uint64))


def beacon_root(ctx: Context, records: bytes, depth: int) -> bytes:
    """BeaconTree(validators, depth).root() (beacon.hpp:102-132); records =
    n x 64-byte ValidatorRecord::encode()"""
    out = C.create_string_buffer(32)
    check(lib().dgkr_beacon_root(ctx.handle, C.c_char_p(bytes(records)), C.c_size_t(len(records) // 64),
                                 C.c_uint(depth), out))
    return out.raw


def beacon_prove(ctx: Context, records: bytes, depth: int, indices) -> Tuple[bytes, bytes, int]:
    """prove_membership for each index (beacon.hpp:136-149) -> (leaves m x 32,
    siblings m x a x 32, a)"""
    idx = _u64_arr(indices)
    m = len(idx)
    n = len(records) // 64
    a_max = max(1, (max(n, 1) - 1).bit_length())
    leaves = C.create_string_buffer(32 * max(m, 1))
    sib = C.create_string_buffer(32 * max(m * a_max, 1))
    a = C.c_uint()
    check(lib().dgkr_beacon_prove(ctx.handle, C.c_char_p(bytes(records)), C.c_size_t(n), C.c_uint(depth),
                                  idx.ctypes.data_as(C.c_void_p), C.c_size_t(m), leaves, sib, C.byref(a)))
    return leaves.raw[: 32 * m], sib.raw[: 32 * m * a.value], a.value


def beacon_verify(ctx: Context, root: bytes, records: bytes, leaves: bytes, siblings: bytes, indices, depth: int,
                  active_log2: int) -> np.ndarray:
    """batched BeaconTree::verify_membership (beacon.hpp:151-174) -> uint8 ok per path"""
    idx = _u64_arr(indices)
    m = len(idx)
    ok = np.zeros(max(m, 1), dtype=np.uint8)
    check(lib().dgkr_beacon_verify(ctx.handle, C.c_char_p(bytes(root)), C.c_char_p(bytes(records)),
                                   C.c_char_p(bytes(leaves)), C.c_char_p(bytes(siblings)),
                                   idx.ctypes.data_as(C.c_void_p), C.c_size_t(m), C.c_uint(depth),
                                   C.c_uint(active_log2), ok.ctypes.data_as(C.c_void_p)))
    return ok[:m]
