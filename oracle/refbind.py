"""ORACLE TEST INFRASTRUCTURE — ctypes binding of oracle/_ref/libdgkr_ref.so.

The library is the UNMODIFIED reference prover (``/root/reference/proj/include``)
compiled against ``oracle/shim`` by ``oracle/Makefile``. Only tests, smoke()
and bench.py's CPU-baseline leg use this module, as the checker / baseline.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from typing import Optional, Sequence

import numpy as np

from . import dgkr_oracle as O

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libdgkr_ref.so")

_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} not built (run `make -C oracle`)")
        _lib = C.CDLL(LIB_PATH)
        _lib.ref_last_error.restype = C.c_char_p
    return _lib


class RefError(RuntimeError):
    pass


def _check(rc: int):
    if rc != 0:
        raise RefError(f"reference error {rc}: {lib().ref_last_error().decode()}")


def _mod(fld: O.Field):
    b = fld.modulus_bytes_min()
    return C.c_char_p(b), C.c_size_t(len(b))


def _pre(pre: Sequence[int]):
    arr = (C.c_uint64 * max(1, len(pre)))(*pre) if pre else (C.c_uint64 * 1)(0)
    return arr, C.c_size_t(len(pre))


def _u8(b: bytes):
    return C.c_char_p(bytes(b))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def transcript_run(fld, label, pre, elems: Sequence[int], n_chal: int, n_idx: int = 0, idx_bound: int = 1):
    w = fld.width
    chal = C.create_string_buffer(max(1, n_chal * w))
    idx = (C.c_uint64 * max(1, n_idx))()
    st = C.create_string_buffer(32)
    pa, pn = _pre(pre)
    _check(lib().ref_transcript_run(*_mod(fld), label.encode(), pa, pn, _u8(fld.elems_to_bytes(elems)),
                                    C.c_size_t(len(elems)), C.c_size_t(n_chal), chal, C.c_size_t(n_idx),
                                    C.c_uint64(idx_bound), idx, st))
    return fld.elems_from_bytes(chal.raw[: n_chal * w]), list(idx)[:n_idx], st.raw


def prove_product_sum(fld, label, pre, pairs, cap: Optional[int] = None):
    n_pairs = len(pairs)
    vars_ = len(pairs[0][0]).bit_length() - 1
    tables = b"".join(fld.elems_to_bytes(f) + fld.elems_to_bytes(g) for f, g in pairs)
    cap = cap or (64 + (vars_ + 2) * 4 * fld.width + 2 * n_pairs * fld.width + 64)
    out = C.create_string_buffer(cap)
    ln = C.c_size_t()
    st = C.create_string_buffer(32)
    pa, pn = _pre(pre)
    _check(lib().ref_prove_product_sum(*_mod(fld), label.encode(), pa, pn, C.c_size_t(n_pairs),
                                       C.c_size_t(vars_), _u8(tables), out, C.c_size_t(cap), C.byref(ln), st))
    return out.raw[: ln.value], st.raw


def prove_layer_sum(fld, label, pre, side_vars, slot_tables, wires: Sequence[O.LayerWire], claimed):
    meta = np.array([(int(w.is_mul), w.x_slot, w.y_slot) for w in wires], dtype=np.uint32).reshape(-1, 3)
    idx = np.array([(w.x_index, w.y_index) for w in wires], dtype=np.uint64).reshape(-1, 2)
    weights = fld.elems_to_bytes([w.weight for w in wires])
    tables = b"".join(fld.elems_to_bytes(t) for t in slot_tables)
    cap = 64 + (2 * side_vars + 2) * 4 * fld.width + 2 * len(slot_tables) * fld.width + 64
    out = C.create_string_buffer(cap)
    ln = C.c_size_t()
    st = C.create_string_buffer(32)
    pa, pn = _pre(pre)
    _check(lib().ref_prove_layer_sum(*_mod(fld), label.encode(), pa, pn, C.c_size_t(side_vars),
                                     C.c_size_t(len(slot_tables)), _u8(tables), C.c_size_t(len(wires)),
                                     _ptr(meta), _ptr(idx), _u8(weights), _u8(fld.to_bytes(claimed)), out,
                                     C.c_size_t(cap), C.byref(ln), st))
    return out.raw[: ln.value], st.raw


def _flat_args(flat):
    lgs, gns, nested, minp = [np.ascontiguousarray(a) for a in flat]
    return (lgs, gns, nested, minp), (_ptr(lgs), _ptr(gns), _ptr(nested), _ptr(minp))


def gkr_prove(fld, label, pre, circuit: O.Circuit, inputs, flat=None):
    flat = flat if flat is not None else circuit.to_flat()
    keep, ptrs = _flat_args(flat)
    depth = len(keep[0]) - 1
    # generous capacity: outputs + per layer (alphas + 2*side rounds + finals)
    out_n = circuit.padded_size(depth)
    cap = 16 + out_n * fld.width + depth * (64 + 4 * fld.width * (2 * 64 + 2) + 2 * (depth + 1) * fld.width)
    out = C.create_string_buffer(cap)
    ln = C.c_size_t()
    st = C.create_string_buffer(32)
    pa, pn = _pre(pre)
    _check(lib().ref_gkr_prove(*_mod(fld), label.encode(), pa, pn, C.c_uint32(circuit.input_size),
                               C.c_uint32(depth), *ptrs, _u8(fld.elems_to_bytes(inputs)), out, C.c_size_t(cap),
                               C.byref(ln), st))
    return out.raw[: ln.value], st.raw


def gkr_verify(fld, label, pre, circuit: O.Circuit, inputs, proof: bytes, flat=None) -> bool:
    flat = flat if flat is not None else circuit.to_flat()
    keep, ptrs = _flat_args(flat)
    depth = len(keep[0]) - 1
    acc = C.c_int()
    pa, pn = _pre(pre)
    _check(lib().ref_gkr_verify(*_mod(fld), label.encode(), pa, pn, C.c_uint32(circuit.input_size),
                                C.c_uint32(depth), *ptrs, _u8(fld.elems_to_bytes(inputs)), _u8(proof),
                                C.c_size_t(len(proof)), C.byref(acc)))
    return bool(acc.value)


def random_general_circuit(seed, input_size, depth, max_gates, max_nested, mul_percent=50) -> O.Circuit:
    lgs = np.zeros(depth + 1, dtype=np.uint64)
    gns = np.zeros(depth * max_gates + 1, dtype=np.uint64)
    nested = np.zeros((depth * max_gates * max_nested, 5), dtype=np.uint32)
    ng = C.c_uint64()
    nn = C.c_uint64()
    _check(lib().ref_random_general_circuit(C.c_uint64(seed), C.c_size_t(input_size), C.c_size_t(depth),
                                            C.c_size_t(max_gates), C.c_size_t(max_nested), C.c_uint(mul_percent),
                                            _ptr(lgs), _ptr(gns), _ptr(nested), C.byref(ng), C.byref(nn)))
    return O.Circuit.from_flat(input_size, lgs, gns[: ng.value + 1], nested[: nn.value])


def pcs_commit(fld, rows) -> bytes:
    data = b"".join(fld.elems_to_bytes(r) for r in rows)
    root = C.create_string_buffer(32)
    _check(lib().ref_pcs_commit(*_mod(fld), C.c_size_t(len(rows)), C.c_size_t(len(rows[0])), _u8(data), root))
    return root.raw


def pcs_open(fld, label, pre, rows, r, q=32):
    data = b"".join(fld.elems_to_bytes(x) for x in rows)
    M, cols = len(rows), len(rows[0])
    depth = O.log2_exact(cols)
    cap = 64 + (len(r) + 2 + M + cols) * fld.width + min(q, cols) * (4 + M * fld.width + 32 * depth) + 64
    out = C.create_string_buffer(cap)
    ln = C.c_size_t()
    st = C.create_string_buffer(32)
    pa, pn = _pre(pre)
    _check(lib().ref_pcs_open(*_mod(fld), label.encode(), pa, pn, C.c_size_t(M), C.c_size_t(cols), _u8(data),
                              _u8(fld.elems_to_bytes(r)), C.c_size_t(len(r)), C.c_size_t(q), out, C.c_size_t(cap),
                              C.byref(ln), st))
    return out.raw[: ln.value], st.raw


def pcs_verify(fld, label, pre, rows_n, cols, root, r, opening: bytes, q=32) -> bool:
    acc = C.c_int()
    pa, pn = _pre(pre)
    _check(lib().ref_pcs_verify(*_mod(fld), label.encode(), pa, pn, C.c_size_t(rows_n), C.c_size_t(cols),
                                _u8(root), _u8(fld.elems_to_bytes(r)), C.c_size_t(len(r)), _u8(opening),
                                C.c_size_t(len(opening)), C.c_size_t(q), C.byref(acc)))
    return bool(acc.value)


def dist_sumcheck(fld, label, pre, n_workers, pairs):
    n_pairs = len(pairs)
    vars_ = len(pairs[0][0]).bit_length() - 1
    tables = b"".join(fld.elems_to_bytes(f) + fld.elems_to_bytes(g) for f, g in pairs)
    cap = 64 + (vars_ + 2) * 4 * fld.width + 2 * n_pairs * fld.width + 64
    out = C.create_string_buffer(cap)
    ln = C.c_size_t()
    st = C.create_string_buffer(32)
    js = C.create_string_buffer(4096)
    pa, pn = _pre(pre)
    _check(lib().ref_dist_sumcheck(*_mod(fld), label.encode(), pa, pn, C.c_size_t(n_workers), C.c_size_t(n_pairs),
                                   C.c_size_t(vars_), _u8(tables), out, C.c_size_t(cap), C.byref(ln), st, js,
                                   C.c_size_t(4096)))
    return out.raw[: ln.value], st.raw, js.value.decode()


def distpc(fld, rows, r, q=32, k=0):
    N = len(rows)
    row_vars = O.log2_exact(len(rows[0]))
    data = b"".join(fld.elems_to_bytes(x) for x in rows)
    roots = C.create_string_buffer(32 * N)
    nr = C.c_size_t()
    cols = len(rows[0])
    cap = N * (64 + (len(r) + 2 + N + cols * N) * fld.width + min(q, cols) * (4 + N * fld.width + 32 * 64)) + 1024
    out = C.create_string_buffer(cap)
    ln = C.c_size_t()
    comb = C.create_string_buffer(fld.width)
    js = C.create_string_buffer(8192)
    _check(lib().ref_distpc(*_mod(fld), C.c_size_t(N), C.c_size_t(k), C.c_size_t(row_vars), _u8(data),
                            _u8(fld.elems_to_bytes(r)), C.c_size_t(len(r)), C.c_size_t(q), roots, C.byref(nr), out,
                            C.c_size_t(cap), C.byref(ln), comb, js, C.c_size_t(8192)))
    raw = out.raw[: ln.value]
    ops = []
    pos = 0
    while pos < len(raw):
        n = int.from_bytes(raw[pos:pos + 4], "little")
        ops.append(raw[pos + 4:pos + 4 + n])
        pos += 4 + n
    return ([roots.raw[32 * i:32 * (i + 1)] for i in range(nr.value)], ops,
            int.from_bytes(comb.raw, "little"), js.value.decode())


def traffic_json_equal(a: str, b: str) -> bool:
    return json.loads(a) == json.loads(b) and a == b


# --- distinct.hpp (config C4) ------------------------------------------------
def distinct_ah(fld, items) -> int:
    out = C.create_string_buffer(fld.width)
    b = fld.elems_to_bytes(items) if not isinstance(items, (bytes, bytearray)) else bytes(items)
    n = len(b) // fld.width
    _check(lib().ref_distinct_ah(*_mod(fld), _u8(b), C.c_size_t(n), out))
    return fld.from_bytes(out.raw)


def distinct_check(fld, a, a_sorted) -> bool:
    ok = C.c_int()
    _check(lib().ref_distinct_check(*_mod(fld), _u8(fld.elems_to_bytes(a)), C.c_size_t(len(a)),
                                    _u8(fld.elems_to_bytes(a_sorted)), C.c_size_t(len(a_sorted)), C.byref(ok)))
    return bool(ok.value)


def distinct_chain_update(fld, h: int, n_max: int, items) -> int:
    out = C.create_string_buffer(fld.width)
    _check(lib().ref_distinct_chain_update(*_mod(fld), _u8(fld.to_bytes(h)), C.c_uint64(n_max),
                                           _u8(fld.elems_to_bytes(items)), C.c_size_t(len(items)), out))
    return fld.from_bytes(out.raw)


def distinct_bitchange(fld, count: int):
    counts = (C.c_uint64 * 512)()
    bits = C.c_size_t()
    _check(lib().ref_distinct_bitchange(*_mod(fld), C.c_size_t(count), counts, C.byref(bits)))
    return list(counts[: bits.value])


def circuit_json(circuit: O.Circuit, flat=None) -> str:
    """the reference's GeneralCircuit::to_json().dump() of a circuit"""
    flat = flat if flat is not None else circuit.to_flat()
    keep, ptrs = _flat_args(flat)
    depth = len(keep[0]) - 1
    cap = 256 + 128 * int(keep[1][-1] if len(keep[1]) else 0) + 64 * int(keep[0][-1])
    out = C.create_string_buffer(cap)
    ln = C.c_size_t()
    _check(lib().ref_circuit_json(C.c_uint32(circuit.input_size), C.c_uint32(depth), *ptrs[:3], out, C.c_size_t(cap),
                                  C.byref(ln)))
    return out.raw[: ln.value].decode()


# --- beacon.hpp (config C3) --------------------------------------------------
def beacon_gen(n: int, seed: int) -> bytes:
    out = C.create_string_buffer(64 * n)
    _check(lib().ref_beacon_gen(C.c_size_t(n), C.c_uint64(seed), out))
    return out.raw


def beacon_root(records: bytes, depth: int) -> bytes:
    out = C.create_string_buffer(32)
    _check(lib().ref_beacon_root(_u8(records), C.c_size_t(len(records) // 64), C.c_size_t(depth), out))
    return out.raw


def beacon_prove(records: bytes, depth: int, index: int):
    leaf = C.create_string_buffer(32)
    sib = C.create_string_buffer(32 * 64)
    a = C.c_size_t()
    _check(lib().ref_beacon_prove(_u8(records), C.c_size_t(len(records) // 64), C.c_size_t(depth), C.c_uint64(index),
                                  leaf, sib, C.byref(a)))
    return leaf.raw, sib.raw[: 32 * a.value], a.value


def beacon_verify(root: bytes, record: bytes, leaf: bytes, siblings: bytes, active_log2: int, index: int,
                  depth: int) -> bool:
    ok = C.c_int()
    _check(lib().ref_beacon_verify(_u8(root), _u8(record), _u8(leaf), _u8(siblings), C.c_size_t(active_log2),
                                   C.c_uint64(index), C.c_size_t(depth), C.byref(ok)))
    return bool(ok.value)
