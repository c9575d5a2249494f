"""Loader for the in-tree CUDA library ``libdgkr_b200.so`` (C ABI in
``include/dgkr_b200.h``). There is no fallback: if the shared object is
missing or fails to load, importing the prover raises."""
from __future__ import annotations

import ctypes as C
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
# DGKR_LIB: an alternative in-tree build of the same library (A/B experiments of
# compile-time variants, e.g. build/variants/); the default is the product build
LIB_PATH = os.environ.get("DGKR_LIB") or os.path.join(_HERE, "libdgkr_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "dgkr_b200.h")

_lib = None

STATUS = {
    0: "DGKR_OK",
    1: "DGKR_INVALID_ARGUMENT",
    2: "DGKR_LOGIC_ERROR",
    3: "DGKR_DOMAIN_ERROR",
    4: "DGKR_OUT_OF_RANGE",
    5: "DGKR_CUDA_ERROR",
    6: "DGKR_UNSUPPORTED",
    7: "DGKR_CAPACITY",
    8: "DGKR_COMM_ERROR",
}


class DgkrError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


# Exception types mirror the reference's (SURVEY.md §8(b) "Errors").
class InvalidArgument(DgkrError, ValueError):
    pass


class LogicError(DgkrError):
    pass


class DomainError(DgkrError, ArithmeticError):
    pass


class OutOfRange(DgkrError, IndexError):
    pass


class CudaError(DgkrError):
    pass


_EXC = {1: InvalidArgument, 2: LogicError, 3: DomainError, 4: OutOfRange, 5: CudaError}


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is not built; run `make -C paper_2404_10404_b200/csrc` "
                "(or __graft_entry__.build()). There is no CPU fallback.")
        _lib = C.CDLL(LIB_PATH)
        _lib.dgkr_last_error.restype = C.c_char_p
        _lib.dgkr_field_width.restype = C.c_size_t
        _lib.dgkr_field_bits.restype = C.c_size_t
        _lib.dgkr_circuit_output_size.restype = C.c_size_t
        _lib.dgkr_gkr_proof_bound.restype = C.c_size_t
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        msg = lib().dgkr_last_error().decode(errors="replace")
        raise _EXC.get(rc, DgkrError)(rc, msg)


def header_symbols():
    """Function names declared in include/dgkr_b200.h."""
    src = open(HEADER_PATH).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dgkr_[a-z0-9_]+)\s*\(", src)))


class Transcript_t(C.Structure):
    _fields_ = [("state", C.c_uint8 * 32), ("draws", C.c_uint64)]


class Profile_t(C.Structure):
    _fields_ = [
        ("launches", C.c_uint64),
        ("round_launches", C.c_uint64),
        ("round_ms", C.c_double),
        ("round_bytes", C.c_uint64),
        ("round_mults", C.c_uint64),
        ("bookkeep_ms", C.c_double),
        ("evaluate_ms", C.c_double),
        ("total_ms", C.c_double),
        ("host_transcript_ms", C.c_double),
        ("output_absorb_ms", C.c_double),
        ("h2d_bytes", C.c_uint64),
        ("d2h_bytes", C.c_uint64),
        ("rounds", C.c_uint64),
        ("ntt_ms", C.c_double),
        ("merkle_ms", C.c_double),
        ("fold_ms", C.c_double),
        ("tail_ms", C.c_double),
        ("tail_rounds", C.c_uint64),
        ("tail_aborts", C.c_uint64),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}
