"""oracle — TEST INFRASTRUCTURE ONLY (see oracle.c header).

ctypes binding for the plain CPU oracle of the recursive Cholesky hot path of
arXiv:1602.06763.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import
this package.  It never imports the product package and the product package
never imports it.

Functions (each follows the passage cited in oracle.c):
  dpotrf(A, uplo)          -> info       unblocked left-looking Cholesky
  dpotrf_cols(A, uplo, c)  -> info       the same loop stopped after c columns (bench sample)
  dpotrf_batched(...)                    per-matrix dpotrf (CFG[4])
  dtrsm_rlt(L, B)                        B := B L^{-T}
  dsyrk_ln(A, C)                         tril(C) -= tril(A A^T)
  dgemm_nt(A, B, C)                      C -= A B^T
  dtrtri(A, uplo, diag)    -> info       A := A^{-1}, triangular
  dlauum(A, uplo)                        A := L^T L (U U^T)
  dpotri(A, uplo)          -> info       A := A^{-1} from its Cholesky factor (trtri + lauum)
  dpotrs(A, B, uplo)                     B := A^{-1} B with the factor in A
  dgetrf(A)                -> (info, ipiv)  P A = L U, partial pivoting

Arrays are numpy float64 in Fortran (column-major) order and are modified in
place, mirroring the LAPACK convention the method uses.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

CFLAGS = ["-O3", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        dp = ctypes.POINTER(ctypes.c_double)
        ip = ctypes.POINTER(ctypes.c_int)
        lp = ctypes.POINTER(ctypes.c_int64)
        c_int, c_char = ctypes.c_int, ctypes.c_char
        lib.oracle_dpotrf.argtypes = [c_char, c_int, dp, c_int]
        lib.oracle_dpotrf.restype = c_int
        lib.oracle_dpotrf_cols.argtypes = [c_char, c_int, dp, c_int, c_int]
        lib.oracle_dpotrf_cols.restype = c_int
        lib.oracle_dpotrf_batched.argtypes = [c_char, c_int, ip, dp, lp, ip, ip]
        lib.oracle_dpotrf_batched.restype = None
        lib.oracle_dtrsm_rlt.argtypes = [c_int, c_int, dp, c_int, dp, c_int]
        lib.oracle_dsyrk_ln.argtypes = [c_int, c_int, dp, c_int, dp, c_int]
        lib.oracle_dgemm_nt.argtypes = [c_int, c_int, c_int, dp, c_int, dp, c_int, dp, c_int]
        lib.oracle_num_threads.restype = c_int
        lib.oracle_dtrtri.argtypes = [c_char, c_char, c_int, dp, c_int]
        lib.oracle_dtrtri.restype = c_int
        lib.oracle_dlauum.argtypes = [c_char, c_int, dp, c_int]
        lib.oracle_dlauum.restype = None
        lib.oracle_dpotri.argtypes = [c_char, c_int, dp, c_int]
        lib.oracle_dpotri.restype = c_int
        lib.oracle_dpotrs.argtypes = [c_char, c_int, c_int, dp, c_int, dp, c_int]
        lib.oracle_dpotrs.restype = None
        lib.oracle_dgetrf.argtypes = [c_int, c_int, dp, c_int, ip]
        lib.oracle_dgetrf.restype = c_int
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _check_f64_fortran(a: np.ndarray, name: str):
    if a.dtype != np.float64:
        raise TypeError(f"{name} must be float64")
    if a.ndim != 2 or not a.flags.f_contiguous:
        raise TypeError(f"{name} must be a 2-D Fortran-ordered array")


def num_threads() -> int:
    return _load().oracle_num_threads()


def dpotrf(A: np.ndarray, uplo: str = "L", n: int | None = None) -> int:
    """In-place Cholesky of the leading n x n block of A (lda = A.shape[0])."""
    _check_f64_fortran(A, "A")
    if n is None:
        n = A.shape[1]
    lda = max(1, A.shape[0])
    return _load().oracle_dpotrf(uplo.encode(), n, _ptr(A), lda)


def dpotrf_raw(uplo: str, n: int, A: np.ndarray, lda: int) -> int:
    """LAPACK-style call on a flat float64 buffer (argument-error paths)."""
    return _load().oracle_dpotrf(uplo.encode(), n, _ptr(A), lda)


def dpotrf_cols(A: np.ndarray, uplo: str, ncols: int) -> int:
    _check_f64_fortran(A, "A")
    return _load().oracle_dpotrf_cols(uplo.encode(), A.shape[1], _ptr(A), max(1, A.shape[0]), ncols)


def dpotrf_cols_panel(P: np.ndarray, ncols: int) -> int:
    """uplo='L' only: the first `ncols` columns of the factorization of an
    n x n matrix given only its first ncols columns P (n x ncols, Fortran, lda
    = n).  The left-looking loop for column j reads columns < j and column j
    only, so the trailing columns it never touches need not exist."""
    _check_f64_fortran(P, "P")
    n, w = P.shape
    assert ncols <= w
    return _load().oracle_dpotrf_cols(b"L", n, _ptr(P), max(1, n), ncols)


def dpotrf_batched(uplo: str, ns: np.ndarray, buf: np.ndarray, offsets: np.ndarray, ldas: np.ndarray) -> np.ndarray:
    """Per-matrix Cholesky of a packed batch; returns the per-matrix info array."""
    ns = np.ascontiguousarray(ns, dtype=np.int32)
    ldas = np.ascontiguousarray(ldas, dtype=np.int32)
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    assert buf.dtype == np.float64 and buf.flags.c_contiguous
    info = np.zeros(len(ns), dtype=np.int32)
    ip = ctypes.POINTER(ctypes.c_int)
    _load().oracle_dpotrf_batched(
        uplo.encode(), len(ns), ns.ctypes.data_as(ip), _ptr(buf),
        offsets.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), ldas.ctypes.data_as(ip), info.ctypes.data_as(ip))
    return info


def dtrsm_rlt(L: np.ndarray, B: np.ndarray) -> None:
    """B := B * L^{-T} (Right, Lower, Trans, NonUnit), in place."""
    _check_f64_fortran(L, "L")
    _check_f64_fortran(B, "B")
    m, k = B.shape
    _load().oracle_dtrsm_rlt(m, k, _ptr(L), max(1, L.shape[0]), _ptr(B), max(1, m))


def dsyrk_ln(A: np.ndarray, C: np.ndarray) -> None:
    """tril(C) -= tril(A A^T), in place; the strict upper triangle is untouched."""
    _check_f64_fortran(A, "A")
    _check_f64_fortran(C, "C")
    n, k = A.shape
    _load().oracle_dsyrk_ln(n, k, _ptr(A), max(1, n), _ptr(C), max(1, C.shape[0]))


def dgemm_nt(A: np.ndarray, B: np.ndarray, C: np.ndarray) -> None:
    """C -= A B^T, in place."""
    for x, nm in ((A, "A"), (B, "B"), (C, "C")):
        _check_f64_fortran(x, nm)
    m, k = A.shape
    n = B.shape[0]
    _load().oracle_dgemm_nt(m, n, k, _ptr(A), max(1, m), _ptr(B), max(1, n), _ptr(C), max(1, C.shape[0]))


def dtrtri(A: np.ndarray, uplo: str = "L", diag: str = "N", n: int | None = None) -> int:
    """In-place inverse of the uplo triangle of A (LAPACK dtrtri semantics)."""
    _check_f64_fortran(A, "A")
    n = A.shape[1] if n is None else n
    return _load().oracle_dtrtri(uplo.encode(), diag.encode(), n, _ptr(A), max(1, A.shape[0]))


def dlauum(A: np.ndarray, uplo: str = "L") -> None:
    """In-place L^T L (uplo 'L') / U U^T (uplo 'U') of the triangular factor in A."""
    _check_f64_fortran(A, "A")
    _load().oracle_dlauum(uplo.encode(), A.shape[1], _ptr(A), max(1, A.shape[0]))


def dpotri(A: np.ndarray, uplo: str = "L") -> int:
    """In-place inverse of the SPD matrix whose Cholesky factor is in A."""
    _check_f64_fortran(A, "A")
    return _load().oracle_dpotri(uplo.encode(), A.shape[1], _ptr(A), max(1, A.shape[0]))


def dpotrs(A: np.ndarray, B: np.ndarray, uplo: str = "L") -> None:
    """B := A^{-1} B with A's Cholesky factor in A (B n x nrhs, Fortran)."""
    _check_f64_fortran(A, "A")
    _check_f64_fortran(B, "B")
    n, nrhs = B.shape
    _load().oracle_dpotrs(uplo.encode(), n, nrhs, _ptr(A), max(1, A.shape[0]), _ptr(B), max(1, n))


def dgetrf(A: np.ndarray):
    """In-place LU with partial pivoting; returns (info, ipiv) with 1-based ipiv."""
    _check_f64_fortran(A, "A")
    m, n = A.shape
    ipiv = np.zeros(max(1, min(m, n)), dtype=np.int32)
    info = _load().oracle_dgetrf(m, n, _ptr(A), max(1, m), ipiv.ctypes.data_as(ctypes.POINTER(ctypes.c_int)))
    return info, ipiv[:min(m, n)]
