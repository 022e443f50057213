"""paper_1602_06763_b200 — B200-native recursive FP64 Cholesky (xpotrf) of
arXiv:1602.06763 (ReLAPACK), behind the C ABI in include/relapack.h.

This module is argument marshalling only: every step of the factorization
runs in the sm_100a kernels of librelapack_b200.so.  There is no CPU
fallback: if the library is missing or a CUDA device is absent the calls
raise.

    import torch, paper_1602_06763_b200 as rl
    A = ...                            # (n, n) float64 CUDA tensor, column-major view (strides (1, lda))
    info = rl.dpotrf(A, "L")           # A's lower triangle := L, A = L L^T
"""
from __future__ import annotations

import ctypes
import os
import re

__all__ = [
    "lib",
    "library_path",
    "dpotrf",
    "dpotrf_raw",
    "dpotrf_async",
    "dpotrf_batched",
    "split_point",
    "profile_enable",
    "profile_reset",
    "profile_read",
    "profile_records",
    "plan_ledger",
    "set_crossover",
    "set_split_tile",
    "set_graphs",
    "get_crossover",
    "last_error",
    "finalize",
    "colmajor",
    "declared_symbols",
    "RelapackError",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
library_path = os.path.join(_HERE, "librelapack_b200.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "relapack.h")
_lib = None


class RelapackError(RuntimeError):
    pass


def lib():
    """Load the in-tree CUDA library (built by __graft_entry__.build()); fail loudly if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(library_path):
            raise RelapackError(
                f"{library_path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        L = ctypes.CDLL(library_path)
        c_int, c_char, c_void_p, c_double = ctypes.c_int, ctypes.c_char, ctypes.c_void_p, ctypes.c_double
        ip = ctypes.POINTER(c_int)
        L.relapack_dpotrf.argtypes = [ctypes.c_char_p, ip, c_void_p, ip, ip]
        L.relapack_dpotrf.restype = None
        L.relapack_dpotrf_async.argtypes = [c_char, c_int, c_void_p, c_int, c_void_p, c_void_p]
        L.relapack_dpotrf_async.restype = c_int
        L.relapack_dpotrf_batched.argtypes = [c_char, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]
        L.relapack_dpotrf_batched.restype = c_int
        L.relapack_comm_unique_id.argtypes = [ctypes.c_char_p]
        L.relapack_comm_unique_id.restype = c_int
        L.relapack_comm_init.argtypes = [ctypes.POINTER(c_void_p), ctypes.c_char_p, c_int, c_int, c_int]
        L.relapack_comm_init.restype = c_int
        L.relapack_comm_destroy.argtypes = [c_void_p]
        L.relapack_comm_destroy.restype = None
        L.relapack_dpotrf_dist.argtypes = [ctypes.c_char_p, ip, c_void_p, ip, c_int, c_int, c_void_p, ip]
        L.relapack_dpotrf_dist.restype = None
        L.relapack_set_stream.argtypes = [c_void_p]
        L.relapack_set_stream.restype = None
        L.relapack_last_error.restype = ctypes.c_char_p
        L.relapack_finalize.restype = None
        for f in ("relapack_set_crossover", "relapack_set_split_tile", "relapack_set_graphs"):
            getattr(L, f).argtypes = [c_int]
            getattr(L, f).restype = c_int
        L.relapack_get_crossover.restype = c_int
        L.relapack_split_point.argtypes = [c_int, c_int]
        L.relapack_split_point.restype = c_int
        L.relapack_plan_ledger.argtypes = [c_int, c_int, c_int, c_int, ctypes.POINTER(c_double), ip]
        L.relapack_plan_ledger.restype = c_int
        L.relapack_version.restype = ctypes.c_char_p
        L.relapack_profile_enable.argtypes = [c_int]
        L.relapack_profile_enable.restype = c_int
        L.relapack_profile_read.argtypes = [c_int, ctypes.POINTER(c_double), ctypes.POINTER(c_double), ip]
        L.relapack_profile_read.restype = c_int
        L.relapack_profile_reset.restype = None
        L.relapack_profile_records.argtypes = [c_int, ctypes.POINTER(c_double)]
        L.relapack_profile_records.restype = c_int
        L.relapack_trace_read.argtypes = [c_int, ctypes.POINTER(c_double)]
        L.relapack_trace_read.restype = c_int
        L.relapack_dpotrf_dist_loopback.argtypes = [ctypes.c_char_p, c_int, c_void_p, c_int, c_int, c_int, c_int, ip]
        L.relapack_dpotrf_dist_loopback.restype = c_int
        L.relapack_dist_schedule.argtypes = [c_int, c_int, c_int, c_int, c_int, c_int, c_int,
                                             ctypes.POINTER(ctypes.c_int64), c_int]
        L.relapack_dist_schedule.restype = c_int
        L.relapack_plan_schedule.argtypes = [c_int, c_int, c_int, c_int, ctypes.POINTER(ctypes.c_int64), c_int,
                                             ctypes.POINTER(c_int), ctypes.POINTER(c_int), c_int]
        L.relapack_plan_schedule.restype = c_int
        i64 = ctypes.c_int64
        L.relapack_update_test.argtypes = [c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_double, c_void_p, i64,
                                           c_void_p, i64, c_void_p, i64, c_int, c_int, c_int, c_int, c_int, c_void_p,
                                           ip]
        L.relapack_update_test.restype = c_int
        L.relapack_trsm_test.argtypes = [c_int, c_int, c_int, c_void_p, i64, c_void_p, i64, c_int, c_void_p]
        L.relapack_trsm_test.restype = c_int
        L.relapack_potf2_test.argtypes = [c_int, c_int, c_void_p, i64, ip, c_void_p]
        L.relapack_potf2_test.restype = c_int
        cp = ctypes.c_char_p
        L.relapack_dtrtri.argtypes = [cp, cp, ip, c_void_p, ip, ip]
        L.relapack_dtrtri.restype = None
        L.relapack_dtrtri_blocked.argtypes = [cp, cp, ip, c_void_p, ip, c_int, ip]
        L.relapack_dtrtri_blocked.restype = None
        L.relapack_dlauum.argtypes = [cp, ip, c_void_p, ip, ip]
        L.relapack_dlauum.restype = None
        L.relapack_dpotri.argtypes = [cp, ip, c_void_p, ip, ip]
        L.relapack_dpotri.restype = None
        L.relapack_dpotrs.argtypes = [cp, ip, ip, c_void_p, ip, c_void_p, ip, ip]
        L.relapack_dpotrs.restype = None
        L.relapack_dgetrf.argtypes = [ip, ip, c_void_p, ip, c_void_p, ip]
        L.relapack_dgetrf.restype = None
        L.relapack_dpotrf_blocked.argtypes = [cp, ip, c_void_p, ip, c_int, ip]
        L.relapack_dpotrf_blocked.restype = None
        L.relapack_xplan_count.argtypes = [c_int, c_int, c_int, ctypes.POINTER(c_int), c_int,
                                           ctypes.POINTER(c_double)]
        L.relapack_xplan_count.restype = c_int
        L.relapack_xprofile_enable.argtypes = [c_int]
        L.relapack_xprofile_enable.restype = c_int
        L.relapack_xprofile_read.argtypes = [c_int, ctypes.POINTER(c_double), ctypes.POINTER(c_double), ip]
        L.relapack_xprofile_read.restype = c_int
        L.relapack_xprofile_reset.restype = None
        L.relapack_xprofile_records.argtypes = [c_int, ctypes.POINTER(c_double)]
        L.relapack_xprofile_records.restype = c_int
        L.relapack_batch_split.argtypes = [c_int, c_void_p, c_int, c_void_p]
        L.relapack_batch_split.restype = c_int
        _lib = L
    return _lib


def declared_symbols() -> list[str]:
    """Function names declared in include/relapack.h (the C ABI)."""
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(relapack_[a-z_0-9]+)\s*\(", src)))


def last_error() -> str:
    return (lib().relapack_last_error() or b"").decode()


def finalize() -> None:
    lib().relapack_finalize()


def set_crossover(c: int) -> None:
    if lib().relapack_set_crossover(int(c)) != 0:
        raise ValueError(f"crossover {c} out of range [16, 256]")


def set_split_tile(t: int) -> None:
    if lib().relapack_set_split_tile(int(t)) != 0:
        raise ValueError(f"split tile {t} not in (8, 16, 32, 64, 128)")


def set_graphs(enabled: bool) -> None:
    lib().relapack_set_graphs(1 if enabled else 0)


def get_crossover() -> int:
    return lib().relapack_get_crossover()


PROFILE_KINDS = {"potf2": 0, "trsm": 1, "gemm": 2, "syrk": 3}


def profile_enable(on: bool) -> None:
    lib().relapack_profile_enable(1 if on else 0)


def profile_reset() -> None:
    lib().relapack_profile_reset()


def profile_read(kind: str):
    """(ms_total, flops_total, launches) recorded for one kernel class since the last reset."""
    ms, fl, cnt = ctypes.c_double(0), ctypes.c_double(0), ctypes.c_int(0)
    if lib().relapack_profile_read(PROFILE_KINDS[kind], ctypes.byref(ms), ctypes.byref(fl), ctypes.byref(cnt)) != 0:
        raise ValueError(kind)
    return ms.value, fl.value, cnt.value


def profile_records(max_records: int = 100000):
    """Per-launch (kind, m, n, k, level, flops, ms) records since the last reset."""
    buf = (ctypes.c_double * (7 * max_records))()
    cnt = lib().relapack_profile_records(max_records, buf)
    kinds = {v: k for k, v in PROFILE_KINDS.items()}
    out = []
    for i in range(cnt):
        r = buf[7 * i: 7 * i + 7]
        out.append(dict(kind=kinds[int(r[0])], m=int(r[1]), n=int(r[2]), k=int(r[3]), level=int(r[4]),
                        flops=r[5], ms=r[6]))
    return out


def trace_records(max_records: int = 100000):
    """Kernel timeline of the last RELAPACK_TRACE=1 factorization: list of dicts
    (kind, m, n, k, flops, t0_us, t1_us) in plan order (see include/relapack.h)."""
    buf = (ctypes.c_double * (7 * max_records))()
    cnt = lib().relapack_trace_read(max_records, buf)
    if cnt < 0:
        raise RelapackError(f"relapack_trace_read failed: {last_error()}")
    names = {0: "potf2", 1: "trsm", 2: "gemm", 3: "syrk", 20: "h2d", 21: "d2h"}
    out = []
    for i in range(cnt):
        r = buf[7 * i: 7 * i + 7]
        out.append(dict(kind=names.get(int(r[0]), str(int(r[0]))), m=int(r[1]), n=int(r[2]), k=int(r[3]),
                        flops=r[4], t0_us=r[5], t1_us=r[6]))
    return out


DIST_KINDS = {0: "potf2", 1: "trsm", 2: "gemm", 3: "syrk", 10: "pack", 11: "allgather", 12: "unpack"}
DIST_FIELDS = ("kind", "level", "c_i", "c_j", "a_i", "a_j", "b_i", "b_j", "m", "n", "k", "info_base",
               "c_buf", "a_buf", "b_buf")


def dist_schedule(n: int, rank: int, nranks: int, nb: int = 512, dist_min: int = 4096, c: int | None = None,
                  T: int = 64):
    """Host-only: rank `rank`'s multi-GPU step list (list of dicts, see include/relapack.h)."""
    c = get_crossover() if c is None else c
    cnt = lib().relapack_dist_schedule(n, c, T, nb, dist_min, rank, nranks, None, 0)
    if cnt < 0:
        raise ValueError("bad schedule arguments")
    buf = (ctypes.c_int64 * (16 * max(cnt, 1)))()
    lib().relapack_dist_schedule(n, c, T, nb, dist_min, rank, nranks, buf, cnt)
    out = []
    for i in range(cnt):
        row = buf[16 * i: 16 * i + 15]
        d = dict(zip(DIST_FIELDS, (int(v) for v in row)))
        d["kind"] = DIST_KINDS[d["kind"]]
        out.append(d)
    return out


def plan_schedule(n: int, c: int = 64, T: int = 64, lookahead: bool = True):
    """Host-only: (ops, deps) of the single-GPU plan — ops as dicts (DIST_FIELDS + deferred),
    deps[i] = direct predecessors of launch i in the captured dependency DAG."""
    L = lib()
    cnt = L.relapack_plan_schedule(n, c, T, int(lookahead), None, 0, None, None, 0)
    if cnt < 0:
        raise ValueError("bad plan arguments")
    buf = (ctypes.c_int64 * (16 * max(cnt, 1)))()
    off = (ctypes.c_int * (cnt + 1))()
    L.relapack_plan_schedule(n, c, T, int(lookahead), buf, cnt, off, None, 0)
    idx = (ctypes.c_int * max(off[cnt], 1))()
    L.relapack_plan_schedule(n, c, T, int(lookahead), buf, cnt, off, idx, off[cnt])
    ops = []
    for i in range(cnt):
        row = buf[16 * i: 16 * i + 16]
        d = dict(zip(DIST_FIELDS + ("deferred",), (int(v) for v in row)))
        d["kind"] = DIST_KINDS[d["kind"]]
        ops.append(d)
    deps = [list(idx[off[i]:off[i + 1]]) for i in range(cnt)]
    return ops, deps


def _locate_nccl() -> None:
    """Point RELAPACK_NCCL_LIB at the NCCL the process uses (torch's bundled one) if not set."""
    if os.environ.get("RELAPACK_NCCL_LIB"):
        return
    try:
        import nvidia.nccl  # the wheel torch links against

        for d in nvidia.nccl.__path__:
            cand = os.path.join(d, "lib", "libnccl.so.2")
            if os.path.exists(cand):
                os.environ["RELAPACK_NCCL_LIB"] = cand
                return
    except Exception:
        pass


class Comm:
    """NCCL communicator for relapack_dpotrf_dist (one process per GPU)."""

    def __init__(self, uid: bytes, nranks: int, rank: int, device: int):
        _locate_nccl()
        self.ptr = ctypes.c_void_p()
        r = lib().relapack_comm_init(ctypes.byref(self.ptr), uid, nranks, rank, device)
        if r != 0:
            raise RelapackError(f"relapack_comm_init failed ({r}): {last_error()}")
        self.nranks, self.rank = nranks, rank

    @staticmethod
    def unique_id() -> bytes:
        _locate_nccl()
        buf = ctypes.create_string_buffer(128)
        r = lib().relapack_comm_unique_id(buf)
        if r != 0:
            raise RelapackError(f"relapack_comm_unique_id failed ({r}): {last_error()}")
        return buf.raw

    def close(self):
        if self.ptr:
            lib().relapack_comm_destroy(self.ptr)
            self.ptr = ctypes.c_void_p()


def dpotrf_dist(A, comm: "Comm", uplo: str = "L", nb: int = 512, dist_min: int = 4096, stream=None) -> int:
    """Distributed factorization of the device matrix A (identical on every rank); returns info."""
    import torch

    ptr, n, lda = _matrix_args(A)
    st = stream if stream is not None else torch.cuda.current_stream(A.device)
    lib().relapack_set_stream(ctypes.c_void_p(st.cuda_stream))
    info = ctypes.c_int(0)
    lib().relapack_dpotrf_dist(uplo.encode(), ctypes.byref(ctypes.c_int(n)), ctypes.c_void_p(ptr),
                               ctypes.byref(ctypes.c_int(lda)), nb, dist_min, comm.ptr, ctypes.byref(info))
    if info.value <= -1000:
        raise RelapackError(f"relapack_dpotrf_dist failed: {last_error()}")
    return info.value


def dpotrf_dist_loopback(As, uplo: str = "L", nb: int = 512, dist_min: int = 4096):
    """Test hook: run the distributed schedule for len(As) virtual ranks on one GPU; returns the infos."""
    ptrs = [_matrix_args(A) for A in As]
    n, lda = ptrs[0][1], ptrs[0][2]
    arr = (ctypes.c_void_p * len(As))(*[p[0] for p in ptrs])
    infos = (ctypes.c_int * len(As))()
    r = lib().relapack_dpotrf_dist_loopback(uplo.encode(), n, arr, lda, nb, dist_min, len(As), infos)
    if r != 0:
        raise RelapackError(f"relapack_dpotrf_dist_loopback failed ({r}): {last_error()}")
    return list(infos)


def _block_args(X):
    """(pointer, ld, layout) of a 2-D float64 CUDA tensor with a unit stride:
    layout 0 when X[r, c] is at ptr + r + c*ld (column-major), 1 when at ptr + c + r*ld."""
    import torch

    if X.dtype != torch.float64 or X.dim() != 2:
        raise TypeError("expected a 2-D float64 tensor")
    rows, cols = X.shape
    if X.stride(0) == 1 and (cols <= 1 or X.stride(1) >= max(1, rows)):
        return X.data_ptr(), max(1, X.stride(1) if cols > 1 else rows), 0
    if X.stride(1) == 1 and (rows <= 1 or X.stride(0) >= max(1, cols)):
        return X.data_ptr(), max(1, X.stride(0) if rows > 1 else cols), 1
    raise ValueError("operand needs a unit stride in one dimension")


def update_test(C, A, B, alpha: float = -1.0, tri: int = 0, tile: int = 0, ksplit: int = 0, tma: bool = True,
                ctas: int = 0, full: int = 0, stream=None):
    """Kernel test hook (K3/K4): C += alpha A B^T on the tri part of C (0 all, 1 lower, 2 upper).
    C: (M, N), A: (M, K), B: (N, K) float64 CUDA tensors, each column- or row-major (its layout).
    ctas > 0 caps the grid (persistent CTAs, several work items each); full > 0 with
    ksplit > 1 splits only the tiles [full, ntiles) (tail split).
    Returns (tile, used_tma, ksplit) the launch used."""
    import torch

    pc, ldc, lc = _block_args(C)
    pa, lda, la = _block_args(A)
    pb, ldb, lb = _block_args(B)
    M, N = C.shape
    K = A.shape[1]
    if A.shape[0] != M or B.shape != (N, K):
        raise ValueError("shape mismatch")
    st = stream if stream is not None else torch.cuda.current_stream(C.device)
    chosen = (ctypes.c_int * 3)()
    r = lib().relapack_update_test(la, lb, lc, tri, M, N, K, float(alpha), ctypes.c_void_p(pc), ldc,
                                   ctypes.c_void_p(pa), lda, ctypes.c_void_p(pb), ldb, tile, ksplit, int(tma),
                                   int(ctas), int(full), ctypes.c_void_p(st.cuda_stream), chosen)
    if r != 0:
        raise RelapackError(f"relapack_update_test failed ({r}): {last_error()}")
    return tuple(chosen)


def trsm_test(Lblk, B, variant: int = 0, stream=None):
    """Kernel test hook (K5): B := B L^{-T} with L the lower triangle of the (t, t) block Lblk.
    Lblk and B must share one layout (column-major: uplo L; row-major: the uplo U L-view)."""
    import torch

    pl, ldl, ll = _block_args(Lblk)
    pb, ldb, lb = _block_args(B)
    if ll != lb:
        raise ValueError("L and B must have the same layout")
    m, t = B.shape
    st = stream if stream is not None else torch.cuda.current_stream(B.device)
    r = lib().relapack_trsm_test(ll, m, t, ctypes.c_void_p(pl), ldl, ctypes.c_void_p(pb), ldb, variant,
                                 ctypes.c_void_p(st.cuda_stream))
    if r != 0:
        raise RelapackError(f"relapack_trsm_test failed ({r}): {last_error()}")


def potf2_test(A, stream=None) -> int:
    """Kernel test hook (K1): base-case factorization of the (n, n) block (n <= 128); returns info."""
    import torch

    pa, lda, la = _block_args(A)
    st = stream if stream is not None else torch.cuda.current_stream(A.device)
    info = ctypes.c_int(0)
    r = lib().relapack_potf2_test(la, A.shape[0], ctypes.c_void_p(pa), lda, ctypes.byref(info),
                                  ctypes.c_void_p(st.cuda_stream))
    if r != 0:
        raise RelapackError(f"relapack_potf2_test failed ({r}): {last_error()}")
    return info.value


def _ci(v: int):
    return ctypes.byref(ctypes.c_int(int(v)))


def _set_stream_for(A, stream):
    import torch

    st = stream if stream is not None else torch.cuda.current_stream(A.device)
    lib().relapack_set_stream(ctypes.c_void_p(st.cuda_stream))


def _check_info(name: str, v: int) -> int:
    if v <= -1000:
        raise RelapackError(f"{name} failed: {last_error()}")
    return v


def dtrtri(A, uplo: str = "L", diag: str = "N", stream=None) -> int:
    """A := A^{-1} for the uplo-triangular device matrix A (column-major); returns info."""
    ptr, n, lda = _matrix_args(A)
    _set_stream_for(A, stream)
    info = ctypes.c_int(0)
    lib().relapack_dtrtri(uplo.encode(), diag.encode(), _ci(n), ctypes.c_void_p(ptr), _ci(lda), ctypes.byref(info))
    return _check_info("relapack_dtrtri", info.value)


def dtrtri_blocked(A, nb: int, uplo: str = "L", diag: str = "N", stream=None) -> int:
    """Blocked (block nb) triangular inverse, for the blocked-vs-recursive comparison; returns info."""
    ptr, n, lda = _matrix_args(A)
    _set_stream_for(A, stream)
    info = ctypes.c_int(0)
    lib().relapack_dtrtri_blocked(uplo.encode(), diag.encode(), _ci(n), ctypes.c_void_p(ptr), _ci(lda), int(nb),
                                  ctypes.byref(info))
    return _check_info("relapack_dtrtri_blocked", info.value)


def dlauum(A, uplo: str = "L", stream=None) -> int:
    """A := L^T L (uplo L) / U U^T (uplo U) in place; returns info."""
    ptr, n, lda = _matrix_args(A)
    _set_stream_for(A, stream)
    info = ctypes.c_int(0)
    lib().relapack_dlauum(uplo.encode(), _ci(n), ctypes.c_void_p(ptr), _ci(lda), ctypes.byref(info))
    return _check_info("relapack_dlauum", info.value)


def dpotri(A, uplo: str = "L", stream=None) -> int:
    """A := A^{-1} from the Cholesky factor in A; returns info."""
    ptr, n, lda = _matrix_args(A)
    _set_stream_for(A, stream)
    info = ctypes.c_int(0)
    lib().relapack_dpotri(uplo.encode(), _ci(n), ctypes.c_void_p(ptr), _ci(lda), ctypes.byref(info))
    return _check_info("relapack_dpotri", info.value)


def dpotrs(A, B, uplo: str = "L", stream=None) -> int:
    """B := A^{-1} B with the Cholesky factor in A; B (n, nrhs) column-major device tensor."""
    ptr, n, lda = _matrix_args(A)
    if B.dim() != 2 or B.shape[0] != n or (B.shape[1] > 1 and B.stride(0) != 1):
        raise ValueError("B must be (n, nrhs) column-major")
    nrhs = B.shape[1]
    ldb = max(1, B.stride(1) if nrhs > 1 else n)
    _set_stream_for(A, stream)
    info = ctypes.c_int(0)
    lib().relapack_dpotrs(uplo.encode(), _ci(n), _ci(nrhs), ctypes.c_void_p(ptr), _ci(lda),
                          ctypes.c_void_p(B.data_ptr()), _ci(ldb), ctypes.byref(info))
    return _check_info("relapack_dpotrs", info.value)


def dgetrf(A, ipiv, stream=None) -> int:
    """P A = L U in place (A (m, n) column-major device tensor); ipiv int32 device tensor of min(m, n)."""
    import torch

    if A.dim() != 2 or A.dtype != torch.float64:
        raise TypeError("A must be a 2-D float64 tensor")
    m, n = A.shape
    if n > 1 and A.stride(0) != 1:
        raise ValueError("A must be column-major")
    lda = max(1, A.stride(1) if n > 1 else m)
    _set_stream_for(A, stream)
    info = ctypes.c_int(0)
    lib().relapack_dgetrf(_ci(m), _ci(n), ctypes.c_void_p(A.data_ptr()), _ci(lda), ctypes.c_void_p(ipiv.data_ptr()),
                          ctypes.byref(info))
    return _check_info("relapack_dgetrf", info.value)


def dpotrf_blocked(A, nb: int, uplo: str = "L", stream=None) -> int:
    """Blocked right-looking Cholesky with block nb on the library's kernels; returns info."""
    ptr, n, lda = _matrix_args(A)
    _set_stream_for(A, stream)
    info = ctypes.c_int(0)
    lib().relapack_dpotrf_blocked(uplo.encode(), _ci(n), ctypes.c_void_p(ptr), _ci(lda), int(nb), ctypes.byref(info))
    return _check_info("relapack_dpotrf_blocked", info.value)


def xplan_count(op: str, n: int, nb: int = 0):
    """Host-only: (launches, kinds, flops) of a §8(f) plan (op in trtri, trtri_blocked, lauum, potri, potrs, getrf,
    getrf_la — the lookahead getrf plan with window nb)."""
    code = {"trtri": 0, "trtri_blocked": 1, "lauum": 2, "potri": 3, "potrs": 4, "getrf": 5, "getrf_la": 6}[op]
    fl = ctypes.c_double(0)
    cnt = lib().relapack_xplan_count(code, n, nb, None, 0, ctypes.byref(fl))
    if cnt < 0:
        raise ValueError("bad plan arguments")
    kinds = (ctypes.c_int * max(cnt, 1))()
    lib().relapack_xplan_count(code, n, nb, kinds, cnt, ctypes.byref(fl))
    return cnt, list(kinds)[:cnt], fl.value


XKINDS = {"gemm": 0, "tri": 1, "trti2": 2, "lauu2": 3, "potf2": 4, "getf2": 5, "laswp": 6, "check": 7, "perm": 8}


def xprofile_records(fn, max_records: int = 200000):
    """Run fn() with the §8(f) plans profiled; per-launch (kind, level, flops, ms) records."""
    L = lib()
    L.relapack_xprofile_reset()
    L.relapack_xprofile_enable(1)
    try:
        fn()
        buf = (ctypes.c_double * (4 * max_records))()
        cnt = L.relapack_xprofile_records(max_records, buf)
        kinds = {v: k for k, v in XKINDS.items()}
        return [dict(kind=kinds[int(buf[4 * i])], level=int(buf[4 * i + 1]), flops=buf[4 * i + 2], ms=buf[4 * i + 3])
                for i in range(cnt)]
    finally:
        L.relapack_xprofile_enable(0)
        L.relapack_xprofile_reset()


def xprofile(fn):
    """Run fn() with the §8(f) plans profiled per kind; returns {kind: (ms, flops, launches)}."""
    L = lib()
    L.relapack_xprofile_reset()
    L.relapack_xprofile_enable(1)
    try:
        fn()
        out = {}
        for k, v in XKINDS.items():
            ms, fl, cnt = ctypes.c_double(0), ctypes.c_double(0), ctypes.c_int(0)
            L.relapack_xprofile_read(v, ctypes.byref(ms), ctypes.byref(fl), ctypes.byref(cnt))
            if cnt.value:
                out[k] = (ms.value, fl.value, cnt.value)
        return out
    finally:
        L.relapack_xprofile_enable(0)
        L.relapack_xprofile_reset()


def batch_split(ns, nranks: int):
    """Host-only: contiguous per-rank ranges of a batch balanced by sum n^3 (list of nranks + 1 bounds)."""
    import numpy as np

    h = np.ascontiguousarray(ns, dtype=np.int32)
    out = np.zeros(nranks + 1, dtype=np.int32)
    if lib().relapack_batch_split(len(h), h.ctypes.data, int(nranks), out.ctypes.data) != 0:
        raise ValueError("bad batch split arguments")
    return [int(x) for x in out]


def split_point(n: int, align: int) -> int:
    return lib().relapack_split_point(int(n), int(align))


def plan_ledger(n: int, c: int, T: int, levels: int):
    """(depth, flops_by_level[levels], base_flops, launches) of the plan the driver builds (host only)."""
    buf = (ctypes.c_double * (levels + 1))()
    cnt = ctypes.c_int(0)
    depth = lib().relapack_plan_ledger(int(n), int(c), int(T), int(levels), buf, ctypes.byref(cnt))
    if depth < 0:
        raise ValueError("bad plan arguments")
    vals = list(buf)
    return depth, vals[:levels], vals[levels], cnt.value


def colmajor(X):
    """A column-major (strides (1, n)) float64 copy of a 2-D torch tensor."""
    return X.t().contiguous().t()


def _matrix_args(A):
    """(pointer, n, lda) of a 2-D float64 torch tensor with unit row stride."""
    import torch

    if not isinstance(A, torch.Tensor) or A.dtype != torch.float64 or A.dim() != 2:
        raise TypeError("A must be a 2-D float64 torch tensor")
    n = A.shape[1]
    if A.shape[0] != n:
        raise ValueError("A must be square")
    if n > 1 and A.stride(0) != 1:
        raise ValueError("A must be column-major (stride(0) == 1); use colmajor(A)")
    lda = max(1, A.stride(1) if n > 1 else max(1, A.shape[0]))
    return A.data_ptr(), n, lda


def dpotrf(A, uplo: str = "L", stream=None) -> int:
    """Factor A in place (LAPACK dpotrf semantics, include/relapack.h); returns info.

    A: (n, n) float64 torch tensor, column-major (strides (1, lda)), on a CUDA
    device (factored in place on the GPU) or on the CPU (pinned or pageable:
    the uplo triangle is staged through the GPU and copied back).
    """
    import torch

    ptr, n, lda = _matrix_args(A)
    if A.is_cuda:
        st = stream if stream is not None else torch.cuda.current_stream(A.device)
        lib().relapack_set_stream(ctypes.c_void_p(st.cuda_stream))
    else:
        st = stream if stream is not None else (torch.cuda.current_stream() if torch.cuda.is_available() else None)
        lib().relapack_set_stream(ctypes.c_void_p(st.cuda_stream if st is not None else 0))
    info = ctypes.c_int(0)
    lib().relapack_dpotrf(uplo.encode(), ctypes.byref(ctypes.c_int(n)), ctypes.c_void_p(ptr),
                          ctypes.byref(ctypes.c_int(lda)), ctypes.byref(info))
    if info.value <= -1000:
        raise RelapackError(f"relapack_dpotrf failed: {last_error()}")
    return info.value


def dpotrf_raw(uplo: str, n: int, ptr: int, lda: int) -> int:
    """Direct C-ABI call with raw arguments (argument-checking tests)."""
    info = ctypes.c_int(0)
    lib().relapack_dpotrf(uplo.encode(), ctypes.byref(ctypes.c_int(n)), ctypes.c_void_p(ptr),
                          ctypes.byref(ctypes.c_int(lda)), ctypes.byref(info))
    return info.value


def dpotrf_async(A, d_info, uplo: str = "L", stream=None) -> int:
    """Stream-ordered factorization; d_info: int32 CUDA tensor (1 element). Returns the argument code."""
    import torch

    ptr, n, lda = _matrix_args(A)
    st = stream if stream is not None else torch.cuda.current_stream(A.device)
    r = lib().relapack_dpotrf_async(uplo.encode(), n, ctypes.c_void_p(ptr), lda, ctypes.c_void_p(d_info.data_ptr()),
                                    ctypes.c_void_p(st.cuda_stream))
    if r <= -1000:
        raise RelapackError(f"relapack_dpotrf_async failed: {last_error()}")
    return r


def dpotrf_batched(ns, ptrs, ldas, infos, uplo: str = "L", stream=None) -> int:
    """Batched small factorizations; ns/ldas/infos int32 and ptrs int64 CUDA tensors of length batch."""
    import torch

    st = stream if stream is not None else torch.cuda.current_stream(ns.device)
    r = lib().relapack_dpotrf_batched(uplo.encode(), int(ns.numel()), ctypes.c_void_p(ns.data_ptr()),
                                      ctypes.c_void_p(ptrs.data_ptr()), ctypes.c_void_p(ldas.data_ptr()),
                                      ctypes.c_void_p(infos.data_ptr()), ctypes.c_void_p(st.cuda_stream))
    if r <= -1000:
        raise RelapackError(f"relapack_dpotrf_batched failed: {last_error()}")
    return r
