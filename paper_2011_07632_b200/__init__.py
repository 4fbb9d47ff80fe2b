"""Thin Python binding of libspdhss.so (the C ABI in include/spdhss.h).

Argument marshalling only: every numeric step runs in the library's CUDA
kernels.  PyTorch provides device memory and the current stream.  There is no
fallback: if libspdhss.so is missing or a CUDA device is absent, calls raise.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libspdhss.so")

SPD_OK, SPD_EINVAL, SPD_ENOTPD, SPD_ENOMEM, SPD_ECUDA, SPD_ENCCL, SPD_ENOCONV = range(7)
GAUSSIAN, MATERN32, EXPONENTIAL, IMQ, K_RPY = range(5)
RPY = K_RPY
LAYOUT_ORIGINAL, LAYOUT_TREE = 0, 1
Q_N, Q_LEVELS, Q_PERM, Q_NODES, Q_BOXES, Q_NNODES, Q_H2_RANKS, Q_SKELETONS = 1, 2, 3, 4, 5, 6, 7, 8
Q_LIST_COUNTS, Q_NEAR, Q_TYPE3, Q_TYPE1 = 9, 10, 11, 12
Q_HSS_RANKS, Q_HSS_EXPORT_SIZE, Q_HSS_EXPORT, Q_HSS_PIVOTS, Q_TIMINGS = 20, 21, 22, 23, 30
Q_SHARD_WORK = 31
Q_SYM_STORE = 32
Q_COMM_BYTES = 33


class SpdError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[spd status {code}] {msg}")
        self.code = code


class NotPositiveDefinite(SpdError):
    pass


class _Kernel(ctypes.Structure):
    _fields_ = [("id", ctypes.c_int), ("l", ctypes.c_double), ("shift", ctypes.c_double)]


class _H2Opts(ctypes.Structure):
    _fields_ = [("n_proxy", ctypes.c_int), ("reserved", ctypes.c_int),
                ("inject_skeletons", ctypes.POINTER(ctypes.c_int32))]


class PcgReport(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int), ("converged", ctypes.c_int),
                ("relres", ctypes.c_double), ("seconds", ctypes.c_double), ("relres_true", ctypes.c_double)]


_lib = None


def lib():
    """Load libspdhss.so (fails loudly if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run __graft_entry__.build() or ./build_lib.sh")
    L = ctypes.CDLL(LIB_PATH)
    vp, i64, c_int, c_double = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
    P = ctypes.POINTER
    sigs = {
        "spd_last_error": ([], ctypes.c_char_p),
        "spd_comm_init": ([vp, c_int, c_int, P(vp)], c_int),
        "spd_comm_unique_id": ([vp], c_int),
        "spd_comm_init_host": ([P(_HostColl), c_int, c_int, P(vp)], c_int),
        "spd_test_shard_owner": ([c_int, c_int, c_int], c_int),
        "spd_comm_free": ([vp], None),
        "h2_build": ([vp, i64, c_int, _Kernel, c_int, c_double, P(_H2Opts), vp, vp, P(vp)], c_int),
        "h2_matvec": ([vp, c_int, vp, i64, vp, i64, i64, vp], c_int),
        "spdhss_build": ([vp, c_int, c_double, c_int, ctypes.c_uint64, vp, vp, P(vp)], c_int),
        "hss_solve": ([vp, c_int, vp, i64, vp, i64, i64, vp], c_int),
        "hss_matvec": ([vp, c_int, vp, i64, vp, i64, i64, vp], c_int),
        "pcg_solve": ([vp, vp, c_int, vp, vp, c_double, c_int, P(PcgReport), vp], c_int),
        "pcg_solve_bj": ([vp, vp, c_int, vp, vp, c_double, c_int, P(PcgReport), vp], c_int),
        "spdhss_build_adaptive": ([vp, c_int, c_int, c_double, c_int, ctypes.c_uint64, vp, vp, P(vp), P(c_int)], c_int),
        "spd_query": ([vp, c_int, vp, ctypes.c_size_t], c_int),
        "h2_free": ([vp], None),
        "h2_release_store": ([vp], c_int),
        "hss_free": ([vp], None),
        "spd_test_gemm": ([c_int, c_int, c_int, c_int, c_int, c_double, vp, c_int, vp, c_int, c_double,
                           vp, c_int, vp], c_int),
        "spd_test_potrf": ([vp, c_int, c_int, P(c_int), vp], c_int),
        "spd_test_trsm": ([ctypes.c_char, c_int, vp, c_int, c_int, vp, c_int, c_int, vp], c_int),
        "spd_test_qrcp": ([c_int, vp, c_int, c_int, c_int, i64, c_int, c_double, vp, vp, vp, i64, vp], c_int),
        "spd_test_proxies": ([vp, c_int, vp, vp], c_int),
        "spd_test_qr_unpivoted": ([c_int, vp, c_int, c_int, c_int, i64, vp], c_int),
        "spd_test_philox_normal": ([vp, i64, c_int, ctypes.c_uint64, vp], c_int),
        "spd_test_tree_host": ([vp, i64, c_int, c_int, vp, vp, vp], c_int),
        "spd_launch_count": ([], ctypes.c_longlong),
        "spd_prof_enable": ([c_int], None),
        "spd_prof_reset": ([], None),
        "spd_prof_count": ([], c_int),
        "spd_prof_get": ([c_int, ctypes.c_char_p, c_int, P(c_double)], c_int),
    }
    for name, (args, res) in sigs.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


EXPORTED = ["spd_comm_unique_id", "spd_comm_init", "spd_comm_init_host", "spd_comm_free", "h2_build", "h2_matvec", "spdhss_build", "hss_solve",
            "hss_matvec", "pcg_solve", "pcg_solve_bj", "spdhss_build_adaptive", "spd_query", "h2_free", "hss_free", "spd_last_error",
            "h2_release_store"]


def _check(status):
    if status in (SPD_OK, SPD_ENOCONV):
        return status
    msg = lib().spd_last_error().decode()
    if status == SPD_ENOTPD:
        raise NotPositiveDefinite(status, msg)
    raise SpdError(status, msg)


def _stream():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dptr(t, name):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64:
        raise TypeError(f"{name} must be a CUDA float64 tensor")
    return ctypes.c_void_p(t.data_ptr())


def _mat(t, name):
    """(n,) or (n, k) column-major CUDA float64 -> (ptr, ld, k)."""
    if t.dim() == 1:
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
        return _dptr(t, name), t.shape[0], 1
    if t.stride(0) != 1:
        raise ValueError(f"{name} must be column-major (use .t().contiguous().t())")
    return _dptr(t, name), max(t.stride(1), t.shape[0]), t.shape[1]


def empty_colmajor(n, k, device="cuda"):
    import torch
    return torch.empty((k, n), dtype=torch.float64, device=device).t()


class H2:
    """Handle of an H2 representation (h2_build)."""

    def __init__(self, ptr, n, d):
        self.ptr = ptr
        self.n = n
        self.d = d

    def __del__(self):
        if getattr(self, "ptr", None) and _lib is not None:
            _lib.h2_free(self.ptr)
            self.ptr = None

    def query(self, what, dtype, count):
        buf = np.zeros(count, dtype=dtype)
        _check(lib().spd_query(self.ptr, what, buf.ctypes.data_as(ctypes.c_void_p), buf.nbytes))
        return buf

    @property
    def levels(self):
        return int(self.query(Q_LEVELS, np.int32, 1)[0])

    @property
    def nnodes(self):
        return int(self.query(Q_NNODES, np.int32, 1)[0])

    @property
    def perm(self):
        return self.query(Q_PERM, np.int64, self.n)

    def nodes(self):
        return self.query(Q_NODES, np.int64, 2 * self.nnodes).reshape(-1, 2)

    def boxes(self):
        return self.query(Q_BOXES, np.float64, 2 * self.d * self.nnodes).reshape(-1, 2, self.d)

    def ranks(self):
        return self.query(Q_H2_RANKS, np.int32, self.nnodes)

    def skeletons(self):
        r = self.ranks()
        flat = self.query(Q_SKELETONS, np.int64, max(1, int(r.sum())))
        out, off = {}, 0
        for i, s in enumerate(r):
            if s:
                out[i] = flat[off:off + s]
                off += s
        return out

    def list_counts(self):
        return self.query(Q_LIST_COUNTS, np.int64, 1 + 2 * self.levels)

    def near_pairs(self):
        c = self.list_counts()
        return self.query(Q_NEAR, np.int32, 2 * int(c[0])).reshape(-1, 2)

    def type3(self):
        c = self.list_counts()
        n3 = int(c[1 + self.levels:].sum())
        return self.query(Q_TYPE3, np.int32, 3 * n3).reshape(-1, 3)

    def type1(self):
        c = self.list_counts()
        n1 = int(c[1:1 + self.levels].sum())
        return self.query(Q_TYPE1, np.int32, 3 * n1).reshape(-1, 3)

    def timings(self):
        return self.query(Q_TIMINGS, np.float64, 16)

    def shard_work(self):
        """(nodes whose per-node work this process computed, nodes with per-node work)."""
        return tuple(int(v) for v in self.query(Q_SHARD_WORK, np.int64, 2))

    def release_store(self):
        """Free the stored symmetric kernel blocks (h2_release_store)."""
        _check(lib().h2_release_store(self.ptr))

    def sym_store(self):
        """(bytes, pieces) of the stored symmetric k = 1 blocks on this process."""
        return tuple(int(v) for v in self.query(Q_SYM_STORE, np.int64, 2))

    def comm_bytes(self):
        """(bytes received through the library's collectives so far, collective calls)."""
        return tuple(int(v) for v in self.query(Q_COMM_BYTES, np.int64, 2))

    def proxies(self, node):
        n_p = 4096 if self.d == 2 else 6144
        return None if node < 0 else _proxies(self, node)


def _proxies(h, node, n_proxy=None):
    import torch
    n_p = n_proxy or (4096 if h.d == 2 else 6144)
    out = np.zeros((n_p, h.d))
    _check(lib().spd_test_proxies(h.ptr, node, out.ctypes.data_as(ctypes.c_void_p), _stream()))
    return out


class Comm:
    """Communicator (spd_comm_init).  Caller-owned; keep it alive while handles use it."""

    def __init__(self, nranks=1, rank=0, unique_id=None):
        self.ptr = ctypes.c_void_p()
        uid = None
        if unique_id is not None:
            uid = ctypes.create_string_buffer(bytes(unique_id), 128)
        _check(lib().spd_comm_init(uid, int(nranks), int(rank), ctypes.byref(self.ptr)))
        self.nranks, self.rank = nranks, rank

    def __del__(self):
        if getattr(self, "ptr", None) and _lib is not None:
            _lib.spd_comm_free(self.ptr)
            self.ptr = None


_F64CB = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.c_size_t)
_I32CB = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int), ctypes.c_size_t)
_BCB = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int)


class _HostColl(ctypes.Structure):
    _fields_ = [("ctx", ctypes.c_void_p), ("allreduce_sum_f64", _F64CB), ("allreduce_sum_i32", _I32CB),
                ("broadcast", _BCB)]


class HostComm(Comm):
    """Host-staged communicator (spd_comm_init_host): the library's sharded path with
    every exchange done by torch.distributed on host tensors (any backend that takes
    CPU tensors, e.g. gloo).  For tests of the sharded path in several processes
    (possibly sharing one GPU); NCCL (Comm) is the production transport."""

    def __init__(self, group=None):
        import numpy as np
        import torch
        import torch.distributed as dist
        self.ptr = ctypes.c_void_p()
        nranks, rank = dist.get_world_size(group), dist.get_rank(group)

        def view(ptr, n, ctype, dtype):
            return torch.from_numpy(np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(ctype)), (n,)))

        def f64(_ctx, buf, n):
            try:
                dist.all_reduce(view(buf, n, ctypes.c_double, None), group=group)
                return 0
            except Exception:          # noqa: BLE001 -- reported to the library as a failed collective
                return 1

        def i32(_ctx, buf, n):
            try:
                dist.all_reduce(view(buf, n, ctypes.c_int, None), group=group)
                return 0
            except Exception:          # noqa: BLE001
                return 1

        def bcast(_ctx, buf, nbytes, root):
            try:
                src = dist.get_global_rank(group, root) if group is not None else root
                dist.broadcast(view(buf, nbytes, ctypes.c_uint8, None), src=src, group=group)
                return 0
            except Exception:          # noqa: BLE001
                return 1

        self._cbs = (_F64CB(f64), _I32CB(i32), _BCB(bcast))      # kept alive with the communicator
        self._ops = _HostColl(None, *self._cbs)
        _check(lib().spd_comm_init_host(ctypes.byref(self._ops), int(nranks), int(rank), ctypes.byref(self.ptr)))
        self.nranks, self.rank = nranks, rank


def comm_unique_id():
    """128-byte NCCL unique id (rank 0), to be shared with the other ranks."""
    buf = ctypes.create_string_buffer(128)
    _check(lib().spd_comm_unique_id(buf))
    return buf.raw


def shard_owner(nranks, count, a):
    """Owner rank of node a of a level with `count` nodes (-1: computed by every rank)."""
    return int(lib().spd_test_shard_owner(int(nranks), int(count), int(a)))


def h2_build(points, kernel_id, ell, shift, leaf, tol, n_proxy=0, comm=None, inject_skeletons=None):
    """points: CUDA float64 (n, d) row-major, original order.  comm: optional Comm
    (subtree-sharded build; every rank ends with the full H2).  inject_skeletons:
    optional dict node -> skeleton tree positions in pivot order for every node at
    levels 1..L-1 (missing nodes: 0), the parity hook of reading R19."""
    if points.dim() != 2 or not points.is_contiguous():
        raise ValueError("points must be a contiguous (n, d) tensor")
    n, d = points.shape
    out = ctypes.c_void_p()
    opts = _H2Opts(int(n_proxy), 0, None)
    if inject_skeletons is not None:
        flat = []
        depth = 0                                  # tree depth of reading R1
        while int(leaf) << depth < n:
            depth += 1
        L = depth + 1
        for i in range((1 << L) - 1):
            if _node_level(i, L) >= L:
                continue
            s = [int(v) for v in inject_skeletons.get(i, [])]
            flat.append(len(s))
            flat.extend(s)
        inj = np.ascontiguousarray(np.array(flat + [0], dtype=np.int32))
        opts.inject_skeletons = inj.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    _check(lib().h2_build(_dptr(points, "points"), n, d, _Kernel(int(kernel_id), float(ell), float(shift)),
                          int(leaf), float(tol), ctypes.byref(opts), comm.ptr if comm is not None else None,
                          _stream(), ctypes.byref(out)))
    h = H2(out, n * (3 if int(kernel_id) == K_RPY else 1), d)      # operator rows (RPY: 3 dofs per point)
    h._comm = comm            # keep the communicator alive as long as the handle
    return h


def _node_level(i, L):
    """Paper level of heap node i in a perfect tree of depth L (root = L, leaves = 1)."""
    return L - ((i + 1).bit_length() - 1)


def h2_matvec(h2, X, layout=LAYOUT_ORIGINAL, out=None):
    x, ldx, k = _mat(X, "X")
    if out is None:
        out = empty_colmajor(h2.n, k) if X.dim() == 2 else X.new_empty(X.shape)
    y, ldy, _ = _mat(out, "out")
    _check(lib().h2_matvec(h2.ptr, layout, x, ldx, y, ldy, k, _stream()))
    return out


class HSS:
    """Handle of an SPD HSS approximation (spdhss_build)."""

    def __init__(self, ptr, h2):
        self.ptr = ptr
        self.h2 = h2          # keeps the H2 alive (freed after the HSS)

    def __del__(self):
        if getattr(self, "ptr", None) and _lib is not None:
            _lib.hss_free(self.ptr)
            self.ptr = None

    def query(self, what, dtype, count):
        buf = np.zeros(count, dtype=dtype)
        _check(lib().spd_query(self.ptr, what, buf.ctypes.data_as(ctypes.c_void_p), buf.nbytes))
        return buf

    def ranks(self):
        return self.query(Q_HSS_RANKS, np.int32, self.h2.nnodes)

    def export(self):
        size = int(self.query(Q_HSS_EXPORT_SIZE, np.int64, 1)[0])
        return self.query(Q_HSS_EXPORT, np.float64, max(1, size))

    def timings(self):
        return self.query(Q_TIMINGS, np.float64, 16)

    def pivots(self, w):
        """QRCP pivots of every node at levels 1..L-1 in heap order: dict node -> (w,)."""
        L, nn = self.h2.levels, self.h2.nnodes
        nodes = [i for i in range(nn) if _node_level(i, L) < L]
        flat = self.query(Q_HSS_PIVOTS, np.int32, max(1, len(nodes) * w))
        order = [i for k in range(1, L) for i in nodes if _node_level(i, L) == k]
        return {i: flat[a * w:(a + 1) * w].astype(np.int64) for a, i in enumerate(order)}

    def shard_work(self):
        """(nodes whose per-node work this process computed, nodes with per-node work)."""
        return tuple(int(v) for v in self.query(Q_SHARD_WORK, np.int64, 2))


def spdhss_build(h2, rank_cap, rel_tol, oversample=10, seed=0, omega=None):
    out = ctypes.c_void_p()
    om = None
    if omega is not None:
        om, ld, w = _mat(omega, "omega")
        if ld != h2.n or w != rank_cap + oversample:
            raise ValueError("omega must be n x (rank_cap + oversample) with ld = n")
    _check(lib().spdhss_build(h2.ptr, int(rank_cap), float(rel_tol), int(oversample), int(seed), om,
                              _stream(), ctypes.byref(out)))
    return HSS(out, h2)


def spdhss_build_adaptive(h2, r0, r_max, rel_tol, oversample=10, seed=0, omega=None):
    """Threshold-driven SPD-HSS (restart form).  Returns (HSS, cap used).
    omega: optional n x (r_max + oversample) tree-order sketch."""
    out = ctypes.c_void_p()
    cap = ctypes.c_int(0)
    om = None
    if omega is not None:
        om, ld, w = _mat(omega, "omega")
        if ld != h2.n or w != r_max + oversample:
            raise ValueError("omega must be n x (r_max + oversample) with ld = n")
    _check(lib().spdhss_build_adaptive(h2.ptr, int(r0), int(r_max), float(rel_tol), int(oversample), int(seed), om,
                                       _stream(), ctypes.byref(out), ctypes.byref(cap)))
    return HSS(out, h2), cap.value


def hss_solve(hss, B, layout=LAYOUT_ORIGINAL, out=None):
    b, ldb, k = _mat(B, "B")
    if out is None:
        out = empty_colmajor(hss.h2.n, k) if B.dim() == 2 else B.new_empty(B.shape)
    x, ldx, _ = _mat(out, "out")
    _check(lib().hss_solve(hss.ptr, layout, b, ldb, x, ldx, k, _stream()))
    return out


def hss_matvec(hss, X, layout=LAYOUT_ORIGINAL, out=None):
    """Y = H X with the SPD-HSS matrix (not its inverse)."""
    x, ldx, k = _mat(X, "X")
    if out is None:
        out = empty_colmajor(hss.h2.n, k) if X.dim() == 2 else X.new_empty(X.shape)
    y, ldy, _ = _mat(out, "out")
    _check(lib().hss_matvec(hss.ptr, layout, x, ldx, y, ldy, k, _stream()))
    return out


def pcg_solve(h2, hss, b, tol=1e-8, maxit=3000, layout=LAYOUT_ORIGINAL, x=None, precond="hss"):
    """Returns (x, PcgReport).  hss=None: unpreconditioned CG.  precond="bj": block
    Jacobi from the SPD-HSS leaf factors (the paper's BJ baseline)."""
    n = h2.n
    if b.dim() != 1 or not b.is_contiguous() or b.numel() != n:
        raise ValueError(f"b must be a contiguous 1-D tensor of length n = {n}")
    if x is None:
        x = b.new_zeros(b.shape)
    if x.dim() != 1 or not x.is_contiguous() or x.numel() != n:
        raise ValueError(f"x must be a contiguous 1-D tensor of length n = {n}")
    rep = PcgReport()
    fn = lib().pcg_solve_bj if precond == "bj" else lib().pcg_solve
    _check(fn(h2.ptr, hss.ptr if hss is not None else None, layout, _dptr(b, "b"),
              _dptr(x, "x"), float(tol), int(maxit), ctypes.byref(rep), _stream()))
    return x, rep


def philox_normal(n, w, seed):
    """Test export: the device Omega generator of spdhss_build (n x w column-major)."""
    import torch
    out = torch.empty((w, n), dtype=torch.float64, device="cuda").t()
    _check(lib().spd_test_philox_normal(ctypes.c_void_p(out.data_ptr()), int(n), int(w), int(seed), _stream()))
    return out


def tree_host(points, leaf):
    """Test export: the host tree / list builder on host points (n, d):
    (perm, boxes (nnodes, 2, d), list counts (1 + 2L))."""
    pts = np.ascontiguousarray(points, dtype=np.float64)
    n, d = pts.shape
    depth = 0
    while int(leaf) << depth < n:
        depth += 1
    L, nn = depth + 1, (1 << (depth + 1)) - 1
    perm = np.zeros(n, np.int64)
    boxes = np.zeros((nn, 2, d))
    counts = np.zeros(1 + 2 * L, np.int64)
    vp = ctypes.c_void_p
    _check(lib().spd_test_tree_host(vp(pts.ctypes.data), n, d, int(leaf), vp(perm.ctypes.data),
                                    vp(boxes.ctypes.data), vp(counts.ctypes.data)))
    return perm, boxes, counts
