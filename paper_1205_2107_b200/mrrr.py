"""Thin Python binding of the C ABI in include/mrrr.h (argument marshalling
only; every step of the solve runs in libmrrr_b200.so's CUDA kernels).

torch is used for device memory and streams only.  There is no CPU fallback:
importing the binding without the built library, or calling it without a
CUDA device, raises.
"""
from __future__ import annotations

import ctypes as C
import os

# Hardware work queues for the solve's streams (csrc/mrrr.cu, mrrr_on_load): read by
# the driver when the CUDA context is created, so it is set at import time, before
# torch initialises CUDA; a value the caller has set is kept.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import torch  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libmrrr_b200.so")

RANGE_ALL, RANGE_INDEX, RANGE_VALUE = 0, 1, 2


class Opts(C.Structure):
    _fields_ = [("tol_relgap", C.c_double), ("rtol_class", C.c_double), ("max_depth", C.c_int),
                ("perturb_root", C.c_int), ("seed", C.c_uint64), ("multisection", C.c_int),
                ("grid_factor", C.c_int), ("rtol_vec", C.c_double), ("rqc_max", C.c_int),
                ("shift_strategy", C.c_int), ("scratch_gb", C.c_double)]


class Stats(C.Structure):
    _fields_ = [("nodes", C.c_int64), ("levels", C.c_int64), ("singletons", C.c_int64),
                ("root_sweeps", C.c_int64), ("refine_sweeps", C.c_int64),
                ("child_sweeps", C.c_int64), ("rqc_iters", C.c_int64),
                ("rqc_fallbacks", C.c_int64), ("safe_resweeps", C.c_int64),
                ("kernel_launches", C.c_int64), ("ms_root", C.c_double), ("ms_tree", C.c_double),
                ("ms_vectors", C.c_double), ("ms_total", C.c_double),
                ("ms_k_root_bisect", C.c_double), ("ms_k_vectors", C.c_double),
                ("vec_tasks", C.c_int64), ("vec_elems", C.c_int64),
                ("ms_k_final_refine", C.c_double), ("vec_nudges", C.c_int64),
                ("vec_items", C.c_int64), ("pool_bytes", C.c_int64), ("workspace_bytes", C.c_int64),
                ("z_copies", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)

_lib = None


class MrrrError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"mrrr error {code}: {msg}")
        self.code = code


def lib():
    """Load libmrrr_b200.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(SO):
            raise RuntimeError(f"{SO} missing: run `python -m paper_1205_2107_b200.build` "
                               "(no CPU fallback exists)")
        L = C.CDLL(SO)
        L.mrrr_default_opts.argtypes = [C.POINTER(Opts)]
        L.mrrr_stemr.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_int, C.c_double, C.c_double,
                                 C.c_int64, C.c_int64, C.POINTER(C.c_int64), C.c_void_p, C.c_void_p,
                                 C.c_int64, C.c_void_p, C.POINTER(Opts)]
        L.mrrr_stemr.restype = C.c_int
        L.mrrr_stemr_host.argtypes = L.mrrr_stemr.argtypes
        L.mrrr_stemr_host.restype = C.c_int
        L.mrrr_stemr_dist.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_int, C.c_double,
                                      C.c_double, C.c_int64, C.c_int64, C.c_int, C.c_int,
                                      ALLGATHER_FN, C.c_void_p, C.POINTER(C.c_int64),
                                      C.POINTER(Opts), C.POINTER(C.c_int64),
                                      C.POINTER(C.c_int64), C.c_void_p, C.c_void_p, C.c_int64,
                                      C.c_void_p]
        L.mrrr_stemr_dist.restype = C.c_int
        L.mrrr_stemr_nccl.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_int, C.c_double,
                                      C.c_double, C.c_int64, C.c_int64, C.c_void_p,
                                      C.POINTER(C.c_int64), C.POINTER(Opts), C.POINTER(C.c_int64),
                                      C.POINTER(C.c_int64), C.c_void_p, C.c_void_p, C.c_int64,
                                      C.c_void_p]
        L.mrrr_stemr_nccl.restype = C.c_int
        L.mrrr_workspace_bytes.argtypes = [C.c_int64, C.c_int64]
        L.mrrr_workspace_bytes.restype = C.c_size_t
        L.mrrr_strerror.argtypes = [C.c_int]
        L.mrrr_strerror.restype = C.c_char_p
        L.mrrr_get_stats.argtypes = [C.POINTER(Stats)]
        L.mrrr_get_stats.restype = C.c_int
        L.mrrr_version.restype = C.c_char_p
        L.mrrr_negcount.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                    C.c_void_p, C.c_int, C.c_void_p]
        L.mrrr_negcount.restype = C.c_int
        L.mrrr_plan_columns.argtypes = [C.c_int64, C.c_int, C.c_void_p, C.c_void_p]
        L.mrrr_plan_columns.restype = C.c_int
        L.mrrr_trim_workspace.restype = C.c_int
        L.mrrr_get_rqc_histogram.argtypes = [C.POINTER(C.c_int64)]
        L.mrrr_get_rqc_histogram.restype = C.c_int
        _lib = L
    return _lib


def default_opts(**kw) -> Opts:
    o = Opts()
    lib().mrrr_default_opts(C.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def last_stats() -> dict:
    st = Stats()
    lib().mrrr_get_stats(C.byref(st))
    return st.as_dict()


def _range_args(n, il, iu, vl, vu):
    if il is not None or iu is not None:
        return RANGE_INDEX, 0.0, 0.0, int(il), int(iu), max(0, int(iu) - int(il) + 1)
    if vl is not None or vu is not None:
        return RANGE_VALUE, float(vl), float(vu), 0, 0, n
    return RANGE_ALL, 0.0, 0.0, 0, 0, n


def _check_out(t, k, device, name, n=None):
    """Caller-supplied output buffers: float64, contiguous, on d's device, with
    room for k eigenvalues (w) or k columns of length n (Z as (k', n), k' >= k)."""
    if t.dtype != torch.float64 or not t.is_contiguous() or t.device != device:
        raise TypeError(f"{name} must be a contiguous float64 tensor on {device}")
    if n is None:
        if t.numel() < k:
            raise ValueError(f"{name} holds {t.numel()} < {k} eigenvalues")
    elif t.dim() != 2 or t.shape[1] != n or t.shape[0] < k:
        raise ValueError(f"{name} must have shape (>= {k}, {n}) (column j of the result is row j)")


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def stemr(d: torch.Tensor, e: torch.Tensor, *, il=None, iu=None, vl=None, vu=None,
          vectors: bool = True, opts: Opts | None = None, w: torch.Tensor | None = None,
          Z: torch.Tensor | None = None, stream=None):
    """Eigenpairs of tridiag(e, d, e) on the GPU of ``d`` (torch.float64 CUDA
    tensors).  Returns ``(w, Z)``: ``w`` ascending (m,), ``Z`` (n, m) with unit
    eigenvector columns (a transposed view of column-major storage), or
    ``None`` when ``vectors=False``.  ``w``/``Z`` may be preallocated: w of
    capacity k and Z as a contiguous (k, n) tensor (column j of the result is
    row j of the buffer)."""
    if not (d.is_cuda and d.dtype == torch.float64):
        raise TypeError("d must be a torch.float64 CUDA tensor (no CPU fallback)")
    n = d.shape[0]
    if n > 1 and not (e.is_cuda and e.dtype == torch.float64 and e.device == d.device):
        raise TypeError("e must be a torch.float64 CUDA tensor on d's device")
    d = d.contiguous()
    e = e.contiguous() if n > 1 else d
    rng, a, b, ilv, iuv, kcap = _range_args(n, il, iu, vl, vu)
    kcap = max(kcap, 1)
    if stream is None:
        stream = torch.cuda.current_stream(d.device)
    if rng == RANGE_VALUE and vectors and Z is None:
        # size Z to the eigenvalues in (vl, vu]: a values-only solve counts them
        # first (instead of an n x n buffer: 80 GB at n = 1e5)
        wv, _ = stemr(d, e, vl=vl, vu=vu, vectors=False, opts=opts, stream=stream)
        kcap = max(int(wv.shape[0]), 1)
    if w is None:
        w = torch.empty(kcap, dtype=torch.float64, device=d.device)
    if vectors and Z is None:
        Z = torch.empty((kcap, n), dtype=torch.float64, device=d.device)
    _check_out(w, kcap, d.device, "w")
    if vectors:
        _check_out(Z, kcap, d.device, "Z", n)
    m = C.c_int64(0)
    o = opts if opts is not None else default_opts()
    with torch.cuda.device(d.device):
        rc = lib().mrrr_stemr(n, _ptr(d), _ptr(e), rng, a, b, ilv, iuv, C.byref(m), _ptr(w),
                              _ptr(Z) if vectors else C.c_void_p(0), n,
                              C.c_void_p(stream.cuda_stream), C.byref(o))
    if rc != 0:
        raise MrrrError(rc, lib().mrrr_strerror(rc).decode())
    k = m.value
    return w[:k], (Z[:k].T if vectors else None)


def stemr_host(d, e, *, il=None, iu=None, vl=None, vu=None, w=None, Z=None, vectors=True,
               opts: Opts | None = None, stream=None):
    """End-to-end entry on HOST tensors (``mrrr_stemr_host``): float64 CPU
    tensors ``d``, ``e`` (pinned for speed); returns host ``(w, Z)`` with the
    same layout as :func:`stemr`.  The copies and the solve run inside the
    library on ``stream`` (default: the current CUDA stream)."""
    n = d.shape[0]
    for t, nm in ((d, "d"), (e, "e")):
        if nm == "e" and n <= 1:
            continue
        if t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
            raise TypeError(f"stemr_host takes contiguous float64 host tensors ({nm})")
    if n > 1 and e.shape[0] < n - 1:
        raise ValueError("e needs n - 1 entries")
    rng, a, b, ilv, iuv, kcap = _range_args(n, il, iu, vl, vu)
    kcap = max(kcap, 1)
    if w is None:
        w = torch.empty(kcap, dtype=torch.float64, pin_memory=True)
    if vectors and Z is None:
        Z = torch.empty((kcap, n), dtype=torch.float64, pin_memory=True)
    for t, nm, nn in ((w, "w", None), (Z if vectors else None, "Z", n)):
        if t is None:
            continue
        if t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
            raise TypeError(f"{nm} must be a contiguous float64 host tensor")
        if (nn is None and t.numel() < kcap) or (nn is not None and (t.dim() != 2 or t.shape[1] != n or t.shape[0] < kcap)):
            raise ValueError(f"{nm} is too small for {kcap} eigenpairs")
    if stream is None:
        stream = torch.cuda.current_stream()
    m = C.c_int64(0)
    o = opts if opts is not None else default_opts()
    e = e if n > 1 else d
    rc = lib().mrrr_stemr_host(n, _ptr(d), _ptr(e), rng, a, b, ilv, iuv, C.byref(m), _ptr(w),
                               _ptr(Z) if vectors else C.c_void_p(0), n,
                               C.c_void_p(stream.cuda_stream), C.byref(o))
    if rc != 0:
        raise MrrrError(rc, lib().mrrr_strerror(rc).decode())
    k = m.value
    return w[:k], (Z[:k].T if vectors else None)


def plan_columns(m: int, nranks: int, free_cut) -> list:
    """The library's shard planner (``mrrr_plan_columns``): the column cuts
    [c_0 = 0, ..., c_P = m] after moving each static cut to the nearest
    cluster boundary (``free_cut[j]`` true: boundary between columns j-1, j)
    within ceil(m/P)/40.  Host only."""
    fc = (C.c_ubyte * (m + 1))(*[1 if x else 0 for x in list(free_cut)[:m + 1]] + [0] * max(0, m + 1 - len(free_cut)))
    cuts = (C.c_int64 * (nranks + 1))()
    rc = lib().mrrr_plan_columns(m, nranks, C.cast(fc, C.c_void_p), C.cast(cuts, C.c_void_p))
    if rc != 0:
        raise MrrrError(rc, lib().mrrr_strerror(rc).decode())
    return list(cuts)


def dist_capacity(k: int, nranks: int) -> int:
    """Columns Z_local must hold: ceil(k/P) + ceil(k/P)/20 (the planner's slack)."""
    epp = (k + max(nranks, 1) - 1) // max(nranks, 1)
    return max(epp + epp // 20, 1)


def shard_columns(m: int, nranks: int, rank: int):
    """Columns [c0, c1) of the m wanted eigenpairs owned by `rank` (the static
    division of PAPER.md L1139-1146 as mrrr_stemr_dist applies it:
    epp = ceil(m / nranks), c0 = rank * epp)."""
    epp = (m + nranks - 1) // nranks
    c0 = min(rank * epp, m)
    return c0, min(c0 + epp, m)


class _DevBuf:
    """Zero-copy view of a device buffer for torch.as_tensor: fp64 by default,
    bytes with ``typestr="|u1"`` (the library's exchanges are byte counts)."""

    def __init__(self, ptr: int, nbytes: int, typestr: str = "<f8"):
        size = nbytes if typestr == "|u1" else nbytes // 8
        self.__cuda_array_interface__ = {"shape": (size,), "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None}


def _ext_stream(handle):
    """torch stream object for a raw cudaStream_t handle (0/None: the legacy default stream)."""
    return torch.cuda.ExternalStream(handle) if handle else torch.cuda.default_stream()


def _host_bytes(ptr: int, nbytes: int):
    arr = (C.c_uint8 * nbytes).from_address(ptr)
    return torch.frombuffer(arr, dtype=torch.uint8)


def _host_view(ptr: int, nbytes: int):
    arr = (C.c_double * (nbytes // 8)).from_address(ptr)
    return torch.frombuffer(arr, dtype=torch.float64)


def torch_allgather(group=None, device: str = "cuda"):
    """An mrrr_allgather_fn over torch.distributed: recv[r * bytes ...] <- rank
    r's send (bytes each).  device="cuda": the library's device buffers, NCCL
    over NVLink; device="cpu": host buffers (gloo; used by the CPU tests of
    the exchange).  Returns the ctypes callback (keep a reference while the
    call runs)."""
    import torch.distributed as dist

    def fn(ctx, send, recv, nbytes, stream):
        try:
            if nbytes == 0:
                return 0
            world = dist.get_world_size(group)
            if device == "cuda":
                # enqueued on the library's stream (the callback's contract,
                # include/mrrr.h): ordered after the kernels that wrote `send`
                # and before the library's reads of `recv`
                with torch.cuda.stream(_ext_stream(stream)):
                    st = torch.as_tensor(_DevBuf(send, nbytes, "|u1"), device="cuda")
                    rt = torch.as_tensor(_DevBuf(recv, nbytes * world, "|u1"), device="cuda")
                    dist.all_gather_into_tensor(rt, st, group=group)
            else:
                st = _host_bytes(send, nbytes)
                parts = [torch.empty_like(st) for _ in range(world)]
                dist.all_gather(parts, st, group=group)
                _host_bytes(recv, nbytes * world).copy_(torch.cat(parts))
            return 0
        except Exception:  # reported as MRRR_ERR_COMM by the library
            return 1
    return ALLGATHER_FN(fn)


def stemr_dist(d: torch.Tensor, e: torch.Tensor, *, il=None, iu=None, vl=None, vu=None,
               vectors: bool = True, opts: Opts | None = None, group=None, rank=None,
               nranks=None, allgather=None, stream=None):
    """Sharded MRRR (``mrrr_stemr_dist``): every rank passes the
    same T and range; returns ``(w_all, Z_local, col_begin)`` where ``w_all``
    holds all m eigenvalues on every rank and ``Z_local`` (n, m_local) the
    eigenvectors of columns ``col_begin .. col_begin + m_local`` (this rank's
    share: the static division with its cuts moved to cluster boundaries).
    The collectives (root grid, root brackets, one bracket exchange per tree
    level, w) go through ``allgather`` (torch.distributed NCCL by default)."""
    import torch.distributed as dist
    if not (d.is_cuda and d.dtype == torch.float64):
        raise TypeError("d must be a torch.float64 CUDA tensor (no CPU fallback)")
    n = d.shape[0]
    if rank is None:
        rank = dist.get_rank(group)
    if nranks is None:
        nranks = dist.get_world_size(group)
    d = d.contiguous()
    e = e.contiguous() if n > 1 else d
    rng, a, b, ilv, iuv, kcap = _range_args(n, il, iu, vl, vu)
    kcap = max(kcap, 1)
    w_all = torch.empty(kcap, dtype=torch.float64, device=d.device)
    Zl = torch.empty((dist_capacity(kcap, nranks), n), dtype=torch.float64, device=d.device) if vectors else None
    if stream is None:
        stream = torch.cuda.current_stream(d.device)
    cb = allgather if allgather is not None else torch_allgather(group)
    m = C.c_int64(0)
    c0 = C.c_int64(0)
    ml = C.c_int64(0)
    o = opts if opts is not None else default_opts()
    with torch.cuda.device(d.device):
        rc = lib().mrrr_stemr_dist(n, _ptr(d), _ptr(e), rng, a, b, ilv, iuv, int(rank), int(nranks),
                                   cb, None, C.byref(m), C.byref(o), C.byref(c0), C.byref(ml),
                                   _ptr(w_all), _ptr(Zl) if vectors else C.c_void_p(0), n,
                                   C.c_void_p(stream.cuda_stream))
    if rc != 0:
        raise MrrrError(rc, lib().mrrr_strerror(rc).decode())
    k = m.value
    return w_all[:k], (Zl[:ml.value].T if vectors else None), c0.value


class _NcclUniqueId(C.Structure):
    _fields_ = [("internal", C.c_char * 128)]  # nccl.h: NCCL_UNIQUE_ID_BYTES


_nccl = None


def _nccl_lib():
    """The NCCL the process already has (torch's bundled libnccl.so.2), else
    the loader path's -- the same one mrrr_stemr_nccl resolves."""
    global _nccl
    if _nccl is None:
        mode = getattr(os, "RTLD_NOLOAD", 4) | os.RTLD_NOW
        try:
            L = C.CDLL("libnccl.so.2", mode=mode)
        except OSError:
            L = C.CDLL("libnccl.so.2")
        L.ncclGetUniqueId.argtypes = [C.POINTER(_NcclUniqueId)]
        L.ncclCommInitRank.argtypes = [C.POINTER(C.c_void_p), C.c_int, _NcclUniqueId, C.c_int]
        L.ncclCommDestroy.argtypes = [C.c_void_p]
        for f in (L.ncclGetUniqueId, L.ncclCommInitRank, L.ncclCommDestroy):
            f.restype = C.c_int
        _nccl = L
    return _nccl


def broadcast_bytes(payload: bytes, rank: int, group=None, device=None) -> bytes:
    """Rank 0's ``payload`` on every rank of ``group`` (the ncclUniqueId
    bootstrap of :class:`NcclComm`; a gloo group broadcasts host memory, an
    nccl group the bytes staged on ``device``)."""
    import torch.distributed as dist
    t = torch.frombuffer(bytearray(payload if rank == 0 else bytes(len(payload))), dtype=torch.uint8)
    if dist.get_backend(group) == "nccl":
        t = t.to(device)
    dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return t.cpu().numpy().tobytes()


class NcclComm:
    """An ncclComm_t owned by the caller of :func:`stemr_nccl` (SURVEY §8(b):
    the communicator is bootstrapped by broadcasting the ncclUniqueId through
    a torch.distributed process group; torch is plumbing only).  ``group`` may
    be a gloo or nccl group; with ``nranks == 1`` no process group is needed."""

    def __init__(self, device, group=None, rank=None, nranks=None):
        import torch.distributed as dist
        self.handle = C.c_void_p(0)
        self.device = torch.device(device)
        if rank is None or nranks is None:
            if dist.is_available() and dist.is_initialized():
                rank, nranks = dist.get_rank(group), dist.get_world_size(group)
            else:
                rank, nranks = 0, 1
        self.rank, self.nranks = int(rank), int(nranks)
        uid = _NcclUniqueId()
        L = _nccl_lib()
        if self.rank == 0 and L.ncclGetUniqueId(C.byref(uid)) != 0:
            raise RuntimeError("ncclGetUniqueId failed")
        if self.nranks > 1:
            raw = broadcast_bytes(C.string_at(C.addressof(uid), 128), self.rank, group, self.device)
            C.memmove(C.byref(uid), raw, 128)
        with torch.cuda.device(self.device):
            rc = L.ncclCommInitRank(C.byref(self.handle), self.nranks, uid, self.rank)
        if rc != 0:
            raise RuntimeError(f"ncclCommInitRank failed ({rc})")

    def destroy(self):
        if self.handle:
            _nccl_lib().ncclCommDestroy(self.handle)
            self.handle = C.c_void_p(0)

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def stemr_nccl(d: torch.Tensor, e: torch.Tensor, comm: NcclComm, *, il=None, iu=None, vl=None, vu=None,
               vectors: bool = True, opts: Opts | None = None, stream=None):
    """Sharded MRRR on an NCCL communicator (``mrrr_stemr_nccl``): the library
    itself issues the protocol's ncclAllGather calls on ``stream``.  Returns
    ``(w_all, Z_local, col_begin)`` as :func:`stemr_dist`."""
    if not (d.is_cuda and d.dtype == torch.float64):
        raise TypeError("d must be a torch.float64 CUDA tensor (no CPU fallback)")
    if d.device != comm.device and not (d.device.index is None or comm.device.index is None):
        raise ValueError("the communicator belongs to another device than d")
    n = d.shape[0]
    d = d.contiguous()
    e = e.contiguous() if n > 1 else d
    rng, a, b, ilv, iuv, kcap = _range_args(n, il, iu, vl, vu)
    kcap = max(kcap, 1)
    w_all = torch.empty(kcap, dtype=torch.float64, device=d.device)
    Zl = torch.empty((dist_capacity(kcap, comm.nranks), n), dtype=torch.float64, device=d.device) if vectors else None
    if stream is None:
        stream = torch.cuda.current_stream(d.device)
    m = C.c_int64(0)
    c0 = C.c_int64(0)
    ml = C.c_int64(0)
    o = opts if opts is not None else default_opts()
    with torch.cuda.device(d.device):
        rc = lib().mrrr_stemr_nccl(n, _ptr(d), _ptr(e), rng, a, b, ilv, iuv, comm.handle,
                                   C.byref(m), C.byref(o), C.byref(c0), C.byref(ml), _ptr(w_all),
                                   _ptr(Zl) if vectors else C.c_void_p(0), n, C.c_void_p(stream.cuda_stream))
    if rc != 0:
        raise MrrrError(rc, lib().mrrr_strerror(rc).decode())
    return w_all[:m.value], (Zl[:ml.value].T if vectors else None), c0.value


def stemr_raw(n, d, e, rng, vl, vu, il, iu, m_ok=True, w=None, Z=None, ldz=None):
    """Direct C call for argument-validation tests (device pointers as tensors)."""
    m = C.c_int64(0)
    return lib().mrrr_stemr(n, _ptr(d), _ptr(e), rng, vl, vu, il, iu,
                            C.byref(m) if m_ok else C.cast(None, C.POINTER(C.c_int64)),
                            _ptr(w), _ptr(Z), ldz if ldz is not None else max(n, 1),
                            C.c_void_p(0), None)


def negcount(D: torch.Tensor, LLD: torch.Tensor, mu: torch.Tensor, mode: int = 0, stream=None):
    """Sturm counts N(mu_q) of the representation (D, LLD) by the library's
    bisection arithmetic (``mrrr_negcount``; mode 0 projective sweep, 1 the qd
    safe path, 2 the refinement's twisted count).  float64 CUDA tensors; returns an int64 CUDA tensor."""
    for t in (D, LLD, mu):
        if not (t.is_cuda and t.dtype == torch.float64):
            raise TypeError("negcount takes float64 CUDA tensors")
    D, LLD, mu = D.contiguous(), LLD.contiguous(), mu.contiguous()
    out = torch.empty(mu.shape[0], dtype=torch.int64, device=D.device)
    if stream is None:
        stream = torch.cuda.current_stream(D.device)
    with torch.cuda.device(D.device):
        rc = lib().mrrr_negcount(D.shape[0], _ptr(D), _ptr(LLD), mu.shape[0], _ptr(mu), _ptr(out),
                                 int(mode), C.c_void_p(stream.cuda_stream))
    if rc != 0:
        raise MrrrError(rc, lib().mrrr_strerror(rc).decode())
    return out


def rqc_histogram() -> list:
    """Eigenpairs of the last solve by the twisted factorizations their RQC
    took (``mrrr_get_rqc_histogram``; index k = factorizations, 15 = 15+)."""
    h = (C.c_int64 * 16)()
    lib().mrrr_get_rqc_histogram(h)
    return list(h)


def trim_workspace() -> None:
    """Release the library's cached device workspace (mrrr_trim_workspace)."""
    rc = lib().mrrr_trim_workspace()
    if rc != 0:
        raise MrrrError(rc, lib().mrrr_strerror(rc).decode())


def version() -> str:
    return lib().mrrr_version().decode()
