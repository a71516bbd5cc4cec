"""ctypes binding of libloopscout_b200.so (the C-ABI in include/loopscout_b200.h).

Device buffers are torch CUDA tensors (PyTorch is plumbing here: allocation,
streams, copies); all compute is in the library's sm_100a kernels.  There is
no CPU fallback: if the library or a GPU is missing, every entry point raises.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from . import abi

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libloopscout_b200.so"


class EngineError(RuntimeError):
    pass


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise EngineError(f"{LIB_PATH.name} is not built; run __graft_entry__.build() "
                          "(there is no CPU fallback)")
    L = C.CDLL(str(LIB_PATH))
    vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int32
    L.ls_last_error.restype = C.c_char_p
    L.ls_task_create.argtypes = [vp, C.c_int, C.POINTER(vp)]
    L.ls_task_destroy.argtypes = [vp]
    L.ls_task_num_features.argtypes = [vp]
    L.ls_task_prepare_unroll.argtypes = [vp, vp, i32]
    L.ls_collect_unroll.argtypes = [vp, vp, i64, vp, i32, vp, vp]
    L.ls_inexact_footprints.argtypes = [vp, vp, i64, vp, vp, vp, vp]
    L.ls_score.argtypes = [vp, vp, i64, vp, vp, vp, vp]
    L.ls_score_topk.argtypes = [vp, vp, i64, i64, i32, vp, vp, vp, vp]
    L.ls_topk_merge.argtypes = [vp, vp, i32, i32, i32, vp, vp, vp]
    L.ls_topk_merge_keys.argtypes = [vp, i64, i32, vp, vp, vp]
    L.ls_topk_allgather_merge.argtypes = [vp, i32, i32, vp, vp, i32, vp, vp, vp, vp]
    L.ls_topk_to_keys.argtypes = [vp, vp, i64, vp, vp]
    L.ls_score_topk_host.argtypes = [vp, vp, i64, i64, i32, vp, vp, vp, vp]
    L.ls_task_set_path.argtypes = [vp, i32]
    L.ls_task_set_space.argtypes = [vp, vp]
    L.ls_score_points.argtypes = [vp, vp, i32, i64, vp, vp, vp, vp]
    L.ls_score_topk_points.argtypes = [vp, vp, i32, i64, i64, i32, vp, vp, vp, vp]
    L.ls_score_topk_points_host.argtypes = [vp, vp, i32, i64, i64, i32, vp, vp, vp, vp]
    L.ls_task_path.argtypes = [vp]
    L.ls_task_points_path.argtypes = [vp]
    L.ls_es_create.argtypes = [vp, vp, vp, C.POINTER(vp)]
    L.ls_es_create_shard.argtypes = [vp, vp, vp, i32, i32, C.POINTER(vp)]
    L.ls_es_begin.argtypes = [vp, vp]
    L.ls_es_step.argtypes = [vp, i32, vp]
    L.ls_es_shard_buffers.argtypes = [vp, vp, vp, vp, vp]
    L.ls_es_run.argtypes = [vp, vp]
    L.ls_es_result.argtypes = [vp, vp, vp, vp, vp, vp, vp]
    L.ls_es_evaluated.argtypes = [vp, vp, vp, i64, vp, vp]
    L.ls_es_noise.argtypes = [vp, i32, vp, vp]
    L.ls_es_sort_state.argtypes = [vp, vp, vp, vp, vp, vp]
    L.ls_es_destroy.argtypes = [vp]
    if L.ls_abi_version() != abi.ABI_VERSION:
        raise EngineError("libloopscout_b200 ABI version mismatch")
    _lib = L
    return L


def _check(rc: int, what: str):
    if rc != 0:
        raise EngineError(f"{what} failed ({rc}): {lib().ls_last_error().decode()}")


_cuda_ok = False


_TORCH = None  # the torch module once CUDA was found usable


def _torch():
    global _cuda_ok, _TORCH
    import torch
    if not _cuda_ok:  # checked once: the per-call wrappers stay a few microseconds
        if not torch.cuda.is_available():
            raise EngineError("no CUDA device visible (there is no CPU fallback)")
        _cuda_ok = True
        _TORCH = torch
    return torch


def _stream(torch, stream, device=None):
    """Raw cudaStream_t: `stream`, else the current stream of `device` (default: current device)."""
    if stream is not None:
        return stream.cuda_stream
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:
        return raw(torch.cuda.current_device() if device is None else device)
    return torch.cuda.current_stream(device).cuda_stream


def _outputs(torch, k, device):
    """Fresh (scores f64[k], indices i64[k], count i64[1]); pass out= to reuse buffers across calls."""
    return (torch.empty(k, dtype=torch.float64, device=device), torch.empty(k, dtype=torch.int64, device=device),
            torch.empty(1, dtype=torch.int64, device=device))


def _dptr(t):
    return None if t is None else t.data_ptr()


def _device_view(torch, ptr: int, n: int, dtype, device):
    """A CUDA tensor aliasing library-owned device memory (no copy; valid while the owner lives)."""
    class _Arr:  # __cuda_array_interface__ shim
        def __init__(self):
            typestr = {torch.int64: "<i8", torch.float64: "<f8"}[dtype]
            self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr, "data": (int(ptr), False),
                                             "version": 3, "strides": None}
    return torch.as_tensor(_Arr(), device=device)


def to_device_records(records: np.ndarray, device=0):
    """Upload packed records as a CUDA uint8 tensor of shape (n, 32)."""
    torch = _torch()
    raw = np.ascontiguousarray(records).view(np.uint8).reshape(-1, abi.RECORD_DTYPE.itemsize)
    return torch.from_numpy(raw).to(f"cuda:{device}", non_blocking=False)


class Task:
    """A device task: one program + schedule template + arch (+ launch)."""

    def __init__(self, desc: abi.TaskDesc, device: int = 0):
        _torch()
        self.device = device
        self.desc = desc
        self.family = desc.family
        self.nfeat = abi.NFEAT_CPU if desc.family == 0 else abi.NFEAT_GPU
        h = C.c_void_p()
        _check(lib().ls_task_create(C.addressof(desc), device, C.byref(h)), "ls_task_create")
        self._h = h
        self._host_points_fn = None
        self._host_out = None
        self._host_out_ptrs = None
        self.has_unroll = any(desc.xforms[i].kind == abi.XF_UNROLL for i in range(desc.n_xforms)) or \
            any(desc.nodes[i].kind == abi.NODE_LOOP and desc.nodes[i].unrolled for i in range(desc.n_nodes))

    def close(self):
        if getattr(self, "_h", None):
            lib().ls_task_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    # -- scoring path -----------------------------------------------------------------
    PATH_AUTO, PATH_GENERIC, PATH_TABULATED, PATH_SPACE = 0, 1, 2, 3

    def set_path(self, path: int):
        """Force a scoring kernel (all bit-identical; LS_PATH_* in include/loopscout_b200.h)."""
        _check(lib().ls_task_set_path(self._h, int(path)), "ls_task_set_path")

    @property
    def path(self) -> int:
        """Path of the record calls (LS_PATH_GENERIC / LS_PATH_TABULATED)."""
        return lib().ls_task_path(self._h)

    @property
    def points_path(self) -> int:
        """Path of the points calls (LS_PATH_GENERIC / LS_PATH_TABULATED / LS_PATH_SPACE)."""
        return lib().ls_task_points_path(self._h)

    def inexact_footprints(self, d_records, stream=None, notes: bool = False):
        """Per record: 1 when the cache model's footprint intervals lose exactness (NodeCost.inexact,
        ls/cache.py:198-202), 0 exact, 255 the record fails apply_schedule (uint8 device tensor);
        with notes=True also the (loop, tensor) masks [n, 2] and the chains [n, 16] of the
        diagnostic (ls_inexact_footprints)."""
        torch = _torch()
        n, dev = int(d_records.shape[0]), f"cuda:{self.device}"
        out = torch.empty(n, dtype=torch.uint8, device=dev)
        masks = torch.empty((n, 2), dtype=torch.int64, device=dev) if notes else None
        chains = torch.empty((n, 16), dtype=torch.uint8, device=dev) if notes else None
        with torch.cuda.device(self.device):
            _check(lib().ls_inexact_footprints(self._h, _dptr(d_records), n, _dptr(out),
                                               _dptr(masks) if notes else None, _dptr(chains) if notes else None,
                                               _stream(torch, stream)), "ls_inexact_footprints")
        return (out, masks, chains) if notes else out

    # -- unroll table ---------------------------------------------------------------
    def prepare_unroll_for(self, d_records, stream=None):
        """Collect the innermost-unroll products these records need and precompute them."""
        if not self.has_unroll:
            return
        torch = _torch()
        n = d_records.shape[0]
        vals = np.zeros(16384, np.int64)
        cnt = np.zeros(1, np.int32)
        _check(lib().ls_collect_unroll(self._h, _dptr(d_records), n, vals.ctypes.data, len(vals),
                                       cnt.ctypes.data, _stream(torch, stream)), "ls_collect_unroll")
        u = vals[:cnt[0]].copy()
        if len(u):
            _check(lib().ls_task_prepare_unroll(self._h, u.ctypes.data, len(u)), "ls_task_prepare_unroll")

    # -- scoring --------------------------------------------------------------------
    def score(self, d_records, features: bool = True, stream=None):
        """(scores f64[n], features f64[n,F] | None, status i32[n]) as CUDA tensors."""
        torch = _torch()
        n = d_records.shape[0]
        dev = d_records.device
        scores = torch.empty(n, dtype=torch.float64, device=dev)
        feats = torch.empty((n, self.nfeat), dtype=torch.float64, device=dev) if features else None
        status = torch.empty(n, dtype=torch.int32, device=dev)
        _check(lib().ls_score(self._h, _dptr(d_records), n, _dptr(scores), _dptr(feats), _dptr(status),
                              _stream(torch, stream)), "ls_score")
        return scores, feats, status

    def score_topk(self, d_records, k: int, base_index: int = 0, stream=None, out=None):
        """k best (score, global index) ascending + number of valid candidates (CUDA tensors)."""
        torch = _torch()
        dev = d_records.device
        s, i, nv = out if out is not None else _outputs(torch, k, dev)  # the count is written by the launch
        _check(lib().ls_score_topk(self._h, _dptr(d_records), d_records.shape[0], int(base_index), int(k),
                                   _dptr(s), _dptr(i), _dptr(nv), _stream(torch, stream, dev.index)),
               "ls_score_topk")
        return s, i, nv

    def score_topk_host(self, h_records, k: int, base_index: int = 0, stream=None):
        """Host records in, host top-k out (H2D staged and overlapped inside the library)."""
        torch = _torch()
        if isinstance(h_records, np.ndarray):
            ptr, n = h_records.ctypes.data, len(h_records)
        else:  # pinned torch uint8 tensor (n, 32)
            ptr, n = h_records.data_ptr(), h_records.shape[0]
        s = np.empty(k, np.float64)
        i = np.empty(k, np.int64)
        nv = np.zeros(1, np.int64)
        _check(lib().ls_score_topk_host(self._h, ptr, n, int(base_index), int(k), s.ctypes.data,
                                        i.ctypes.data, nv.ctypes.data, _stream(torch, stream, self.device)),
               "ls_score_topk_host")
        return s, i, int(nv[0])


    # -- points API (candidates as space points) --------------------------------------
    def set_space(self, space: "abi.SpaceDesc"):
        """Attach a schedule space (pack.SpaceTemplate.space_desc()) for the points API."""
        _check(lib().ls_task_set_space(self._h, C.addressof(space)), "ls_task_set_space")

    def score_points(self, d_points, features: bool = True, stream=None):
        """ls_score over a CUDA tensor of space points: int32 / int64, or uint8 [n, 3] (packed
        3-byte points, pack.pack_points)."""
        torch = _torch()
        n, eb = _points_shape(d_points)
        dev = d_points.device
        scores = torch.empty(n, dtype=torch.float64, device=dev)
        feats = torch.empty((n, self.nfeat), dtype=torch.float64, device=dev) if features else None
        status = torch.empty(n, dtype=torch.int32, device=dev)
        _check(lib().ls_score_points(self._h, _dptr(d_points), eb, n, _dptr(scores),
                                     _dptr(feats), _dptr(status), _stream(torch, stream)), "ls_score_points")
        return scores, feats, status

    def score_topk_points(self, d_points, k: int, base_index: int = 0, stream=None, out=None):
        torch = _torch()
        dev = d_points.device
        n, eb = _points_shape(d_points)
        s, i, nv = out if out is not None else _outputs(torch, k, dev)  # the count is written by the launch
        _check(lib().ls_score_topk_points(self._h, _dptr(d_points), eb, n,
                                          int(base_index), int(k), _dptr(s), _dptr(i), _dptr(nv),
                                          _stream(torch, stream, dev.index)), "ls_score_topk_points")
        return s, i, nv

    def score_topk_points_host(self, h_points, k: int, base_index: int = 0, stream=None, out=None):
        """Host points (numpy uint32 / uint64 / uint8 [n, 3], or a pinned torch tensor) in, host
        top-k out; `out` = preallocated (f64[k], i64[k], i64[1]) numpy arrays."""
        if isinstance(h_points, np.ndarray):
            if not h_points.flags.c_contiguous:
                h_points = np.ascontiguousarray(h_points)
            ptr = h_points.ctypes.data
        else:
            ptr = h_points.data_ptr()
        n, eb = _points_shape(h_points)
        if out is None:
            out = (np.empty(k, np.float64), np.empty(k, np.int64), np.zeros(1, np.int64))
        s, i, nv = out
        if out is self._host_out:  # the caller's preallocated outputs: their addresses are cached
            sp, ip, nvp = self._host_out_ptrs
        else:
            sp, ip, nvp = s.ctypes.data, i.ctypes.data, nv.ctypes.data
            self._host_out, self._host_out_ptrs = out, (sp, ip, nvp)
        fn = self._host_points_fn
        if fn is None:  # (native call helper, address of the C entry point)
            try:
                from . import _packer  # csrc/packer.cpp (built by build.py)
                call = getattr(_packer, "call_points_host", None)
            except ImportError:
                call = None
            fn = self._host_points_fn = (call, C.cast(lib().ls_score_topk_points_host, C.c_void_p).value,
                                         self._h.value)
        call, addr, h = fn
        st = _stream(_TORCH or _torch(), stream, self.device)
        if call is not None:
            rc = call(addr, h, ptr, eb, n, base_index, k, sp, ip, nvp, st or 0)
        else:
            rc = lib().ls_score_topk_points_host(self._h, ptr, eb, n, base_index, k, sp, ip, nvp, st)
        if rc:
            _check(rc, "ls_score_topk_points_host")
        return s, i, int(nv[0])


def _points_shape(p):
    """(count, point_bytes) of a points buffer: 1-D 4/8-byte integers, or uint8 [n, 3]."""
    shape = p.shape
    if len(shape) == 2:
        if shape[1] != 3 or p.dtype not in (np.uint8, getattr(_TORCH, "uint8", None)):
            raise ValueError("2-D points must be packed uint8 [n, 3] (pack.pack_points)")
        return shape[0], 3
    eb = p.itemsize if isinstance(p, np.ndarray) else p.element_size()
    return shape[0], eb


def topk_merge(scores, index, n_lists: int, k_in: int, k_out: int, stream=None):
    """Merge n_lists (score, index) lists of k_in each into the k_out best (CUDA tensors)."""
    torch = _torch()
    out_s = torch.empty(k_out, dtype=torch.float64, device=scores.device)
    out_i = torch.empty(k_out, dtype=torch.int64, device=scores.device)
    _check(lib().ls_topk_merge(_dptr(scores), _dptr(index), int(n_lists), int(k_in), int(k_out),
                               _dptr(out_s), _dptr(out_i), _stream(torch, stream)), "ls_topk_merge")
    return out_s, out_i


def topk_to_keys(scores, index, out, stream=None):
    """Pack (score, index) lists into 16-byte ls_topk_key rows of `out` (int64 CUDA tensor [m, 2])."""
    torch = _torch()
    m = scores.shape[0]
    assert out.dtype == torch.int64 and out.shape[0] >= m and out.is_contiguous()
    _check(lib().ls_topk_to_keys(_dptr(scores), _dptr(index), m, _dptr(out), _stream(torch, stream)),
           "ls_topk_to_keys")
    return out


def topk_merge_keys(keys, k_out: int, out=None, stream=None):
    """Merge gathered ls_topk_key rows (int64 CUDA tensor [m, 2]) into the k_out best (score, index)."""
    torch = _torch()
    if out is None:
        out = (torch.empty(k_out, dtype=torch.float64, device=keys.device),
               torch.empty(k_out, dtype=torch.int64, device=keys.device))
    _check(lib().ls_topk_merge_keys(_dptr(keys), keys.shape[0], int(k_out), _dptr(out[0]), _dptr(out[1]),
                                    _stream(torch, stream)), "ls_topk_merge_keys")
    return out


def topk_allgather_merge(nccl_comm: int, rank: int, world: int, scores, index, k: int, scratch=None, out=None,
                         stream=None):
    """The C-ABI multi-GPU merge over a caller-owned NCCL communicator (ncclComm_t as an int):
    pack this rank's k best, one in-place ncclAllGather, the merge kernel (ls_topk_allgather_merge).
    torch.distributed users go through dist.gather_topk (same keys, same merge kernel)."""
    torch = _torch()
    dev = scores.device
    if scratch is None:
        scratch = torch.empty((world * k, 2), dtype=torch.int64, device=dev)
    if out is None:
        out = (torch.empty(k, dtype=torch.float64, device=dev), torch.empty(k, dtype=torch.int64, device=dev))
    _check(lib().ls_topk_allgather_merge(C.c_void_p(nccl_comm), int(rank), int(world), _dptr(scores), _dptr(index),
                                         int(k), _dptr(scratch), _dptr(out[0]), _dptr(out[1]),
                                         _stream(torch, stream, dev.index)), "ls_topk_allgather_merge")
    return out


class EsRun:
    """A device ES run over a task's attached space (ls_es_* in include/loopscout_b200.h).

    rank/world shard the population (ls_es_create_shard): drive it with run_sharded."""

    def __init__(self, task: Task, alpha: float, sigma: float, population: int, iterations: int, seed: int,
                 rank_normalize: bool = True, theta0=None, rank: int = 0, world: int = 1):
        self.task = task
        self.dim = None
        self.rank, self.world = int(rank), int(world)
        p = abi.EsParams(alpha=float(alpha), sigma=float(sigma), population=int(population),
                         iterations=int(iterations), seed=int(seed) & (2 ** 64 - 1),
                         rank_normalize=1 if rank_normalize else 0)
        self.params = p
        th = None if theta0 is None else np.ascontiguousarray(theta0, np.float64)
        h = C.c_void_p()
        with _torch().cuda.device(task.device):
            _check(lib().ls_es_create_shard(task._h, C.addressof(p), None if th is None else th.ctypes.data,
                                            self.rank, self.world, C.byref(h)), "ls_es_create_shard")
        self._h = h

    def run(self, stream=None):
        torch = _torch()
        with torch.cuda.device(self.task.device):
            _check(lib().ls_es_run(self._h, _stream(torch, stream)), "ls_es_run")

    def shard_buffers(self):
        """(keys u64 [world * keys_per_rank], partials f64 [world * partials_per_rank]) as CUDA tensors
        aliasing the run's exchange buffers (zero-copy views), plus the per-rank slice lengths."""
        torch = _torch()
        kp, pp = C.c_void_p(), C.c_void_p()
        kn, pn = C.c_int64(), C.c_int64()
        _check(lib().ls_es_shard_buffers(self._h, C.byref(kp), C.byref(kn), C.byref(pp), C.byref(pn)),
               "ls_es_shard_buffers")
        dev = f"cuda:{self.task.device}"
        keys = _device_view(torch, kp.value, kn.value * self.world, torch.int64, dev)
        parts = _device_view(torch, pp.value, pn.value * self.world, torch.float64, dev)
        return keys, parts, kn.value, pn.value

    def begin(self, stream=None):
        """Fresh state and the start point (ls_es_begin)."""
        torch = _torch()
        with torch.cuda.device(self.task.device):
            _check(lib().ls_es_begin(self._h, _stream(torch, stream)), "ls_es_begin")

    def step(self, stage: int, stream=None):
        """One stage of a generation (ls_es_step): 0 local members, 1 ranks + local chunks, 2 update."""
        torch = _torch()
        with torch.cuda.device(self.task.device):
            _check(lib().ls_es_step(self._h, int(stage), _stream(torch, stream)), "ls_es_step")

    def run_sharded(self, exchange, stream=None, generations: "int | None" = None):
        """Every generation stage by stage, with exchange(full_tensor, per_rank) an in-place all-gather
        of the rank slices between stages 0/1 and 1/2 (not called for world 1).  generations=0 for a
        one-schedule space (only the start point, ls/es.py:187-188)."""
        keys, parts, kn, pn = self.shard_buffers()
        self.begin(stream)
        for _ in range(self.params.iterations if generations is None else generations):
            self.step(0, stream)
            if self.world > 1:
                exchange(keys, kn)
            self.step(1, stream)
            if self.world > 1:
                exchange(parts, pn)
            self.step(2, stream)

    def result(self, dim: int, stream=None):
        """(theta history [iters+1, dim], trace [iters], evaluations, error code, best score)."""
        torch = _torch()
        it = self.params.iterations
        hist = np.zeros((it + 1, dim), np.float64)
        trace = np.zeros(it, np.float64)
        ev = np.zeros(1, np.int64)
        err = np.zeros(1, np.int64)
        best = np.zeros(1, np.float64)
        with torch.cuda.device(self.task.device):
            _check(lib().ls_es_result(self._h, hist.ctypes.data, trace.ctypes.data, ev.ctypes.data,
                                      err.ctypes.data, best.ctypes.data, _stream(torch, stream)), "ls_es_result")
        return hist, trace, int(ev[0]), int(err[0]), float(best[0])

    def evaluated(self, stream=None):
        """Distinct evaluated (points uint64, scores float64) in discovery order."""
        torch = _torch()
        cnt = np.zeros(1, np.int64)
        with torch.cuda.device(self.task.device):
            _check(lib().ls_es_evaluated(self._h, None, None, 0, cnt.ctypes.data, _stream(torch, stream)),
                   "ls_es_evaluated")
            m = int(cnt[0])
            pts = np.zeros(m, np.uint64)
            sc = np.zeros(m, np.float64)
            _check(lib().ls_es_evaluated(self._h, pts.ctypes.data, sc.ctypes.data, m, cnt.ctypes.data,
                                         _stream(torch, stream)), "ls_es_evaluated")
        return pts, sc

    def noise(self, generation: int, dim: int, stream=None):
        torch = _torch()
        out = torch.empty((self.params.population, dim), dtype=torch.float64, device=f"cuda:{self.task.device}")
        with torch.cuda.device(self.task.device):
            _check(lib().ls_es_noise(self._h, int(generation), _dptr(out), _stream(torch, stream)), "ls_es_noise")
        return out

    def sort_state(self, stream=None):
        """The last generation's rank sort (diagnostic): (keys in member order, sorted keys,
        member at each sorted position, each member's sorted position) as device tensors."""
        torch = _torch()
        n, dev = self.params.population, f"cuda:{self.task.device}"
        kin = torch.empty(n, dtype=torch.int64, device=dev)
        kout = torch.empty(n, dtype=torch.int64, device=dev)
        mem = torch.empty(n, dtype=torch.int32, device=dev)
        rk = torch.empty(n, dtype=torch.int32, device=dev)
        with torch.cuda.device(self.task.device):
            _check(lib().ls_es_sort_state(self._h, _dptr(kin), _dptr(kout), _dptr(mem), _dptr(rk),
                                          _stream(torch, stream)), "ls_es_sort_state")
        return kin, kout, mem, rk

    def close(self):
        if getattr(self, "_h", None):
            lib().ls_es_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass
