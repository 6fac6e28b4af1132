"""paper_2401_00672_b200 -- B200-native POBK orthogonal-category Kaczmarz sweep (arXiv 2401.00672).

Python face of libpobk.so (include/pobk.h): a Plan is built once per system by
pobk_preprocess (RCM + first-fit partition + device layout, native C++), then solved any number of
times on the GPU with pobk_solve (hand-written sm_100a kernels).  Device vectors are torch CUDA
float64 tensors; the library only sees raw pointers and the current CUDA stream.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib as L
from ._lib import PobkError, Report, KERNEL, STOP, TERM_NAME  # noqa: F401

__all__ = ["Plan", "PobkError", "Report", "solve_batch", "solve_batch_host", "lane_tile_rows", "half_gpu_tile_rows", "KERNEL", "STOP"]


def _torch():
    import torch
    return torch


def _dev_ptr(t, name: str, m: int):
    torch = _torch()
    if t is None:
        return None
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous() \
            or t.numel() != m:
        raise TypeError(f"{name} must be a contiguous CUDA float64 tensor with {m} elements")
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        torch = _torch()
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    return ctypes.c_void_p(int(stream))


def _solve_opts(tol, max_sweeps, stop, check_every, sweep_offset=0, order="schedule") -> L.SolveOpts:
    o = L.SolveOpts()
    L.lib.pobk_solve_opts_default(ctypes.byref(o))
    o.tol = float(tol)
    o.max_sweeps = int(max_sweeps)
    o.stop = L.STOP[stop] if isinstance(stop, str) else int(stop)
    o.check_every = int(check_every)
    o.sweep_offset = int(sweep_offset)
    o.order = L.ORDER[order] if isinstance(order, str) else int(order)
    return o


class Plan:
    """One preprocessed system (pobk_preprocess).  device=-1 builds a host-only plan (queries only)."""

    def __init__(self, handle, device: int):
        self._h = handle
        self.device = device
        m, nnz, ns, no, b0, b1, t = (ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int32(),
                                     ctypes.c_int64(), ctypes.c_int64(), ctypes.c_double())
        L.check(L.lib.pobk_plan_info(self._h, ctypes.byref(m), ctypes.byref(nnz), ctypes.byref(ns), ctypes.byref(no),
                                     ctypes.byref(b0), ctypes.byref(b1), ctypes.byref(t)))
        self.m, self.nnz, self.nsteps, self.n_oclass = m.value, nnz.value, ns.value, no.value
        self.bw_before, self.bw_after, self.preprocess_seconds = b0.value, b1.value, t.value

    @classmethod
    def from_csr(cls, m: int, indptr, indices, data, thr: float = 0.0, reorder: int = 1, kernel: str = "auto",
                 tile_rows: int = 0, guard: int = 0, device: int | None = None) -> "Plan":
        if device is None:
            device = _torch().cuda.current_device()
        ip = L.as_host(indptr, np.int64)
        ix = L.as_host(indices, np.int32)
        vd = L.as_host(data, np.float64)
        o = L.PreprocessOpts()
        L.lib.pobk_preprocess_opts_default(ctypes.byref(o))
        o.thr, o.reorder, o.kernel, o.tile_rows, o.guard = float(thr), int(reorder), L.KERNEL[kernel], int(tile_rows), int(guard)
        h = ctypes.c_void_p()
        L.check(L.lib.pobk_preprocess(int(m), L.ptr(ip), L.ptr(ix), L.ptr(vd), ctypes.byref(o), int(device), ctypes.byref(h)))
        return cls(h, device)

    @classmethod
    def from_system(cls, system, **kw) -> "Plan":
        return cls.from_csr(system.m, system.indptr, system.indices, system.data, **kw)

    @classmethod
    def from_csr_blocks(cls, m: int, indptr, indices, data, k: int, thr: float, reorder: int = 1,
                        device: int | None = None) -> "Plan":
        """The paper-literal variant (pobk_blocks_preprocess): k uniform row blocks, centroid
        cosine table, Oclass pairs / Nclass (Alg 5 as written); solved with Plan.solve."""
        if device is None:
            device = _torch().cuda.current_device()
        ip = L.as_host(indptr, np.int64)
        ix = L.as_host(indices, np.int32)
        vd = L.as_host(data, np.float64)
        o = L.BlocksOpts(int(k), float(thr), int(reorder))
        h = ctypes.c_void_p()
        L.check(L.lib.pobk_blocks_preprocess(int(m), L.ptr(ip), L.ptr(ix), L.ptr(vd), ctypes.byref(o), int(device),
                                             ctypes.byref(h)))
        return cls(h, device)

    @classmethod
    def from_system_blocks(cls, system, **kw) -> "Plan":
        return cls.from_csr_blocks(system.m, system.indptr, system.indices, system.data, **kw)

    def blocks_info(self) -> dict:
        """k, block boundaries, the cosine table C, Oclass pairs, Nclass blocks, zn, nn."""
        k = ctypes.c_int32()
        L.check(L.lib.pobk_blocks_info(self._h, ctypes.byref(k), None, None, None, None, None, None, None, None))
        k = k.value
        ptr = np.empty(k + 1, np.int64)
        C = np.empty((k, k), np.float64)
        pairs = np.empty(2 * k, np.int32)
        ncl = np.empty(k, np.int32)
        npair, nn_, zn, nn = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_double(), ctypes.c_double()
        L.check(L.lib.pobk_blocks_info(self._h, None, L.ptr(ptr), L.ptr(C), L.ptr(pairs), ctypes.byref(npair), L.ptr(ncl),
                                       ctypes.byref(nn_), ctypes.byref(zn), ctypes.byref(nn)))
        return {"k": k, "ptr": ptr, "C": C, "pairs": [tuple(map(int, pairs[2 * i:2 * i + 2])) for i in range(npair.value)],
                "nclass": ncl[:nn_.value].tolist(), "zn": zn.value, "nn": nn.value}

    # ------------------------------------------------------------ queries
    def perm(self) -> np.ndarray:
        out = np.empty(self.m, dtype=np.int32)
        L.check(L.lib.pobk_plan_get_perm(self._h, L.ptr(out)))
        return out

    def partition(self):
        colour = np.empty(self.m, dtype=np.int32)
        cat_ptr = np.empty(self.nsteps + 1, dtype=np.int32)
        cat_rows = np.empty(self.m, dtype=np.int32)
        L.check(L.lib.pobk_plan_get_partition(self._h, L.ptr(colour), L.ptr(cat_ptr), L.ptr(cat_rows)))
        return colour, cat_ptr, cat_rows

    def tiles(self):
        n = ctypes.c_int32()
        L.check(L.lib.pobk_plan_get_tiles(self._h, ctypes.byref(n), None))
        if n.value == 0:
            return 0, None
        t = np.empty(self.m, dtype=np.int32)
        L.check(L.lib.pobk_plan_get_tiles(self._h, ctypes.byref(n), L.ptr(t)))
        return n.value, t

    def layout_stats(self) -> dict:
        st = L.LayoutStats()
        L.check(L.lib.pobk_plan_get_layout_stats(self._h, ctypes.byref(st)))
        return st.as_dict()

    # ------------------------------------------------------------ solves
    def solve(self, f, x, x_star=None, tol: float = 1e-6, max_sweeps: int = 500000, stop="rse", check_every: int = 1,
              stream=None, sweep_offset: int = 0, order: str = "schedule") -> Report:
        """x (CUDA float64, user frame) is x0 on entry and the solution on exit; sweep_offset > 0
        resumes a solve whose x0 already had that many sweeps (same check numbering and total cap)."""
        rep = L.Report()
        o = _solve_opts(tol, max_sweeps, stop, check_every, sweep_offset, order)
        L.check(L.lib.pobk_solve(self._h, _dev_ptr(f, "f", self.m), _dev_ptr(x, "x", self.m),
                                 _dev_ptr(x_star, "x_star", self.m), ctypes.byref(o), _stream(stream), ctypes.byref(rep)))
        return rep

    def solve_host(self, f: np.ndarray, x: np.ndarray, x_star=None, tol: float = 1e-6, max_sweeps: int = 500000,
                   stop="rse", check_every: int = 1, stream=None, sweep_offset: int = 0) -> Report:
        """End-to-end path with host arrays (x is updated in place)."""
        for name, a in (("f", f), ("x", x), ("x_star", x_star)):
            if a is not None and (not isinstance(a, np.ndarray) or a.dtype != np.float64 or not a.flags.c_contiguous
                                  or a.size != self.m):
                raise TypeError(f"{name} must be a contiguous float64 numpy array of length {self.m}")
        rep = L.Report()
        o = _solve_opts(tol, max_sweeps, stop, check_every, sweep_offset)
        L.check(L.lib.pobk_solve_host(self._h, L.ptr(f), L.ptr(x), L.ptr(x_star) if x_star is not None else None,
                                      ctypes.byref(o), _stream(stream), ctypes.byref(rep)))
        return rep

    def solve_multi(self, fs, xs, x_stars=None, tol: float = 1e-6, max_sweeps: int = 500000, stop="rse",
                    check_every: int = 1, stream=None, sweep_offset: int = 0) -> list[Report]:
        """pobk_solve_multi: R <= 8 right-hand sides of this plan's matrix in one sweep loop (A read
        once per step for all of them); each stops on its own rule; bitwise the single solves."""
        R = len(fs)
        F = (ctypes.c_void_p * R)(*[_dev_ptr(f, "f", self.m).value for f in fs])
        X = (ctypes.c_void_p * R)(*[_dev_ptr(x, "x", self.m).value for x in xs])
        XS = (ctypes.c_void_p * R)(*[_dev_ptr(x, "x_star", self.m).value for x in x_stars]) if x_stars else None
        reps = (L.Report * R)()
        o = _solve_opts(tol, max_sweeps, stop, check_every, sweep_offset)
        L.check(L.lib.pobk_solve_multi(self._h, R, ctypes.cast(F, ctypes.c_void_p), ctypes.cast(X, ctypes.c_void_p),
                                       ctypes.cast(XS, ctypes.c_void_p) if XS is not None else None, ctypes.byref(o),
                                       _stream(stream), ctypes.cast(reps, ctypes.c_void_p)))
        return list(reps)

    def residual_norm(self, f, x, stream=None) -> float:
        out = ctypes.c_double()
        L.check(L.lib.pobk_residual_norm(self._h, _dev_ptr(f, "f", self.m), _dev_ptr(x, "x", self.m), _stream(stream),
                                         ctypes.byref(out)))
        return out.value

    def residual_sumsq_rows(self, row_begin: int, row_end: int, f, x, stream=None) -> float:
        out = ctypes.c_double()
        L.check(L.lib.pobk_residual_sumsq_rows(self._h, int(row_begin), int(row_end), _dev_ptr(f, "f", self.m),
                                               _dev_ptr(x, "x", self.m), _stream(stream), ctypes.byref(out)))
        return out.value

    def close(self):
        if self._h:
            L.lib.pobk_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def solve_batch(plans, fs, xs, x_stars=None, tol: float = 1e-6, max_sweeps: int = 500000, stop="rse",
                check_every: int = 1, stream=None) -> list[Report]:
    """pobk_solve_batch: independent systems on one device (two concurrent lanes when every plan is a
    K2 plan filling at most half the SMs, e.g. built with tile_rows = half_gpu_tile_rows(m))."""
    nb = len(plans)
    H = (ctypes.c_void_p * nb)(*[p._h.value for p in plans])
    F = (ctypes.c_void_p * nb)(*[_dev_ptr(f, "f", p.m).value for f, p in zip(fs, plans)])
    X = (ctypes.c_void_p * nb)(*[_dev_ptr(x, "x", p.m).value for x, p in zip(xs, plans)])
    XS = (ctypes.c_void_p * nb)(*[_dev_ptr(x, "x_star", p.m).value for x, p in zip(x_stars, plans)]) if x_stars else None
    reps = (L.Report * nb)()
    o = _solve_opts(tol, max_sweeps, stop, check_every)
    L.check(L.lib.pobk_solve_batch(H, nb, ctypes.cast(F, ctypes.c_void_p), ctypes.cast(X, ctypes.c_void_p),
                                   ctypes.cast(XS, ctypes.c_void_p) if XS is not None else None, ctypes.byref(o),
                                   _stream(stream), ctypes.cast(reps, ctypes.c_void_p)))
    return list(reps)


def solve_batch_host(plans, fs, xs, x_stars=None, tol: float = 1e-6, max_sweeps: int = 500000, stop="rse",
                     check_every: int = 1, stream=None) -> list[Report]:
    """pobk_solve_batch_host: solve_batch with host (numpy float64) vectors; xs are updated in
    place.  On concurrent lanes the copies of other systems overlap the sweeps (pinned memory)."""
    nb = len(plans)
    for j, (p, f, x) in enumerate(zip(plans, fs, xs)):
        for name, a in (("f", f), ("x", x), ("x_star", x_stars[j] if x_stars else None)):
            if a is not None and (not isinstance(a, np.ndarray) or a.dtype != np.float64 or not a.flags.c_contiguous
                                  or a.size != p.m):
                raise TypeError(f"system {j}: {name} must be a contiguous float64 numpy array of length {p.m}")
    H = (ctypes.c_void_p * nb)(*[p._h.value for p in plans])
    F = (ctypes.c_void_p * nb)(*[L.ptr(f).value for f in fs])
    X = (ctypes.c_void_p * nb)(*[L.ptr(x).value for x in xs])
    XS = (ctypes.c_void_p * nb)(*[L.ptr(x).value for x in x_stars]) if x_stars else None
    reps = (L.Report * nb)()
    o = _solve_opts(tol, max_sweeps, stop, check_every)
    L.check(L.lib.pobk_solve_batch_host(H, nb, ctypes.cast(F, ctypes.c_void_p), ctypes.cast(X, ctypes.c_void_p),
                                        ctypes.cast(XS, ctypes.c_void_p) if XS is not None else None, ctypes.byref(o),
                                        _stream(stream), ctypes.cast(reps, ctypes.c_void_p)))
    return list(reps)


def lane_tile_rows(m: int, lanes: int = 2, device: int | None = None) -> int:
    """tile_rows for a K2 plan whose tiles fill at most 1/lanes of the device's SMs, so that
    pobk_solve_batch runs `lanes` systems (or right-hand sides of one matrix, one plan each)
    side by side.  The tiles must still keep their columns in shared memory: 2 lanes suit the 1M-row
    configs, 4 lanes the 262k-row config 3."""
    import torch
    sms = torch.cuda.get_device_properties(device if device is not None else torch.cuda.current_device()).multi_processor_count
    return -(-int(m) // max(1, sms // max(1, int(lanes)) - 2))


def half_gpu_tile_rows(m: int, device: int | None = None) -> int:
    """lane_tile_rows(m, 2): tiles filling at most half of the device's SMs (two lanes)."""
    return lane_tile_rows(m, 2, device)
