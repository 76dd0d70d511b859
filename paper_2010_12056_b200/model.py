"""Python view of a cpd_ctx: the C-ABI entry points of include/cpd.h as methods.

Names follow the ABI (cp_als_init, msdt_sweep, dt_sweep, pp_init, pp_approx_sweep,
fitness, ...).  Only marshalling happens here.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import check, dptr, dptr_array, load_library


class CPDecomposition:
    """One rank's CP-ALS state on the device (a cpd_ctx).

    T: torch CUDA float64 contiguous tensor = this rank's block [s_1/I_1, ..., s_N/I_N] of the
       processor grid (default 1 x .. x 1 x world: the slab [s_1..s_{N-1}, s_N/world])
       (borrowed: keep it alive as long as this object).
    shape: global mode sizes; R: rank; A0: N global s_n x R host arrays.
    """

    def __init__(self, T, shape, R, A0, *, device=0, rank=0, world=1, nccl_id=None, stream=None,
                 pp_eps=0.1, reuse_root_in_pp_init=True, profile_phases=False, local_group=None,
                 ttm_impl=2, grid=None, fused_rs=False, msdt_levels=1):
        lib = load_library()
        self.N = len(shape)
        self.shape = tuple(int(s) for s in shape)
        self.R = int(R)
        self.world = world
        self._T = T  # keep alive
        o = _lib.cpd_opts()
        check(lib.cpd_opts_default(C.byref(o)))
        o.device, o.rank, o.world = device, rank, world
        self._nccl_buf = None
        if nccl_id is not None:
            self._nccl_buf = C.create_string_buffer(bytes(nccl_id), _lib.CPD_NCCL_ID_BYTES)
            o.nccl_unique_id = C.cast(self._nccl_buf, C.c_void_p)
        o.stream = _lib._stream_ptr(stream)
        o.pp_eps = float(pp_eps)
        o.reuse_root_in_pp_init = int(bool(reuse_root_in_pp_init))
        o.profile_phases = int(profile_phases)
        o.local_group = local_group.value if local_group is not None else None
        o.ttm_impl = int(ttm_impl)
        o.fused_rs = int(bool(fused_rs))
        o.msdt_levels = int(msdt_levels)
        self.grid = tuple(grid) if grid is not None else (1,) * (self.N - 1) + (world,)
        if grid is not None:
            for n, g in enumerate(grid):
                o.grid[n] = int(g)
        A0 = [np.ascontiguousarray(a, dtype=np.float64) for a in A0]
        shp = (C.c_int64 * self.N)(*self.shape)
        ctx = C.c_void_p()
        check(lib.cp_als_init(C.byref(ctx), self.N, shp, self.R, C.c_void_p(T.data_ptr()),
                              dptr_array(A0), C.byref(o)))
        self._ctx = ctx
        self._lib = lib

    # -- sweeps ---------------------------------------------------------------------------
    def msdt_sweep(self) -> float:
        f = C.c_double()
        check(self._lib.msdt_sweep(self._ctx, C.byref(f)), self._ctx)
        return f.value

    def dt_sweep(self) -> float:
        f = C.c_double()
        check(self._lib.dt_sweep(self._ctx, C.byref(f)), self._ctx)
        return f.value

    def pp_init(self):
        check(self._lib.pp_init(self._ctx), self._ctx)

    def pp_approx_sweep(self):
        f, v = C.c_double(), C.c_int()
        check(self._lib.pp_approx_sweep(self._ctx, C.byref(f), C.byref(v)), self._ctx)
        return f.value, bool(v.value)

    def fitness(self) -> float:
        f = C.c_double()
        check(self._lib.fitness(self._ctx, C.byref(f)), self._ctx)
        return f.value

    def pp_condition(self) -> bool:
        v = C.c_int()
        check(self._lib.cpd_pp_condition(self._ctx, C.byref(v)), self._ctx)
        return bool(v.value)

    # -- accessors ------------------------------------------------------------------------
    def get_factor(self, n, out=None):
        out = np.empty((self.shape[n], self.R)) if out is None else out
        check(self._lib.cpd_get_factor(self._ctx, n, dptr(out)), self._ctx)
        return out

    def get_last_mttkrp(self, n):
        out = np.empty((self.shape[n], self.R))
        check(self._lib.cpd_get_last_mttkrp(self._ctx, n, dptr(out)), self._ctx)
        return out

    def set_factors(self, A):
        A = [np.ascontiguousarray(a, dtype=np.float64) for a in A]
        check(self._lib.cpd_set_factors(self._ctx, dptr_array(A)), self._ctx)

    def phase_ms(self):
        out = np.zeros(5)
        check(self._lib.cpd_get_phase_ms(self._ctx, dptr(out)), self._ctx)
        return dict(zip(["ttm", "mttv", "solve", "hadamard", "other"], out.tolist()))

    def counters(self):
        out = np.zeros(6)
        check(self._lib.cpd_get_counters(self._ctx, dptr(out)), self._ctx)
        tb = np.zeros(1)
        check(self._lib.cpd_get_ttm_bytes(self._ctx, dptr(tb)), self._ctx)
        return dict(zip(["ttm_flops", "ttm_launches", "stream_bytes", "stream_launches", "roots",
                         "kernel_launches", "ttm_bytes"],
                        out.tolist() + [float(tb[0])]))

    def filler_counters(self):
        """cpd_get_filler_counters: PP operator streams on the filler stream (bytes, launches)."""
        out = np.zeros(2)
        check(self._lib.cpd_get_filler_counters(self._ctx, dptr(out)), self._ctx)
        return {"bytes": float(out[0]), "launches": int(out[1])}

    def get_memory(self):
        """cpd_get_memory: auxiliary device memory (peak and live bytes of tree nodes / PP operators /
        block KRPs since init or reset_counters) and the bytes of T's digit planes."""
        out = np.zeros(3)
        check(self._lib.cpd_get_memory(self._ctx, dptr(out)), self._ctx)
        return {"peak": float(out[0]), "live": float(out[1]), "digits": float(out[2])}

    def set_profile_level(self, level):
        check(self._lib.cpd_set_profile_level(self._ctx, int(level)), self._ctx)

    def reset_counters(self):
        check(self._lib.cpd_reset_counters(self._ctx), self._ctx)

    def debug_pp_operator(self, a, b):
        out = np.empty((self.shape[a] // self.grid[a], self.shape[b] // self.grid[b], self.R))
        check(self._lib.cpd_debug_get_pp_operator(self._ctx, a, b, dptr(out)), self._ctx)
        return out

    def set_tensor(self):
        """The borrowed T's contents changed: recompute ||T||^2 and the TTM engine's view of T."""
        check(self._lib.cpd_set_tensor(self._ctx), self._ctx)

    def ttm_engine(self) -> str:
        """The first-level TTM engine chosen at init: "dmma", "int8-digits" or "int8-convert"."""
        e = C.c_int()
        check(self._lib.cpd_ttm_engine(self._ctx, C.byref(e)), self._ctx)
        return {0: "dmma", 1: "int8-digits", 2: "int8-convert"}[e.value]

    def last_sweep_status(self) -> dict:
        """Eq. 3 status of the last sweep: {"radicand_negative": bool, "radicand_rel": float}
        (cpd_last_sweep_status; a set flag means the reported fitness is the clamped 1)."""
        fl, rr = C.c_int(), C.c_double()
        check(self._lib.cpd_last_sweep_status(self._ctx, C.byref(fl), C.byref(rr)), self._ctx)
        return {"radicand_negative": bool(fl.value & 1), "radicand_rel": rr.value}

    def close(self):
        if getattr(self, "_ctx", None) is not None and self._ctx.value:
            self._lib.cpd_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def cp_als_init(T, shape, R, A0, **kw) -> CPDecomposition:
    """cp_als_init of include/cpd.h returning the ctx wrapper."""
    return CPDecomposition(T, shape, R, A0, **kw)
