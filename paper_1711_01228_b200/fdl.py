"""ctypes binding of libfdl.so (include/fdl.h) -- argument marshalling only.

Every step of the layout runs in the CUDA library; this module converts numpy
arrays to pointers, checks status codes and raises.  There is no fallback:
if libfdl.so cannot be loaded, importing the binding fails loudly.
"""
from __future__ import annotations

import ctypes
import math
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FDL_LIB") or os.path.join(_PKG, "lib", "libfdl.so")  # FDL_LIB: A/B builds in tests

FDL_TILE = 128
STATUS = {
    0: "FDL_OK", -1: "FDL_E_INVALID_ARG", -2: "FDL_E_SELF_LOOP", -3: "FDL_E_DUPLICATE_EDGE",
    -4: "FDL_E_ASYMMETRIC", -5: "FDL_E_DISCONNECTED", -6: "FDL_E_BAD_LENGTH", -7: "FDL_E_DIAMETER",
    -8: "FDL_E_OOM", -9: "FDL_E_CUDA", -10: "FDL_E_NCCL", -11: "FDL_E_SOLVER", -12: "FDL_E_NONFINITE",
    -13: "FDL_E_UNSUPPORTED", -14: "FDL_E_STATE",
}
STOP = {0: "none", 1: "rel_tol", 2: "zero_stress", 3: "max_iter"}
STRAT_FIXED, STRAT_ENUM, STRAT_PROB = 0, 1, 2  # include/fdl.h fdl_strategy

EXPORTS = [
    "fdl_abi_version", "fdl_params_default", "fdl_create", "fdl_create_sharded", "fdl_shard_tiles",
    "fdl_nccl_unique_id", "fdl_set_stream", "fdl_step", "fdl_run_until_converged", "fdl_get_positions",
    "fdl_set_positions", "fdl_eval_forces", "fdl_get_hop_rows", "fdl_get_diag", "fdl_get_info",
    "fdl_set_timing", "fdl_get_stats", "fdl_reset_stats", "fdl_bench_ffma", "fdl_bench_p1s_mix", "fdl_bench_p2_mix", "fdl_status_str",
    "fdl_last_error", "fdl_destroy", "fdl_eval_partial", "fdl_set_omega_vertex", "fdl_get_dist_rows",
    "fdl_group_create", "fdl_group_destroy", "fdl_create_loopback",
]


class FdlError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        self.name = STATUS.get(status, str(status))
        super().__init__(f"{self.name}: {msg}")


class Params(ctypes.Structure):
    _fields_ = [
        ("struct_size", ctypes.c_uint32), ("dim", ctypes.c_int32), ("k", ctypes.c_double),
        ("omega", ctypes.c_double), ("step", ctypes.c_double), ("tol", ctypes.c_double),
        ("max_iter", ctypes.c_int32), ("weight_exp", ctypes.c_double), ("cg_rtol", ctypes.c_double),
        ("cg_max_iter", ctypes.c_int32), ("strategy", ctypes.c_int32), ("seed", ctypes.c_uint64),
        ("device", ctypes.c_int32), ("a_refresh", ctypes.c_int32), ("hop_bits", ctypes.c_int32),
        ("cg_extrap", ctypes.c_int32), ("enum_count", ctypes.c_int32), ("enum_step", ctypes.c_double),
        ("p1_split", ctypes.c_int32), ("use_graphs", ctypes.c_int32), ("cg_history", ctypes.c_int32),
    ]


class IterInfo(ctypes.Structure):
    _fields_ = [
        ("it", ctypes.c_int32), ("accepted", ctypes.c_int32), ("cg_iters", ctypes.c_int32),
        ("stop", ctypes.c_int32), ("omega", ctypes.c_double), ("f_before", ctypes.c_double),
        ("f_next", ctypes.c_double), ("f_relaxed", ctypes.c_double), ("f_after", ctypes.c_double),
        ("rel_decrease", ctypes.c_double), ("cg_relres", ctypes.c_double), ("maxdisp", ctypes.c_double),
    ]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class RunInfo(ctypes.Structure):
    _fields_ = [
        ("iterations", ctypes.c_int32), ("accepted", ctypes.c_int32), ("stop", ctypes.c_int32),
        ("cg_iters", ctypes.c_int32), ("f_initial", ctypes.c_double), ("f_final", ctypes.c_double),
    ]


class CtxInfo(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int32), ("dim", ctypes.c_int32), ("diameter", ctypes.c_int32),
        ("hop_bits", ctypes.c_int32), ("rank", ctypes.c_int32), ("world", ctypes.c_int32),
        ("tile0", ctypes.c_int64), ("tile1", ctypes.c_int64), ("iterations", ctypes.c_int32),
        ("k", ctypes.c_double), ("f", ctypes.c_double), ("hop_matrix_bytes", ctypes.c_uint64),
        ("local_pairs", ctypes.c_uint64), ("device_bytes", ctypes.c_uint64), ("setup_ms", ctypes.c_double),
        ("setup_dist_ms", ctypes.c_double), ("bfs_bytes", ctypes.c_uint64),
    ]


class Stats(ctypes.Structure):
    _fields_ = [
        ("launches", ctypes.c_uint64), ("p1_launches", ctypes.c_uint64), ("p2_launches", ctypes.c_uint64),
        ("p1_pairs", ctypes.c_uint64), ("p2_pairs", ctypes.c_uint64), ("p1_pairs_x2", ctypes.c_uint64),
        ("p1_ms", ctypes.c_double), ("p2_ms", ctypes.c_double), ("other_ms", ctypes.c_double),
        ("steps", ctypes.c_uint64), ("cg_iters", ctypes.c_uint64), ("p1_pairs_nor", ctypes.c_uint64),
        ("p1_rejected", ctypes.c_uint64), ("p1s_launches", ctypes.c_uint64), ("p1s_ms", ctypes.c_double),
        ("p1_predicted", ctypes.c_uint64), ("p1_predicted_rejected", ctypes.c_uint64),
    ]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not found: build it with __graft_entry__.build() "
                          "(no CPU fallback exists)")
    L = ctypes.CDLL(LIB_PATH)
    P, i32, u64, dbl, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint64, ctypes.c_double, ctypes.c_size_t
    sig = {
        "fdl_abi_version": (i32, []),
        "fdl_params_default": (None, [ctypes.POINTER(Params)]),
        "fdl_create": (i32, [i32, P, P, P, ctypes.POINTER(Params), P, ctypes.POINTER(P)]),
        "fdl_create_sharded": (i32, [i32, P, P, P, ctypes.POINTER(Params), P, P, i32, i32, ctypes.POINTER(P)]),
        "fdl_shard_tiles": (i32, [i32, i32, i32, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]),
        "fdl_nccl_unique_id": (i32, [P]),
        "fdl_set_stream": (i32, [P, P]),
        "fdl_step": (i32, [P, ctypes.POINTER(IterInfo)]),
        "fdl_run_until_converged": (i32, [P, ctypes.POINTER(RunInfo)]),
        "fdl_get_positions": (i32, [P, P, sz]),
        "fdl_set_positions": (i32, [P, P, sz]),
        "fdl_eval_forces": (i32, [P, P, P, P]),
        "fdl_set_omega_vertex": (i32, [P, P, sz]),
        "fdl_get_dist_rows": (i32, [P, i32, i32, P]),
        "fdl_group_create": (i32, [i32, ctypes.POINTER(P)]),
        "fdl_group_destroy": (None, [P]),
        "fdl_create_loopback": (i32, [i32, P, P, P, ctypes.POINTER(Params), P, P, i32, ctypes.POINTER(P)]),
        "fdl_get_hop_rows": (i32, [P, i32, i32, P]),
        "fdl_get_diag": (i32, [P, P, sz]),
        "fdl_get_info": (i32, [P, ctypes.POINTER(CtxInfo)]),
        "fdl_set_timing": (i32, [P, i32]),
        "fdl_get_stats": (i32, [P, ctypes.POINTER(Stats)]),
        "fdl_reset_stats": (i32, [P]),
        "fdl_bench_ffma": (i32, [i32, ctypes.POINTER(dbl), ctypes.POINTER(dbl)]),
        "fdl_bench_p1s_mix": (i32, [i32, ctypes.POINTER(dbl), ctypes.POINTER(dbl)]),
        "fdl_bench_p2_mix": (i32, [i32, ctypes.POINTER(dbl), ctypes.POINTER(dbl)]),
        "fdl_status_str": (ctypes.c_char_p, [i32]),
        "fdl_last_error": (ctypes.c_char_p, [P]),
        "fdl_destroy": (None, [P]),
        "fdl_eval_partial": (i32, [P, i32, P, P, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    return L


lib = _load()


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def params_default() -> Params:
    p = Params()
    lib.fdl_params_default(ctypes.byref(p))
    return p


def make_params(dim=2, k=0.0, omega=1.5, step=math.inf, tol=1e-4, max_iter=500, cg_rtol=0.0,
                cg_max_iter=0, strategy=STRAT_FIXED, seed=1, device=0, a_refresh=0, hop_bits=0, cg_extrap=2, enum_count=19, weight_exp=-2.0,
                enum_step=0.5, p1_split=-1, use_graphs=-1, cg_history=0) -> Params:
    p = params_default()
    p.dim, p.k, p.omega, p.step, p.tol, p.max_iter = dim, k, omega, step, tol, max_iter
    p.cg_rtol, p.cg_max_iter, p.strategy, p.seed, p.device = cg_rtol, cg_max_iter, strategy, seed, device
    p.a_refresh = a_refresh
    p.hop_bits = hop_bits
    p.cg_extrap = cg_extrap
    p.enum_count, p.enum_step = enum_count, enum_step
    p.weight_exp = weight_exp
    p.p1_split = p1_split
    p.use_graphs = use_graphs
    p.cg_history = cg_history
    return p


def shard_tiles(n: int, world: int, rank: int):
    a, b = ctypes.c_int64(), ctypes.c_int64()
    _check(None, lib.fdl_shard_tiles(n, world, rank, ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def nccl_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(None, lib.fdl_nccl_unique_id(buf))
    return bytes(buf)


def bench_p1s_mix(device: int = 0):
    """(TFLOP/s, ms) of the line-6 pass's per-tile arithmetic on a resident tile."""
    tf, ms = ctypes.c_double(), ctypes.c_double()
    _check(None, lib.fdl_bench_p1s_mix(device, ctypes.byref(tf), ctypes.byref(ms)))
    return tf.value, ms.value


def bench_p2_mix(device: int = 0):
    """(hop GB/s, ms) of the PCG matvec pass's per-tile work on a resident tile."""
    gbs, ms = ctypes.c_double(), ctypes.c_double()
    _check(None, lib.fdl_bench_p2_mix(device, ctypes.byref(gbs), ctypes.byref(ms)))
    return gbs.value, ms.value


def bench_ffma(device: int = 0):
    tf, ms = ctypes.c_double(), ctypes.c_double()
    _check(None, lib.fdl_bench_ffma(device, ctypes.byref(tf), ctypes.byref(ms)))
    return tf.value, ms.value


def _check(ctx, status):
    if status != 0:
        msg = lib.fdl_last_error(ctx).decode() if ctx else ""
        raise FdlError(status, msg)


class LoopbackGroup:
    """In-process loopback transport of `world` ranks (include/fdl.h test hook)."""

    def __init__(self, world: int):
        self.world = int(world)
        self._h = ctypes.c_void_p()
        _check(None, lib.fdl_group_create(self.world, ctypes.byref(self._h)))

    def close(self):
        if self._h:
            lib.fdl_group_destroy(self._h)
            self._h = ctypes.c_void_p()


class Layout:
    """One layout context (fdl_ctx) on one GPU; names follow include/fdl.h."""

    def __init__(self, n: int, row_ptr, col_idx, params: Params | None = None, init_pos=None,
                 nccl_id: bytes | None = None, rank: int = 0, world: int = 1, edge_len=None,
                 group: "LoopbackGroup | None" = None):
        self._h = ctypes.c_void_p()
        self.n = int(n)
        self._rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        self._col = np.ascontiguousarray(col_idx, dtype=np.int32)
        self.params = params if params is not None else params_default()
        self.dim = int(self.params.dim)
        X0 = None if init_pos is None else np.ascontiguousarray(init_pos, dtype=np.float64)
        self._len = None if edge_len is None else np.ascontiguousarray(edge_len, dtype=np.float64)
        if self._len is not None and self._len.size != self._col.size:
            raise ValueError("edge_len must have one entry per stored CSR direction")
        if X0 is not None and X0.size != self.n * self.dim:
            raise ValueError("init_pos must have n*dim entries")
        if group is not None:
            st = lib.fdl_create_loopback(self.n, _ptr(self._rp), _ptr(self._col), _ptr(self._len),
                                         ctypes.byref(self.params), _ptr(X0), group._h, rank, ctypes.byref(self._h))
        elif world == 1 and nccl_id is None:
            st = lib.fdl_create(self.n, _ptr(self._rp), _ptr(self._col), _ptr(self._len), ctypes.byref(self.params),
                                _ptr(X0), ctypes.byref(self._h))
        else:
            # nccl_id None -> emulated rank (test hook: fdl_eval_partial only);
            # world 1 with an id -> one-rank communicator
            idbuf = None if nccl_id is None else (ctypes.c_uint8 * 128).from_buffer_copy(nccl_id)
            st = lib.fdl_create_sharded(self.n, _ptr(self._rp), _ptr(self._col), _ptr(self._len),
                                        ctypes.byref(self.params),
                                        _ptr(X0), idbuf, rank, world, ctypes.byref(self._h))
        if st != 0:
            raise FdlError(st, "fdl_create failed (see stderr)")
        self.info = self.get_info()

    @classmethod
    def from_graph(cls, g, **kw):
        return cls(g.n, g.row_ptr, g.col, **kw)

    def close(self):
        if self._h:
            lib.fdl_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ------------------------------------------------------------ ABI calls
    def set_stream(self, stream_ptr: int | None):
        _check(self._h, lib.fdl_set_stream(self._h, ctypes.c_void_p(stream_ptr) if stream_ptr else None))

    def step(self) -> IterInfo:
        info = IterInfo()
        _check(self._h, lib.fdl_step(self._h, ctypes.byref(info)))
        return info

    def run_until_converged(self) -> RunInfo:
        info = RunInfo()
        _check(self._h, lib.fdl_run_until_converged(self._h, ctypes.byref(info)))
        return info

    def get_positions(self, out: np.ndarray | None = None) -> np.ndarray:
        if out is None:
            out = np.empty((self.n, self.dim), dtype=np.float64)
        _check(self._h, lib.fdl_get_positions(self._h, _ptr(out), out.size))
        return out

    def set_positions(self, X) -> None:
        X = np.ascontiguousarray(X, dtype=np.float64)
        _check(self._h, lib.fdl_set_positions(self._h, _ptr(X), X.size))

    def set_omega_vertex(self, omega) -> None:
        """Per-vertex relax factors; None restores the scalar omega."""
        if omega is None:
            _check(self._h, lib.fdl_set_omega_vertex(self._h, None, 0))
            return
        w = np.ascontiguousarray(omega, dtype=np.float64)
        _check(self._h, lib.fdl_set_omega_vertex(self._h, _ptr(w), w.size))

    def eval_forces(self):
        R = np.empty((self.n, self.dim))
        A = np.empty((self.n, self.dim))
        f = ctypes.c_double()
        _check(self._h, lib.fdl_eval_forces(self._h, _ptr(R), _ptr(A), ctypes.byref(f)))
        return R, A, f.value

    def eval_partial(self, mode: int, X):
        """This rank's partial L^X X (mode 0, with partial stress) or L^W X (mode 1) at X."""
        X = np.ascontiguousarray(X, dtype=np.float64)
        out = np.empty((self.n, self.dim))
        f = ctypes.c_double()
        _check(self._h, lib.fdl_eval_partial(self._h, mode, _ptr(X), _ptr(out), ctypes.byref(f)))
        return out, f.value

    def get_hop_rows(self, r0: int, nrows: int) -> np.ndarray:
        out = np.empty((nrows, self.n), dtype=np.uint16)
        _check(self._h, lib.fdl_get_hop_rows(self._h, r0, nrows, _ptr(out)))
        return out

    def get_dist_rows(self, r0: int, nrows: int) -> np.ndarray:
        """d_ij = k x shortest path length for rows [r0, r0 + nrows) (original units)."""
        out = np.empty((nrows, self.n), dtype=np.float64)
        _check(self._h, lib.fdl_get_dist_rows(self._h, r0, nrows, _ptr(out)))
        return out

    def get_diag(self) -> np.ndarray:
        out = np.empty(self.n, dtype=np.float64)
        _check(self._h, lib.fdl_get_diag(self._h, _ptr(out), self.n))
        return out

    def get_info(self) -> CtxInfo:
        info = CtxInfo()
        _check(self._h, lib.fdl_get_info(self._h, ctypes.byref(info)))
        return info

    def set_timing(self, on: bool = True):
        _check(self._h, lib.fdl_set_timing(self._h, 1 if on else 0))

    def get_stats(self) -> Stats:
        s = Stats()
        _check(self._h, lib.fdl_get_stats(self._h, ctypes.byref(s)))
        return s

    def reset_stats(self):
        _check(self._h, lib.fdl_reset_stats(self._h))

    @property
    def f(self) -> float:
        return self.get_info().f
