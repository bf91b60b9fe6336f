"""Thin ctypes binding of include/mwu.h (argument marshalling only — every step of the hot path
runs in libmwu.so's CUDA kernels).  torch is used for device memory of inputs/outputs only.

Fails loudly if the CUDA library is missing: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libmwu.so")

OK, ERR_ARG, ERR_CUDA, ERR_OOM, ERR_NCCL, ERR_STATE, ERR_NUMERIC = range(7)
RUNNING, FEASIBLE, INFEASIBLE, ITER_LIMIT = range(4)
OUTCOME_NAMES = {RUNNING: "running", FEASIBLE: "feasible", INFEASIBLE: "infeasible", ITER_LIMIT: "iter_limit"}
REASON_NAMES = {0: "", 1: "MAXD_ZERO", 2: "ALPHA_LT_1", 3: "EMPTY_COVER_ROW", 4: "ITER_LIMIT", 5: "MIN_Z"}
MIXED, PURE_PACKING, PURE_COVERING = range(3)
STEP_RULES = {"binary": 0, "newton": 1, "standard": 2}
GRAPH_KINDS = {"bmatch": 0, "match": 1, "vcover": 2, "domset": 3, "densest": 4}
VEC = {"x": 0, "d": 1, "y": 2, "z": 3, "dy": 4, "dz": 5, "wp": 6, "wc": 7, "g": 8, "h": 9, "xbest": 10}
ST = {"inc_rowptr": 0, "inc_slots": 1, "degree": 2, "prow": 3, "c_rowptr": 4, "c_colidx": 5,
      "ct_rowptr": 6, "ct_rowidx": 7, "pt_rowptr": 8, "pt_rowidx": 9, "p_rowptr": 10, "p_colidx": 11}
ST_DTYPE = {0: torch.int64, 1: torch.int32, 2: torch.int32, 3: torch.int32, 4: torch.int64, 5: torch.int32,
            6: torch.int64, 7: torch.int32, 8: torch.int64, 9: torch.int32, 10: torch.int64, 11: torch.int32}


class MwuError(RuntimeError):
    pass


class _Csr(ctypes.Structure):
    _fields_ = [("rows", ctypes.c_int64), ("cols", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("rowptr", ctypes.c_void_p), ("colidx", ctypes.c_void_p), ("vals", ctypes.c_void_p)]


class _Graph(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("n_vertices", ctypes.c_int64), ("n_edges", ctypes.c_int64),
                ("n_left", ctypes.c_int64), ("src", ctypes.c_void_p), ("dst", ctypes.c_void_p)]


class Options(ctypes.Structure):
    _fields_ = [("eta_factor", ctypes.c_double), ("max_iter", ctypes.c_int64), ("tol_prose", ctypes.c_int),
                ("max_evals", ctypes.c_int), ("outer_rel_tol", ctypes.c_double), ("use_graph", ctypes.c_int),
                ("bisect_depth", ctypes.c_int), ("device", ctypes.c_int), ("world", ctypes.c_int),
                ("rank", ctypes.c_int), ("nccl_id", ctypes.c_void_p), ("comm_group", ctypes.c_void_p),
                ("deterministic", ctypes.c_int), ("stream", ctypes.c_void_p), ("block_l", ctypes.c_int),
                ("block_r", ctypes.c_int), ("compact_cover", ctypes.c_int), ("step_rule", ctypes.c_int)]


class Stats(ctypes.Structure):
    _fields_ = [("outcome", ctypes.c_int32), ("reason", ctypes.c_int32), ("probes", ctypes.c_int64),
                ("iters_total", ctypes.c_int64), ("iters_last", ctypes.c_int64), ("search_evals", ctypes.c_int64),
                ("search_passes", ctypes.c_int64), ("bound", ctypes.c_double), ("objective", ctypes.c_double),
                ("certificate", ctypes.c_double), ("eta", ctypes.c_double), ("alpha_last", ctypes.c_double),
                ("n", ctypes.c_int64), ("m_P", ctypes.c_int64), ("m_C", ctypes.c_int64), ("nnz_P", ctypes.c_int64),
                ("nnz_C", ctypes.c_int64), ("empty_rows_dropped", ctypes.c_int64), ("t_create_ms", ctypes.c_double),
                ("t_solve_ms", ctypes.c_double), ("t_loop_ms", ctypes.c_double),
                ("bytes_alg_per_iter", ctypes.c_double), ("kernel_launches", ctypes.c_int64),
                ("near_tie_count", ctypes.c_int64), ("t_phase_ms", ctypes.c_double * 4),
                ("max_Px_raw", ctypes.c_double), ("min_Cx_raw", ctypes.c_double), ("max_Px", ctypes.c_double),
                ("min_Cx", ctypes.c_double), ("probe_graph", ctypes.c_int64)]


EXPORTS = ["mwu_default_options", "mwu_create_csr", "mwu_create_graph", "mwu_solve", "mwu_get_x",
           "mwu_get_stats", "mwu_destroy", "mwu_last_error", "mwu_probe_begin", "mwu_step", "mwu_run_probe",
           "mwu_run_iters", "mwu_get_vec", "mwu_vec_len", "mwu_set_record", "mwu_get_structure",
           "mwu_get_scalars", "mwu_get_unique_id", "mwu_profile_iters", "mwu_shard_range",
           "mwu_simgroup_create", "mwu_simgroup_destroy", "mwu_set_stream", "mwu_create_gmatch"]

_lib = None


def lib():
    """Load libmwu.so (raises if it was not built — no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            raise MwuError(f"{_SO} not found: build it with `python -m paper_2307_03307_b200.build` "
                           "(there is no CPU fallback)")
        L = ctypes.CDLL(_SO)
        vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
        L.mwu_default_options.argtypes = [ctypes.POINTER(Options)]
        L.mwu_default_options.restype = None
        L.mwu_create_csr.argtypes = [ctypes.POINTER(_Csr), ctypes.POINTER(_Csr), ctypes.c_int,
                                     ctypes.POINTER(Options), ctypes.POINTER(vp)]
        L.mwu_create_graph.argtypes = [ctypes.POINTER(_Graph), ctypes.POINTER(Options), ctypes.POINTER(vp)]
        L.mwu_create_gmatch.argtypes = [ctypes.POINTER(_Graph), vp, vp, ctypes.POINTER(Options), ctypes.POINTER(vp)]
        L.mwu_solve.argtypes = [vp, dbl, i64, ctypes.POINTER(i32)]
        L.mwu_get_x.argtypes = [vp, vp, i64]
        L.mwu_get_stats.argtypes = [vp, ctypes.POINTER(Stats)]
        L.mwu_destroy.argtypes = [vp]
        L.mwu_destroy.restype = None
        L.mwu_last_error.argtypes = [vp]
        L.mwu_last_error.restype = ctypes.c_char_p
        L.mwu_probe_begin.argtypes = [vp, dbl, dbl]
        L.mwu_step.argtypes = [vp, dbl, ctypes.POINTER(i32)]
        L.mwu_run_probe.argtypes = [vp, ctypes.POINTER(i32)]
        L.mwu_run_iters.argtypes = [vp, i64, ctypes.POINTER(i32)]
        L.mwu_get_vec.argtypes = [vp, ctypes.c_int, vp, i64]
        L.mwu_vec_len.argtypes = [vp, ctypes.c_int]
        L.mwu_vec_len.restype = i64
        L.mwu_set_record.argtypes = [vp, ctypes.c_int]
        L.mwu_set_stream.argtypes = [vp, vp]
        L.mwu_get_structure.argtypes = [vp, ctypes.c_int, vp, ctypes.POINTER(i64)]
        L.mwu_get_scalars.argtypes = [vp, ctypes.POINTER(dbl)]
        L.mwu_get_unique_id.argtypes = [vp]
        L.mwu_profile_iters.argtypes = [vp, i64, ctypes.POINTER(dbl)]
        L.mwu_shard_range.argtypes = [i64, ctypes.c_int, ctypes.c_int, ctypes.POINTER(i64), ctypes.POINTER(i64)]
        L.mwu_simgroup_create.argtypes = [ctypes.c_int, ctypes.POINTER(vp)]
        L.mwu_simgroup_destroy.argtypes = [vp]
        L.mwu_simgroup_destroy.restype = None
        for name in EXPORTS:
            getattr(L, name)
        _lib = L
    return _lib


def _current_stream():
    """cudaStream_t of torch's current stream (None without CUDA): the caller-side ordering of
    every ABI call that reads or writes tensors (mwu_options.stream)."""
    if torch.cuda.is_available() and torch.cuda.is_initialized():
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    return None


def default_options(keep=None, **kw) -> Options:
    o = Options()
    lib().mwu_default_options(ctypes.byref(o))
    o.stream = _current_stream()
    for k, v in kw.items():
        if not hasattr(o, k):
            raise TypeError(f"unknown option {k}")
        if k == "nccl_id" and isinstance(v, (bytes, bytearray)):
            buf = ctypes.create_string_buffer(bytes(v), 128)
            if keep is not None:
                keep.append(buf)
            v = ctypes.cast(buf, ctypes.c_void_p)
        elif k == "comm_group" and isinstance(v, SimGroup):
            v = v.handle
        elif k == "step_rule" and isinstance(v, str):
            v = STEP_RULES[v]
        setattr(o, k, v)
    return o


def get_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 creates it; share it with torch.distributed)."""
    buf = ctypes.create_string_buffer(128)
    st = lib().mwu_get_unique_id(buf)
    if st != OK:
        raise MwuError(f"mwu_get_unique_id: status {st}: {lib().mwu_last_error(None).decode()}")
    return buf.raw


def share_unique_id(make_id) -> bytes:
    """Rank 0 calls make_id() and every rank of the torch.distributed group receives it."""
    import torch.distributed as dist
    box = [make_id() if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(box, src=0)
    return box[0]


def shard_range(n_edges: int, world: int, rank: int):
    """The internal edge range [e0, e1) rank `rank` of `world` owns (mwu_shard_range)."""
    a, b = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().mwu_shard_range(int(n_edges), int(world), int(rank), ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


class SimGroup:
    """In-process group of `world` ranks on one device (tests of the sharded engine)."""

    def __init__(self, world: int):
        h = ctypes.c_void_p()
        _check(lib().mwu_simgroup_create(int(world), ctypes.byref(h)))
        self.handle, self.world = h, world

    def close(self):
        if self.handle:
            lib().mwu_simgroup_destroy(self.handle)
            self.handle = None


def _ptr(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _check(st: int, ctx=None):
    if st != OK:
        msg = lib().mwu_last_error(ctx).decode()
        raise MwuError(f"mwu status {st}: {msg}")


class Solver:
    """One C-ABI context.  Inputs may be CUDA or CPU tensors (the library copies them)."""

    def __init__(self, handle, keep):
        self._h = handle
        self._keep = keep
        self.n = int(lib().mwu_vec_len(handle, VEC["x"]))

    # ---------------------------------------------------------------- creation
    @classmethod
    def graph(cls, kind: str, src: torch.Tensor, dst: torch.Tensor, n_vertices: int, n_left: int = 0,
              **opts) -> "Solver":
        src = src.to(torch.int32).contiguous()
        dst = dst.to(torch.int32).contiguous()
        g = _Graph(GRAPH_KINDS[kind], int(n_vertices), int(src.numel()), int(n_left), _ptr(src), _ptr(dst))
        keep = [src, dst]
        o = default_options(keep, **opts)
        h = ctypes.c_void_p()
        _check(lib().mwu_create_graph(ctypes.byref(g), ctypes.byref(o), ctypes.byref(h)))
        return cls(h, keep)

    @classmethod
    def graph_distributed(cls, kind: str, src, dst, n_vertices: int, n_left: int = 0, **opts) -> "Solver":
        """Edge-sharded context over the torch.distributed process group (one GPU per rank):
        rank 0 creates the NCCL id, every rank passes the same full edge list."""
        import torch.distributed as dist
        ws, rk = dist.get_world_size(), dist.get_rank()
        uid = share_unique_id(get_unique_id)     # world 1 too: the exchange runs through NCCL
        return cls.graph(kind, src, dst, n_vertices, n_left, world=ws, rank=rk, nccl_id=uid, **opts)

    @classmethod
    def gmatch(cls, src: torch.Tensor, dst: torch.Tensor, n_vertices: int, lb: torch.Tensor, ub: torch.Tensor,
               **opts) -> "Solver":
        """Generalized matching l <= M x <= u (mwu_create_gmatch; solve() runs one MIXED probe)."""
        src = src.to(torch.int32).contiguous()
        dst = dst.to(torch.int32).contiguous()
        lb = lb.to(torch.float64).contiguous()
        ub = ub.to(torch.float64).contiguous()
        g = _Graph(GRAPH_KINDS["match"], int(n_vertices), int(src.numel()), 0, _ptr(src), _ptr(dst))
        keep = [src, dst, lb, ub]
        o = default_options(keep, **opts)
        h = ctypes.c_void_p()
        _check(lib().mwu_create_gmatch(ctypes.byref(g), _ptr(lb), _ptr(ub), ctypes.byref(o), ctypes.byref(h)))
        return cls(h, keep)

    @classmethod
    def csr(cls, mode: int, n: int, P=None, C=None, **opts) -> "Solver":
        """P, C: (rowptr int64, colidx int32, vals float64 or None) tuples (canonical CSR)."""
        keep = []

        def mk(A):
            if A is None:
                return None
            rp, ci, va = A
            rp = rp.to(torch.int64).contiguous()
            ci = ci.to(torch.int32).contiguous()
            va = None if va is None else va.to(torch.float64).contiguous()
            keep.extend([rp, ci, va])
            return _Csr(rp.numel() - 1, int(n), ci.numel(), _ptr(rp), _ptr(ci), _ptr(va))

        cp, cc = mk(P), mk(C)
        o = default_options(**opts)
        h = ctypes.c_void_p()
        _check(lib().mwu_create_csr(ctypes.byref(cp) if cp else None, ctypes.byref(cc) if cc else None,
                                    int(mode), ctypes.byref(o), ctypes.byref(h)))
        return cls(h, keep)

    # ---------------------------------------------------------------- solve
    def solve(self, eps: float, max_iter: int = 0) -> str:
        out = ctypes.c_int32()
        _check(lib().mwu_solve(self._h, float(eps), int(max_iter), ctypes.byref(out)), self._h)
        return OUTCOME_NAMES[out.value]

    def _sync_stream(self):
        st = _current_stream()
        _check(lib().mwu_set_stream(self._h, st), self._h)

    def x(self, device="cuda") -> torch.Tensor:
        self._sync_stream()
        t = torch.empty(self.n, dtype=torch.float64, device=device)
        _check(lib().mwu_get_x(self._h, _ptr(t), t.numel()), self._h)
        return t

    def stats(self) -> dict:
        s = Stats()
        _check(lib().mwu_get_stats(self._h, ctypes.byref(s)), self._h)
        d = {k: getattr(s, k) for k, _ in Stats._fields_}
        d["t_phase_ms"] = dict(zip(("column", "step", "search", "update"), list(s.t_phase_ms)))
        d["outcome"] = OUTCOME_NAMES.get(d["outcome"], str(d["outcome"]))
        d["reason"] = REASON_NAMES.get(d["reason"], str(d["reason"]))
        return d

    # ---------------------------------------------------------------- probe hooks
    def probe_begin(self, bound: float, eps: float):
        _check(lib().mwu_probe_begin(self._h, float(bound), float(eps)), self._h)

    def step(self, alpha: float = 0.0) -> str:
        st = ctypes.c_int32()
        _check(lib().mwu_step(self._h, float(alpha), ctypes.byref(st)), self._h)
        return OUTCOME_NAMES[st.value]

    def run_probe(self) -> str:
        st = ctypes.c_int32()
        _check(lib().mwu_run_probe(self._h, ctypes.byref(st)), self._h)
        return OUTCOME_NAMES[st.value]

    def run_iters(self, k: int) -> str:
        st = ctypes.c_int32()
        _check(lib().mwu_run_iters(self._h, int(k), ctypes.byref(st)), self._h)
        return OUTCOME_NAMES[st.value]

    def set_record(self, on: bool = True):
        _check(lib().mwu_set_record(self._h, int(bool(on))), self._h)

    def vec(self, which: str, device="cuda") -> torch.Tensor:
        w = VEC[which]
        L = int(lib().mwu_vec_len(self._h, w))
        if L <= 0:
            raise MwuError(f"vector {which} unavailable")
        self._sync_stream()
        t = torch.empty(L, dtype=torch.float64, device=device)
        _check(lib().mwu_get_vec(self._h, w, _ptr(t), L), self._h)
        return t

    def structure(self, which: str, device="cpu") -> torch.Tensor:
        w = ST[which]
        nb = ctypes.c_int64(0)
        lib().mwu_get_structure(self._h, w, None, ctypes.byref(nb))
        if nb.value <= 0:
            raise MwuError(f"structure {which} unavailable")
        dt = ST_DTYPE[w]
        t = torch.empty(nb.value // torch.empty(0, dtype=dt).element_size(), dtype=dt, device=device)
        _check(lib().mwu_get_structure(self._h, w, _ptr(t), ctypes.byref(nb)), self._h)
        return t

    def profile_iters(self, k: int) -> dict:
        a = (ctypes.c_double * 10)()
        _check(lib().mwu_profile_iters(self._h, int(k), a), self._h)
        names = ["column", "step", "search", "update"]
        out = {n: {"ms": a[2 * i], "launches": a[2 * i + 1]} for i, n in enumerate(names)}
        out["iters"], out["passes"] = a[8], a[9]
        return out

    def scalars(self) -> dict:
        a = (ctypes.c_double * 10)()
        _check(lib().mwu_get_scalars(self._h, a), self._h)
        keys = ["eta", "sigma", "sP", "SP", "sC", "SC", "t", "alpha_last", "evals", "passes"]
        return dict(zip(keys, list(a)))

    def close(self):
        if self._h:
            lib().mwu_destroy(self._h)
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
