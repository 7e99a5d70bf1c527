"""B200-native ParaQAOA hot path — Python mirror of the reference's qcut:: API.

The compute lives in ``libqcgpu.so`` (CUDA sm_100a kernels + C++ host engine, built
from ``csrc/``) behind the C-ABI declared in ``include/qcgpu.h``. This module binds it
with ctypes and mirrors the reference's entry points (``/root/reference/proj/include/
qcut``) with the same names, argument meaning and error behaviour: ``ConfigError`` /
``ResourceError`` / ``IoError`` stand for qcut::config_error / resource_error /
io_error (errors.hpp:8-24).

There is no CPU fallback: constructing an :class:`Engine` without the built library or
without a CUDA device raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "Engine", "QcError", "ConfigError", "ResourceError", "IoError", "InternalError",
    "EDGE_DTYPE", "edges_array", "library_path", "load_library", "SolveResult", "MergeResult",
    "RunReport", "Partition", "partition_chain", "derive_subgraph_count", "Comm",
    "run_pipeline_multi", "run_record_bytes", "unpack_records",
]

HERE = os.path.dirname(os.path.abspath(__file__))
EDGE_DTYPE = np.dtype([("u", "<u4"), ("v", "<u4"), ("w", "<f8")])  # qc_edge == qcut::Edge


class QcError(RuntimeError):
    code = 4


class ConfigError(QcError):
    code = 1


class ResourceError(QcError):
    code = 2


class IoError(QcError):
    code = 3


class InternalError(QcError):
    code = 4


_ERRS = {1: ConfigError, 2: ResourceError, 3: IoError, 4: InternalError}


def library_path() -> str:
    return os.path.join(HERE, "libqcgpu.so")


# ---- C structs (include/qcgpu.h) ---------------------------------------------------
class _Graph(C.Structure):
    _fields_ = [("n", C.c_int32), ("m", C.c_int32), ("edges", C.c_void_p)]


class _SolveOptions(C.Structure):
    _fields_ = [("top_k", C.c_int32), ("layers", C.c_int32), ("budget", C.c_int32),
                ("fold", C.c_int32), ("seed", C.c_uint64), ("qubit_cap", C.c_uint64),
                ("tolerance", C.c_double), ("threads", C.c_int32), ("reserved", C.c_int32)]


class _SolveResult(C.Structure):
    _fields_ = [("width", C.c_int32), ("folded", C.c_int32), ("count", C.c_int32),
                ("evals", C.c_int32), ("expectation", C.c_double), ("bits", C.c_void_p),
                ("probs", C.c_void_p), ("params", C.c_void_p)]


class _Pool(C.Structure):
    _fields_ = [("levels", C.c_int32), ("widths", C.c_void_p), ("counts", C.c_void_p),
                ("bits", C.c_void_p)]


class _Chain(C.Structure):
    _fields_ = [("pieces", C.c_int32), ("first", C.c_void_p), ("last", C.c_void_p)]


class _MergeOptions(C.Structure):
    _fields_ = [("start_level", C.c_int32), ("workers", C.c_int32), ("incremental", C.c_int32),
                ("halve_symmetry", C.c_int32), ("path_budget", C.c_double)]


class _ChainedMergeOptions(C.Structure):
    _fields_ = [("window", C.c_int64), ("window_leaves", C.c_int64), ("workers", C.c_int32),
                ("halve_symmetry", C.c_int32)]


class _MergeResult(C.Structure):
    _fields_ = [("best_value", C.c_double), ("candidates_evaluated", C.c_uint64),
                ("assignment", C.c_void_p)]


class _RunConfig(C.Structure):
    _fields_ = [("qubit_cap", C.c_int32), ("subgraphs", C.c_int32), ("top_k", C.c_int32),
                ("start_level", C.c_int32), ("layers", C.c_int32), ("budget", C.c_int32),
                ("seed", C.c_uint64), ("fold", C.c_int32), ("halve_symmetry", C.c_int32),
                ("partition_mode", C.c_int32), ("merge_incremental", C.c_int32),
                ("merge_mode", C.c_int32), ("shard_index", C.c_int32),
                ("shard_count", C.c_int32), ("reserved", C.c_int32),
                ("path_budget", C.c_double), ("nm_tolerance", C.c_double)]


class _RunReport(C.Structure):
    _fields_ = [("cut", C.c_double), ("candidates_evaluated", C.c_uint64),
                ("partition_s", C.c_double), ("qaoa_s", C.c_double), ("merge_s", C.c_double),
                ("total_s", C.c_double), ("subgraphs", C.c_int32), ("windowed", C.c_int32),
                ("evals", C.c_uint64)]


EXPORTED_SYMBOLS = [
    "qc_engine_create", "qc_engine_destroy", "qc_last_error", "qc_abi_version", "qc_qubit_cap",
    "qc_engine_launches", "qc_engine_set_memory_budget", "qc_cost_table", "qc_plus_state",
    "qc_apply_cost_layer", "qc_apply_mixer_layer", "qc_expectation", "qc_norm_sq",
    "qc_linear_ramp", "qc_run_ansatz", "qc_eval_batch", "qc_optimize_batch",
    "qc_top_candidates", "qc_solve_subgraph", "qc_solve_batch", "qc_level_merge",
    "qc_chained_merge", "qc_run_pipeline", "qc_record_bytes", "qc_shard_range",
    "qc_shard_solve", "qc_merge_records", "qc_engine_profile", "qc_engine_profile_read",
    "qc_engine_transfers", "qc_engine_stream", "qc_pipeline_prepare", "qc_pipeline_execute",
    "qc_pipeline_destroy", "qc_simplex_create", "qc_simplex_ask", "qc_simplex_tell",
    "qc_simplex_result", "qc_simplex_destroy", "qc_optimizer_create", "qc_optimizer_ask",
    "qc_optimizer_tell", "qc_optimizer_result", "qc_optimizer_destroy", "qc_generate_er",
    "qc_generate_regular", "qc_engine_host_stats", "qc_engine_phase_times",
    "qc_engine_set_precision", "qc_engine_profile_read_fp64", "qc_run_record_bytes",
    "qc_pipeline_records", "qc_comm_id", "qc_comm_create", "qc_comm_create_all",
    "qc_comm_rank", "qc_comm_destroy", "qc_gather_topk", "qc_run_pipeline_multi",
    "qc_engine_set_mixer", "qc_engine_host_split",
]

KERNEL_KINDS = ["levels", "onchip", "pass_low", "pass_high", "blocksum", "finalsum", "topk",
                "merge_tables", "merge_search", "merge_other"]

_LIB = None


def load_library(path: str | None = None) -> C.CDLL:
    """Load libqcgpu.so (raises if it was not built — there is no fallback)."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    p = path or library_path()
    if not os.path.exists(p):
        raise ImportError(f"{p} not built: run __graft_entry__.build() "
                          "(make -C paper_2603_26232_b200/csrc)")
    lib = C.CDLL(p)
    lib.qc_last_error.restype = C.c_char_p
    lib.qc_engine_launches.restype = C.c_uint64
    lib.qc_record_bytes.restype = C.c_int64
    lib.qc_engine_destroy.restype = None
    lib.qc_engine_stream.restype = C.c_void_p
    lib.qc_pipeline_destroy.restype = None
    lib.qc_comm_destroy.restype = None
    if path is None:
        _LIB = lib
    return lib


def _check(lib, rc: int):
    if rc != 0:
        raise _ERRS.get(rc, InternalError)(lib.qc_last_error().decode())


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def edges_array(edges) -> np.ndarray:
    """(u, v[, w]) triples or an EDGE_DTYPE array -> contiguous EDGE_DTYPE array."""
    if isinstance(edges, np.ndarray) and edges.dtype == EDGE_DTYPE:
        return np.ascontiguousarray(edges)
    out = np.zeros(len(edges), dtype=EDGE_DTYPE)
    for i, e in enumerate(edges):
        out[i] = (e[0], e[1], e[2] if len(e) > 2 else 1.0)
    return out


def _graph(n: int, edges) -> tuple[_Graph, np.ndarray]:
    e = edges_array(edges)
    return _Graph(int(n), len(e), e.ctypes.data if len(e) else None), e


@dataclass
class SolveResult:  # qaoa.hpp:147-152 (+ CandidateSet qaoa.hpp:130-134)
    width: int
    folded: bool
    bits: np.ndarray
    probs: np.ndarray
    params: np.ndarray  # packed [gammas..., betas...]
    expectation: float
    evals: int


@dataclass
class MergeResult:  # merge.hpp:93-97
    best_value: float
    assignment: np.ndarray
    candidates_evaluated: int


@dataclass
class RunReport:
    cut: float
    candidates_evaluated: int
    partition_s: float
    qaoa_s: float
    merge_s: float
    total_s: float
    subgraphs: int
    windowed: bool
    evals: int
    assignment: str = ""


@dataclass
class Partition:  # partition.hpp:22-34 (chain pieces as global id ranges)
    first: np.ndarray
    last: np.ndarray
    local: list = field(default_factory=list)  # (n_local, EDGE_DTYPE array in local ids)
    inter: int = 0


def generate_er(n: int, p: float, seed: int) -> np.ndarray:
    """graph.hpp:146-160 generate_er_graph (host, qc_generate_er)."""
    lib = load_library()
    m = C.c_int64(0)
    _check(lib, lib.qc_generate_er(C.c_int(n), C.c_double(p), C.c_uint64(seed), None,
                                   C.c_int64(0), C.byref(m)))
    out = np.zeros(m.value, dtype=EDGE_DTYPE)
    _check(lib, lib.qc_generate_er(C.c_int(n), C.c_double(p), C.c_uint64(seed), _p(out),
                                   C.c_int64(m.value), C.byref(m)))
    return out


def generate_regular(n: int, d: int, seed: int, wlo: int = 1, whi: int = 10) -> np.ndarray:
    """Weighted random d-regular graph, integer weights U{wlo..whi} (BASELINE config 3)."""
    lib = load_library()
    m = C.c_int64(0)
    _check(lib, lib.qc_generate_regular(C.c_int(n), C.c_int(d), C.c_uint64(seed), C.c_int(wlo),
                                        C.c_int(whi), None, C.c_int64(0), C.byref(m)))
    out = np.zeros(m.value, dtype=EDGE_DTYPE)
    _check(lib, lib.qc_generate_regular(C.c_int(n), C.c_int(d), C.c_uint64(seed), C.c_int(wlo),
                                        C.c_int(whi), _p(out), C.c_int64(m.value), C.byref(m)))
    return out


def derive_subgraph_count(n: int, cap: int) -> int:  # partition.hpp:163-167
    if cap < 2:
        raise ConfigError("qubit cap must be at least 2")
    return 1 if n <= cap else (n - 1 + cap - 2) // (cap - 1)


def partition_chain(n: int, edges, M: int, mode: int = 0, cap: int = 0) -> Partition:
    """partition.hpp:111-160 (host prep; same chain as the engine's pipeline)."""
    if M < 1:
        raise ConfigError("subgraph count must be positive")
    if n == 0:
        raise ConfigError("cannot partition an empty graph")
    if M == 1:
        first, last = [0], [n - 1]
    else:
        if n < M + 1:
            raise ConfigError(f"need at least {M + 1} vertices for {M} chained subgraphs, got {n}")
        total = n - 1
        if mode == 1:
            s = n // M - 1
            if s < 1:
                raise ConfigError(f"tail-remainder split needs n >= 2*M, got n={n} M={M}")
            spans = [s] * (M - 1) + [total - (M - 1) * s]
        else:
            s = (total + M - 1) // M
            if (M - 1) * s <= total - 1:
                spans = [s] * (M - 1) + [total - (M - 1) * s]
            else:
                q, r = divmod(total, M)
                spans = [q + (1 if i < r else 0) for i in range(M)]
        first, last, a = [], [], 0
        for sp in spans:
            first.append(a)
            last.append(a + sp)
            a += sp
    if cap > 0:
        largest = max(b - a + 1 for a, b in zip(first, last))
        if largest > cap:
            need = (n - 1 + cap - 2) // (cap - 1)
            raise ResourceError(f"largest subgraph has {largest} vertices, over the {cap}-qubit "
                                f"cap; use at least {need} subgraphs")
    e = edges_array(edges)
    last_piece = np.zeros(n, np.int64)
    for i, (a, b) in enumerate(zip(first, last)):
        last_piece[a:b + 1] = i
    u = np.minimum(e["u"], e["v"]).astype(np.int64)
    v = np.maximum(e["u"], e["v"]).astype(np.int64)
    piece = last_piece[u] if len(e) else np.zeros(0, np.int64)
    intra = v <= np.asarray(last, np.int64)[piece] if len(e) else np.zeros(0, bool)
    local = []
    sel = np.nonzero(intra)[0] if len(e) else np.zeros(0, np.int64)
    sel = sel[np.argsort(piece[sel], kind="stable")]  # by piece, edge-list order inside
    bounds = np.searchsorted(piece[sel], np.arange(len(first) + 1))
    for i, (a, b) in enumerate(zip(first, last)):
        s_i = sel[bounds[i]:bounds[i + 1]]
        le = np.zeros(len(s_i), EDGE_DTYPE)
        le["u"] = u[s_i] - a
        le["v"] = v[s_i] - a
        le["w"] = e["w"][s_i]
        local.append((b - a + 1, le))
    return Partition(np.asarray(first, np.int32), np.asarray(last, np.int32), local,
                     int((~intra).sum()) if len(e) else 0)


class Engine:
    """One CUDA device's engine (qc_engine_create). All methods take host arrays."""

    def __init__(self, device: int = 0, library: str | None = None):
        self.lib = load_library(library)
        h = C.c_void_p()
        _check(self.lib, self.lib.qc_engine_create(C.c_int(device), C.byref(h)))
        self._h = h
        self.device = device

    def close(self):
        if getattr(self, "_h", None):
            self.lib.qc_engine_destroy(self._h)
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

    def _call(self, name, *args):
        _check(self.lib, getattr(self.lib, name)(self._h, *args))

    @property
    def launches(self) -> int:
        return int(self.lib.qc_engine_launches(self._h))

    def set_precision(self, bits: int):
        """64: exact fp64 (default); 32: optional fp32 mode for solve/eval (1e-4)."""
        self._call("qc_engine_set_precision", C.c_int(bits))

    def set_mixer(self, mixer: str | int):
        """fp32 mode's mixer form: "rx" (0, mixer_pair rotations) or "wht" (1, the
        Walsh-Hadamard form H diag H with add/sub butterflies); precision 32 first."""
        m = {"rx": 0, "wht": 1}.get(mixer, mixer) if isinstance(mixer, str) else int(mixer)
        self._call("qc_engine_set_mixer", C.c_int(m))

    def set_memory_budget(self, nbytes: int):
        self._call("qc_engine_set_memory_budget", C.c_uint64(nbytes))

    # ---- instrumentation -----------------------------------------------------------
    def profile(self, on: bool | int = True):
        """Start (and reset) live per-kernel CUDA-event timing; on=N>1 samples one launch
        in N per kernel kind (keeps the event overhead out of a timed region)."""
        self._call("qc_engine_profile", C.c_int(int(on)))

    def profile_read(self) -> dict:
        out = {}
        for k, name in enumerate(KERNEL_KINDS):
            n = C.c_uint64(0)
            ms = C.c_double(0)
            b = C.c_double(0)
            f = C.c_double(0)
            self._call("qc_engine_profile_read", C.c_int(k), C.byref(n), C.byref(ms), C.byref(b))
            self._call("qc_engine_profile_read_fp64", C.c_int(k), C.byref(f))
            out[name] = dict(launches=int(n.value), ms=ms.value, bytes=b.value,
                             fp64_ops=f.value)  # sampled
        return out

    def host_stats(self, reset: bool = False):
        w, p_, n = C.c_double(0), C.c_double(0), C.c_uint64(0)
        ph = (C.c_double * 4)()
        _check(self.lib, self.lib.qc_engine_phase_times(self._h, ph))
        sp = (C.c_double * 3)()
        _check(self.lib, self.lib.qc_engine_host_split(self._h, sp))
        _check(self.lib, self.lib.qc_engine_host_stats(self._h, C.byref(w), C.byref(p_), C.byref(n),
                                                       C.c_int(int(reset))))
        return dict(wait_s=w.value, prep_s=p_.value, chunk_steps=int(n.value),
                    optimize_s=ph[0], final_s=ph[1], merge_s=ph[2], execute_s=ph[3],
                    tell_s=sp[0], stage_s=sp[1], launch_s=sp[2])

    def transfers(self):
        h = C.c_uint64(0)
        d = C.c_uint64(0)
        _check(self.lib, self.lib.qc_engine_transfers(self._h, C.byref(h), C.byref(d)))
        return int(h.value), int(d.value)

    def stream_handle(self) -> int:
        return int(self.lib.qc_engine_stream(self._h) or 0)

    def prepare_pipeline(self, n: int, edges, **cfg) -> "PipelineSession":
        return PipelineSession(self, n, edges, **cfg)

    # ---- statevector.hpp -----------------------------------------------------------
    def cost_table(self, n: int, edges, cap: int = 24):
        g, keep = _graph(n, edges)
        out = np.zeros(1 << max(n, 0), np.float64)
        integral = C.c_int(0)
        mx = C.c_double(0)
        self._call("qc_cost_table", C.byref(g), C.c_int(cap), _p(out), C.byref(integral),
                   C.byref(mx))
        return out, bool(integral.value), mx.value

    def plus_state(self, q: int, cap: int = 24) -> np.ndarray:
        out = np.zeros(1 << max(min(q, 40), 0), np.complex128) if 1 <= q <= cap else \
            np.zeros(1, np.complex128)
        self._call("qc_plus_state", C.c_int(q), C.c_int(cap), _p(out))
        return out

    def apply_cost_layer(self, amps: np.ndarray, n: int, edges, gamma: float) -> np.ndarray:
        a = np.ascontiguousarray(amps, np.complex128).copy()
        g, keep = _graph(n, edges)
        q = int(np.log2(len(a))) if len(a) else 0
        self._call("qc_apply_cost_layer", C.c_int(q), _p(a), C.byref(g), C.c_double(gamma))
        return a

    def apply_mixer_layer(self, amps: np.ndarray, beta: float) -> np.ndarray:
        a = np.ascontiguousarray(amps, np.complex128).copy()
        q = int(np.log2(len(a))) if len(a) else 0
        self._call("qc_apply_mixer_layer", C.c_int(q), _p(a), C.c_double(beta))
        return a

    def expectation(self, amps: np.ndarray, n: int, edges) -> float:
        a = np.ascontiguousarray(amps, np.complex128)
        g, keep = _graph(n, edges)
        out = C.c_double(0)
        self._call("qc_expectation", C.c_int(int(np.log2(len(a)))), _p(a), C.byref(g),
                   C.byref(out))
        return out.value

    def norm_sq(self, amps: np.ndarray) -> float:
        a = np.ascontiguousarray(amps, np.complex128)
        out = C.c_double(0)
        self._call("qc_norm_sq", C.c_int(int(np.log2(len(a)))), _p(a), C.byref(out))
        return out.value

    # ---- qaoa.hpp ------------------------------------------------------------------
    def linear_ramp(self, p: int):
        g = np.zeros(max(p, 1))
        b = np.zeros(max(p, 1))
        _check(self.lib, self.lib.qc_linear_ramp(C.c_int(p), _p(g), _p(b)))
        return g, b

    def run_ansatz(self, n: int, edges, gammas, betas, want_amps: bool = True):
        g, keep = _graph(n, edges)
        ga = np.ascontiguousarray(gammas, np.float64)
        be = np.ascontiguousarray(betas, np.float64)
        if len(ga) != len(be):
            raise ConfigError("gamma and beta schedules must have equal length")
        amps = np.zeros(1 << n, np.complex128) if want_amps else None
        ex = C.c_double(0)
        self._call("qc_run_ansatz", C.byref(g), C.c_int(len(ga)), _p(ga), _p(be), _p(amps),
                   C.byref(ex))
        return amps, ex.value

    def eval_batch(self, graphs, p: int, index, params) -> np.ndarray:
        """graphs: [(n, edges)], index[k] -> graph, params[k] packed 2p."""
        structs = (_Graph * len(graphs))()
        keep = []
        for i, (n, edges) in enumerate(graphs):
            gs, e = _graph(n, edges)
            structs[i] = gs
            keep.append(e)
        idx = np.ascontiguousarray(index, np.int32)
        prm = np.ascontiguousarray(params, np.float64).reshape(len(idx), 2 * p)
        out = np.zeros(len(idx))
        self._call("qc_eval_batch", structs, C.c_int(len(graphs)), C.c_int(p),
                   C.c_int(len(idx)), _p(idx), _p(prm), _p(out))
        return out

    def optimize_batch(self, graphs, p: int, budget: int, seeds, tol: float = 1e-5,
                       trace: bool = False):
        n = len(graphs)
        structs = (_Graph * n)()
        keep = []
        for i, (nv, edges) in enumerate(graphs):
            gs, e = _graph(nv, edges)
            structs[i] = gs
            keep.append(e)
        sd = np.ascontiguousarray(seeds, np.uint64)
        params = np.zeros((n, 2 * p))
        ex = np.zeros(n)
        ev = np.zeros(n, np.int32)
        tx = np.zeros((n, budget, 2 * p)) if trace else None
        tf = np.zeros((n, budget)) if trace else None
        self._call("qc_optimize_batch", structs, C.c_int(n), C.c_int(p), C.c_int(budget),
                   _p(sd), C.c_double(tol), _p(params), _p(ex), _p(ev), _p(tx), _p(tf))
        out = dict(params=params, expectation=ex, evals=ev)
        if trace:
            out["trace_x"], out["trace_f"] = tx, tf
        return out

    def top_candidates(self, amps: np.ndarray, top_k: int, fold: bool = True):
        a = np.ascontiguousarray(amps, np.complex128)
        k = max(int(top_k), 1)
        bits = np.zeros(k, np.uint32)
        probs = np.zeros(k)
        self._call("qc_top_candidates", C.c_int(int(np.log2(len(a)))), _p(a), C.c_int(top_k),
                   C.c_int(int(fold)), _p(bits), _p(probs))
        return bits, probs

    @staticmethod
    def _opts(top_k=2, layers=3, budget=200, seed=0, fold=True, threads=1, qubit_cap=20,
              tolerance=1e-5):
        return _SolveOptions(int(top_k), int(layers), int(budget), int(bool(fold)), int(seed),
                             int(qubit_cap), float(tolerance), int(threads), 0)

    def solve_batch(self, graphs, options) -> list[SolveResult]:
        """graphs: [(n, edges)]; options: list of dicts (SolveOptions fields) or one dict."""
        n = len(graphs)
        if isinstance(options, dict):
            options = [options] * n
        structs = (_Graph * n)()
        opts = (_SolveOptions * n)()
        res = (_SolveResult * n)()
        keep, bufs = [], []
        for i, ((nv, edges), o) in enumerate(zip(graphs, options)):
            gs, e = _graph(nv, edges)
            structs[i] = gs
            keep.append(e)
            so = self._opts(**o)
            opts[i] = so
            k = max(so.top_k, 1)
            b = np.zeros(k, np.uint32)
            pr = np.zeros(k)
            pa = np.zeros(2 * max(so.layers, 1))
            bufs.append((b, pr, pa))
            res[i] = _SolveResult(0, 0, 0, 0, 0.0, b.ctypes.data, pr.ctypes.data, pa.ctypes.data)
        self._call("qc_solve_batch", structs, C.c_int(n), opts, res)
        out = []
        for i in range(n):
            r = res[i]
            b, pr, pa = bufs[i]
            out.append(SolveResult(r.width, bool(r.folded), b[: r.count].copy(),
                                   pr[: r.count].copy(), pa[: 2 * opts[i].layers].copy(),
                                   r.expectation, r.evals))
        return out

    def solve_subgraph(self, n: int, edges, **opts) -> SolveResult:
        return self.solve_batch([(n, edges)], [opts])[0]

    # ---- merge.hpp -----------------------------------------------------------------
    @staticmethod
    def _pool(pool):
        widths = np.array([w for w, _ in pool], np.int32)
        counts = np.array([len(b) for _, b in pool], np.int32)
        bits = np.concatenate([np.asarray(b, np.uint32) for _, b in pool]) if pool else \
            np.zeros(0, np.uint32)
        bits = np.ascontiguousarray(bits, np.uint32)
        return _Pool(len(pool), widths.ctypes.data, counts.ctypes.data,
                     bits.ctypes.data if len(bits) else None), (widths, counts, bits)

    def level_merge(self, n: int, edges, chain, pool, start_level: int = 1, workers: int = 1,
                    incremental: bool = False, path_budget: float = 1e9,
                    halve: bool = False) -> MergeResult:
        g, ke = _graph(n, edges)
        P, kp = self._pool(pool)
        first = np.ascontiguousarray(chain[0], np.int32)
        last = np.ascontiguousarray(chain[1], np.int32)
        ch = _Chain(len(first), first.ctypes.data, last.ctypes.data)
        o = _MergeOptions(start_level, workers, int(incremental), int(halve), path_budget)
        asg = np.zeros(max(n, 1), np.uint8)
        r = _MergeResult(0.0, 0, asg.ctypes.data)
        self._call("qc_level_merge", C.byref(P), C.byref(g), C.byref(ch), C.byref(o), C.byref(r))
        return MergeResult(r.best_value, asg[:n].copy(), r.candidates_evaluated)

    def chained_merge(self, n: int, edges, chain, pool, window: int = 0,
                      window_leaves: int = 1 << 16, workers: int = 1,
                      halve: bool = True) -> MergeResult:
        g, ke = _graph(n, edges)
        P, kp = self._pool(pool)
        first = np.ascontiguousarray(chain[0], np.int32)
        last = np.ascontiguousarray(chain[1], np.int32)
        ch = _Chain(len(first), first.ctypes.data, last.ctypes.data)
        o = _ChainedMergeOptions(window, window_leaves, workers, int(halve))
        asg = np.zeros(max(n, 1), np.uint8)
        r = _MergeResult(0.0, 0, asg.ctypes.data)
        self._call("qc_chained_merge", C.byref(P), C.byref(g), C.byref(ch), C.byref(o),
                   C.byref(r))
        return MergeResult(r.best_value, asg[:n].copy(), r.candidates_evaluated)

    # ---- pipeline ------------------------------------------------------------------
    @staticmethod
    def run_config(qubit_cap=20, subgraphs=0, top_k=2, start_level=1, layers=3, budget=200,
                   seed=0, fold=True, halve_symmetry=False, partition_mode=0,
                   merge_incremental=True, merge_mode=0, shard_index=0, shard_count=1,
                   path_budget=1e9, nm_tolerance=1e-5, **_ignored) -> _RunConfig:
        return _RunConfig(qubit_cap, subgraphs, top_k, start_level, layers, budget, seed,
                          int(fold), int(halve_symmetry), partition_mode, int(merge_incremental),
                          merge_mode, shard_index, shard_count, 0, path_budget, nm_tolerance)

    def run_pipeline(self, n: int, edges, **cfg) -> RunReport:
        g, ke = _graph(n, edges)
        c = self.run_config(**cfg)
        rep = _RunReport()
        asg = C.create_string_buffer(n + 1)
        self._call("qc_run_pipeline", C.byref(g), C.byref(c), C.byref(rep), asg)
        return RunReport(rep.cut, rep.candidates_evaluated, rep.partition_s, rep.qaoa_s,
                         rep.merge_s, rep.total_s, rep.subgraphs, bool(rep.windowed), rep.evals,
                         asg.value.decode())

    def record_bytes(self, kcap: int, layers: int) -> int:
        return int(self.lib.qc_record_bytes(C.c_int(kcap), C.c_int(layers)))

    def shard_range(self, M: int, index: int, count: int):
        b = C.c_int32(0)
        e = C.c_int32(0)
        _check(self.lib, self.lib.qc_shard_range(C.c_int(M), C.c_int(index), C.c_int(count),
                                                 C.byref(b), C.byref(e)))
        return b.value, e.value

    def subgraph_count(self, n: int, edges, **cfg) -> int:
        g, ke = _graph(n, edges)
        c = self.run_config(**cfg)
        M = C.c_int32(0)
        self._call("qc_shard_solve", C.byref(g), C.byref(c), C.c_int32(0), C.c_int32(0), None,
                   C.c_int64(0), C.byref(M))
        return M.value

    def run_record_bytes(self, n: int, edges, **cfg) -> tuple[int, int]:
        """(record bytes, M) of the run: the geometry qc_shard_solve / qc_gather_topk /
        qc_merge_records use (widest piece of the same chain partition)."""
        return run_record_bytes(n, edges, **cfg)

    def shard_solve(self, n: int, edges, begin: int, end: int, record_bytes: int,
                    **cfg) -> np.ndarray:
        g, ke = _graph(n, edges)
        c = self.run_config(**cfg)
        buf = np.zeros(max((end - begin) * record_bytes, 1), np.uint8)
        M = C.c_int32(0)
        self._call("qc_shard_solve", C.byref(g), C.byref(c), C.c_int32(begin), C.c_int32(end),
                   _p(buf), C.c_int64(buf.size), C.byref(M))
        return buf[: (end - begin) * record_bytes]

    def merge_records(self, n: int, edges, records: np.ndarray, M: int, **cfg) -> RunReport:
        g, ke = _graph(n, edges)
        c = self.run_config(**cfg)
        rec = np.ascontiguousarray(records, np.uint8)
        rep = _RunReport()
        asg = C.create_string_buffer(n + 1)
        self._call("qc_merge_records", C.byref(g), C.byref(c), _p(rec), C.c_int64(rec.size),
                   C.c_int32(M), C.byref(rep), asg)
        return RunReport(rep.cut, rep.candidates_evaluated, rep.partition_s, rep.qaoa_s,
                         rep.merge_s, rep.total_s, rep.subgraphs, bool(rep.windowed), rep.evals,
                         asg.value.decode())


def run_record_bytes(n: int, edges, **cfg) -> tuple[int, int]:
    """qc_run_record_bytes (host only): (record bytes, subgraph count M) of (graph, cfg)."""
    lib = load_library()
    g, ke = _graph(n, edges)
    c = Engine.run_config(**cfg)
    rb = C.c_int64(0)
    M = C.c_int32(0)
    _check(lib, lib.qc_run_record_bytes(C.byref(g), C.byref(c), C.byref(rb), C.byref(M)))
    return int(rb.value), int(M.value)


def unpack_records(records: np.ndarray, M: int, record_bytes: int, layers: int) -> list:
    """Solve records (include/qcgpu.h layout) -> SolveResult per subgraph."""
    rec = np.ascontiguousarray(records, np.uint8)[: M * record_bytes].reshape(M, record_bytes)
    body = record_bytes - 24 - 16 * layers  # = 8*ceil(kcap/2) + 8*kcap, strictly increasing
    kcap = 0
    while 8 * ((kcap * 4 + 7) // 8) + 8 * kcap < body:
        kcap += 1
    if 8 * ((kcap * 4 + 7) // 8) + 8 * kcap != body:
        raise ConfigError(f"{record_bytes} bytes is not a record size for {layers} layers")
    boff = 24
    poff = boff + 8 * ((kcap * 4 + 7) // 8)
    aoff = poff + 8 * kcap
    out = []
    for r in rec:
        width, count, evals, folded = (int(x) for x in r[:16].view(np.int32))
        out.append(SolveResult(width, bool(folded), r[boff:boff + 4 * count].view(np.uint32).copy(),
                               r[poff:poff + 8 * count].view(np.float64).copy(),
                               r[aoff:aoff + 16 * layers].view(np.float64).copy(),
                               float(r[16:24].view(np.float64)[0]), evals))
    return out


class Comm:
    """qc_comm: one rank of the NCCL record-gather communicator (include/qcgpu.h)."""

    ID_BYTES = 128

    def __init__(self, engine: Engine, handle):
        self.engine = engine
        self._h = handle

    @staticmethod
    def unique_id() -> bytes:
        lib = load_library()
        buf = C.create_string_buffer(Comm.ID_BYTES)
        _check(lib, lib.qc_comm_id(buf))
        return buf.raw

    @classmethod
    def create(cls, engine: Engine, nranks: int, rank: int, uid: bytes) -> "Comm":
        h = C.c_void_p()
        buf = C.create_string_buffer(bytes(uid), Comm.ID_BYTES)
        _check(engine.lib, engine.lib.qc_comm_create(engine._h, C.c_int(nranks), C.c_int(rank),
                                                     buf, C.byref(h)))
        return cls(engine, h)

    @classmethod
    def create_all(cls, engines) -> list:
        n = len(engines)
        hs = (C.c_void_p * n)(*[e._h.value for e in engines])
        out = (C.c_void_p * n)()
        lib = engines[0].lib
        _check(lib, lib.qc_comm_create_all(hs, C.c_int(n), out))
        return [cls(e, C.c_void_p(out[i])) for i, e in enumerate(engines)]

    def rank(self) -> tuple[int, int]:
        r, nr = C.c_int32(0), C.c_int32(0)
        _check(self.engine.lib, self.engine.lib.qc_comm_rank(self._h, C.byref(r), C.byref(nr)))
        return r.value, nr.value

    def gather_topk(self, local: np.ndarray, count: int, M: int, record_bytes: int) -> np.ndarray:
        loc = np.ascontiguousarray(local, np.uint8)
        out = np.zeros(max(M * record_bytes, 1), np.uint8)
        _check(self.engine.lib, self.engine.lib.qc_gather_topk(
            self._h, _p(loc) if loc.size else None, C.c_int32(count), C.c_int32(M),
            C.c_int64(record_bytes), _p(out)))
        return out[: M * record_bytes]

    def close(self):
        if getattr(self, "_h", None):
            self.engine.lib.qc_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_pipeline_multi(engines, n: int, edges, comms=None, **cfg) -> RunReport:
    """qc_run_pipeline_multi: one process, one engine per GPU; NCCL record gather over
    `comms` (Comm.create_all), or a host-memory gather when comms is None."""
    lib = engines[0].lib
    k = len(engines)
    hs = (C.c_void_p * k)(*[e._h.value for e in engines])
    cs = (C.c_void_p * k)(*[c._h.value for c in comms]) if comms else None
    g, ke = _graph(n, edges)
    c = Engine.run_config(**cfg)
    rep = _RunReport()
    asg = C.create_string_buffer(n + 1)
    _check(lib, lib.qc_run_pipeline_multi(hs, cs, C.c_int(k), C.byref(g), C.byref(c),
                                          C.byref(rep), asg))
    return RunReport(rep.cut, rep.candidates_evaluated, rep.partition_s, rep.qaoa_s,
                     rep.merge_s, rep.total_s, rep.subgraphs, bool(rep.windowed), rep.evals,
                     asg.value.decode())


class PipelineSession:
    """qc_pipeline_*: partition + resident device cut tables, then repeatable execute()."""

    def __init__(self, engine: Engine, n: int, edges, **cfg):
        self.engine = engine
        self.n = n
        self.layers = int(cfg.get("layers", 3))
        g, self._edges = _graph(n, edges)
        c = engine.run_config(**cfg)
        h = C.c_void_p()
        _check(engine.lib, engine.lib.qc_pipeline_prepare(engine._h, C.byref(g), C.byref(c),
                                                          C.byref(h)))
        self._h = h

    def execute(self) -> RunReport:
        rep = _RunReport()
        asg = C.create_string_buffer(self.n + 1)
        _check(self.engine.lib, self.engine.lib.qc_pipeline_execute(self._h, C.byref(rep), asg))
        return RunReport(rep.cut, rep.candidates_evaluated, rep.partition_s, rep.qaoa_s,
                         rep.merge_s, rep.total_s, rep.subgraphs, bool(rep.windowed), rep.evals,
                         asg.value.decode())

    def geometry(self) -> tuple[int, int]:
        """(record bytes, M) of the session's run (qc_pipeline_records without a buffer)."""
        rb = C.c_int64(0)
        M = C.c_int32(0)
        _check(self.engine.lib, self.engine.lib.qc_pipeline_records(self._h, None, C.c_int64(0),
                                                                    C.byref(rb), C.byref(M)))
        return int(rb.value), int(M.value)

    def execute_shard(self) -> np.ndarray:
        """Sharded session (shard_count > 1): this rank's block of the QAOA stage
        (qc_pipeline_execute_shard) -> its packed solve records (uint8)."""
        lib = self.engine.lib
        rb, _ = self.geometry()
        b = C.c_int32(0)
        e = C.c_int32(0)
        _check(lib, lib.qc_pipeline_execute_shard(self._h, None, C.c_int64(0), C.byref(b), C.byref(e),
                                                  None))
        n = e.value - b.value
        buf = np.zeros(max(n * rb, 1), np.uint8)
        q = C.c_double(0)
        _check(lib, lib.qc_pipeline_execute_shard(self._h, _p(buf), C.c_int64(buf.size), C.byref(b),
                                                  C.byref(e), C.byref(q)))
        return buf[: n * rb]

    def merge_records(self, records: np.ndarray) -> RunReport:
        """pipeline.hpp:298-334 on all M gathered records (qc_pipeline_merge_records)."""
        rec = np.ascontiguousarray(records, np.uint8)
        rep = _RunReport()
        asg = C.create_string_buffer(self.n + 1)
        _check(self.engine.lib, self.engine.lib.qc_pipeline_merge_records(
            self._h, _p(rec), C.c_int64(rec.size), C.byref(rep), asg))
        return RunReport(rep.cut, rep.candidates_evaluated, rep.partition_s, rep.qaoa_s,
                         rep.merge_s, rep.total_s, rep.subgraphs, bool(rep.windowed), rep.evals,
                         asg.value.decode())

    def records(self) -> list:
        """SolveResults of the last execute() (qc_pipeline_records), in subgraph order."""
        lib = self.engine.lib
        rb = C.c_int64(0)
        M = C.c_int32(0)
        _check(lib, lib.qc_pipeline_records(self._h, None, C.c_int64(0), C.byref(rb), C.byref(M)))
        buf = np.zeros(max(rb.value * M.value, 1), np.uint8)
        _check(lib, lib.qc_pipeline_records(self._h, _p(buf), C.c_int64(buf.size), C.byref(rb),
                                            C.byref(M)))
        return unpack_records(buf, M.value, rb.value, self.layers)

    def close(self):
        if getattr(self, "_h", None):
            self.engine.lib.qc_pipeline_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def kcap_for(n_max_width: int, top_k: int, fold: bool = True) -> int:
    classes = 1 << (n_max_width - 1) if fold else 1 << n_max_width
    return classes if top_k == 0 else min(classes, top_k)
