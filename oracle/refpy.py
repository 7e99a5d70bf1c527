"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the parity checkers.

Two backends with the same Python surface:

* ``RefLib``  — ``oracle/_ref/libqcut_ref{,26}.so``: the unmodified reference headers
  (/root/reference/proj/include/qcut) behind oracle/ref_driver.cpp. Exists only where
  the reference tree was present at build time (this container; the .so travels to
  the GPU box inside the repo snapshot).
* ``OracleLib`` — ``oracle/_build/libqcut_oracle.so``: our C restatement
  (oracle/qcut_oracle.c), pinned against RefLib and tests/golden/.

Only tests/, oracle/gen_golden.py, __graft_entry__.smoke() and bench.py's
reference/cpu_baseline legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libqcut_ref.so")
REF26_SO = os.path.join(HERE, "_ref", "libqcut_ref26.so")
ORACLE_SO = os.path.join(HERE, "_build", "libqcut_oracle.so")

EDGE_DTYPE = np.dtype([("u", "<u4"), ("v", "<u4"), ("w", "<f8")])  # == qcut::Edge layout


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class ConfigError(OracleError):
    pass


class ResourceError(OracleError):
    pass


_ERR = {1: ConfigError, 2: ResourceError}


def edges_array(edges) -> np.ndarray:
    """(u, v, w) triples or an EDGE_DTYPE array -> contiguous EDGE_DTYPE array."""
    if isinstance(edges, np.ndarray) and edges.dtype == EDGE_DTYPE:
        return np.ascontiguousarray(edges)
    out = np.zeros(len(edges), dtype=EDGE_DTYPE)
    for i, e in enumerate(edges):
        out[i] = (e[0], e[1], e[2] if len(e) > 2 else 1.0)
    return out


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


class _SolveOpts(C.Structure):
    _fields_ = [("top_k", C.c_int), ("layers", C.c_int), ("budget", C.c_int),
                ("seed", C.c_uint64), ("fold", C.c_int), ("threads", C.c_int),
                ("qubit_cap", C.c_uint64), ("tolerance", C.c_double)]


class _RunConfig(C.Structure):
    _fields_ = [("qubit_cap", C.c_int), ("solvers", C.c_int), ("subgraphs", C.c_int),
                ("top_k", C.c_int), ("start_level", C.c_int), ("layers", C.c_int),
                ("budget", C.c_int), ("seed", C.c_uint64), ("fold", C.c_int),
                ("halve_symmetry", C.c_int), ("partition_mode", C.c_int),
                ("merge_incremental", C.c_int), ("merge_mode", C.c_int), ("workers", C.c_int),
                ("path_budget", C.c_double), ("nm_tolerance", C.c_double),
                ("baseline", C.c_int)]


class _RunResult(C.Structure):
    _fields_ = [("cut", C.c_double), ("leaves", C.c_uint64), ("partition_s", C.c_double),
                ("qaoa_s", C.c_double), ("merge_s", C.c_double), ("total_s", C.c_double),
                ("baseline_value", C.c_double), ("subgraphs", C.c_int), ("windowed", C.c_int)]


@dataclass
class SolveOut:
    bits: np.ndarray
    probs: np.ndarray
    params: np.ndarray
    expectation: float
    evals: int
    width: int = 0


@dataclass
class MergeOut:
    value: float
    assignment: np.ndarray  # uint8 per vertex
    leaves: int


class _Lib:
    prefix = ""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.path = path
        self.lib = C.CDLL(path)
        getattr(self.lib, self.prefix + "last_error").restype = C.c_char_p

    def _call(self, name, *args):
        rc = getattr(self.lib, self.prefix + name)(*args)
        if rc != 0:
            msg = getattr(self.lib, self.prefix + "last_error")().decode()
            raise _ERR.get(rc, OracleError)(rc, msg)

    # --- graph / partition ---------------------------------------------------
    def generate_er(self, n: int, p: float, seed: int) -> np.ndarray:
        m = C.c_longlong(0)
        self._call("generate_er", C.c_int(n), C.c_double(p), C.c_uint64(seed), None,
                   C.c_longlong(0), C.byref(m))
        out = np.zeros(m.value, dtype=EDGE_DTYPE)
        self._call("generate_er", C.c_int(n), C.c_double(p), C.c_uint64(seed), _p(out),
                   C.c_longlong(m.value), C.byref(m))
        return out

    def partition(self, n: int, edges, M: int, mode: int = 0, cap: int = 0):
        e = edges_array(edges)
        first = np.zeros(M, np.int32)
        last = np.zeros(M, np.int32)
        local_m = np.zeros(M, np.int32)
        inter = C.c_longlong(0)
        self._call("partition", C.c_int(n), C.c_int(len(e)), _p(e), C.c_int(M), C.c_int(mode),
                   C.c_int(cap), _p(first), _p(last), _p(local_m), C.byref(inter))
        return first, last, local_m, inter.value

    def derive_subgraph_count(self, n: int, cap: int) -> int:
        out = C.c_int(0)
        self._call("derive_subgraph_count", C.c_longlong(n), C.c_longlong(cap), C.byref(out))
        return out.value

    # --- statevector ---------------------------------------------------------
    def cost_table(self, n: int, edges, cap: int = 24):
        e = edges_array(edges)
        out = np.zeros(1 << n, np.float64)
        integral = C.c_int(0)
        mx = C.c_double(0)
        self._call("cost_table", C.c_int(n), C.c_int(len(e)), _p(e), C.c_int(cap), _p(out),
                   C.byref(integral), C.byref(mx))
        return out, bool(integral.value), mx.value

    def plus_state(self, q: int, cap: int = 24) -> np.ndarray:
        out = np.zeros(1 << q, np.complex128)
        self._call("plus_state", C.c_int(q), C.c_int(cap), _p(out))
        return out

    def apply_cost_layer(self, amps: np.ndarray, n: int, edges, gamma: float, threads: int = 1):
        a = np.ascontiguousarray(amps, np.complex128).copy()
        e = edges_array(edges)
        q = int(np.log2(len(a)))
        self._call("apply_cost_layer", C.c_int(q), _p(a), C.c_int(n), C.c_int(len(e)), _p(e),
                   C.c_double(gamma), C.c_int(threads))
        return a

    def apply_mixer_layer(self, amps: np.ndarray, beta: float, threads: int = 1):
        a = np.ascontiguousarray(amps, np.complex128).copy()
        q = int(np.log2(len(a)))
        self._call("apply_mixer_layer", C.c_int(q), _p(a), C.c_double(beta), C.c_int(threads))
        return a

    def expectation(self, amps: np.ndarray, n: int, edges, threads: int = 1) -> float:
        a = np.ascontiguousarray(amps, np.complex128)
        e = edges_array(edges)
        out = C.c_double(0)
        q = int(np.log2(len(a)))
        self._call("expectation", C.c_int(q), _p(a), C.c_int(n), C.c_int(len(e)), _p(e),
                   C.c_int(threads), C.byref(out))
        return out.value

    def norm_sq(self, amps: np.ndarray, threads: int = 1) -> float:
        a = np.ascontiguousarray(amps, np.complex128)
        out = C.c_double(0)
        self._call("norm_sq", C.c_int(int(np.log2(len(a)))), _p(a), C.c_int(threads), C.byref(out))
        return out.value

    def run_ansatz(self, n: int, edges, gammas, betas, threads: int = 1, want_amps=True):
        e = edges_array(edges)
        g = np.ascontiguousarray(gammas, np.float64)
        b = np.ascontiguousarray(betas, np.float64)
        amps = np.zeros(1 << n, np.complex128) if want_amps else None
        ex = C.c_double(0)
        self._call("run_ansatz", C.c_int(n), C.c_int(len(e)), _p(e), C.c_int(len(g)), _p(g),
                   _p(b), C.c_int(threads), _p(amps), C.byref(ex))
        return amps, ex.value

    def linear_ramp(self, p: int):
        g = np.zeros(p)
        b = np.zeros(p)
        self._call("linear_ramp", C.c_int(p), _p(g), _p(b))
        return g, b

    def optimize(self, n: int, edges, p: int, budget: int, seed: int = 0, threads: int = 1,
                 tol: float = 1e-5, trace: bool = False):
        e = edges_array(edges)
        params = np.zeros(2 * p)
        ex = C.c_double(0)
        ev = C.c_int(0)
        tx = np.zeros((budget, 2 * p)) if trace else None
        tf = np.zeros(budget) if trace else None
        tl = C.c_int(0)
        self._call("optimize", C.c_int(n), C.c_int(len(e)), _p(e), C.c_int(p), C.c_int(budget),
                   C.c_uint64(seed), C.c_int(threads), C.c_double(tol), _p(params), C.byref(ex),
                   C.byref(ev), _p(tx), _p(tf), C.byref(tl))
        out = dict(params=params, expectation=ex.value, evals=ev.value)
        if trace:
            out["trace_x"] = tx[: tl.value]
            out["trace_f"] = tf[: tl.value]
        return out

    def top_candidates(self, amps: np.ndarray, top_k: int, fold: bool = True):
        a = np.ascontiguousarray(amps, np.complex128)
        bits = np.zeros(max(top_k, 1), np.uint32)
        probs = np.zeros(max(top_k, 1), np.float64)
        self._call("top_candidates", C.c_int(int(np.log2(len(a)))), _p(a), C.c_int(top_k),
                   C.c_int(int(fold)), _p(bits), _p(probs))
        return bits, probs

    def solve_subgraph(self, n: int, edges, top_k=2, layers=3, budget=200, seed=0, fold=True,
                       threads=1, qubit_cap=20, tolerance=1e-5) -> SolveOut:
        e = edges_array(edges)
        o = _SolveOpts(top_k, layers, budget, seed, int(fold), threads, qubit_cap, tolerance)
        cap = max(top_k, 1)
        bits = np.zeros(cap, np.uint32)
        probs = np.zeros(cap)
        cnt = C.c_int(0)
        params = np.zeros(2 * max(layers, 1))
        ex = C.c_double(0)
        ev = C.c_int(0)
        self._call("solve_subgraph", C.c_int(n), C.c_int(len(e)), _p(e), C.byref(o), _p(bits),
                   _p(probs), C.byref(cnt), _p(params), C.byref(ex), C.byref(ev))
        return SolveOut(bits[: cnt.value], probs[: cnt.value], params, ex.value, ev.value)

    # --- merge ---------------------------------------------------------------
    @staticmethod
    def _pool_arrays(pool):
        widths = np.array([w for w, _ in pool], np.int32)
        counts = np.array([len(b) for _, b in pool], np.int32)
        bits = np.concatenate([np.asarray(b, np.uint32) for _, b in pool]) if pool else \
            np.zeros(0, np.uint32)
        return widths, counts, np.ascontiguousarray(bits, np.uint32)

    def level_merge(self, n: int, edges, M: int, pool, mode: int = 0, start_level: int = 1,
                    workers: int = 1, incremental: bool = False, path_budget: float = 1e9,
                    halve: bool = False) -> MergeOut:
        e = edges_array(edges)
        w, c, b = self._pool_arrays(pool)
        val = C.c_double(0)
        asg = np.zeros(n, np.uint8)
        leaves = C.c_uint64(0)
        self._call("level_merge", C.c_int(n), C.c_int(len(e)), _p(e), C.c_int(M), C.c_int(mode),
                   _p(w), _p(c), _p(b), C.c_int(start_level), C.c_int(workers),
                   C.c_int(int(incremental)), C.c_double(path_budget), C.c_int(int(halve)),
                   C.byref(val), _p(asg), C.byref(leaves))
        return MergeOut(val.value, asg, leaves.value)

    def chained_merge(self, n: int, edges, M: int, pool, mode: int = 0, window: int = 0,
                      window_leaves: int = 1 << 16, workers: int = 1,
                      halve: bool = True) -> MergeOut:
        e = edges_array(edges)
        w, c, b = self._pool_arrays(pool)
        val = C.c_double(0)
        asg = np.zeros(n, np.uint8)
        leaves = C.c_uint64(0)
        self._call("chained_merge", C.c_int(n), C.c_int(len(e)), _p(e), C.c_int(M),
                   C.c_int(mode), _p(w), _p(c), _p(b), C.c_longlong(window),
                   C.c_longlong(window_leaves), C.c_int(workers), C.c_int(int(halve)),
                   C.byref(val), _p(asg), C.byref(leaves))
        return MergeOut(val.value, asg, leaves.value)

    # --- pipeline ------------------------------------------------------------
    def run_pipeline(self, n: int, edges, qubit_cap=20, solvers=0, subgraphs=0, top_k=2,
                     start_level=1, layers=3, budget=200, seed=0, fold=True,
                     halve_symmetry=False, partition_mode=0, merge_incremental=True,
                     merge_mode=0, workers=1, path_budget=1e9, nm_tolerance=1e-5,
                     baseline=3):
        e = edges_array(edges)
        cfg = _RunConfig(qubit_cap, solvers, subgraphs, top_k, start_level, layers, budget, seed,
                         int(fold), int(halve_symmetry), partition_mode, int(merge_incremental),
                         merge_mode, workers, path_budget, nm_tolerance, baseline)
        res = _RunResult()
        asg = C.create_string_buffer(n + 1)
        mcap = 4096
        sub_ex = np.zeros(mcap)
        sub_ev = np.zeros(mcap, np.int32)
        self._call("run_pipeline", C.c_int(n), C.c_int(len(e)), _p(e), C.byref(cfg),
                   C.byref(res), asg, _p(sub_ex), _p(sub_ev), C.c_int(mcap))
        M = res.subgraphs
        return dict(cut=res.cut, leaves=res.leaves, partition_s=res.partition_s,
                    qaoa_s=res.qaoa_s, merge_s=res.merge_s, total_s=res.total_s,
                    subgraphs=M, windowed=bool(res.windowed), assignment=asg.value.decode(),
                    sub_expectation=sub_ex[:M].copy(), sub_evals=sub_ev[:M].copy())


class RefLib(_Lib):
    prefix = "ref_"

    def __init__(self, cap26: bool = False):
        super().__init__(REF26_SO if cap26 else REF_SO)

    def qubit_cap(self) -> int:
        return self.lib.ref_qubit_cap()

    def solve_stage(self, n, edges, M, indices, top_k, layers, budget, seed=0, fold=True,
                    slots=1, threads=1, qubit_cap=20, tol=1e-5, mode=0):
        """pipeline.hpp:219-296's QAOA stage for the subgraphs `indices` of the reference's
        own partition (ref_solve_stage): one SolveOut per index, plus wall seconds."""
        e = edges_array(edges)
        idx = np.ascontiguousarray(indices, np.int32)
        cnt = len(idx)
        kcap = max(int(top_k), 1) if top_k else (1 << (qubit_cap - 1 if fold else qubit_cap))
        widths = np.zeros(cnt, np.int32)
        counts = np.zeros(cnt, np.int32)
        bits = np.zeros((cnt, kcap), np.uint32)
        probs = np.zeros((cnt, kcap))
        params = np.zeros((cnt, 2 * layers))
        ex = np.zeros(cnt)
        ev = np.zeros(cnt, np.int32)
        secs = C.c_double(0)
        self._call("solve_stage", C.c_int(n), C.c_int(len(e)), _p(e), C.c_int(M), C.c_int(mode),
                   C.c_int(qubit_cap), _p(idx), C.c_int(cnt), C.c_int(top_k), C.c_int(layers),
                   C.c_int(budget), C.c_uint64(seed), C.c_int(int(fold)), C.c_int(slots),
                   C.c_int(threads), C.c_double(tol), C.c_int(kcap), _p(widths), _p(counts),
                   _p(bits), _p(probs), _p(params), _p(ex), _p(ev), C.byref(secs))
        out = [SolveOut(bits[k, : counts[k]].copy(), probs[k, : counts[k]].copy(), params[k].copy(),
                        float(ex[k]), int(ev[k])) for k in range(cnt)]
        for o, w in zip(out, widths):
            o.width = int(w)
        return out, secs.value

    def eval_timing(self, n, edges, gammas, betas, threads=1, reps=3):
        """Seconds per objective evaluation (run_ansatz + expectation on a prebuilt
        CostTable, qaoa.hpp:89-91) at fixed angles, and the expectation."""
        e = edges_array(edges)
        g = np.ascontiguousarray(gammas, np.float64)
        b = np.ascontiguousarray(betas, np.float64)
        sec = C.c_double(0)
        ex = C.c_double(0)
        self._call("eval_timing", C.c_int(n), C.c_int(len(e)), _p(e), C.c_int(len(g)), _p(g),
                   _p(b), C.c_int(threads), C.c_int(reps), C.byref(sec), C.byref(ex))
        return sec.value, ex.value


class RefChecker:
    """The parity checker of the -m gpu tests: the reference build itself (RefLib over
    oracle/_ref/libqcut_ref.so; libqcut_ref26.so once set_qubit_cap(26), BASELINE config 5),
    with the C restatement (OracleLib) only for what the reference has no function for
    (the config-3 regular generator). Same Python surface as OracleLib."""

    kind = "reference"

    def __init__(self):
        self._r24 = RefLib()
        self._r26 = RefLib(cap26=True) if ref_available(True) else None
        self._cur = self._r24
        self._orc = OracleLib() if oracle_available() else None

    def set_qubit_cap(self, cap: int):
        if cap > 24 and self._r26 is None:
            raise FileNotFoundError(REF26_SO)
        self._cur = self._r26 if cap > 24 else self._r24

    def qubit_cap(self) -> int:
        return self._cur.qubit_cap()

    def generate_regular(self, *a, **kw):
        return self._orc.generate_regular(*a, **kw)

    def __getattr__(self, name):
        return getattr(self._cur, name)


def checker():
    """RefChecker when oracle/_ref was built (this container; the .so files travel to the
    GPU box in the repo snapshot), else the C restatement."""
    if ref_available() and ref_available(True):
        return RefChecker()
    return OracleLib()


class OracleLib(_Lib):
    prefix = "orc_"

    def __init__(self):
        super().__init__(ORACLE_SO)

    def generate_regular(self, n: int, d: int, seed: int, wlo: int = 1, whi: int = 10) -> np.ndarray:
        m = C.c_longlong(0)
        self._call("generate_regular", C.c_int(n), C.c_int(d), C.c_uint64(seed), C.c_int(wlo),
                   C.c_int(whi), None, C.c_longlong(0), C.byref(m))
        out = np.zeros(m.value, dtype=EDGE_DTYPE)
        self._call("generate_regular", C.c_int(n), C.c_int(d), C.c_uint64(seed), C.c_int(wlo),
                   C.c_int(whi), _p(out), C.c_longlong(m.value), C.byref(m))
        return out

    def set_qubit_cap(self, cap: int):
        """kQubitCap (statevector.hpp:20): 24 in the reference, 26 for config 5."""
        self.lib.orc_set_qubit_cap(C.c_int(cap))

    def qubit_cap(self) -> int:
        return self.lib.orc_qubit_cap()


def ref_available(cap26: bool = False) -> bool:
    return os.path.exists(REF26_SO if cap26 else REF_SO)


def oracle_available() -> bool:
    return os.path.exists(ORACLE_SO)
