"""oracle -- TEST INFRASTRUCTURE ONLY.

ctypes front-ends over two CPU checkers of the reference mlnmf solver path:

* ``Restated``  -- oracle/_build/libmlnmf_oracle.so, the serial C restatement
  (oracle/mlnmf_oracle.c, every function cites the reference file:line).
* ``Reference`` -- oracle/_ref/libmlnmf_ref.so, the UNMODIFIED reference
  (/root/reference/proj/src) compiled by oracle/Makefile with OpenMP, behind
  the extern "C" shim oracle/ref_capi.cpp.  Present only where it was built
  (this container builds it; the .so travels to the GPU box via gpurun).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this package.  The product
(paper_1009_0881_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATED_SO = os.path.join(HERE, "_build", "libmlnmf_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmlnmf_ref.so")

ANLS, MU, HALS = 0, 1, 2
NONE, NI, VC, FMG = 0, 1, 2, 3
KINDS = {"anls": ANLS, "mu": MU, "hals": HALS}
CYCLES = {"none": NONE, "ni": NI, "vc": VC, "fmg": FMG}

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_sz = C.c_size_t


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


def _d(a):
    return a.ctypes.data_as(_dp)


def _i(a):
    return a.ctypes.data_as(_ip)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


@dataclass
class Trace:
    """Mirror of mlnmf::RunTrace (proj/include/mlnmf/solvers.hpp:14-35)."""
    elapsed: np.ndarray
    work: np.ndarray
    level: np.ndarray
    error: np.ndarray
    alloc_level: np.ndarray
    alloc_amount: np.ndarray
    counts: np.ndarray
    degenerate: int
    phase_level: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    phase_steps: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))


class _OrcTrace(C.Structure):
    _fields_ = [
        ("n_samples", _sz), ("cap_samples", _sz),
        ("elapsed", _dp), ("work", _dp), ("level", _ip), ("error", _dp),
        ("n_alloc", _sz), ("alloc_level", _ip), ("alloc_amount", _dp),
        ("n_counts", _sz), ("counts", _ip), ("hals_degenerate", C.c_int),
        ("n_phases", _sz), ("phase_level", _ip), ("phase_steps", C.POINTER(C.c_long)),
    ]


class _OrcGen(C.Structure):
    _fields_ = [
        ("h", _sz), ("w", _sz), ("r", _sz), ("blobs", _sz),
        ("sigma_min", C.c_double), ("sigma_max", C.c_double),
        ("noise_kind", C.c_int), ("noise_scale", C.c_double), ("seed", C.c_uint64),
    ]


def _arr(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


class _Common:
    lib: C.CDLL
    prefix: str

    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self._errmsg())

    def _errmsg(self):
        return ""

    # ---- core ----
    def random_init(self, m, n, r, seed):
        V = np.empty((m, r)); W = np.empty((r, n))
        self._check(self._fn("random_init")(_sz(m), _sz(n), _sz(r), C.c_uint64(seed), _d(V), _d(W)))
        return V, W

    def iteration_cost(self, m, n, r, kind):
        f = self._fn("iteration_cost")
        f.restype = C.c_double
        return f(_sz(m), _sz(n), _sz(r), C.c_int(KINDS.get(kind, kind)))

    def mu_step(self, M, V, W):
        M = _f64(M); V = _f64(V).copy(); W = _f64(W).copy()
        m, n = M.shape; r = V.shape[1]
        rc = self._fn("mu_step")(_d(M), _d(V), _d(W), _sz(m), _sz(n), _sz(r))
        if rc not in (None, 0):
            self._check(rc)
        return V, W

    def hals_step(self, M, V, W):
        M = _f64(M); V = _f64(V).copy(); W = _f64(W).copy()
        m, n = M.shape; r = V.shape[1]
        deg = C.c_int(0)
        rc = self._fn("hals_step")(_d(M), _d(V), _d(W), _sz(m), _sz(n), _sz(r), C.byref(deg))
        if rc not in (None, 0):
            self._check(rc)
        return V, W, deg.value

    def anls_step(self, M, V, W):
        M = _f64(M); V = _f64(V).copy(); W = _f64(W).copy()
        m, n = M.shape; r = V.shape[1]
        counts = np.zeros(m + n, np.int32)
        self._check(self._fn("anls_step")(_d(M), _d(V), _d(W), _sz(m), _sz(n), _sz(r), _i(counts)))
        return V, W, counts

    def nnls_active_set(self, G, h, x0):
        G = _f64(G); h = _f64(h); x0 = _f64(x0)
        r = h.shape[0]
        x = np.zeros(r); it = C.c_int(0)
        self._check(self._fn("nnls_active_set")(_d(G), _d(h), _d(x0), _sz(r), _d(x), C.byref(it)))
        return x, it.value

    # ---- diagnostics (transfer.cpp:128-153) ----
    def smoothness(self, M, h, w):
        M = _f64(M)
        out = C.c_double()
        self._check(self._fn("smoothness")(_d(M), _sz(h), _sz(w), _sz(M.shape[1]), C.byref(out)))
        return out.value

    def initialization_bound(self, M, h, w, Vc, W):
        M = _f64(M); Vc = _f64(Vc); W = _f64(W)
        lhs = C.c_double(); rhs = C.c_double()
        self._check(self._fn("initialization_bound")(_d(M), _sz(h), _sz(w), _sz(M.shape[1]), _d(Vc), _d(W),
                                                     _sz(Vc.shape[1]), C.byref(lhs), C.byref(rhs)))
        return lhs.value, rhs.value


class Restated(_Common):
    """The serial C restatement (oracle/mlnmf_oracle.c)."""
    prefix = "orc_"

    def __init__(self, path: str = RESTATED_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = C.CDLL(path)
        L = self.lib
        L.orc_frobenius_error.restype = C.c_double
        L.orc_frobenius_norm.restype = C.c_double
        L.orc_mu_step.restype = None
        L.orc_hals_step.restype = None
        L.orc_op_apply.restype = None
        L.orc_build_restriction.restype = C.c_void_p
        L.orc_build_prolongation.restype = C.c_void_p
        L.orc_generate.restype = None
        L.orc_trace_free.argtypes = [C.c_void_p]
        L.orc_op_free.argtypes = [C.c_void_p]
        L.orc_splitmix_next.restype = C.c_uint64

    def splitmix_first(self, seed):
        s = C.c_uint64(seed)
        return self.lib.orc_splitmix_next(C.byref(s))

    def frobenius_error(self, M, V, W):
        M = _f64(M); V = _f64(V); W = _f64(W)
        return self.lib.orc_frobenius_error(_d(M), _d(V), _d(W), _sz(M.shape[0]), _sz(M.shape[1]), _sz(V.shape[1]))

    def coarsen(self, h, w):
        hc = _sz(); wc = _sz()
        self._check(self.lib.orc_coarsen(_sz(h), _sz(w), C.byref(hc), C.byref(wc)))
        return hc.value, wc.value

    def operator_dense(self, h, w, which):
        hc, wc = self.coarsen(h, w)
        fine, coarse = h * w, hc * wc
        op = (self.lib.orc_build_restriction if which == 0 else self.lib.orc_build_prolongation)(_sz(h), _sz(w))
        out_dim, in_dim = (coarse, fine) if which == 0 else (fine, coarse)
        D = np.zeros((out_dim, in_dim))
        for j in range(in_dim):
            e = np.zeros((in_dim, 1)); e[j, 0] = 1.0
            y = np.zeros((out_dim, 1))
            self.lib.orc_op_apply(C.c_void_p(op), _d(e), _sz(1), _d(y))
            D[:, j] = y[:, 0]
        self.lib.orc_op_free(C.c_void_p(op))
        return D

    def apply_operator(self, h, w, which, X):
        X = _f64(X)
        op = (self.lib.orc_build_restriction if which == 0 else self.lib.orc_build_prolongation)(_sz(h), _sz(w))
        hc, wc = self.coarsen(h, w)
        out_dim = hc * wc if which == 0 else h * w
        Y = np.zeros((out_dim, X.shape[1]))
        self.lib.orc_op_apply(C.c_void_p(op), _d(X), _sz(X.shape[1]), _d(Y))
        self.lib.orc_op_free(C.c_void_p(op))
        return Y

    def _take_trace(self, tp):
        t = C.cast(tp, C.POINTER(_OrcTrace)).contents
        tr = Trace(
            _arr(t.elapsed, t.n_samples, np.float64), _arr(t.work, t.n_samples, np.float64),
            _arr(t.level, t.n_samples, np.int32), _arr(t.error, t.n_samples, np.float64),
            _arr(t.alloc_level, t.n_alloc, np.int32), _arr(t.alloc_amount, t.n_alloc, np.float64),
            _arr(t.counts, t.n_counts, np.int32), int(t.hals_degenerate),
            _arr(t.phase_level, t.n_phases, np.int32), _arr(t.phase_steps, t.n_phases, np.int64))
        self.lib.orc_trace_free(C.c_void_p(tp))
        return tr

    def run_configuration(self, M, h, w, levels, kind, cycle, rank, seed, amount,
                          trace_every=1, mode=0):
        M = _f64(M); m, n = M.shape
        V = np.zeros((m, rank)); W = np.zeros((rank, n))
        tp = C.c_void_p()
        rc = self.lib.orc_run_configuration(
            _d(M), _sz(m), _sz(n), _sz(h), _sz(w), _sz(levels), C.c_int(KINDS.get(kind, kind)),
            C.c_int(CYCLES.get(cycle, cycle)), _sz(rank), C.c_uint64(seed), C.c_int(mode),
            C.c_double(amount), _sz(trace_every), _d(V), _d(W), C.byref(tp))
        tr = self._take_trace(tp.value) if tp.value else None
        self._check(rc)
        return V, W, tr

    def run_solver(self, M, V0, W0, kind, amount, trace_every=1, mode=0):
        M = _f64(M); V = _f64(V0).copy(); W = _f64(W0).copy()
        m, n = M.shape
        tp = C.c_void_p()
        rc = self.lib.orc_run_solver(_d(M), _sz(m), _sz(n), _sz(V.shape[1]), _d(V), _d(W),
                                     C.c_int(KINDS.get(kind, kind)), C.c_int(mode), C.c_double(amount),
                                     _sz(trace_every), C.byref(tp))
        tr = self._take_trace(tp.value) if tp.value else None
        self._check(rc)
        return V, W, tr

    def run_cycle_on(self, M, h, w, hierarchy_levels, levels, V0, W0, kind, cycle, amount,
                     trace_every=1, mode=0):
        M = _f64(M); V0 = _f64(V0); W0 = _f64(W0)
        m, n = M.shape; r = V0.shape[1]
        V = np.zeros_like(V0); W = np.zeros_like(W0)
        tp = C.c_void_p()
        rc = self.lib.orc_run_cycle_on(
            _d(M), _sz(m), _sz(n), _sz(h), _sz(w), _sz(hierarchy_levels), _sz(levels),
            _d(V0), _d(W0), _sz(r), C.c_int(KINDS.get(kind, kind)), C.c_int(CYCLES.get(cycle, cycle)),
            C.c_int(mode), C.c_double(amount), _sz(trace_every), _d(V), _d(W), C.byref(tp))
        tr = self._take_trace(tp.value) if tp.value else None
        self._check(rc)
        return V, W, tr

    def generate(self, h, w, r, blobs, sigma_min, sigma_max, noise_kind, noise_scale, seed,
                 n_total, col0=0, n_cols=None):
        n_cols = n_total - col0 if n_cols is None else n_cols
        p = _OrcGen(h, w, r, blobs, sigma_min, sigma_max, noise_kind, noise_scale, seed)
        M = np.zeros((h * w, n_cols))
        self.lib.orc_generate(C.byref(p), _sz(n_total), _sz(col0), _sz(n_cols), _d(M))
        return M


class Reference(_Common):
    """The unmodified reference library (oracle/_ref/libmlnmf_ref.so)."""
    prefix = "ref_"

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_splitmix_first.restype = C.c_uint64
        for nm in ("ref_trace_n_samples", "ref_trace_n_alloc", "ref_trace_n_counts"):
            getattr(L, nm).restype = _sz
            getattr(L, nm).argtypes = [C.c_void_p]
        L.ref_trace_degenerate.argtypes = [C.c_void_p]
        L.ref_trace_free.argtypes = [C.c_void_p]
        L.ref_trace_copy.restype = None

    @staticmethod
    def available(path: str = REF_SO) -> bool:
        return os.path.exists(path)

    def _errmsg(self):
        return self.lib.ref_last_error().decode()

    def splitmix_first(self, seed):
        return self.lib.ref_splitmix_first(C.c_uint64(seed))

    def frobenius_error(self, M, V, W):
        M = _f64(M); V = _f64(V); W = _f64(W)
        out = C.c_double()
        self._check(self.lib.ref_frobenius_error(_d(M), _d(V), _d(W), _sz(M.shape[0]), _sz(M.shape[1]),
                                                 _sz(V.shape[1]), C.byref(out)))
        return out.value

    def operator_dense(self, h, w, which):
        hc, wc = (h + 1) // 2, (w + 1) // 2
        fine, coarse = h * w, hc * wc
        shape = (coarse, fine) if which == 0 else (fine, coarse)
        D = np.zeros(shape)
        self._check(self.lib.ref_operator_dense(_sz(h), _sz(w), C.c_int(which), _d(D)))
        return D

    def apply_operator(self, h, w, which, X):
        X = _f64(X)
        hc, wc = (h + 1) // 2, (w + 1) // 2
        out_dim = hc * wc if which == 0 else h * w
        Y = np.zeros((out_dim, X.shape[1]))
        self._check(self.lib.ref_apply_operator(_sz(h), _sz(w), C.c_int(which), _d(X), _sz(X.shape[1]), _d(Y)))
        return Y

    def _take_trace(self, tp):
        L = self.lib
        ns, na, nc = L.ref_trace_n_samples(tp), L.ref_trace_n_alloc(tp), L.ref_trace_n_counts(tp)
        el = np.zeros(ns); wk = np.zeros(ns); lv = np.zeros(ns, np.int32); er = np.zeros(ns)
        al = np.zeros(na, np.int32); aa = np.zeros(na); cn = np.zeros(max(nc, 1), np.int32)
        L.ref_trace_copy(C.c_void_p(tp), _d(el), _d(wk), _i(lv), _d(er), _i(al), _d(aa), _i(cn))
        deg = L.ref_trace_degenerate(C.c_void_p(tp))
        L.ref_trace_free(C.c_void_p(tp))
        return Trace(el, wk, lv, er, al, aa, cn[:nc], int(deg))

    def run_configuration(self, M, h, w, levels, kind, cycle, rank, seed, amount,
                          trace_every=1, mode=0):
        M = _f64(M); m, n = M.shape
        V = np.zeros((m, rank)); W = np.zeros((rank, n))
        tp = C.c_void_p()
        rc = self.lib.ref_run_configuration(
            _d(M), _sz(m), _sz(n), _sz(h), _sz(w), _sz(levels), C.c_int(KINDS.get(kind, kind)),
            C.c_int(CYCLES.get(cycle, cycle)), _sz(rank), C.c_uint64(seed), C.c_int(mode),
            C.c_double(amount), _sz(trace_every), _d(V), _d(W), C.byref(tp))
        self._check(rc)
        return V, W, self._take_trace(tp.value)

    def run_solver(self, M, V0, W0, kind, amount, trace_every=1, mode=0):
        M = _f64(M); V = _f64(V0).copy(); W = _f64(W0).copy()
        m, n = M.shape
        tp = C.c_void_p()
        rc = self.lib.ref_run_solver(_d(M), _sz(m), _sz(n), _sz(V.shape[1]), _d(V), _d(W),
                                     C.c_int(KINDS.get(kind, kind)), C.c_int(mode), C.c_double(amount),
                                     _sz(trace_every), C.byref(tp))
        self._check(rc)
        return V, W, self._take_trace(tp.value)

    def run_cycle_on(self, M, h, w, hierarchy_levels, levels, V0, W0, kind, cycle, amount,
                     trace_every=1, mode=0):
        M = _f64(M); V0 = _f64(V0); W0 = _f64(W0)
        m, n = M.shape; r = V0.shape[1]
        V = np.zeros_like(V0); W = np.zeros_like(W0)
        tp = C.c_void_p()
        rc = self.lib.ref_run_cycle_on(
            _d(M), _sz(m), _sz(n), _sz(h), _sz(w), _sz(hierarchy_levels), _sz(levels),
            _d(V0), _d(W0), _sz(r), C.c_int(KINDS.get(kind, kind)), C.c_int(CYCLES.get(cycle, cycle)),
            C.c_int(mode), C.c_double(amount), _sz(trace_every), _d(V), _d(W), C.byref(tp))
        self._check(rc)
        return V, W, self._take_trace(tp.value)


# ---------------------------------------------------------------------------
# BASELINE.json configurations (DESIGN.md section 3 restates them).
# ---------------------------------------------------------------------------
CONFIGS = {
    0: dict(h=32, w=32, n=1000, r=20, levels=3, blobs=3, sigma=(2.0, 6.0), noise=(0, 0.01),
            scale_to_unit=False, budget=100.0),
    1: dict(h=19, w=19, n=2429, r=49, levels=2, blobs=3, sigma=(2.0, 6.0), noise=(0, 0.01),
            scale_to_unit=True, budget=500.0),
    2: dict(h=112, w=92, n=400, r=40, levels=4, blobs=5, sigma=(2.0, 6.0), noise=(1, 0.02),
            scale_to_unit=False, budget=100.0),
    3: dict(h=243, w=320, n=165, r=49, levels=5, blobs=3, sigma=(4.0, 20.0), noise=(0, 0.01),
            scale_to_unit=False, budget=100.0),
    4: dict(h=256, w=256, n=262144, r=64, levels=5, blobs=3, sigma=(4.0, 20.0), noise=(0, 0.01),
            scale_to_unit=False, budget=20.0),
}


def generate_config(cfg: int, seed: int = 0, n: int | None = None, col0: int = 0,
                    n_cols: int | None = None, restated: Restated | None = None):
    """Host twin of the product's device generator for BASELINE config `cfg`."""
    c = CONFIGS[cfg]
    n_total = c["n"] if n is None else n
    o = restated or Restated()
    M = o.generate(c["h"], c["w"], c["r"], c["blobs"], c["sigma"][0], c["sigma"][1],
                   c["noise"][0], c["noise"][1], seed, n_total, col0, n_cols)
    if c["scale_to_unit"]:
        M /= M.max()
    return M
