"""paper_1009_0881_b200 -- B200-native multilevel NMF (Gillis & Glineur, arXiv 1009.0881).

Python mirror of the reference library's public solver API
(/root/reference/proj/include/mlnmf/{matrix,solvers,multilevel,transfer,cost_model}.hpp)
over the C-ABI in include/mlnmf_b200.h.  Every call runs on the GPU through
the in-tree CUDA extension ``_lib/libmlnmf_b200.so``; there is no CPU
fallback -- importing this package without the built library raises.

Same names, argument meaning and error behaviour as the reference:
  std::invalid_argument  -> ValueError
  mlnmf::DataError       -> DataError
  mlnmf::NnlsCapExceeded -> NnlsCapExceeded
  std::runtime_error     -> RuntimeError
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field
from typing import NamedTuple, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# MLNMF_B200_LIB: a kernel-variant build of the same library (tools/ab_variant.sh)
LIB_PATH = os.environ.get("MLNMF_B200_LIB") or os.path.join(_HERE, "_lib", "libmlnmf_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the sm_100a extension first "
        "(python -c 'import __graft_entry__ as g; g.build()' or python paper_1009_0881_b200/build.py)")

_lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_lp = C.POINTER(C.c_long)
_sz = C.c_size_t
_vp = C.c_void_p


# ---------------------------------------------------------------------------
# enums and small types (reference names)
# ---------------------------------------------------------------------------
class SolverKind(enum.IntEnum):  # cost_model.hpp:9
    kAnls = 0
    kMu = 1
    kHals = 2


class CycleKind(enum.IntEnum):  # multilevel.hpp:11
    kSingleLevel = 0
    kNestedIteration = 1
    kVCycle = 2
    kFullMultigrid = 3


class BudgetMode(enum.IntEnum):  # solvers.hpp:37-41
    kWorkUnits = 0
    kWallClockSeconds = 1


F32, F64 = 0, 1
GEMM_AUTO, GEMM_SIMT, GEMM_TCGEN05 = 0, 1, 2
ERROR_AUTO, ERROR_GRAM, ERROR_DIRECT = 0, 1, 2

KIND_NAMES = {"anls": SolverKind.kAnls, "mu": SolverKind.kMu, "hals": SolverKind.kHals}
CYCLE_NAMES = {"none": CycleKind.kSingleLevel, "ni": CycleKind.kNestedIteration,
               "vc": CycleKind.kVCycle, "fmg": CycleKind.kFullMultigrid}


def _kind(k):
    return int(KIND_NAMES[k] if isinstance(k, str) else k)


def _cycle(c):
    return int(CYCLE_NAMES[c] if isinstance(c, str) else c)


@dataclass
class Budget:
    """mlnmf::Budget (solvers.hpp:37-41)."""
    mode: BudgetMode = BudgetMode.kWorkUnits
    amount: float = 0.0


@dataclass
class ImageGrid:
    """mlnmf::ImageGrid (transfer.hpp:13-21): pixel (i, j) -> row j*height + i."""
    height: int = 0
    width: int = 0

    def pixels(self) -> int:
        return self.height * self.width

    def index(self, i: int, j: int) -> int:
        return j * self.height + i


def coarsen_grid(g: ImageGrid) -> ImageGrid:
    """coarsen_grid (transfer.cpp:55-59)."""
    if g.height < 2 or g.width < 2:
        raise ValueError("coarsen_grid: grid below 2x2 cannot be coarsened")
    return ImageGrid((g.height + 1) // 2, (g.width + 1) // 2)


@dataclass
class TraceSample:
    elapsed_s: float
    work_units: float
    level: int
    error: float


@dataclass
class RunTrace:
    """mlnmf::RunTrace (solvers.hpp:14-35) plus the realised steps per phase."""
    elapsed_s: np.ndarray
    work_units: np.ndarray
    level: np.ndarray
    error: np.ndarray
    alloc_level: np.ndarray
    alloc_amount: np.ndarray
    nnls_iteration_counts: np.ndarray
    hals_degenerate_columns: int
    phase_level: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    phase_steps: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))

    @property
    def samples(self):
        return [TraceSample(float(a), float(b), int(c), float(d))
                for a, b, c, d in zip(self.elapsed_s, self.work_units, self.level, self.error)]

    @property
    def allocations(self):
        return list(zip(self.alloc_level.tolist(), self.alloc_amount.tolist()))

    def final_error(self) -> float:
        return float(self.error[-1])


@dataclass
class MultilevelResult:
    V: np.ndarray
    W: np.ndarray
    trace: RunTrace


SolveResult = MultilevelResult


class DataError(RuntimeError):
    pass


class NnlsCapExceeded(RuntimeError):
    pass


class _Options(C.Structure):
    _fields_ = [("device", C.c_int), ("dtype", C.c_int), ("exact", C.c_int), ("gemm_path", C.c_int),
                ("error_mode", C.c_int), ("world", C.c_int), ("rank", C.c_int), ("nccl_id", _vp)]


class _GenParams(C.Structure):
    _fields_ = [("h", _sz), ("w", _sz), ("r", _sz), ("blobs", _sz), ("sigma_min", C.c_double),
                ("sigma_max", C.c_double), ("noise_kind", C.c_int), ("noise_scale", C.c_double),
                ("seed", C.c_uint64), ("scale_to_unit", C.c_int)]


# ---------------------------------------------------------------------------
# ctypes prototypes
# ---------------------------------------------------------------------------
def _proto(name, restype, *args):
    f = getattr(_lib, name)
    f.restype = restype
    f.argtypes = list(args)
    return f


_lib.mlnmf_last_error.restype = C.c_char_p
_proto("mlnmf_set_default_options", C.c_int, C.POINTER(_Options))
_proto("mlnmf_nccl_unique_id", C.c_int, _vp)
_proto("mlnmf_iteration_cost", C.c_double, _sz, _sz, _sz, C.c_int)
_proto("mlnmf_plan_configuration", C.c_int, _sz, _sz, _sz, _sz, C.c_int, C.c_int, _sz, C.c_double, _sz,
       C.POINTER(_vp))
_proto("mlnmf_run_configuration", C.c_int, _dp, _sz, _sz, _sz, _sz, _sz, C.c_int, C.c_int, _sz, C.c_uint64,
       C.c_int, C.c_double, _sz, _dp, _dp, C.POINTER(_vp))
_proto("mlnmf_run_cycle", C.c_int, _dp, _sz, _sz, _sz, _sz, _sz, _sz, _dp, _dp, _sz, C.c_int, C.c_int, C.c_int,
       C.c_double, _sz, _dp, _dp, C.POINTER(_vp))
_proto("mlnmf_run_seeds", C.c_int, C.POINTER(_Options), _dp, _sz, _sz, _sz, _sz, _sz, C.c_int, C.c_int, _sz,
       C.c_uint64, _sz, C.c_int, C.c_double, _sz, _dp)
_proto("mlnmf_run_solver", C.c_int, _dp, _sz, _sz, _dp, _dp, _sz, C.c_int, C.c_int, C.c_double, _sz, _dp, _dp,
       C.POINTER(_vp))
_proto("mlnmf_mu_step", C.c_int, _dp, _sz, _sz, _dp, _dp, _sz)
_proto("mlnmf_hals_step", C.c_int, _dp, _sz, _sz, _dp, _dp, _sz, _ip)
_proto("mlnmf_anls_step", C.c_int, _dp, _sz, _sz, _dp, _dp, _sz, _ip)
_proto("mlnmf_nnls_active_set", C.c_int, _dp, _dp, _dp, _sz, _dp, _ip)
_proto("mlnmf_frobenius_error", C.c_int, _dp, _dp, _dp, _sz, _sz, _sz, _dp)
_proto("mlnmf_random_init", C.c_int, _sz, _sz, _sz, C.c_uint64, _dp, _dp)
_proto("mlnmf_restrict_columns", C.c_int, _sz, _sz, _dp, _sz, _dp)
_proto("mlnmf_prolong_columns", C.c_int, _sz, _sz, _dp, _sz, _dp)
_proto("mlnmf_smoothness", C.c_int, _dp, _sz, _sz, _sz, _sz, _dp)
_proto("mlnmf_initialization_bound", C.c_int, _dp, _sz, _sz, _sz, _sz, _dp, _dp, _sz, _dp, _dp)
_proto("mlnmf_session_create", C.c_int, C.POINTER(_Options), C.POINTER(_vp))
_proto("mlnmf_session_destroy", None, _vp)
_HOST_ALLREDUCE = C.CFUNCTYPE(C.c_int, _vp, C.POINTER(C.c_double), _sz, C.c_int)
_proto("mlnmf_session_create_host_comm", C.c_int, C.POINTER(_Options), _HOST_ALLREDUCE, _vp, C.POINTER(_vp))
_proto("mlnmf_session_set_data", C.c_int, _vp, _vp, C.c_int, _sz, _sz, _sz, _sz, _sz, _sz)
_proto("mlnmf_session_generate", C.c_int, _vp, C.POINTER(_GenParams), _sz, _sz, _sz)
_proto("mlnmf_session_run_configuration", C.c_int, _vp, _sz, C.c_int, C.c_int, _sz, C.c_uint64, C.c_int,
       C.c_double, _sz, C.POINTER(_vp))
_proto("mlnmf_session_run_cycle", C.c_int, _vp, _sz, _sz, _vp, _vp, C.c_int, _sz, C.c_int, C.c_int, C.c_int,
       C.c_double, _sz, C.POINTER(_vp))
_proto("mlnmf_session_get_factors", C.c_int, _vp, _vp, _vp, C.c_int)
_proto("mlnmf_session_set_factors", C.c_int, _vp, _vp, _vp, C.c_int, _sz)
_proto("mlnmf_session_steps", C.c_int, _vp, C.c_int, _sz)
_proto("mlnmf_session_build_levels", C.c_int, _vp, _sz)
_proto("mlnmf_session_num_levels", _sz, _vp)
_proto("mlnmf_session_level_shape", C.c_int, _vp, _sz, C.POINTER(_sz), C.POINTER(_sz))
_proto("mlnmf_session_init_random", C.c_int, _vp, _sz, C.c_uint64)
_proto("mlnmf_session_set_factors_level", C.c_int, _vp, _sz, _vp, _vp, C.c_int, _sz)
_proto("mlnmf_session_get_factors_level", C.c_int, _vp, _sz, _vp, _vp, C.c_int)
_proto("mlnmf_session_restrict_V", C.c_int, _vp, _sz)
_proto("mlnmf_session_prolong_V", C.c_int, _vp, _sz)
_proto("mlnmf_session_run_phase", C.c_int, _vp, _sz, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, _sz,
       _dp, _dp, C.POINTER(_vp))
_proto("mlnmf_session_sync", C.c_int, _vp)
_proto("mlnmf_session_error", C.c_int, _vp, _dp)
_proto("mlnmf_session_norm2", C.c_int, _vp, _sz, _dp)
_proto("mlnmf_session_smoothness", C.c_int, _vp, _sz, _dp)
_proto("mlnmf_session_initialization_bound", C.c_int, _vp, _sz, _vp, _vp, C.c_int, _sz, _dp, _dp)
_proto("mlnmf_session_gram_w", C.c_int, _vp, _vp)
_proto("mlnmf_session_gram_v", C.c_int, _vp, _vp)
_proto("mlnmf_session_export_data", C.c_int, _vp, _vp, C.c_int)
_proto("mlnmf_session_export_level", C.c_int, _vp, C.c_size_t, _vp, C.POINTER(C.c_int))
_proto("mlnmf_session_products", C.c_int, _vp, _dp, _dp)
_proto("mlnmf_session_set_profiling", C.c_int, _vp, C.c_int)
_proto("mlnmf_session_kernel_times", C.c_int, _vp, _dp, _lp, _dp, _lp)
_proto("mlnmf_session_launches", C.c_long, _vp)
_proto("mlnmf_session_stream", _vp, _vp)
_proto("mlnmf_session_tc_active", C.c_int, _vp)
_proto("mlnmf_session_gram_error", C.c_int, _vp)
_proto("mlnmf_trace_num_samples", _sz, _vp)
_proto("mlnmf_trace_samples", None, _vp, _dp, _dp, _ip, _dp)
_proto("mlnmf_trace_num_allocations", _sz, _vp)
_proto("mlnmf_trace_allocations", None, _vp, _ip, _dp)
_proto("mlnmf_trace_num_nnls_counts", _sz, _vp)
_proto("mlnmf_trace_nnls_counts", None, _vp, _ip)
_proto("mlnmf_trace_degenerate", C.c_int, _vp)
_proto("mlnmf_trace_num_phases", _sz, _vp)
_proto("mlnmf_trace_phases", None, _vp, _ip, _lp)
_proto("mlnmf_trace_free", None, _vp)
_proto("mlnmf_session_comm_time", C.c_int, _vp, _dp, _lp)
_proto("mlnmf_session_phase_times", C.c_int, _vp, _dp, _lp)
_proto("mlnmf_load_pgm_dir", C.c_int, C.c_char_p, C.POINTER(_vp), C.POINTER(_sz), C.POINTER(_sz), C.POINTER(_sz),
       C.POINTER(_sz))
_proto("mlnmf_load_csv", C.c_int, C.c_char_p, C.POINTER(_vp), C.POINTER(_sz), C.POINTER(_sz))
_proto("mlnmf_save_matrix_csv", C.c_int, _dp, _sz, _sz, C.c_char_p)
_proto("mlnmf_save_basis_mosaic", C.c_int, _dp, _sz, _sz, _sz, _sz, C.c_char_p)
_proto("mlnmf_synth_smooth_dataset", C.c_int, _sz, _sz, _sz, _sz, C.c_uint64, _dp)
_proto("mlnmf_free", None, _vp)

EXPORTED_SYMBOLS = sorted(n for n in dir(_lib) if n.startswith("mlnmf_"))


def _check(rc: int):
    if rc == 0:
        return
    msg = _lib.mlnmf_last_error().decode()
    if rc == 2:
        raise ValueError(msg)
    if rc == 3:
        raise DataError(msg)
    if rc == 4:
        raise NnlsCapExceeded(msg)
    raise RuntimeError(msg)


def _d(a):
    return a.ctypes.data_as(_dp)


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None and a.shape != shape:
        raise ValueError(f"expected shape {shape}, got {a.shape}")
    return a


def _take_trace(tp: int) -> RunTrace:
    ns = _lib.mlnmf_trace_num_samples(tp)
    el, wk, er = np.zeros(ns), np.zeros(ns), np.zeros(ns)
    lv = np.zeros(ns, np.int32)
    _lib.mlnmf_trace_samples(tp, _d(el), _d(wk), lv.ctypes.data_as(_ip), _d(er))
    na = _lib.mlnmf_trace_num_allocations(tp)
    al, aa = np.zeros(na, np.int32), np.zeros(na)
    _lib.mlnmf_trace_allocations(tp, al.ctypes.data_as(_ip), _d(aa))
    nc = _lib.mlnmf_trace_num_nnls_counts(tp)
    cn = np.zeros(max(nc, 1), np.int32)
    _lib.mlnmf_trace_nnls_counts(tp, cn.ctypes.data_as(_ip))
    nph = _lib.mlnmf_trace_num_phases(tp)
    pl, ps = np.zeros(nph, np.int32), np.zeros(nph, np.int64)
    _lib.mlnmf_trace_phases(tp, pl.ctypes.data_as(_ip), ps.ctypes.data_as(_lp))
    deg = _lib.mlnmf_trace_degenerate(tp)
    _lib.mlnmf_trace_free(tp)
    return RunTrace(el, wk, lv, er, al, aa, cn[:nc].copy(), int(deg), pl, ps)


# ---------------------------------------------------------------------------
# default-session options of the one-shot calls
# ---------------------------------------------------------------------------
_default_opts = [0, F64, 0, GEMM_AUTO, ERROR_AUTO, 1, 0, None]


def set_default_options(device=0, dtype=F64, exact=False, gemm_path=GEMM_AUTO, error_mode=ERROR_AUTO):
    o = _Options(device, dtype, int(bool(exact)), gemm_path, error_mode, 1, 0, None)
    _check(_lib.mlnmf_set_default_options(C.byref(o)))
    _default_opts[:] = [device, dtype, int(bool(exact)), gemm_path, error_mode, 1, 0, None]


# ---------------------------------------------------------------------------
# reference-shaped API
# ---------------------------------------------------------------------------
def _budget(b):
    if isinstance(b, Budget):
        return int(b.mode), float(b.amount)
    return int(BudgetMode.kWorkUnits), float(b)


def run_configuration(M, grid: ImageGrid, level_count: int, kind, cycle, rank: int, seed: int, budget,
                      trace_every: int = 1) -> MultilevelResult:
    """run_configuration (multilevel.hpp:43-47, multilevel.cpp:116-132)."""
    M = _f64(M)
    m, n = M.shape
    V = np.zeros((m, rank))
    W = np.zeros((rank, n))
    mode, amount = _budget(budget)
    tp = _vp()
    rc = _lib.mlnmf_run_configuration(_d(M), m, n, grid.height, grid.width, level_count, _kind(kind),
                                      _cycle(cycle), rank, seed, mode, amount, trace_every, _d(V), _d(W),
                                      C.byref(tp))
    _check(rc)
    return MultilevelResult(V, W, _take_trace(tp.value))


# ---------------------------------------------------------------------------
# run_bench (proj/include/mlnmf/bench.hpp:15-45, proj/src/bench.cpp:28-84)
# ---------------------------------------------------------------------------
@dataclass
class BenchConfig:
    algorithms: list = field(default_factory=lambda: ["hals"])
    cycles: list = field(default_factory=lambda: ["none"])
    level_counts: list = field(default_factory=lambda: [1])
    rank: int = 1
    runs: int = 1
    budget: object = None
    base_seed: int = 0


@dataclass
class BenchEntry:
    algorithm: str
    cycle: str
    levels: int
    runs: int = 0
    mean: float = 0.0
    stddev: float = 0.0
    min: float = 0.0
    max: float = 0.0
    skipped: bool = False
    note: str = ""
    errors: Optional[np.ndarray] = None


def run_seeds(M, grid: ImageGrid, level_count: int, kind, cycle, rank: int, base_seed: int, runs: int, budget,
              workers: int = 8, dtype=None, exact=None) -> np.ndarray:
    """Final errors of run_configuration(..., seed = base_seed + i, trace_every = 0)
    for i < runs, batched over `workers` concurrent device sessions."""
    M = _f64(M)
    m, n = M.shape
    mode, amount = _budget(budget)
    o = _Options(*_default_opts)
    if dtype is not None:
        o.dtype = dtype
    if exact is not None:
        o.exact = int(bool(exact))
    out = np.zeros(runs)
    _check(_lib.mlnmf_run_seeds(C.byref(o), _d(M), m, n, grid.height, grid.width, level_count, _kind(kind),
                                _cycle(cycle), rank, base_seed, runs, mode, amount, workers, _d(out)))
    return out


def run_bench(M, grid: Optional[ImageGrid], cfg: BenchConfig, workers: int = 8, dtype=None, exact=None):
    """run_bench (bench.cpp:28-84): for every algorithm x cycle x level count,
    `runs` seeded run_configuration calls (trace_every = 0), summarised by the
    mean / sample stddev / min / max of the final error; the same skip rules.
    The runs of one entry execute concurrently on `workers` device sessions."""
    if cfg.runs < 1:
        raise ValueError("run_bench: runs >= 1")
    M = _f64(M)
    entries = []
    for algo in cfg.algorithms:
        for cycle in cfg.cycles:
            for levels in cfg.level_counts:
                e = BenchEntry(str(algo), str(cycle), int(levels))
                if _cycle(cycle) == CycleKind.kSingleLevel and levels != 1:
                    e.skipped, e.note = True, "single-level runs use exactly one level"
                    entries.append(e)
                    continue
                if levels > 1 and grid is None:
                    e.skipped, e.note = True, "dataset has no pixel grid"
                    entries.append(e)
                    continue
                g = grid if grid is not None else ImageGrid(M.shape[0], 1)
                try:
                    errs = run_seeds(M, g, levels, algo, cycle, cfg.rank, cfg.base_seed, cfg.runs, cfg.budget,
                                     workers, dtype, exact)
                except ValueError as ex:
                    e.skipped, e.note = True, str(ex)
                    entries.append(e)
                    continue
                e.runs = len(errs)
                e.mean = float(errs.sum() / len(errs))
                e.stddev = float(np.sqrt(((errs - e.mean) ** 2).sum() / (len(errs) - 1))) if len(errs) > 1 else 0.0
                e.min, e.max, e.errors = float(errs.min()), float(errs.max()), errs
                entries.append(e)
    return entries


@dataclass
class GridHierarchy:
    """GridHierarchy (transfer.hpp:87-99).  The restricted data lives on the
    device inside each cycle call; this object carries M, the grid and depth."""
    M: np.ndarray
    grid: ImageGrid
    level_count: int

    @staticmethod
    def build(M, grid: ImageGrid, level_count: int) -> "GridHierarchy":
        if level_count < 1:
            raise ValueError("GridHierarchy: need at least one level")
        M = _f64(M)
        if grid.pixels() != M.shape[0]:
            raise ValueError("GridHierarchy: grid does not match matrix rows")
        g = grid
        for _ in range(level_count - 1):
            if g.height < 2 or g.width < 2:
                raise ValueError("GridHierarchy: too many levels for this grid")
            g = coarsen_grid(g)
        return GridHierarchy(M, grid, level_count)

    @property
    def levels(self):
        out, g = [self.grid], self.grid
        for _ in range(self.level_count - 1):
            g = coarsen_grid(g)
            out.append(g)
        return out


def _run_cycle(h: GridHierarchy, levels, V0, W0, kind, cycle, budget, trace_every):
    M = h.M
    m, n = M.shape
    V0 = _f64(V0)
    r = V0.shape[1]
    W0 = _f64(W0, (r, n))
    if V0.shape[0] != m:
        raise ValueError("solver step: dimension mismatch")
    V = np.zeros_like(V0)
    W = np.zeros_like(W0)
    mode, amount = _budget(budget)
    tp = _vp()
    rc = _lib.mlnmf_run_cycle(_d(M), m, n, h.grid.height, h.grid.width, h.level_count, levels, _d(V0), _d(W0), r,
                              _kind(kind), _cycle(cycle), mode, amount, trace_every, _d(V), _d(W), C.byref(tp))
    _check(rc)
    return MultilevelResult(V, W, _take_trace(tp.value))


def nested_iteration(h, levels, V0, W0, kind, budget, trace_every=1):
    """nested_iteration (multilevel.hpp:22-26)."""
    return _run_cycle(h, levels, V0, W0, kind, CycleKind.kNestedIteration, budget, trace_every)


def v_cycle(h, levels, V0, W0, kind, budget, trace_every=1):
    """v_cycle (multilevel.hpp:28-32)."""
    return _run_cycle(h, levels, V0, W0, kind, CycleKind.kVCycle, budget, trace_every)


def full_multigrid(h, levels, V0, W0, kind, budget, trace_every=1):
    """full_multigrid (multilevel.hpp:34-38)."""
    return _run_cycle(h, levels, V0, W0, kind, CycleKind.kFullMultigrid, budget, trace_every)


def run_solver(M, V0, W0, kind, budget, trace_every=1) -> SolveResult:
    """run_solver (solvers.hpp:101-103)."""
    M = _f64(M)
    m, n = M.shape
    V0 = _f64(V0)
    r = V0.shape[1]
    if V0.shape[0] != m:
        raise ValueError("solver step: dimension mismatch")
    W0 = _f64(W0)
    if W0.shape != (r, n):
        raise ValueError("solver step: dimension mismatch")
    V = np.zeros_like(V0)
    W = np.zeros_like(W0)
    mode, amount = _budget(budget)
    tp = _vp()
    _check(_lib.mlnmf_run_solver(_d(M), m, n, _d(V0), _d(W0), r, _kind(kind), mode, amount, trace_every, _d(V),
                                 _d(W), C.byref(tp)))
    return SolveResult(V, W, _take_trace(tp.value))


def _step_args(M, V, W):
    M = _f64(M)
    m, n = M.shape
    V = _f64(V).copy()
    W = _f64(W).copy()
    r = V.shape[1]
    if V.shape[0] != m or W.shape != (r, n):
        raise ValueError("solver step: dimension mismatch")
    return M, V, W, m, n, r


def mu_step(M, V, W):
    """mu_step (solvers.hpp:45); returns the updated (V, W)."""
    M, V, W, m, n, r = _step_args(M, V, W)
    _check(_lib.mlnmf_mu_step(_d(M), m, n, _d(V), _d(W), r))
    return V, W


def hals_step(M, V, W):
    """hals_step (solvers.hpp:50); returns (V, W, degenerate_count)."""
    M, V, W, m, n, r = _step_args(M, V, W)
    deg = C.c_int(0)
    _check(_lib.mlnmf_hals_step(_d(M), m, n, _d(V), _d(W), r, C.byref(deg)))
    return V, W, deg.value


def anls_step(M, V, W):
    """anls_step (solvers.hpp:68); returns (V, W, exchange counts m + n)."""
    M, V, W, m, n, r = _step_args(M, V, W)
    counts = np.zeros(m + n, np.int32)
    _check(_lib.mlnmf_anls_step(_d(M), m, n, _d(V), _d(W), r, counts.ctypes.data_as(_ip)))
    return V, W, counts


def nnls_active_set(G, h, x0):
    """nnls_active_set (solvers.hpp:61-63); returns (x, iterations)."""
    h = _f64(h)
    r = h.shape[0]
    G = _f64(G)
    x0 = _f64(x0)
    if G.shape != (r, r) or x0.shape != (r,):
        raise ValueError("nnls_active_set: dimension mismatch")
    x = np.zeros(r)
    it = C.c_int(0)
    _check(_lib.mlnmf_nnls_active_set(_d(G), _d(h), _d(x0), r, _d(x), C.byref(it)))
    return x, it.value


def frobenius_error(M, V, W) -> float:
    """frobenius_error (matrix.hpp:99-101)."""
    M = _f64(M)
    V = _f64(V)
    W = _f64(W)
    m, n = M.shape
    r = V.shape[1]
    if V.shape[0] != m or W.shape != (r, n):
        raise ValueError("column_sq_errors: dimension mismatch")
    out = C.c_double()
    _check(_lib.mlnmf_frobenius_error(_d(M), _d(V), _d(W), m, n, r, C.byref(out)))
    return out.value


def random_init(m: int, n: int, r: int, seed: int):
    """random_init (matrix.hpp:106-107)."""
    if r < 1 or r > min(m, n):
        raise ValueError("random_init: rank must satisfy 1 <= r <= min(m,n)")
    V = np.zeros((m, r))
    W = np.zeros((r, n))
    _check(_lib.mlnmf_random_init(m, n, r, seed, _d(V), _d(W)))
    return V, W


def restrict_columns(grid: ImageGrid, X):
    """restrict_columns(build_restriction(grid), X) (transfer.hpp:68)."""
    X = _f64(X)
    if X.ndim == 1:
        X = X[:, None]
    if X.shape[0] != grid.pixels():
        raise ValueError("TransferOperator::apply: dimension mismatch")
    c = coarsen_grid(grid)
    Y = np.zeros((c.pixels(), X.shape[1]))
    _check(_lib.mlnmf_restrict_columns(grid.height, grid.width, _d(X), X.shape[1], _d(Y)))
    return Y


def prolong_columns(grid: ImageGrid, X):
    """prolong_columns(build_prolongation(grid), X) (transfer.hpp:69); grid is the fine grid."""
    X = _f64(X)
    if X.ndim == 1:
        X = X[:, None]
    c = coarsen_grid(grid)
    if X.shape[0] != c.pixels():
        raise ValueError("TransferOperator::apply: dimension mismatch")
    Y = np.zeros((grid.pixels(), X.shape[1]))
    _check(_lib.mlnmf_prolong_columns(grid.height, grid.width, _d(X), X.shape[1], _d(Y)))
    return Y


def smoothness(M, grid: ImageGrid) -> float:
    """smoothness(M, build_restriction(grid), build_prolongation(grid))
    (transfer.hpp:75-76): ||M - P R M||_F / ||M||_F, on the device."""
    M = _f64(M)
    if M.ndim == 1:
        M = M[:, None]
    if M.shape[0] != grid.pixels():
        raise ValueError("TransferOperator::apply: dimension mismatch")
    out = C.c_double()
    _check(_lib.mlnmf_smoothness(_d(M), M.shape[0], M.shape[1], grid.height, grid.width, C.byref(out)))
    return out.value


class BoundCheck(NamedTuple):  # transfer.hpp:78-81
    lhs: float  # ||M - P(V')W||_F
    rhs: float  # s_M ||M||_F + ||P||_F ||R(M) - V'W||_F


def initialization_bound(M, grid: ImageGrid, V_coarse, W) -> BoundCheck:
    """initialization_bound(M, R, P, V_coarse, W) with R, P built on `grid`
    (transfer.hpp:85-87, transfer.cpp:143-153), on the device."""
    M, Vc, W = _f64(M), _f64(V_coarse), _f64(W)
    c = coarsen_grid(grid)
    if M.shape[0] != grid.pixels() or Vc.shape[0] != c.pixels() or W.shape != (Vc.shape[1], M.shape[1]):
        raise ValueError("initialization_bound: dimension mismatch")
    lhs, rhs = C.c_double(), C.c_double()
    _check(_lib.mlnmf_initialization_bound(_d(M), M.shape[0], M.shape[1], grid.height, grid.width, _d(Vc), _d(W),
                                           Vc.shape[1], C.byref(lhs), C.byref(rhs)))
    return BoundCheck(lhs.value, rhs.value)


def iteration_cost(m: int, n: int, r: int, kind) -> float:
    """iteration_cost with CostParams::with_default_sr (cost_model.hpp:36)."""
    return _lib.mlnmf_iteration_cost(m, n, r, _kind(kind))


def plan_configuration(grid: ImageGrid, n: int, level_count: int, kind, cycle, rank: int, amount: float,
                       trace_every: int = 1) -> RunTrace:
    """Host-only dry run of the scheduler (no GPU needed): allocations, steps per
    phase and the work/level stamps of every sample of a work-unit run."""
    tp = _vp()
    _check(_lib.mlnmf_plan_configuration(grid.height, grid.width, n, level_count, _kind(kind), _cycle(cycle), rank,
                                         float(amount), trace_every, C.byref(tp)))
    return _take_trace(tp.value)


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(_lib.mlnmf_nccl_unique_id(buf))
    return buf.raw


# ---------------------------------------------------------------------------
# Session: device-resident data, fp32/fp64 storage, sharding over ranks
# ---------------------------------------------------------------------------
GEN_CONFIGS = {
    # BASELINE.json configs -> generator parameters
    0: dict(h=32, w=32, n=1000, r=20, levels=3, blobs=3, sigma=(2.0, 6.0), noise=(0, 0.01), scale_to_unit=0),
    1: dict(h=19, w=19, n=2429, r=49, levels=2, blobs=3, sigma=(2.0, 6.0), noise=(0, 0.01), scale_to_unit=1),
    2: dict(h=112, w=92, n=400, r=40, levels=4, blobs=5, sigma=(2.0, 6.0), noise=(1, 0.02), scale_to_unit=0),
    3: dict(h=243, w=320, n=165, r=49, levels=5, blobs=3, sigma=(4.0, 20.0), noise=(0, 0.01), scale_to_unit=0),
    4: dict(h=256, w=256, n=262144, r=64, levels=5, blobs=3, sigma=(4.0, 20.0), noise=(0, 0.01), scale_to_unit=0),
}


def shard_columns(n_total: int, world: int, rank: int):
    """Column shard [col0, col0 + n_local) of rank `rank` (contiguous blocks,
    the first n_total % world ranks one column larger)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    base, extra = divmod(n_total, world)
    n_local = base + (1 if rank < extra else 0)
    col0 = rank * base + min(rank, extra)
    return col0, n_local


class HostGroup:
    """In-process collective for `world` sessions (ranks), each driven from
    its own thread (mlnmf_session_create_host_comm): every allreduce deposits
    the rank's buffer, waits for all ranks, and leaves the element-wise sum
    (ranks added in rank order: deterministic, identical on every rank) or
    max.  It lets the real sharded engine run world > 1 in one process, on
    one GPU, with no device-side waits between ranks."""

    def __init__(self, world: int, timeout: float = 300.0):
        import threading
        self.world = world
        self._bufs = [None] * world
        self._barrier = threading.Barrier(world, timeout=timeout)

    def allreduce(self, rank: int, buf: np.ndarray, op: int):
        self._bufs[rank] = buf.copy()
        self._barrier.wait()
        out = self._bufs[0].copy()
        for b in self._bufs[1:]:
            out = out + b if op == 0 else np.maximum(out, b)
        self._barrier.wait()  # every rank has read the deposits before the next exchange
        buf[:] = out

    def abort(self):
        self._barrier.abort()


class Session:
    """A device-resident solver instance (one per GPU / rank).  world > 1
    needs an NCCL id (one process per GPU) or a HostGroup (ranks as threads
    of one process)."""

    def __init__(self, device=0, dtype=F64, exact=False, gemm_path=GEMM_AUTO, error_mode=ERROR_AUTO,
                 world=1, rank=0, nccl_id: Optional[bytes] = None, host_group: Optional[HostGroup] = None):
        self._idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id else None
        o = _Options(device, dtype, int(bool(exact)), gemm_path, error_mode, world, rank,
                     C.cast(self._idbuf, _vp) if self._idbuf is not None else None)
        h = _vp()
        if host_group is not None:
            def _cb(ctx, buf, count, op, _g=host_group, _r=rank):
                try:
                    _g.allreduce(_r, np.ctypeslib.as_array(buf, shape=(count,)), op)
                    return 0
                except Exception:
                    _g.abort()  # release the other ranks (their exchange fails too)
                    return 1
            self._cb = _HOST_ALLREDUCE(_cb)
            _check(_lib.mlnmf_session_create_host_comm(C.byref(o), self._cb, None, C.byref(h)))
        else:
            _check(_lib.mlnmf_session_create(C.byref(o), C.byref(h)))
        self._h = h.value
        self.dtype = dtype
        self.world, self.rank = world, rank
        self.m = self.n_local = self.n_total = self.col0 = 0
        self.r = 0

    def close(self):
        if getattr(self, "_h", None):
            _lib.mlnmf_session_destroy(self._h)
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

    @property
    def np_dtype(self):
        return np.float32 if self.dtype == F32 else np.float64

    def set_data(self, M_local, grid: ImageGrid, n_total=None, col0=0):
        M_local = np.asarray(M_local)
        hd = F32 if M_local.dtype == np.float32 else F64
        M_local = np.ascontiguousarray(M_local, dtype=np.float32 if hd == F32 else np.float64)
        m, nl = M_local.shape
        n_total = nl if n_total is None else n_total
        _check(_lib.mlnmf_session_set_data(self._h, M_local.ctypes.data, hd, m, nl, n_total, col0, grid.height,
                                           grid.width))
        self.m, self.n_local, self.n_total, self.col0 = m, nl, n_total, col0
        self.grid = grid

    def set_data_ptr(self, ptr: int, host_dtype: int, m: int, n_local: int, grid: ImageGrid, n_total=None, col0=0):
        """set_data from a raw host pointer (e.g. pinned memory)."""
        n_total = n_local if n_total is None else n_total
        _check(_lib.mlnmf_session_set_data(self._h, ptr, host_dtype, m, n_local, n_total, col0, grid.height,
                                           grid.width))
        self.m, self.n_local, self.n_total, self.col0 = m, n_local, n_total, col0
        self.grid = grid

    def generate(self, cfg: int, seed: int = 0, n_total=None, col0=0, n_local=None, r=None):
        c = GEN_CONFIGS[cfg]
        n_total = c["n"] if n_total is None else n_total
        n_local = n_total - col0 if n_local is None else n_local
        g = _GenParams(c["h"], c["w"], c["r"] if r is None else r, c["blobs"], c["sigma"][0], c["sigma"][1],
                       c["noise"][0], c["noise"][1], seed, c["scale_to_unit"])
        _check(_lib.mlnmf_session_generate(self._h, C.byref(g), n_total, col0, n_local))
        self.m, self.n_local, self.n_total, self.col0 = c["h"] * c["w"], n_local, n_total, col0
        self.grid = ImageGrid(c["h"], c["w"])
        return self.grid

    def run_configuration(self, level_count, kind, cycle, rank, seed, budget, trace_every=1) -> RunTrace:
        mode, amount = _budget(budget)
        tp = _vp()
        _check(_lib.mlnmf_session_run_configuration(self._h, level_count, _kind(kind), _cycle(cycle), rank, seed,
                                                    mode, amount, trace_every, C.byref(tp)))
        self.r = rank
        return _take_trace(tp.value)

    def run_cycle(self, hierarchy_levels, levels, V0, W0_local, kind, cycle, budget, trace_every=1) -> RunTrace:
        V0 = np.ascontiguousarray(V0, dtype=np.float64)
        W0 = np.ascontiguousarray(W0_local, dtype=np.float64)
        mode, amount = _budget(budget)
        tp = _vp()
        _check(_lib.mlnmf_session_run_cycle(self._h, hierarchy_levels, levels, V0.ctypes.data, W0.ctypes.data, F64,
                                            V0.shape[1], _kind(kind), _cycle(cycle), mode, amount, trace_every,
                                            C.byref(tp)))
        self.r = V0.shape[1]
        return _take_trace(tp.value)

    def set_factors(self, V, W_local):
        V = np.ascontiguousarray(V, dtype=np.float64)
        W = np.ascontiguousarray(W_local, dtype=np.float64)
        _check(_lib.mlnmf_session_set_factors(self._h, V.ctypes.data, W.ctypes.data, F64, V.shape[1]))
        self.r = V.shape[1]

    def get_factors(self, dtype=np.float64):
        hd = F32 if dtype == np.float32 else F64
        V = np.zeros((self.m, self.r), dtype=dtype)
        W = np.zeros((self.r, self.n_local), dtype=dtype)
        _check(_lib.mlnmf_session_get_factors(self._h, V.ctypes.data, W.ctypes.data, hd))
        return V, W

    def get_factors_ptr(self, V_ptr: int, W_ptr: int, host_dtype: int):
        _check(_lib.mlnmf_session_get_factors(self._h, V_ptr, W_ptr, host_dtype))

    # ---- resident per-level pieces of a multilevel cycle ----
    def build_levels(self, level_count: int):
        """GridHierarchy::build on the device (transfer.cpp:155-174)."""
        _check(_lib.mlnmf_session_build_levels(self._h, level_count))

    @property
    def num_levels(self) -> int:
        return int(_lib.mlnmf_session_num_levels(self._h))

    def level_grid(self, level: int) -> ImageGrid:
        h, w = _sz(), _sz()
        _check(_lib.mlnmf_session_level_shape(self._h, level, C.byref(h), C.byref(w)))
        return ImageGrid(h.value, w.value)

    def init_random(self, r: int, seed: int):
        """random_init(m, n_total, r, seed) at level 0 (matrix.cpp:51-60)."""
        _check(_lib.mlnmf_session_init_random(self._h, r, seed))
        self.r = r

    def set_factors_level(self, level: int, V, W_local):
        V = np.ascontiguousarray(V, dtype=np.float64)
        W = np.ascontiguousarray(W_local, dtype=np.float64)
        _check(_lib.mlnmf_session_set_factors_level(self._h, level, V.ctypes.data, W.ctypes.data, F64, V.shape[1]))
        self.r = V.shape[1]

    def get_factors_level(self, level: int):
        g = self.level_grid(level)
        V = np.zeros((g.pixels(), self.r))
        W = np.zeros((self.r, self.n_local))
        _check(_lib.mlnmf_session_get_factors_level(self._h, level, V.ctypes.data, W.ctypes.data, F64))
        return V, W

    def restrict_V(self, level: int):
        """V_{level+1} = R V_level (multilevel.cpp:39)."""
        _check(_lib.mlnmf_session_restrict_V(self._h, level))

    def prolong_V(self, level: int):
        """V_level = P V_{level+1} (multilevel.cpp:41)."""
        _check(_lib.mlnmf_session_prolong_V(self._h, level))

    def run_phase(self, level: int, kind, budget, step_flops: float, unit_flops: float, trace_every: int = 1,
                  work_consumed: float = 0.0):
        """run_solver_phase (solvers.cpp:300-341) on the resident level.
        Returns (leftover, work_consumed, trace): the unconsumed amount, the
        run's advanced cumulative work and the phase trace (sample times
        relative to the phase start)."""
        mode, amount = _budget(budget)
        wc, left, tp = C.c_double(work_consumed), C.c_double(), _vp()
        _check(_lib.mlnmf_session_run_phase(self._h, level, _kind(kind), mode, amount, step_flops, unit_flops,
                                            trace_every, C.byref(wc), C.byref(left), C.byref(tp)))
        return left.value, wc.value, _take_trace(tp.value)

    def steps(self, kind, n_steps: int):
        _check(_lib.mlnmf_session_steps(self._h, _kind(kind), n_steps))

    def sync(self):
        _check(_lib.mlnmf_session_sync(self._h))

    def error(self) -> float:
        out = C.c_double()
        _check(_lib.mlnmf_session_error(self._h, C.byref(out)))
        return out.value

    def norm2(self, level: int = 0) -> float:
        """||M_level||_F^2 over all ranks."""
        out = C.c_double()
        _check(_lib.mlnmf_session_norm2(self._h, level, C.byref(out)))
        return out.value

    def smoothness(self, level: int = 0) -> float:
        """s_M of the resident level-`level` data over all ranks (transfer.cpp:128-141)."""
        out = C.c_double()
        _check(_lib.mlnmf_session_smoothness(self._h, level, C.byref(out)))
        return out.value

    def initialization_bound(self, V_coarse, W_local, level: int = 0) -> BoundCheck:
        """Both sides of the coarse-initialization bound at `level` over all ranks
        (transfer.cpp:143-153); V_coarse has level+1's rows, W_local this rank's
        columns.  Leaves V_coarse / P V_coarse / W as the session's factors."""
        g = self.grid
        for _ in range(level + 1):
            g = coarsen_grid(g)
        Vc = np.ascontiguousarray(V_coarse, dtype=np.float64)
        W = np.ascontiguousarray(W_local, dtype=np.float64)
        if Vc.ndim != 2 or Vc.shape[0] != g.pixels() or W.shape != (Vc.shape[1], self.n_local):
            raise ValueError("initialization_bound: dimension mismatch")
        lhs, rhs = C.c_double(), C.c_double()
        _check(_lib.mlnmf_session_initialization_bound(self._h, level, Vc.ctypes.data, W.ctypes.data, F64,
                                                       Vc.shape[1], C.byref(lhs), C.byref(rhs)))
        self.r = Vc.shape[1]
        return BoundCheck(lhs.value, rhs.value)

    def products(self):
        """(A, C) = (M W^T, V^T M) at level 0 with the current factors, through
        the active implementation (SIMT or tcgen05); this rank's partials."""
        A = np.zeros((self.m, self.r))
        Cm = np.zeros((self.r, self.n_local))
        _check(_lib.mlnmf_session_products(self._h, _d(A), _d(Cm)))
        return A, Cm

    def gram_v(self):
        """D = V^T V of the level-0 V through the active kernel."""
        D = np.zeros((self.r, self.r))
        _check(_lib.mlnmf_session_gram_v(self._h, _d(D)))
        return D

    def gram_w(self):
        """B = W W^T of this rank's W shard through the active kernel (not allreduced)."""
        B = np.zeros((self.r, self.r))
        _check(_lib.mlnmf_session_gram_w(self._h, _d(B)))
        return B

    def export_data(self, ptr: Optional[int] = None):
        """Level-0 M (m x n_local) to a host buffer (numpy array if ptr is None)."""
        if ptr is None:
            M = np.zeros((self.m, self.n_local), dtype=self.np_dtype)
            _check(_lib.mlnmf_session_export_data(self._h, M.ctypes.data, self.dtype))
            return M
        _check(_lib.mlnmf_session_export_data(self._h, ptr, self.dtype))
        return None

    def export_level(self, level: int):
        """This rank's level data R(...R(M)) (m_level x n_local) in the level's storage type."""
        dt = C.c_int(0)
        _check(_lib.mlnmf_session_export_level(self._h, level, None, C.byref(dt)))
        g = self.level_grid(level)
        M = np.zeros((g.pixels(), self.n_local), dtype=np.float32 if dt.value == F32 else np.float64)
        _check(_lib.mlnmf_session_export_level(self._h, level, M.ctypes.data, C.byref(dt)))
        return M

    def set_profiling(self, on: bool):
        _check(_lib.mlnmf_session_set_profiling(self._h, int(on)))

    def kernel_times(self):
        a, c = C.c_double(), C.c_double()
        an, cn = C.c_long(), C.c_long()
        _check(_lib.mlnmf_session_kernel_times(self._h, C.byref(a), C.byref(an), C.byref(c), C.byref(cn)))
        x, xn = C.c_double(), C.c_long()
        _check(_lib.mlnmf_session_comm_time(self._h, C.byref(x), C.byref(xn)))
        return dict(mwt_ms=a.value, mwt_n=an.value, vtm_ms=c.value, vtm_n=cn.value, comm_ms=x.value, comm_n=xn.value)

    STEP_PHASES = ("B = W W^T", "A = M W^T", "allreduce [A|B]", "V update", "D = V^T V", "C = V^T M", "W update")

    def phase_times(self):
        """Mean ms per timed interval of each step phase (profiling on; CUDA
        events on the engine stream), keyed by STEP_PHASES; phases that did
        not run are omitted."""
        ms = (C.c_double * 7)()
        cnt = (C.c_long * 7)()
        _check(_lib.mlnmf_session_phase_times(self._h, ms, cnt))
        return {k: ms[i] / cnt[i] for i, k in enumerate(self.STEP_PHASES) if cnt[i] > 0}

    @property
    def launches(self) -> int:
        return int(_lib.mlnmf_session_launches(self._h))

    @property
    def stream(self) -> int:
        return int(_lib.mlnmf_session_stream(self._h) or 0)

    @property
    def tc_active(self) -> bool:
        return bool(_lib.mlnmf_session_tc_active(self._h))

    @property
    def gram_error(self) -> bool:
        return bool(_lib.mlnmf_session_gram_error(self._h))


# ---------------------------------------------------------------------------
# dataset / result I/O (proj/include/mlnmf/io.hpp) -- host code in the library
# (csrc/host_io.cpp), the same formats as the mlnmf_b200 CLI
# ---------------------------------------------------------------------------
@dataclass
class Dataset:
    """mlnmf::Dataset (io.hpp:16-21): one column per image; grid None for CSV."""
    matrix: np.ndarray
    grid: Optional[ImageGrid]
    name: str


def _take_matrix(ptr, m, n):
    try:
        return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_double)), shape=(m, n)).copy() if m * n else \
            np.zeros((m, n))
    finally:
        _lib.mlnmf_free(ptr)


def load_pgm_dir(path) -> Dataset:
    """load_pgm_dir (io.hpp:46-48): every P5 image in byte-wise filename order."""
    ptr, m, n, h, w = C.c_void_p(), C.c_size_t(), C.c_size_t(), C.c_size_t(), C.c_size_t()
    _check(_lib.mlnmf_load_pgm_dir(os.fsencode(str(path)), C.byref(ptr), C.byref(m), C.byref(n), C.byref(h),
                                   C.byref(w)))
    M = _take_matrix(ptr, m.value, n.value)
    return Dataset(M, ImageGrid(h.value, w.value), os.path.basename(os.path.normpath(str(path))))


def load_csv(path) -> Dataset:
    """load_csv (io.hpp:50-51): rectangular nonnegative CSV, no header."""
    ptr, m, n = C.c_void_p(), C.c_size_t(), C.c_size_t()
    _check(_lib.mlnmf_load_csv(os.fsencode(str(path)), C.byref(ptr), C.byref(m), C.byref(n)))
    return Dataset(_take_matrix(ptr, m.value, n.value), None, os.path.splitext(os.path.basename(str(path)))[0])


def save_matrix_csv(M, path):
    """save_matrix_csv (io.hpp:53): one row per line, %.17g."""
    M = np.ascontiguousarray(M, dtype=np.float64)
    _check(_lib.mlnmf_save_matrix_csv(_d(M), M.shape[0], M.shape[1], os.fsencode(str(path))))


def save_trace_csv(trace: RunTrace, path):
    """save_trace_csv (io.hpp:55-57): header elapsed_s,work_units,level,error,
    %.17g values (the same bytes as the C writer)."""
    with open(path, "w") as f:
        f.write("elapsed_s,work_units,level,error\n")
        for a, b, c, d in zip(trace.elapsed_s, trace.work_units, trace.level, trace.error):
            f.write("%.17g,%.17g,%d,%.17g\n" % (a, b, c, d))


def save_basis_mosaic(V, grid: ImageGrid, path):
    """save_basis_mosaic (io.hpp:60-63): basis_kkk.pgm per column + mosaic.pgm."""
    V = np.ascontiguousarray(V, dtype=np.float64)
    _check(_lib.mlnmf_save_basis_mosaic(_d(V), V.shape[0], V.shape[1], grid.height, grid.width,
                                        os.fsencode(str(path))))


def synth_smooth_dataset(height: int, width: int, n: int, blobs: int, seed: int) -> Dataset:
    """synth_smooth_dataset (io.hpp:69-75): the reference's seeded PGM image set."""
    M = np.empty((height * width, n))
    _check(_lib.mlnmf_synth_smooth_dataset(height, width, n, blobs, C.c_uint64(seed), _d(M)))
    return Dataset(M, ImageGrid(height, width), "synth")
