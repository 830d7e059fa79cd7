"""Python mirror of the reference's public C++ interface for the hot path.

Names, argument meaning and error behaviour follow proj/include/skridge/
(sketch.hpp, precond.hpp, svrg.hpp, ridge.hpp, bench.hpp); every call runs on
the B200 through the C-ABI in include/skr.h.  There is no CPU fallback: the
CUDA library must load or the first call raises.

Orientation: data is handed over as an (n, d) row-major array — byte-identical
to the reference's d x n column-major DenseMatrix — and factors come back as
(d, k) arrays whose column j is basis vector j (``left[:, j]``), as in
SketchedSvd::left.
"""
from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, field
from enum import Enum
from typing import Optional

import numpy as np

from . import _lib
from ._lib import EpochRecordC, SvrgConfigC, SynthSpecC, f64, i64, cint, vp

# ---------------------------------------------------------------------------
# errors.hpp:10-60, svrg.hpp:27-35 (+ DeviceError for CUDA/NCCL failures)


class SkridgeError(Exception):
    pass


class DimensionError(SkridgeError, ValueError):
    pass


class ParameterError(SkridgeError, ValueError):
    pass


class InputError(SkridgeError, ValueError):
    pass


class EmptyBasisError(SkridgeError, ValueError):
    pass


class ScaleGuardError(SkridgeError, RuntimeError):
    pass


class DeviceError(SkridgeError, RuntimeError):
    pass


class DivergenceError(SkridgeError, RuntimeError):
    def __init__(self, what: str, trace: list):
        super().__init__(what)
        self.trace = trace


_ERR = {1: DimensionError, 2: ParameterError, 3: InputError, 4: ScaleGuardError, 6: DeviceError,
        7: DeviceError, 8: EmptyBasisError, 9: DeviceError, 10: DeviceError}


def _check(rc: int):
    if rc != 0:
        msg = _lib.last_error()
        raise _ERR.get(rc, DeviceError)(msg)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


# ---------------------------------------------------------------------------
class Context:
    """One per process and GPU (the C-ABI's skr_ctx)."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, nccl_id: bytes | None = None):
        lib = _lib.load()
        h = vp()
        if world > 1 or nccl_id is not None:  # world == 1 with an id: the sharded path on one GPU
            if nccl_id is None or len(nccl_id) != 128:
                raise ParameterError("distributed context needs the 128-byte NCCL id")
            _check(lib.skr_ctx_create_dist(device, rank, world, nccl_id, C.byref(h)))
        else:
            _check(lib.skr_ctx_create(device, C.byref(h)))
        self.h = h
        self.device, self.rank, self.world = device, rank, world

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(_lib.load().skr_nccl_unique_id(buf))
        return buf.raw

    def synchronize(self):
        _check(_lib.load().skr_ctx_synchronize(self.h))

    @property
    def stream(self) -> int:
        return _lib.load().skr_ctx_stream(self.h) or 0

    @property
    def kernel_launches(self) -> int:
        return int(_lib.load().skr_ctx_kernel_launches(self.h))

    def profile(self, enable: bool = True):
        """Enable (and reset) CUDA-event timing of the hot kernels."""
        _check(_lib.load().skr_ctx_profile(self.h, int(enable)))

    def trim(self) -> int:
        """Return the parked >= 1 GiB buffers to the driver; bytes released (skr_ctx_trim)."""
        out = i64()
        _check(_lib.load().skr_ctx_trim(self.h, C.byref(out)))
        return int(out.value)

    def set_prep_cap(self, ctas: int):
        """Cap the inner loop's PREP grid (0 = uncapped); see skr_ctx_set_prep_cap."""
        _check(_lib.load().skr_ctx_set_prep_cap(self.h, int(ctas)))

    def profile_read(self, key: str):
        """(total device ms, launches) of a profiled kernel key."""
        ms, cnt = f64(), i64()
        _check(_lib.load().skr_ctx_profile_read(self.h, key.encode(), C.byref(ms), C.byref(cnt)))
        return ms.value, cnt.value

    def close(self):
        if getattr(self, "h", None):
            _lib.load().skr_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Optional[Context] = None


def shard_rows(n: int, world: int, rank: int) -> tuple:
    """(row0, n_local) of `rank` when the library shards n rows over `world` ranks
    (skr_shard_rows: the layout skr_data_generate uses; host only)."""
    r0, nl = C.c_int64(), C.c_int64()
    _check(_lib.load().skr_shard_rows(int(n), int(world), int(rank), C.byref(r0), C.byref(nl)))
    return r0.value, nl.value


def shard_layout(counts, rank: int) -> tuple:
    """(n_global, row0) of `rank` from every rank's local row count in rank order
    (skr_shard_layout: what skr_data_create derives after gathering the counts)."""
    c = np.ascontiguousarray(counts, dtype=np.int64)
    ng, r0 = C.c_int64(), C.c_int64()
    _check(_lib.load().skr_shard_layout(c, len(c), int(rank), C.byref(ng), C.byref(r0)))
    return ng.value, r0.value


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


# ---------------------------------------------------------------------------
class DataMatrix:
    """DataMatrix (data_matrix.hpp:18-61): immutable device storage + uniform scale.

    ``rows()`` is the dimension d and ``cols()`` the point count n, as in the
    reference (points are its columns).
    """

    def __init__(self, x=None, scale: float = 1.0, ctx: Context | None = None, _handle=None,
                 _owner=None):
        self.ctx = ctx or default_context()
        self._owner = _owner
        if _handle is not None:
            self.h = _handle
        else:
            x = np.asarray(x)
            if x.ndim != 2:
                raise DimensionError("data matrix: expected an (n, d) array")
            if x.dtype == np.float32:
                dt, arr = 1, np.ascontiguousarray(x)
            else:
                dt, arr = 0, _f64(x)
            if not np.all(np.isfinite(arr)):
                raise InputError("data matrix: entries must be finite")
            h = vp()
            _check(_lib.load().skr_data_create(self.ctx.h, arr.ctypes.data, arr.shape[0], arr.shape[1],
                                               dt, C.byref(h)))
            self.h = h
            if scale != 1.0:
                h2 = vp()
                _check(_lib.load().skr_data_scaled(self.h, float(scale), C.byref(h2)))
                _lib.load().skr_data_destroy(self.h)
                self.h = h2
        n, d, dt, sc, ng, r0 = i64(), i64(), cint(), f64(), i64(), i64()
        _check(_lib.load().skr_data_info(self.h, C.byref(n), C.byref(d), C.byref(dt), C.byref(sc),
                                         C.byref(ng), C.byref(r0)))
        self.n_local, self.d, self.dtype = n.value, d.value, dt.value
        self._scale, self.n_global, self.row0 = sc.value, ng.value, r0.value

    @classmethod
    def from_csr(cls, row_ptr, col_idx, values, d: int, ctx: Context | None = None) -> "DataMatrix":
        """DataMatrix(SparseMatrix) (data_matrix.hpp:24): this rank's points as CSR
        (= the reference's CSC over points; strictly increasing indices, finite
        nonzero values, sparse_matrix.hpp:12-14).  Accepts scipy.sparse too."""
        ctx = ctx or default_context()
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(col_idx, dtype=np.int32)
        va = _f64(values)
        h = vp()
        _check(_lib.load().skr_data_create_csr(ctx.h, len(rp) - 1, int(d), rp, ci, va, C.byref(h)))
        return cls(ctx=ctx, _handle=h)

    @classmethod
    def from_scipy(cls, m, ctx: Context | None = None) -> "DataMatrix":
        """Points as the rows of a scipy.sparse matrix (converted to canonical CSR)."""
        m = m.tocsr()
        m.sum_duplicates()
        m.sort_indices()
        m.eliminate_zeros()
        return cls.from_csr(m.indptr, m.indices, m.data, m.shape[1], ctx)

    @property
    def sparse(self) -> bool:
        sp, nnz = cint(), i64()
        _check(_lib.load().skr_data_is_sparse(self.h, C.byref(sp), C.byref(nnz)))
        return bool(sp.value)

    @classmethod
    def generate(cls, spec: "SynthSpec", ctx: Context | None = None) -> "DataMatrix":
        ctx = ctx or default_context()
        c = SynthSpecC(spec.n, spec.d, 1 if spec.dtype == "f32" else 0, spec.seed, spec.spectrum,
                       spec.spectrum_param, int(spec.t_scale), spec.tau)
        h = vp()
        _check(_lib.load().skr_data_generate(ctx.h, C.byref(c), C.byref(h)))
        return cls(ctx=ctx, _handle=h)

    def rows(self) -> int:
        return self.d

    def cols(self) -> int:
        return self.n_global

    def scale(self) -> float:
        return self._scale

    def scaled(self, factor: float) -> "DataMatrix":
        h = vp()
        _check(_lib.load().skr_data_scaled(self.h, float(factor), C.byref(h)))
        return DataMatrix(ctx=self.ctx, _handle=h, _owner=self)

    def download(self) -> np.ndarray:
        out = np.empty((self.n_local, self.d), dtype=np.float32 if self.dtype == 1 else np.float64)
        _check(_lib.load().skr_data_download(self.h, out.ctypes.data))
        return out

    def labels(self) -> np.ndarray:
        out = np.empty(self.n_local)
        _check(_lib.load().skr_data_labels(self.h, out))
        return out

    def __del__(self):
        if getattr(self, "h", None):
            try:
                _lib.load().skr_data_destroy(self.h)
            except Exception:
                pass
            self.h = None


@dataclass
class SynthSpec:
    n: int
    d: int
    dtype: str = "f64"
    seed: int = 0
    spectrum: int = 0          # 0: 1/j, 1: r^j, 2: j^-p, 3: 1/j (j<=50), 0.02/j beyond
    spectrum_param: float = 0.0
    t_scale: bool = False
    tau: float = 0.1


# ---------------------------------------------------------------------------
@dataclass
class RidgeProblem:
    """RidgeProblem (ridge.hpp:17-27)."""
    data: DataMatrix
    labels: np.ndarray
    lam: float

    def __post_init__(self):
        self.labels = _f64(self.labels)
        if len(self.labels) != self.data.n_local:
            raise DimensionError("ridge problem: label count must equal point count")
        if not (self.lam > 0.0):
            raise ParameterError("ridge problem: lambda must be positive")

    def dim(self) -> int:
        return self.data.d

    def count(self) -> int:
        return self.data.n_global


def scaled_design(p: RidgeProblem) -> DataMatrix:
    """ridge.cpp:54-56: the data scaled by 1/sqrt(n), storage shared."""
    return p.data.scaled(1.0 / math.sqrt(p.count()))


def objective(p: RidgeProblem, w) -> float:
    """ridge.cpp:33-43 on the device."""
    w = _f64(w)
    if len(w) != p.dim():
        raise DimensionError("objective: vector length mismatch")
    out = f64()
    _check(_lib.load().skr_ridge_objective(p.data.ctx.h, p.data.h, p.labels, p.lam, w, C.byref(out)))
    return out.value


# ---------------------------------------------------------------------------
@dataclass
class LanczosConfig:
    """sketch.hpp:27-32."""
    k: int = 0
    eps_prime: float = 0.5
    seed: int = 0
    q_override: Optional[int] = None


@dataclass
class SketchedSvd:
    """sketch.hpp:18-25.  left is (d, k); right is (n_local, k) or None."""
    left: np.ndarray
    singular_values: np.ndarray
    right: Optional[np.ndarray]
    k: int
    q: int
    rank_reduced: bool = False


def lanczos_iterations(n: int, eps_prime: float) -> int:
    """sketch.cpp:13-16."""
    return max(2, int(math.ceil(math.log(n) / math.sqrt(eps_prime))))


def block_lanczos(a: DataMatrix, cfg: LanczosConfig, want_right: bool = True) -> SketchedSvd:
    """sketch.cpp:41-90 on the device (Pi from the reference's mt19937_64 stream)."""
    k, d, n = int(cfg.k), a.d, a.n_local
    U = np.zeros(d * max(k, 1))
    sig = np.zeros(max(k, 1))
    V = np.zeros(n * max(k, 1)) if want_right else None
    ku, qu, rr = i64(), i64(), cint()
    q = int(cfg.q_override) if cfg.q_override else 0
    _check(_lib.load().skr_lanczos(a.ctx.h, a.h, k, q, float(cfg.eps_prime), int(cfg.seed), U, sig,
                                   V.ctypes.data if V is not None else None, C.byref(ku), C.byref(qu),
                                   C.byref(rr)))
    kk = ku.value
    left = U[: d * kk].reshape(kk, d).T
    right = V[: n * kk].reshape(kk, n).T if V is not None else None
    return SketchedSvd(left, sig[:kk].copy(), right, kk, qu.value, bool(rr.value))


# ---------------------------------------------------------------------------
class PreconditionerKind(Enum):
    Sketched = 0
    Exact = 1
    Identity = 2
    Optimal = 3


class Preconditioner:
    """precond.hpp:28-67: P^{-1/2} v = c v + U (diag(inv_sqrt) - c) U^T v (a host value type)."""

    def __init__(self, kind, dim, basis, inv_sqrt, tail, lam):
        self._kind, self._dim, self._basis = kind, dim, basis
        self._inv_sqrt, self._tail, self._lambda = inv_sqrt, tail, lam

    @staticmethod
    def identity(dim: int, lam: float) -> "Preconditioner":
        _check_lambda(lam)
        return Preconditioner(PreconditionerKind.Identity, dim, np.zeros((dim, 0)), np.zeros(0), 1.0, lam)

    def kind(self):
        return self._kind

    def dim(self) -> int:
        return self._dim

    def rank(self) -> int:
        return len(self._inv_sqrt)

    def lam(self) -> float:
        return self._lambda

    def tail_coeff(self) -> float:
        return self._tail

    def inv_sqrt_diag(self) -> np.ndarray:
        return self._inv_sqrt

    def basis(self) -> np.ndarray:
        return self._basis

    def min_inv_eigenvalue(self) -> float:
        lead = self._inv_sqrt[0] if self.rank() else self._tail
        return lead * lead

    def singular_values(self) -> np.ndarray:
        """sigma~ recovered from the coefficients (what the C-ABI takes)."""
        return self._sigma

    # precond.cpp:67-118: O(dk) host maps of the value type (off the hot path; the
    # device applies P^{-1/2} inside the problem and PreconditionedRidge.apply_inv_sqrt)
    def _apply(self, v, sqrt_map: bool) -> np.ndarray:
        v = _f64(v)
        if len(v) != self._dim:
            raise DimensionError(("apply_sqrt" if sqrt_map else "apply_inv_sqrt") + ": vector length mismatch")
        c = 1.0 / self._tail if sqrt_map else self._tail
        out = c * v
        if self.rank():
            proj = self._basis.T @ v
            coef = (1.0 / self._inv_sqrt if sqrt_map else self._inv_sqrt) - c
            out = out + self._basis @ (proj * coef)
        return out

    def apply_inv_sqrt(self, v) -> np.ndarray:
        return self._apply(v, False)

    def apply_sqrt(self, v) -> np.ndarray:
        return self._apply(v, True)

    def inv_sqrt_sq_norm(self, v_sq_norm: float, proj) -> float:
        proj = _f64(proj)
        if len(proj) != self.rank():
            raise DimensionError("inv_sqrt_sq_norm: projection length mismatch")
        c2 = self._tail * self._tail
        s = c2 * v_sq_norm
        for j in range(len(proj)):
            s += (self._inv_sqrt[j] * self._inv_sqrt[j] - c2) * proj[j] * proj[j]
        return s


def _check_lambda(lam):
    if not (lam > 0.0) or not math.isfinite(lam):
        raise ParameterError("preconditioner: lambda must be positive")


def build_sketched(sv: SketchedSvd, lam: float) -> Preconditioner:
    """precond.cpp:120-136 (+ validate, :34-49)."""
    _check_lambda(lam)
    if sv.k < 1:
        raise ParameterError("build_sketched: factors must have rank >= 1")
    s = np.asarray(sv.singular_values[: sv.k], dtype=np.float64)
    inv = 1.0 / np.sqrt(s * s + lam)
    cap = 1.0 / math.sqrt(lam) * (1.0 + 1e-12)
    if np.any(~(inv > 0.0)) or np.any(inv > cap):
        raise InputError("preconditioner: coefficient out of range")
    if np.any(np.diff(inv) < 0):
        raise InputError("preconditioner: coefficients must be non-decreasing")
    p = Preconditioner(PreconditionerKind.Sketched, sv.left.shape[0], np.asarray(sv.left), inv,
                       float(inv[-1]), lam)
    p._sigma = s
    return p


class ApplyMode(Enum):
    Dense = 0
    Lazy = 1
    Auto = 2


kDenseModeMaxEntries = 200_000_000  # ridge.hpp:65 (the Dense-mode guard, ridge.cpp:110-113)


# ---------------------------------------------------------------------------
class SvrgMode(Enum):
    """svrg.hpp:37 — provenance label of a config; the solve is identical."""
    Theoretical = 0
    Tuned = 1


@dataclass
class SvrgConfig:
    """svrg.hpp:39-45."""
    epochs: int = 1
    epoch_length: int = 1
    step_size: float = 0.1
    seed: int = 0
    mode: "SvrgMode" = None  # label only (svrg.hpp:37,44); defaults to Tuned

    def __post_init__(self):
        if self.mode is None:
            self.mode = SvrgMode.Tuned




@dataclass
class EpochRecord:
    """svrg.hpp:16-21."""
    epoch: int
    objective: float
    suboptimality: Optional[float]
    elapsed_ms: float


@dataclass
class SvrgResult:
    iterate: np.ndarray
    trace: list


class GpuEpochState:
    """EpochState (svrg.hpp:53-62) for an external engine: step() only records
    (index, inv_nq); epoch_average() runs the whole epoch as one K10 launch."""

    def __init__(self, p: "PreconditionedRidge"):
        self.p = p
        self._idx: list[int] = []

    def begin_epoch(self, snapshot, full_grad):
        self._snap, self._mu = _f64(snapshot), _f64(full_grad)
        self._idx = []

    def step(self, index: int, eta: float, inv_nq: float = 0.0):
        self._eta = eta
        self._idx.append(int(index))

    def epoch_average(self) -> np.ndarray:
        out = np.empty(self.p.d)
        idx = np.asarray(self._idx, dtype=np.int64)
        _check(_lib.load().skr_epoch(self.p.h, self._snap, self._mu, idx, len(idx), float(self._eta), out))
        return out


class PreconditionedRidge:
    """PreconditionedRidge (ridge.hpp:78-119) — the FiniteSumProblem plugin on the B200.

    ApplyMode (skr_problem_create_mode): Dense materialises X~ in HBM (and, like
    ridge.cpp:110-113, raises ScaleGuardError above 2e8 entries; sparse data are
    densified on the device); Lazy keeps X and the k x n projections and runs the
    device Lazy chain (ridge.cpp:283-400; dense data go through a CSR view); Auto
    is the device's choice — Dense for dense data (180 GB of HBM holds X~ at every
    BASELINE size), Lazy for sparse.  mode() reports what the device runs.
    """

    def __init__(self, p: RidgeProblem, precond: Preconditioner, mode: ApplyMode = ApplyMode.Auto):
        if precond.dim() != p.dim():
            raise DimensionError("preconditioned components: dimension mismatch")
        self.problem_ = p
        self.precond_ = precond
        k = precond.rank()
        self.k = k
        U = np.ascontiguousarray(np.asarray(precond.basis()).T) if k else None  # (k, d): row j = u_j
        sig = _f64(precond._sigma) if k else None
        h = vp()
        _check(_lib.load().skr_problem_create_mode(p.data.ctx.h, p.data.h, p.labels, float(p.lam),
                                                   U.ctypes.data if k else None,
                                                   sig.ctypes.data if k else None, k, int(ApplyMode(mode).value),
                                                   C.byref(h)))
        self.h = h
        n, d, kk, a, b, m = i64(), i64(), i64(), f64(), f64(), f64()
        _check(_lib.load().skr_problem_info(self.h, C.byref(n), C.byref(d), C.byref(kk), C.byref(a),
                                            C.byref(b), C.byref(m)))
        self.n, self.d = n.value, d.value
        self._alpha, self._beta_hat, self._max_row_sq = a.value, b.value, m.value
        self._betas = None

    # FiniteSumProblem (svrg.hpp:67-80)
    def component_count(self) -> int:
        return self.n + self.d

    def dimension(self) -> int:
        return self.d

    def betas(self) -> np.ndarray:
        if self._betas is None:
            out = np.empty(self.n + self.d)
            _check(_lib.load().skr_problem_betas(self.h, out))
            self._betas = out
        return self._betas

    def strong_convexity(self) -> float:
        return self._alpha

    def objective(self, w) -> float:
        out = f64()
        _check(_lib.load().skr_objective(self.h, _f64(w), C.byref(out)))
        return out.value

    def full_gradient(self, w, with_objective: bool = False):
        mu = np.empty(self.d)
        obj = f64()
        _check(_lib.load().skr_full_gradient(self.h, _f64(w), mu, C.byref(obj) if with_objective else None))
        return (mu, obj.value) if with_objective else mu

    def component_gradient(self, i: int, w) -> np.ndarray:
        out = np.empty(self.d)
        _check(_lib.load().skr_component_gradient(self.h, int(i), _f64(w), out))
        return out

    def make_epoch_state(self) -> GpuEpochState:
        return GpuEpochState(self)

    # PreconditionedRidge extras
    def mode(self) -> ApplyMode:
        """ridge.hpp:96: the mode the device problem runs in (skr_problem_mode)."""
        m = C.c_int()
        _check(_lib.load().skr_problem_mode(self.h, C.byref(m)))
        return ApplyMode(m.value)

    def preconditioner(self) -> Preconditioner:
        return self.precond_

    def problem(self) -> RidgeProblem:
        return self.problem_

    def max_row_sq(self) -> float:
        """max_i ||x~_i||^2 over the data rows (the BASELINE step-size rule)."""
        return self._max_row_sq

    def mean_beta(self) -> float:
        return self._beta_hat

    def apply_inv_sqrt(self, v) -> np.ndarray:
        out = np.empty(self.d)
        _check(_lib.load().skr_apply_inv_sqrt(self.h, _f64(v), out))
        return out

    def transformed(self) -> np.ndarray:
        out = np.empty((self.problem_.data.n_local, self.d),
                       dtype=np.float32 if self.problem_.data.dtype == 1 else np.float64)
        _check(_lib.load().skr_problem_transformed(self.h, out.ctypes.data))
        return out

    def index_stream(self, seed: int, count: int) -> np.ndarray:
        out = np.empty(count, dtype=np.int64)
        _check(_lib.load().skr_index_stream(self.h, int(seed), int(count), out))
        return out

    def __del__(self):
        if getattr(self, "h", None):
            try:
                _lib.load().skr_problem_destroy(self.h)
            except Exception:
                pass
            self.h = None



def build_exact(sv: SketchedSvd, lam: float) -> Preconditioner:
    """precond.cpp:138-142: build_sketched on exact factors, kind Exact."""
    p = build_sketched(sv, lam)
    p._kind = PreconditionerKind.Exact
    return p


CONDITION_GUARD_DIM = 2000  # kConditionGuardDim (precond.cpp:14)


def build_optimal(data: DataMatrix, lam: float) -> Preconditioner:
    """precond.cpp:144-162: the full-rank preconditioner from sym_eigs(data.gram())
    (device SYRK + eigensolve, reference sign/order conventions); guarded at d <= 2000."""
    _check_lambda(lam)
    d = data.d
    if d > CONDITION_GUARD_DIM:
        raise ScaleGuardError("build_optimal: dimension exceeds the dense diagnostic guard")
    vals = np.empty(d)
    vecs = np.empty(d * d)
    _check(_lib.load().skr_gram_eigs(data.ctx.h, data.h, vals, vecs))
    U = vecs.reshape(d, d).T.copy()  # column j = eigenvector j
    inv = 1.0 / np.sqrt(np.maximum(vals, 0.0) + lam)
    p = Preconditioner(PreconditionerKind.Optimal, d, U, inv, float(inv[-1]), lam)
    p._sigma = np.sqrt(np.maximum(vals, 0.0))
    return p

def preconditioned_components(p: RidgeProblem, precond: Preconditioner,
                              mode: ApplyMode = ApplyMode.Auto) -> PreconditionedRidge:
    """ridge.hpp:121-123."""
    return PreconditionedRidge(p, precond, mode)


def mean_beta(p: PreconditionedRidge) -> float:
    """svrg.cpp:213-217."""
    return p.mean_beta()


def theoretical_params(p: PreconditionedRidge, w0_gap: float, epsilon: float) -> SvrgConfig:
    """svrg.cpp:219-232: S = max(1, ceil(ln(gap/eps))), m = max(1, ceil(beta_hat/alpha)),
    eta = 0.1/beta_hat, mode Theoretical."""
    if not (epsilon > 0.0) or not (w0_gap > 0.0):
        raise ParameterError("theoretical_params: w0_gap and epsilon must be positive")
    bh = mean_beta(p)
    return SvrgConfig(int(max(1.0, math.ceil(math.log(w0_gap / epsilon)))),
                      int(max(1.0, math.ceil(bh / p.strong_convexity()))), 0.1 / bh, 0, SvrgMode.Theoretical)


def eta_grid(beta_hat: float) -> list:
    """bench.cpp:96-100: 2^j / beta_hat, j = -3..3."""
    return [math.ldexp(1.0, j) / beta_hat for j in range(-3, 4)]


def svrg_solve(p: PreconditionedRidge, cfg: SvrgConfig, w0=None,
               reference_value: Optional[float] = None, stop_suboptimality: Optional[float] = None) -> SvrgResult:
    """svrg.cpp:152-211 — GPU-native: the index stream is the reference's
    NormalSampler(cfg.seed) stream, drawn on the device.  `stop_suboptimality`
    (needs reference_value) ends the solve after the first epoch at or below it
    (time-to-epsilon, bench.cpp:182-189); the reference always runs cfg.epochs."""
    w0 = np.zeros(p.d) if w0 is None else _f64(w0)
    if len(w0) != p.d:
        raise DimensionError("svrg: start point length mismatch")
    c = SvrgConfigC(int(cfg.epochs), int(cfg.epoch_length), float(cfg.step_size), int(cfg.seed))
    tr = (EpochRecordC * max(1, int(cfg.epochs)))()
    w = np.empty(p.d)
    done = i64()
    ref = float("nan") if reference_value is None else float(reference_value)
    if stop_suboptimality is None:
        rc = _lib.load().skr_svrg(p.h, C.byref(c), w0, ref, w, tr, C.byref(done))
    else:
        rc = _lib.load().skr_svrg_until(p.h, C.byref(c), w0, ref, float(stop_suboptimality), w, tr, C.byref(done))
    trace = [EpochRecord(int(r.epoch), float(r.objective),
                         None if math.isnan(r.suboptimality) else float(r.suboptimality),
                         float(r.elapsed_ms)) for r in tr[: done.value]]
    if rc == 5:
        raise DivergenceError(_lib.last_error(), trace)
    _check(rc)
    return SvrgResult(w, trace)


# ---------------------------------------------------------------------------
@dataclass
class SketchedSolveDiagnostics:
    """ridge.hpp:125-136."""
    singular_values: np.ndarray = field(default_factory=lambda: np.zeros(0))
    k_used: int = 0
    q_used: int = 0
    rank_reduced: bool = False
    mode: ApplyMode = ApplyMode.Dense
    beta_hat: float = 0.0
    sketch_ms: float = 0.0
    precompute_ms: float = 0.0
    solve_ms: float = 0.0
    max_projection_drift: float = 0.0


@dataclass
class SketchedSolveResult:
    iterate: np.ndarray
    trace: list
    diagnostics: SketchedSolveDiagnostics


def sketched_preconditioned_svrg(p: RidgeProblem, k: int, cfg: SvrgConfig, sketch_seed: int,
                                 mode: ApplyMode = ApplyMode.Auto,
                                 reference_value: Optional[float] = None,
                                 q_override: Optional[int] = None) -> SketchedSolveResult:
    """ridge.cpp:413-454.  q_override lets the BASELINE configs fix q (the
    reference's pipeline hard-codes eps' = 0.5)."""
    if k < 1 or k > min(p.dim(), p.count()):
        raise ParameterError("sketched svrg: k must satisfy 1 <= k <= min(d, n)")
    diag = SketchedSolveDiagnostics()
    t0 = time.perf_counter()
    sv = block_lanczos(scaled_design(p), LanczosConfig(k, 0.5, sketch_seed, q_override), want_right=False)
    diag.sketch_ms = (time.perf_counter() - t0) * 1e3
    diag.singular_values, diag.k_used, diag.q_used, diag.rank_reduced = sv.singular_values, sv.k, sv.q, sv.rank_reduced
    t0 = time.perf_counter()
    pc = build_sketched(sv, p.lam)
    comp = preconditioned_components(p, pc, mode)
    diag.precompute_ms = (time.perf_counter() - t0) * 1e3
    diag.mode = comp.mode()
    diag.beta_hat = comp.mean_beta()
    t0 = time.perf_counter()
    res = svrg_solve(comp, cfg, np.zeros(p.dim()), reference_value)
    diag.solve_ms = (time.perf_counter() - t0) * 1e3
    return SketchedSolveResult(comp.apply_inv_sqrt(res.iterate), res.trace, diag)


@dataclass
class ReferenceSolution:
    minimizer: np.ndarray
    minimum: float


def reference_minimum_cg(p: RidgeProblem, rel_residual_tol: float, max_iterations: int):
    """bench.hpp:26 / bench.cpp:56-82 on the device: CG from w = 0 on the normal
    equations; returns (w, iterations run)."""
    w = np.empty(p.dim())
    it = i64()
    _check(_lib.load().skr_reference_minimum_cg(p.data.ctx.h, p.data.h, p.labels, float(p.lam),
                                                float(rel_residual_tol), int(max_iterations), w, C.byref(it)))
    return w, it.value


def reference_minimum(p: RidgeProblem) -> ReferenceSolution:
    """bench.cpp:84-94 on the device: SYRK + Cholesky for d <= 5000, else the CG
    route reference_minimum_cg(p, 1e-12, 20 d)."""
    w = np.empty(p.dim())
    mn = f64()
    _check(_lib.load().skr_reference_minimum(p.data.ctx.h, p.data.h, p.labels, float(p.lam), w, C.byref(mn)))
    return ReferenceSolution(w, mn.value)


def conditioned_condition_number(data: DataMatrix, lam: float, precond: Preconditioner) -> float:
    """precond.cpp:196-206 without the d <= 2000 guard (the device has the memory)."""
    k = precond.rank()
    U = np.ascontiguousarray(np.asarray(precond.basis()).T) if k else None
    sig = _f64(precond._sigma) if k else None
    out = f64()
    _check(_lib.load().skr_conditioned_cond(data.ctx.h, data.h, float(lam), U.ctypes.data if k else None,
                                            sig.ctypes.data if k else None, k, C.byref(out)))
    return out.value


# test hooks for the reference streams
def mt_uniforms(seed: int, count: int, ctx: Context | None = None) -> np.ndarray:
    ctx = ctx or default_context()
    out = np.empty(count)
    _check(_lib.load().skr_mt_uniforms(ctx.h, int(seed), int(count), out))
    return out


def make_cumulative_weights(beta, sequential: bool = False, ctx: Context | None = None):
    """svrg.cpp:90-106 on the device: (cum, total) of the sampling weights, bit-identical to the
    reference's sequential fp64 loops (block-scan form, or the one-thread chains)."""
    ctx = ctx or default_context()
    beta = np.ascontiguousarray(beta, dtype=np.float64)
    if beta.size == 0:
        raise InputError("sampling: no weights")
    cum, tot = np.empty(beta.size), f64()
    _check(_lib.load().skr_cumulative_weights(ctx.h, beta, beta.size, int(sequential), cum, C.byref(tot)))
    return cum, tot.value


def gaussian_matrix(rows: int, cols: int, seed: int, ctx: Context | None = None) -> np.ndarray:
    """random.cpp:28-41 on the device; returns (rows, cols)."""
    ctx = ctx or default_context()
    out = np.empty(rows * cols)
    _check(_lib.load().skr_gaussian_matrix(ctx.h, int(rows), int(cols), int(seed), out))
    return out.reshape(cols, rows).T


# ---------------------------------------------------------------------------
# Convergence experiment (bench.hpp:31-59, bench.cpp:96-193) with the eta-grid
# runs of one (method, seed) executed CONCURRENTLY on one GPU: each grid point
# is an independent SVRG chain on a clone of the problem (skr_problem_clone:
# shared X~, private workspaces) bound to its own context (own streams).  A
# chain occupies one thread-block cluster (<= 16 SMs), so the 7 grid points fill
# the GPU instead of running back to back as in the reference.
@dataclass
class BenchConfig:
    """bench.hpp:31-38."""
    lam: float = 1e-6
    k: int = 30
    epochs: int = 20
    eta: Optional[float] = None
    seeds: list = field(default_factory=lambda: [0])
    mode: ApplyMode = ApplyMode.Auto


@dataclass
class ConvergenceRow:
    """bench.hpp:40-46."""
    method: str
    seed: int
    epoch: int
    suboptimality: float
    elapsed_ms: float


def _clone_problem(pre: PreconditionedRidge, ctx: Context) -> PreconditionedRidge:
    h = vp()
    _check(_lib.load().skr_problem_clone(pre.h, ctx.h, C.byref(h)))
    c = object.__new__(PreconditionedRidge)
    c.__dict__.update(pre.__dict__)
    c.h = h
    return c


def run_convergence(p: RidgeProblem, cfg: BenchConfig, lanes: int = 7, prep_cap: Optional[int] = None) -> list:
    """bench.cpp:140-193: both methods, one row per (method, seed, epoch) with the
    suboptimality against one shared reference solve; epoch length 2(n+d); eta
    tuned over eta_grid (bench.cpp:96-100) unless fixed — the grid point with the
    lowest final suboptimality wins (first in grid order on ties), divergent
    runs are discarded.  The sketched method runs block_lanczos with eps' = 0.5
    and the seed, as sketched_preconditioned_svrg does (ridge.cpp:427-431)."""
    from concurrent.futures import ThreadPoolExecutor
    if not cfg.seeds:
        raise ParameterError("bench: at least one seed required")
    problem = RidgeProblem(p.data, p.labels, cfg.lam)
    ref = reference_minimum(problem)
    n, d = problem.count(), problem.dim()
    m = 2 * (n + d)
    start = max(objective(problem, np.zeros(d)) - ref.minimum, 0.0)
    plain = preconditioned_components(problem, Preconditioner.identity(d, cfg.lam))
    ctxs = [Context(p.data.ctx.device) for _ in range(max(1, int(lanes)))]
    if prep_cap is not None:  # optional PREP grid cap per lane (measured: no gain at c2, see DESIGN)
        for cx in ctxs:
            cx.set_prep_cap(prep_cap)
    rows = []
    # Contexts are checked out per job: calls on one Context must be serialised
    # (skr.h), and the pool hands a job to whichever worker is free.
    import queue
    free = queue.Queue()
    for cx in ctxs:
        free.put(cx)

    def run_once(job):
        pre, eta, seed = job
        cx = free.get()
        clone = _clone_problem(pre, cx)
        try:
            res = svrg_solve(clone, SvrgConfig(cfg.epochs, m, eta, seed, SvrgMode.Tuned), np.zeros(d), ref.minimum)
            tr = res.trace
            final = tr[-1].suboptimality if tr and tr[-1].suboptimality is not None else math.inf
            return (final if math.isfinite(final) else math.inf), tr
        except DivergenceError:
            return math.inf, []
        finally:
            del clone
            free.put(cx)

    with ThreadPoolExecutor(max_workers=len(ctxs)) as pool:
        for sketched in (False, True):
            method = "sketched-svrg" if sketched else "svrg"
            for seed in cfg.seeds:
                if sketched:
                    sv = block_lanczos(scaled_design(problem), LanczosConfig(cfg.k, 0.5, int(seed)))
                    pre = preconditioned_components(problem, build_sketched(sv, cfg.lam), cfg.mode)
                else:
                    pre = plain
                grid = [cfg.eta] if cfg.eta is not None else eta_grid(mean_beta(pre))
                jobs = [(pre, eta, int(seed)) for eta in grid]
                results = list(pool.map(run_once, jobs))
                best, best_tr = math.inf, []
                for final, tr in results:  # strict '<' in grid order, as bench.cpp:180
                    if final < best:
                        best, best_tr = final, tr
                if not best_tr:
                    raise DivergenceError("bench: every step size diverged for method " + method, [])
                rows.append(ConvergenceRow(method, int(seed), 0, start, 0.0))
                for rec in best_tr:
                    rows.append(ConvergenceRow(method, int(seed), rec.epoch,
                                               max(rec.suboptimality or 0.0, 0.0), rec.elapsed_ms))
    return rows


# ---------------------------------------------------------------------------
# Ratio / spectrum diagnostics (precond.hpp:13-20,81-91; precond.cpp:23-32,165-172,
# 208-219; bench.cpp:195-212).  The spectrum is one device SYRK + eigensolve;
# the rest is O(d) host arithmetic.
class DegenerateSpectrumError(SkridgeError, RuntimeError):
    """errors.hpp:45-49."""


class DegenerateDataError(SkridgeError, RuntimeError):
    """errors.hpp:39-43."""


class ParseError(SkridgeError, RuntimeError):
    """errors.hpp:51-61: carries the 1-based line number."""

    def __init__(self, line: int, what: str):
        super().__init__(f"line {line}: {what}")
        self.line = line


@dataclass
class SpectrumSummary:
    """precond.hpp:13-20: eigenvalues descending and >= 0 (round-off clamped)."""
    eigenvalues: np.ndarray
    lam: float = 0.0

    def __post_init__(self):
        e = _f64(self.eigenvalues).copy()
        floor = -1e-10 * max(1.0, float(e[0])) if len(e) else 0.0
        prev = math.inf
        for i, v in enumerate(e):
            if v < floor:
                raise InputError("spectrum: negative eigenvalue")
            if v < 0.0:
                e[i] = v = 0.0
            if v > prev:
                raise InputError("spectrum: eigenvalues must be descending")
            prev = v
        self.eigenvalues = e

    def dim(self) -> int:
        return len(self.eigenvalues)


@dataclass
class RatioRow:
    """bench.hpp:50-53."""
    k: int
    ratio: float


def dataset_spectrum(p: RidgeProblem) -> SpectrumSummary:
    """bench.cpp:205-212 on the device: all d eigenvalues of X^T X / n, zero past rank."""
    out = np.empty(p.dim())
    _check(_lib.load().skr_dataset_spectrum(p.data.ctx.h, p.data.h, out))
    return SpectrumSummary(out, p.lam)


def avg_condition_number(spec: SpectrumSummary) -> float:
    """precond.cpp:165-172: sum_i (lam_i + lambda) / (lam_min + lambda)."""
    if spec.dim() == 0:
        raise InputError("avg_condition_number: empty spectrum")
    denom = spec.eigenvalues[-1] + spec.lam
    if not (denom > 0.0):
        raise InputError("avg_condition_number: lam_min + lambda must be positive")
    tr = 0.0
    for v in spec.eigenvalues:
        tr += v + spec.lam
    return tr / denom


def theoretical_ratio(spec: SpectrumSummary, k: int) -> float:
    """precond.cpp:208-219: (head + tail) / (k lam_k + tail), sums in index order."""
    d = spec.dim()
    if k < 1 or k > d:
        raise ParameterError("theoretical_ratio: k must satisfy 1 <= k <= d")
    head = 0.0
    for i in range(k):
        head += spec.eigenvalues[i]
    tail = 0.0
    for i in range(k, d):
        tail += spec.eigenvalues[i]
    denom = float(k) * spec.eigenvalues[k - 1] + tail
    if denom == 0.0:
        raise DegenerateSpectrumError("theoretical_ratio: zero denominator")
    return (head + tail) / denom


def run_ratio_curve(spec: SpectrumSummary, k_max: int) -> list:
    """bench.cpp:195-203."""
    if k_max < 1 or k_max > spec.dim():
        raise ParameterError("ratio curve: k_max must satisfy 1 <= k_max <= d")
    return [RatioRow(k, theoretical_ratio(spec, k)) for k in range(1, k_max + 1)]


# ---------------------------------------------------------------------------
# Sparse corpus I/O (dataset.hpp:37-49, dataset.cpp:80-198): host text parsing
# into a device CSR DataMatrix.
@dataclass
class LabeledDataset:
    data: DataMatrix
    labels: np.ndarray
    provenance: str = ""


def _strict_float(tok: str) -> float:
    if "_" in tok or tok != tok.strip():
        raise ValueError(tok)
    return float(tok)


def read_sparse_corpus(path: str, ctx: Context | None = None) -> LabeledDataset:
    """dataset.cpp:87-162: lines "label idx:value ...", 1-based strictly increasing
    indices, '#' comments, blank lines skipped, zero values dropped, d = the
    largest index seen."""
    try:
        f = open(path)
    except OSError:
        raise InputError("corpus: cannot open " + path)
    rp, ci, va, labels = [0], [], [], []
    max_index = 0
    with f:
        for lineno, raw in enumerate(f, start=1):
            toks = raw.split("#", 1)[0].split()
            if not toks:
                continue
            try:
                labels.append(_strict_float(toks[0]))
            except ValueError:
                raise ParseError(lineno, f"bad label '{toks[0]}'")
            prev = 0
            for tok in toks[1:]:
                colon = tok.find(":")
                if colon <= 0 or colon + 1 >= len(tok):
                    raise ParseError(lineno, f"bad feature '{tok}'")
                try:
                    head = tok[:colon]
                    if "_" in head or not head.lstrip("+-").isdigit():
                        raise ValueError(tok)
                    index = int(head)
                    if index < 1:
                        raise ValueError(tok)
                    value = _strict_float(tok[colon + 1:])
                except ValueError:
                    raise ParseError(lineno, f"bad feature '{tok}'")
                if index <= prev:
                    raise ParseError(lineno, "feature indices must be strictly increasing")
                if not math.isfinite(value):
                    raise ParseError(lineno, "non-finite value")
                prev = index
                max_index = max(max_index, index)
                if value != 0.0:
                    ci.append(index - 1)
                    va.append(value)
            rp.append(len(va))
    if not labels:
        raise InputError("corpus: no data lines in " + path)
    if max_index == 0:
        raise DegenerateDataError("corpus: no features seen")
    data = DataMatrix.from_csr(np.asarray(rp, dtype=np.int64), np.asarray(ci, dtype=np.int32),
                               np.asarray(va, dtype=np.float64), max_index, ctx)
    return LabeledDataset(data, np.asarray(labels, dtype=np.float64), path)


def write_sparse_corpus(row_ptr, col_idx, values, labels, path: str, scale: float = 1.0):
    """dataset.cpp:164-186 for CSR rows: "%.17g" labels and values, 1-based indices."""
    rp = np.asarray(row_ptr)
    with open(path, "w") as out:
        for i in range(len(labels)):
            parts = ["%.17g" % labels[i]]
            for t in range(rp[i], rp[i + 1]):
                parts.append("%d:%s" % (int(col_idx[t]) + 1, "%.17g" % (scale * values[t])))
            out.write(" ".join(parts) + "\n")


def average_norm_normalize(ds: LabeledDataset, row_ptr=None, values=None) -> LabeledDataset:
    """dataset.cpp:188-198: scale the data by 1 / (mean point norm), summed in point
    order.  Needs the host CSR arrays the DataMatrix was built from."""
    rp, va = np.asarray(row_ptr), np.asarray(values, dtype=np.float64)
    n = len(rp) - 1
    if n == 0:
        raise DegenerateDataError("normalize: empty dataset")
    total = 0.0
    for i in range(n):
        seg = va[rp[i]:rp[i + 1]]
        total += math.sqrt(float(np.dot(seg, seg)))
    mean = total / n
    if mean == 0.0:
        raise DegenerateDataError("normalize: all columns are zero")
    return LabeledDataset(ds.data.scaled(1.0 / mean), ds.labels.copy(), ds.provenance)
