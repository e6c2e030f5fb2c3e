"""BSGD-TV solver on a B200 (drop-in for `bsgdtv.solvers`, `pkg/src/bsgdtv/solvers.py`).

Same entry points, types and semantics as the reference:
`SolverConfig`, `Problem`, `TraceSample`, `ConvergenceTrace`,
`read_trace_csv`, `DivergenceError`, `schedule_pairs`,
`sufficient_decrease_holds`, `SolverState`, `init_bsgd_state`,
`bsgd_tv_iteration` and `run_solver`.

What changes is where the state lives.  `SolverState` keeps x, r, g (and the
z cache when the stochastic path needs it) in HBM; its fields read back as
numpy arrays on access, exactly like the reference dataclass, and accept
numpy assignments.  One epoch (`bsgd_tv_iteration`, `solvers.py:259-341`)
is one `bsgd_epoch` call: K2 (A^T r_k with the step epilogue) -> TV prox
(one cooperative kernel) -> K1 (A x_{k+1}, which is both the monitor's
fidelity product and the next epoch's residual) -> a one-warp tail that
evaluates the Eq. 9 test and records the epoch's statistics.

Algebraic identity used (no approximation): the reference computes
r_{k+1} = y - A x_k at epoch k and, with the default monitor, the uncharged
f_next = ||y - A x_{k+1}||^2.  The latter product IS epoch k+1's residual, so
it is computed once and carried ("lookahead"); a user assignment to
`state.x` invalidates it and the next epoch recomputes y - A x_k.
Charged matvec units follow the reference's bookkeeping exactly.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import NamedTuple

import numpy as np

from . import _native as nat
from .blockops import BlockOperator
from .tv import PixelLayout, ProxSettings

SOLVER_KINDS = ("bsgd", "ista", "gd", "admm")


@dataclass(frozen=True)
class SolverConfig:
    """Run parameters (`solvers.py:33-73`), identical fields and validation."""

    mu: float
    lam: float = 0.0
    alpha: float = 1.0
    gamma: float = 1.0
    epochs: float = 200
    seed: int = 0
    prox: ProxSettings = field(default_factory=ProxSettings)
    rho: float = 1.0
    cg_iters: int = 5
    monitor_decrease: bool = True
    enforce_decrease: bool = False
    max_halvings: int = 20
    divergence_limit: float = 1e6

    def __post_init__(self) -> None:
        if not self.mu > 0:
            raise ValueError("mu must be positive")
        if self.lam < 0:
            raise ValueError("lam must be nonnegative")
        for name, frac in (("alpha", self.alpha), ("gamma", self.gamma)):
            if not 0 < frac <= 1:
                raise ValueError(f"{name} must lie in (0, 1]")
        if self.epochs < 0:
            raise ValueError("epochs must be nonnegative")
        if self.cg_iters < 1:
            raise ValueError("cg_iters must be >= 1")
        if self.max_halvings < 0:
            raise ValueError("max_halvings must be nonnegative")
        if not self.divergence_limit > 0:
            raise ValueError("divergence_limit must be positive")


@dataclass
class Problem:
    """Inverse-problem instance handed to `run_solver` (`solvers.py:76-99`)."""

    op: BlockOperator
    y: np.ndarray
    x_true: np.ndarray | None = None
    layout: PixelLayout | None = None

    def __post_init__(self) -> None:
        t = nat.torch()
        rows, cols = self.op.shape
        if not isinstance(self.y, t.Tensor):
            self.y = np.asarray(self.y, dtype=np.float64)
        if tuple(self.y.shape) != (rows,):
            raise ValueError(f"y has shape {tuple(self.y.shape)}, expected ({rows},)")
        if self.x_true is not None:
            if not isinstance(self.x_true, t.Tensor):
                self.x_true = np.asarray(self.x_true, dtype=np.float64)
            if tuple(self.x_true.shape) != (cols,):
                raise ValueError(f"x_true has shape {tuple(self.x_true.shape)}, expected ({cols},)")
        if self.layout is not None and self.layout.size != cols:
            raise ValueError("layout pixel count does not match the column dimension")


class TraceSample(NamedTuple):
    epoch: float
    relative_error: float
    objective: float
    matvec_units: float


@dataclass
class ConvergenceTrace:
    """Sampled run history plus per-iteration decrease flags (`solvers.py:109-144`)."""

    samples: list = field(default_factory=list)
    decrease_flags: list = field(default_factory=list)
    final_x: np.ndarray | None = None

    def append(self, sample: TraceSample) -> None:
        if self.samples and not sample.epoch > self.samples[-1].epoch:
            raise ValueError("trace epochs must be strictly increasing")
        self.samples.append(sample)

    def epochs(self) -> np.ndarray:
        return np.array([s.epoch for s in self.samples])

    def relative_errors(self) -> np.ndarray:
        return np.array([s.relative_error for s in self.samples])

    def objectives(self) -> np.ndarray:
        return np.array([s.objective for s in self.samples])

    def matvec_units(self) -> np.ndarray:
        return np.array([s.matvec_units for s in self.samples])

    def to_csv_string(self) -> str:
        lines = ["epoch,relative_error,objective,matvec_units"]
        for s in self.samples:
            lines.append(f"{s.epoch:.17g},{s.relative_error:.17g},{s.objective:.17g},{s.matvec_units:.17g}")
        return "\n".join(lines) + "\n"

    def write_csv(self, path) -> None:
        with open(path, "w") as fh:
            fh.write(self.to_csv_string())


def read_trace_csv(path) -> ConvergenceTrace:
    trace = ConvergenceTrace()
    with open(path) as fh:
        header = fh.readline().strip()
        if header != "epoch,relative_error,objective,matvec_units":
            raise ValueError(f"unexpected trace header in {path}")
        for line in fh:
            line = line.strip()
            if not line:
                continue
            parts = line.split(",")
            if len(parts) != 4:
                raise ValueError(f"bad trace row in {path}: {line}")
            trace.append(TraceSample(*(float(p) for p in parts)))
    return trace


class DivergenceError(RuntimeError):
    """Iterates left the admissible region; carries the trace so far (`solvers.py:164-169`)."""

    def __init__(self, message: str, trace: ConvergenceTrace):
        super().__init__(message)
        self.trace = trace


def _round_half_up(value: float) -> int:
    return int(math.floor(value + 0.5))


def schedule_pairs(num_row_blocks: int, num_col_blocks: int, alpha: float, gamma: float,
                   rng: np.random.Generator):
    """Pair draw of one iteration (`solvers.py:176-195`): host RNG, unchanged, so the
    numpy Generator state advances exactly as in the reference."""
    if alpha == 1.0 and gamma == 1.0:
        flat = rng.permutation(num_row_blocks * num_col_blocks)
        return [(int(k) // num_col_blocks, int(k) % num_col_blocks) for k in flat]
    picked_rows = _round_half_up(gamma * num_row_blocks)
    picked_cols = _round_half_up(alpha * num_col_blocks)
    if picked_rows < 1 or picked_cols < 1:
        raise ValueError("alpha/gamma select no blocks after rounding")
    i_sel = rng.choice(num_row_blocks, size=picked_rows, replace=False)
    j_sel = rng.choice(num_col_blocks, size=picked_cols, replace=False)
    return [(int(i), int(j)) for i in i_sel for j in j_sel]


def sufficient_decrease_holds(f_next: float, f_curr: float, x_next, x_curr, grad_prev, mu: float) -> bool:
    """Eq. 9 test (`solvers.py:198-215`), dot products on the device."""
    if not mu > 0:
        raise ValueError("mu must be positive")
    t = nat.torch()
    dev = nat.require_cuda()
    xn = nat.as_f64(x_next, dev)
    xc = nat.as_f64(x_curr, dev)
    gp = nat.as_f64(grad_prev, dev)
    delta = xn - xc
    scratch = t.empty(nat.SCRATCH_BYTES // 8, dtype=t.float64, device=dev)
    out = t.empty(2, dtype=t.float64, device=dev)
    n = delta.numel()
    nat.call("bsgd_dot", n, nat.ptr(delta), nat.ptr(gp), nat.ptr(out[0:1]), nat.ptr(scratch), nat.stream_ptr(dev))
    nat.call("bsgd_dot", n, nat.ptr(delta), nat.ptr(delta), nat.ptr(out[1:2]), nat.ptr(scratch), nat.stream_ptr(dev))
    dg, dd = (float(v) for v in out.cpu().tolist())
    bound = f_curr + dg
    bound += dd / (2.0 * mu)
    return bool(f_next < bound)


# ---------------------------------------------------------------------------
# device-resident state
# ---------------------------------------------------------------------------

class SolverState:
    """Per-run state of the block-stochastic iteration, resident in HBM.

    Field names and meaning follow the reference dataclass (`solvers.py:218-237`):
    ``x``, ``z_cache``, ``r_vec``, ``g`` read back as numpy float64 arrays and
    accept assignment; ``epoch``, ``matvec_units``, ``rng``, ``mu_eff``,
    ``f_curr`` and ``last_decrease_ok`` behave as there.  ``*_device``
    accessors return the CUDA tensors without a copy.
    """

    def __init__(self, op: BlockOperator, y, cfg: SolverConfig, history_capacity: int = 64):
        t = nat.torch()
        self._op = op
        self._dev = op.device
        rows, cols = op.shape
        self._rows, self._cols = rows, cols
        self._y_src = y
        self._y = nat.as_f64(y, self._dev, rows)
        f64 = dict(dtype=t.float64, device=self._dev)
        self._x = t.zeros(2, cols, **f64)
        self._r = t.empty(2, rows, **f64)
        self._r[0].copy_(self._y)
        self._r[1].copy_(self._y)   # y - A 0 = y exactly: the lookahead of x_0
        self._xi = 0
        self._ri = 0
        self._la_valid = True
        self._la_policy = True
        self._version = 0           # bumped by every epoch and every state write
        self._host_reads = False    # x / r_vec read back since the last epoch
        self._spec = None           # readback started during the last epoch (see _speculative_epoch)
        self._side = None
        self._pending_r = None      # pinned host r_vec assigned, copy deferred (see r_vec.setter)
        self._copy = None
        self._g = t.zeros(cols, **f64)
        self._z = None              # explicit z cache (N, rows) once the stochastic path ran
        self._z_explicit = False
        self._f_curr = t.empty(1, **f64)
        scratch = t.empty(nat.SCRATCH_BYTES // 8, **f64)
        nat.call("bsgd_dot", rows, nat.ptr(self._y), nat.ptr(self._y), nat.ptr(self._f_curr), nat.ptr(scratch),
                 nat.stream_ptr(self._dev))
        self._counter = t.zeros(1, dtype=t.int64, device=self._dev)
        self._hist = t.zeros(max(1, history_capacity), nat.HIST_COLS, **f64)
        self._rows_used = 0
        self._ws = None
        self._ws_key = None
        self._x_true = None
        self._last_row = None
        self._last_ok_static = None
        self.epoch = 0.0
        self.matvec_units = 0.0
        self.rng = np.random.default_rng(cfg.seed)
        self.mu_eff = cfg.mu

    # --- reference-style fields ---------------------------------------------
    # Reads return numpy arrays backed by pinned host memory (torch's caching
    # host allocator), so a read -> modify -> assign round trip moves data by
    # DMA without an extra host copy; each read is a fresh array.  A caller that
    # reads x / r_vec after every epoch gets them copied back while the epoch is
    # still running (r behind K1, x behind the step), see `_speculative_epoch`.

    def _read(self, which: str, dev_tensor) -> np.ndarray:
        self._host_reads = True
        sp = self._spec
        if sp is not None and sp["version"] == self._version and which in sp:
            h, ev = sp.pop(which)
            ev.synchronize()
            return h.numpy()
        return self._to_host(dev_tensor)

    def _touch(self) -> None:
        self._version += 1
        self._spec = None

    @staticmethod
    def _to_host(t) -> np.ndarray:
        tt = nat.torch()
        h = tt.empty(t.shape, dtype=tt.float64, pin_memory=True)
        h.copy_(t, non_blocking=True)
        tt.cuda.current_stream(t.device).synchronize()
        return h.numpy()

    def _from_host(self, dst, value, length) -> None:
        tt = nat.torch()
        if isinstance(value, tt.Tensor):
            dst.copy_(nat.as_f64(value, self._dev, length))
            return
        arr = np.asarray(value, dtype=np.float64)
        if arr.shape != (length,):
            raise ValueError(f"expected vector of length {length}, got {arr.shape}")
        src = tt.from_numpy(np.ascontiguousarray(arr))
        pinned = src.is_pinned()
        dst.copy_(src, non_blocking=pinned)
        if pinned:  # the caller may reuse its array right away
            tt.cuda.current_stream(self._dev).synchronize()

    @property
    def x(self) -> np.ndarray:
        return self._read("x", self._x[self._xi])

    @x.setter
    def x(self, value) -> None:
        self._from_host(self._x[self._xi], value, self._cols)
        self._touch()
        # a new x voids the lookahead product y - A x_next; a caller that writes x
        # between epochs would void every one, so stop computing it eagerly (without
        # the monitor, each epoch then runs K1(x_k) and K2(r_k) merged: still two
        # products, none wasted)
        if self._la_valid:
            self._la_policy = False
        self._la_valid = False

    @property
    def r_vec(self) -> np.ndarray:
        self._flush_r()
        return self._read("r", self._r[self._ri])

    @r_vec.setter
    def r_vec(self, value) -> None:
        # A pinned, contiguous float64 array (what the getters hand out) is copied
        # lazily: a full-pass epoch moves it over PCIe while K1, which does not
        # read r_k, runs, and waits for the copy before it returns, so the caller
        # may reuse the array afterwards exactly as with an eager copy.
        t = nat.torch()
        self._pending_r = None
        if not isinstance(value, t.Tensor):
            arr = np.asarray(value)
            if (arr.dtype == np.float64 and arr.shape == (self._rows,) and arr.flags.c_contiguous
                    and t.from_numpy(arr).is_pinned()):
                self._pending_r = arr
                self._touch()
                return
        self._from_host(self._r[self._ri], value, self._rows)
        self._touch()

    def _flush_r(self) -> None:
        if self._pending_r is not None:
            arr, self._pending_r = self._pending_r, None
            self._from_host(self._r[self._ri], arr, self._rows)

    @property
    def g(self) -> np.ndarray:
        return self._to_host(self._g)

    @g.setter
    def g(self, value) -> None:
        self._from_host(self._g, value, self._cols)
        self._touch()

    @property
    def z_cache(self) -> np.ndarray:
        return self._z_device().cpu().numpy()

    @z_cache.setter
    def z_cache(self, value) -> None:
        t = nat.torch()
        z = t.as_tensor(np.asarray(value, dtype=np.float64)).to(self._dev)
        if tuple(z.shape) != (self._op.num_col_blocks, self._rows):
            raise ValueError("z_cache shape mismatch")
        self._z = z.contiguous()
        self._z_explicit = True

    @property
    def f_curr(self) -> float:
        return float(self._f_curr.item())

    @f_curr.setter
    def f_curr(self, value: float) -> None:
        self._f_curr.fill_(float(value))

    @property
    def last_decrease_ok(self):
        if self._last_row is None:
            return self._last_ok_static
        h = float(self._hist[self._last_row, nat.H_HOLDS].item())
        return None if h < 0 else bool(h > 0.5)

    @last_decrease_ok.setter
    def last_decrease_ok(self, value) -> None:
        self._last_row = None
        self._last_ok_static = value

    # --- device accessors ----------------------------------------------------

    @property
    def x_device(self):
        return self._x[self._xi]

    @property
    def r_device(self):
        self._flush_r()
        return self._r[self._ri]

    @property
    def g_device(self):
        return self._g

    def history(self, rows: int | None = None) -> np.ndarray:
        n = self._rows_used if rows is None else rows
        return self._hist[:n].cpu().numpy()

    # --- internals -----------------------------------------------------------

    def _ensure_history(self, extra: int) -> None:
        need = self._rows_used + extra
        if need <= self._hist.shape[0]:
            return
        t = nat.torch()
        new = t.zeros(max(need, 2 * self._hist.shape[0]), nat.HIST_COLS, dtype=t.float64, device=self._dev)
        new[: self._hist.shape[0]].copy_(self._hist)
        self._hist = new

    def _workspace(self, layout: PixelLayout | None, lam: float):
        hw = (layout.height, layout.width) if (lam > 0 and layout is not None) else (0, 0)
        if self._ws is None or self._ws_key != hw:
            t = nat.torch()
            nbytes = int(nat.load().bsgd_epoch_workspace_bytes(self._op.plan, hw[0], hw[1]))
            self._ws = t.zeros((nbytes + 7) // 8, dtype=t.float64, device=self._dev)
            self._ws_key = hw
        return self._ws

    def _y_for(self, y):
        if y is self._y_src or y is self._y:
            return self._y
        return nat.as_f64(y, self._dev, self._rows)

    def _z_device(self):
        """Explicit z cache; materialised from x_{k-1} (the x behind r_vec) when implicit."""
        if self._z_explicit:
            return self._z
        t = nat.torch()
        op = self._op
        part = op.partition
        z = t.zeros(op.num_col_blocks, self._rows, dtype=t.float64, device=self._dev)
        x_prev = self._x[1 - self._xi]
        st = nat.stream_ptr(self._dev)
        for i in range(part.num_row_blocks):
            r0, r1 = part.row_range(i)
            for j in range(part.num_col_blocks):
                c0, c1 = part.col_range(j)
                xs = x_prev[c0:c1].contiguous()
                nat.call("bsgd_block_matvec", op.plan, i, j, nat.ptr(xs), nat.ptr(z[j, r0:r1]), st)
        return z


def init_bsgd_state(op: BlockOperator, y, cfg: SolverConfig) -> SolverState:
    """x = 0, z cache = 0, r = y, f_curr = y.y (`solvers.py:240-256`)."""
    rows, _ = op.shape
    shp = tuple(y.shape) if hasattr(y, "shape") else np.asarray(y).shape
    if shp != (rows,):
        raise ValueError(f"y has shape {shp}, expected ({rows},)")
    return SolverState(op, y, cfg)


# ---------------------------------------------------------------------------
# one epoch
# ---------------------------------------------------------------------------

def _epoch_args(state: SolverState, cfg: SolverConfig, layout, y_dev, xi: int, ri: int, flags: int,
                mu: float, ws) -> nat.EpochArgs:
    lam = cfg.lam
    perm = layout.device_perm(state._dev) if (lam > 0 and layout is not None) else None
    a = nat.EpochArgs()
    a.x_k = nat.ptr(state._x[xi])
    a.x_next = nat.ptr(state._x[1 - xi])
    a.r_k = nat.ptr(state._r[ri])
    a.r_next = nat.ptr(state._r[1 - ri])
    a.r_ahead = nat.ptr(state._r[ri])
    a.y = nat.ptr(y_dev)
    a.g = nat.ptr(state._g)
    a.x_true = nat.ptr(state._x_true) if state._x_true is not None else None
    a.perm = nat.ptr(perm) if perm is not None else None
    a.mu = mu
    a.lam = lam
    a.height = layout.height if (lam > 0 and layout is not None) else 0
    a.width = layout.width if (lam > 0 and layout is not None) else 0
    a.depth = getattr(layout, "depth", 1) if (lam > 0 and layout is not None) else 0
    a.max_inner_iters = cfg.prox.max_inner_iters
    a.tol = cfg.prox.tol
    a.f_curr = nat.ptr(state._f_curr)
    a.history = nat.ptr(state._hist)
    a.epoch_counter = nat.ptr(state._counter)
    a.history_capacity = state._hist.shape[0]
    a.dual_objectives = None
    a.workspace = nat.ptr(ws)
    a.workspace_bytes = ws.numel() * 8
    a.flags = flags
    return a


def _launch(state: SolverState, args: nat.EpochArgs) -> None:
    nat.call("bsgd_epoch", state._op.plan, ctypes.byref(args), nat.stream_ptr(state._dev))


def _read_holds(state: SolverState, row: int) -> bool:
    return float(state._hist[row, nat.H_HOLDS].item()) > 0.5


def bsgd_tv_iteration(state: SolverState, op: BlockOperator, y, cfg: SolverConfig,
                      layout: PixelLayout | None = None, executor=None) -> SolverState:
    """One outer iteration (`solvers.py:259-341`); mutates and returns ``state``.

    ``executor`` is accepted for signature compatibility; the per-pair work
    runs as GPU kernels, and all reductions are fixed-order, so results do not
    depend on it.
    """
    if cfg.lam > 0 and layout is None:
        raise ValueError("layout required when lam > 0")
    if op is not state._op:
        raise ValueError("state was initialised for a different operator")
    part = op.partition
    m, n = part.num_row_blocks, part.num_col_blocks
    pairs = schedule_pairs(m, n, cfg.alpha, cfg.gamma, state.rng)
    y_dev = state._y_for(y)
    monitor = cfg.monitor_decrease or cfg.enforce_decrease
    ws = state._workspace(layout, cfg.lam)
    state._ensure_history(cfg.max_halvings + 2)
    xi, ri = state._xi, state._ri
    full = len(pairs) == m * n
    want_la = monitor or state._la_policy
    flags = (nat.EP_LOOKAHEAD if want_la else 0) | (nat.EP_MONITOR if monitor else 0)
    f_before = state._f_curr.clone() if cfg.enforce_decrease else None
    if full:
        if not state._la_valid:
            flags |= nat.EP_R_NEXT
        op._charge(2 * op.nnz)
    else:
        state._flush_r()
        _pair_products(state, op, pairs, y_dev, xi, ri)
        flags |= nat.EP_SKIP_GRAD
    mu = state.mu_eff
    split = full and not monitor and bool(flags & nat.EP_R_NEXT) and not (flags & nat.EP_LOOKAHEAD)
    speculate = state._host_reads and split
    pending_r = state._pending_r if split else None
    if pending_r is None:
        state._flush_r()
    state._pending_r = None
    state._host_reads = False
    state._touch()
    if speculate or pending_r is not None:
        _speculative_epoch(state, cfg, layout, y_dev, xi, ri, flags, mu, ws, pending_r, speculate)
    else:
        args = _epoch_args(state, cfg, layout, y_dev, xi, ri, flags, mu, ws)
        _launch(state, args)
    row = state._rows_used
    state._rows_used += 1
    if cfg.enforce_decrease:
        halvings = 0
        holds = _read_holds(state, row)
        retry_flags = nat.EP_SKIP_GRAD | nat.EP_LOOKAHEAD | nat.EP_MONITOR
        while not holds and halvings < cfg.max_halvings:
            mu *= 0.5
            halvings += 1
            state._f_curr.copy_(f_before)
            state._counter.fill_(row)
            retry = _epoch_args(state, cfg, layout, y_dev, xi, ri, retry_flags, mu, ws)
            _launch(state, retry)
            holds = _read_holds(state, row)
        state.mu_eff = mu
    state._xi = 1 - xi
    state._ri = 1 - ri
    state._la_valid = bool(flags & nat.EP_LOOKAHEAD)
    if full:
        state._z_explicit = False
    state._last_row = row if monitor else None
    state._last_ok_static = None
    state.epoch += len(pairs) / (m * n)
    pend = getattr(state, "_spec_pending", None)
    if pend is not None:
        pend["version"] = state._version
        state._spec = pend
        state._spec_pending = None
    return state


def _speculative_epoch(state: SolverState, cfg: SolverConfig, layout, y_dev, xi: int, ri: int, flags: int,
                       mu: float, ws, pending_r=None, readback: bool = True) -> None:
    """The same epoch as one `bsgd_epoch` with R_NEXT, split so the host copies overlap it.

    The caller read x / r_vec back after the previous epoch, so it will again:
    K1 (r_next = y - A x_k, `bsgd_epoch_forward`) runs first and r_next starts
    streaming to pinned host memory on a side stream while K2, the step and the
    prox run; x_next follows as soon as it exists.  The getters hand these
    buffers out (once) while the state version is unchanged.  An r_vec assigned
    from pinned host memory (``pending_r``) crosses PCIe on a copy stream while
    K1 runs; K2 waits for it.
    """
    t = nat.torch()
    dev = state._dev
    cur = t.cuda.current_stream(dev)
    if state._side is None:
        state._side = t.cuda.Stream(device=dev)
    side = state._side
    args = _epoch_args(state, cfg, layout, y_dev, xi, ri, flags & ~nat.EP_R_NEXT, mu, ws)
    r_next, x_next = state._r[1 - ri], state._x[1 - xi]
    copied = None
    if pending_r is not None:
        if state._copy is None:
            state._copy = t.cuda.Stream(device=dev)
        start = t.cuda.Event()
        start.record(cur)   # work queued earlier may still read the r_k slot
        with t.cuda.stream(state._copy):
            state._copy.wait_event(start)
            state._r[ri].copy_(t.from_numpy(pending_r), non_blocking=True)
            copied = t.cuda.Event()
            copied.record(state._copy)
    nat.call("bsgd_epoch_forward", state._op.plan, nat.ptr(state._x[xi]), nat.ptr(y_dev), nat.ptr(r_next),
             ctypes.byref(args), nat.stream_ptr(dev))
    if readback:
        ev_r = t.cuda.Event()
        ev_r.record(cur)
        rh = t.empty(r_next.shape, dtype=t.float64, pin_memory=True)
        with t.cuda.stream(side):
            side.wait_event(ev_r)
            rh.copy_(r_next, non_blocking=True)
            done_r = t.cuda.Event()
            done_r.record(side)
    if copied is not None:
        cur.wait_event(copied)
    _launch(state, args)
    if readback:
        ev_x = t.cuda.Event()
        ev_x.record(cur)
        xh = t.empty(x_next.shape, dtype=t.float64, pin_memory=True)
        with t.cuda.stream(side):
            side.wait_event(ev_x)
            xh.copy_(x_next, non_blocking=True)
            done_x = t.cuda.Event()
            done_x.record(side)
        # no wait on the main stream: the next epoch writes the other ring slots, and
        # anything that does overwrite these (a setter, the epoch after next) bumps the
        # state version first, so a copy it could race with is never handed out
        state._spec_pending = {"x": (xh, done_x), "r": (rh, done_r)}
    if copied is not None:
        copied.synchronize()   # the caller may reuse its r_vec array from here on


def _pair_products(state: SolverState, op: BlockOperator, pairs, y_dev, xi: int, ri: int) -> None:
    """Stochastic alpha/gamma < 1 products (`solvers.py:274-303`): z cache commit,
    residual from the cache, gradient over the selected pairs."""
    z = state._z_device()
    state._z = z
    state._z_explicit = True
    rows_sel = np.array(sorted({i for i, _ in pairs}), dtype=np.int64)
    cols_sel = np.array(sorted({j for _, j in pairs}), dtype=np.int64)
    nat.call("bsgd_pair_products", op.plan, rows_sel.size, rows_sel.ctypes.data, cols_sel.size,
             cols_sel.ctypes.data, nat.ptr(state._x[xi]), nat.ptr(state._r[ri]), nat.ptr(y_dev), nat.ptr(z),
             nat.ptr(state._g), nat.ptr(state._r[1 - ri]), nat.stream_ptr(state._dev))
    op._charge(2 * sum(op.block_nnz(i, j) for i, j in pairs))


# ---------------------------------------------------------------------------
# run_solver
# ---------------------------------------------------------------------------

class _GraphRunner:
    """CUDA-graph replay of full-sweep epochs (alpha = gamma = 1, no enforcement).

    The x / r rings flip every epoch, so a captured pair of epochs (one per
    parity) replays any even number of epochs; the history row index lives
    on the device, so replays write consecutive rows.
    """

    def __init__(self, state: SolverState, cfg: SolverConfig, layout, y_dev, epochs_per_graph: int):
        self.state = state
        self.cfg = cfg
        self.layout = layout
        self.y_dev = y_dev
        self.k = epochs_per_graph
        self.graph = None
        self.parity = None

    def _flags(self, monitor):
        return nat.EP_LOOKAHEAD | (nat.EP_MONITOR if monitor else 0)

    def capture(self, monitor: bool) -> bool:
        t = nat.torch()
        st = self.state
        st._flush_r()
        ws = st._workspace(self.layout, self.cfg.lam)
        xi, ri = st._xi, st._ri
        args = [_epoch_args(st, self.cfg, self.layout, self.y_dev, (xi + e) % 2, (ri + e) % 2,
                            self._flags(monitor), st.mu_eff, ws) for e in range(2)]
        self._args = args
        g = t.cuda.CUDAGraph()
        try:
            side = t.cuda.Stream(device=st._dev)
            side.wait_stream(t.cuda.current_stream(st._dev))
            with t.cuda.graph(g, stream=side):
                for e in range(self.k):
                    _launch(st, args[e % 2])
        except Exception:  # capture unsupported: eager launches still run on the GPU
            self.graph = None
            return False
        self.graph = g
        self.parity = (xi, ri)
        return True

    def replay(self) -> None:
        self.graph.replay()


def run_solver(kind: str, problem: Problem, cfg: SolverConfig, sample_every: int = 1, workers: int = 1,
               *, use_graphs: bool = True, chunk_epochs: int = 64, group=None) -> ConvergenceTrace:
    """Drive the solver to the epoch budget, sampling the trace (`solvers.py:445-533`).

    Samples, decrease flags, divergence checks and matvec units follow the
    reference exactly; per-epoch quantities are produced on the device and
    read back once per chunk of ``chunk_epochs`` epochs (no per-epoch host
    synchronisation).  ``workers`` is validated and otherwise unused (the
    products already use the whole GPU).

    Multi-GPU (one process per GPU): pass ``group`` (a torch.distributed process
    group, or "default" for the world group) and a `Problem` whose ``op`` is this
    rank's `parallel.CudaShard`; the run is `parallel.run_solver_distributed`
    (row slabs, one NCCL all-reduce per epoch) and returns the same trace on
    every rank.  A plain BlockOperator with a group of more than one rank raises.
    """
    if kind not in SOLVER_KINDS:
        raise ValueError(f"unknown solver kind {kind!r}; expected one of {SOLVER_KINDS}")
    if sample_every < 1:
        raise ValueError("sample_every must be >= 1")
    if workers < 1:
        raise ValueError("workers must be >= 1")
    if kind != "bsgd":
        raise NotImplementedError(
            f"solver kind {kind!r} is a reference baseline outside this drop-in's scope (SURVEY.md §2 #13)")
    if group is not None:
        from . import parallel
        grp = None if group == "default" else group
        if isinstance(problem.op, BlockOperator):
            import torch.distributed as dist
            if dist.is_initialized() and dist.get_world_size(grp) > 1:
                raise ValueError("multi-GPU run_solver needs this rank's shard (parallel.CudaShard) as problem.op")
        else:
            return parallel.run_solver_distributed(problem, cfg, sample_every, grp, use_graphs=use_graphs,
                                                   chunk_epochs=chunk_epochs)
    op = problem.op
    lam = cfg.lam
    if lam > 0 and problem.layout is None:
        raise ValueError("problem layout required when lam > 0")
    layout = problem.layout
    units0 = op.matvec_units
    trace = ConvergenceTrace()
    state = init_bsgd_state(op, problem.y, cfg)
    y_dev = state._y
    xt_norm = None
    if problem.x_true is not None:
        xt = problem.x_true
        xt_host = xt.detach().cpu().numpy() if hasattr(xt, "detach") else np.asarray(xt, dtype=np.float64)
        xt_norm = float(np.linalg.norm(xt_host))
        if xt_norm == 0.0:
            raise ValueError("reference vector is zero; relative error undefined")
        state._x_true = nat.as_f64(xt, state._dev, op.shape[1])
    monitor = cfg.monitor_decrease or cfg.enforce_decrease
    state._la_policy = True

    # sample at initialisation: x = 0, objective = ||y||^2 (+ 2 lam TV(0) = 0), one charged unit
    units = op.matvec_units - units0
    rel0 = 1.0 if xt_norm is not None else float("nan")
    trace.append(TraceSample(0.0, rel0, state.f_curr, units))
    op._charge(op.nnz)

    full_sweep = cfg.alpha == 1.0 and cfg.gamma == 1.0
    graphs_ok = use_graphs and full_sweep and not cfg.enforce_decrease
    est_epochs = int(math.ceil(cfg.epochs / (1.0 if full_sweep else _pair_fraction(op, cfg)) + 2))
    state._ensure_history(est_epochs + cfg.max_halvings + 4)
    runner = None
    pending = []  # (history row, epoch, sampled, applied-before-sample)
    epoch = 0.0
    next_sample = float(sample_every)

    def charge_epoch_bookkeeping(ep, row, applied_before_epoch):
        nonlocal next_sample
        sampled = ep >= next_sample - 1e-9
        entry = {"row": row, "epoch": ep, "sampled": sampled, "applied_epoch": op._nnz_applied,
                 "units": None}
        if sampled:
            entry["units"] = op.matvec_units - units0
            op._charge(op.nnz)
            next_sample = (math.floor(ep / sample_every + 1e-9) + 1) * sample_every
        pending.append(entry)

    def drain():
        if not pending:
            return None
        hist = state.history(state._rows_used)
        for k, e in enumerate(pending):
            h = hist[e["row"]]
            norm = math.sqrt(h[nat.H_XX]) if h[nat.H_XX] >= 0 else float("nan")
            if monitor:
                trace.decrease_flags.append(bool(h[nat.H_HOLDS] > 0.5))
            if not math.isfinite(norm) or norm > cfg.divergence_limit:
                trace.final_x = None
                with op._lock:  # the reference stops charging at the divergent epoch
                    op._nnz_applied = e["applied_epoch"]
                pending.clear()
                return DivergenceError(
                    f"iterate norm {norm:.3e} left the admissible region at epoch {e['epoch']:.6g}", trace)
            if e["sampled"]:
                rel = math.sqrt(max(h[nat.H_XE], 0.0)) / xt_norm if xt_norm is not None else float("nan")
                obj = float(h[nat.H_FNEXT])
                if lam > 0:
                    obj += 2.0 * lam * float(h[nat.H_TV])
                trace.append(TraceSample(e["epoch"], rel, obj, e["units"]))
        pending.clear()
        return None

    while epoch < cfg.epochs - 1e-9:
        remaining = int(math.ceil(cfg.epochs - epoch - 1e-9)) if full_sweep else 1
        if graphs_ok and state._rows_used >= 1 and remaining >= 2:
            if runner is None:
                runner = _GraphRunner(state, cfg, layout, y_dev, 2)
                if not runner.capture(monitor):
                    graphs_ok = False
                    runner = None
                    continue
            # parity of the captured pair must match the current ring state
            n_pairs = min(remaining // 2, max(1, chunk_epochs // 2))
            for _ in range(n_pairs):
                for _e in range(2):
                    schedule_pairs(op.num_row_blocks, op.num_col_blocks, cfg.alpha, cfg.gamma, state.rng)
                    applied_before = op._nnz_applied
                    op._charge(2 * op.nnz)
                    row = state._rows_used
                    state._rows_used += 1
                    epoch += 1.0
                    state.epoch = epoch
                    charge_epoch_bookkeeping(epoch, row, applied_before)
                runner.replay()
            state._last_row = state._rows_used - 1 if monitor else None
        else:
            applied_before = op._nnz_applied
            bsgd_tv_iteration(state, op, y_dev, cfg, layout=layout)
            epoch = state.epoch
            charge_epoch_bookkeeping(epoch, state._rows_used - 1, applied_before)
        if len(pending) >= chunk_epochs or not (epoch < cfg.epochs - 1e-9):
            err = drain()
            if err is not None:
                raise err
    err = drain()
    if err is not None:
        raise err
    trace.final_x = state.x.copy()
    return trace


def _pair_fraction(op: BlockOperator, cfg: SolverConfig) -> float:
    m, n = op.num_row_blocks, op.num_col_blocks
    return (_round_half_up(cfg.gamma * m) * _round_half_up(cfg.alpha * n)) / (m * n)
