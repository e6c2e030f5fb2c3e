"""Multi-GPU BSGD-TV: row-slab ownership over NCCL (SURVEY.md §8 e).

One process per GPU (torchrun).  Rank p owns a contiguous range of whole row
blocks I_i of the M x N partition (`make_partition`, `blockops.py:96-109`): it
holds A[I_p, :] and its transpose, y[I_p] and its slice of the residual, and a
replicated copy of x.  One epoch (Algorithm 1, `solvers.py:259-341`):

    g_p   = 2 A[I_p,:]^T r[I_p]                 K2 on the local rows   (bsgd_grad)
    g     = sum_p g_p                            NCCL all-reduce, cols doubles
    x'    = prox(x + mu g)                       replicated              (bsgd_step)
    r'[I_p] = y[I_p] - A[I_p,:] x'               K1 on the local rows    (bsgd_epoch_forward)
    f'    = sum_p ||r'[I_p]||^2                  NCCL all-reduce, 1 double
    tail: Eq. 9 test, f_curr, history row        replicated              (bsgd_epoch_tail)

The only exchange of the epoch is the cols-length all-reduce (4 MB at
configs[1]) plus one scalar.  The sums over row blocks become a local sum plus
an all-reduce: same value up to floating-point association, like every other
reduction order change in this path (tolerance parity).

The compute backend is pluggable so the host choreography (ownership,
collectives, bookkeeping) is testable on CPU with the gloo backend; the
production backend is `CudaShard`, which calls the C ABI and fails loudly if
the CUDA library is unavailable.
"""

from __future__ import annotations

import ctypes
import math
import os

import numpy as np

from . import _native as nat
from .blockops import BlockOperator, make_partition


def row_block_ownership(num_row_blocks: int, world: int):
    """Contiguous row-block ranges per rank (near-equal, extra blocks to the first ranks)."""
    if world < 1:
        raise ValueError("world size must be >= 1")
    if world > num_row_blocks:
        raise ValueError(f"{world} ranks cannot own whole blocks of a {num_row_blocks}-row-block partition")
    base, extra = divmod(num_row_blocks, world)
    out, start = [], 0
    for p in range(world):
        stop = start + base + (1 if p < extra else 0)
        out.append((start, stop))
        start = stop
    return out


class ShardSpec:
    """Which rows / row blocks a rank owns.

    ``granularity`` > 1 is for slice-stacked operators (A = A2 (x) I_D,
    granularity D): a rank then owns whole stored rows of A2 (all D slices of
    each), split near-evenly, and its local block bounds are the global row
    blocks clipped to that range (configs[4]'s 16 row blocks are not multiples
    of D, so whole-block ownership would split stored rows).
    """

    def __init__(self, partition, rank: int, world: int, granularity: int = 1):
        self.partition = partition
        self.rank, self.world = rank, world
        self.granularity = granularity
        if granularity <= 1:
            b0, b1 = row_block_ownership(partition.num_row_blocks, world)[rank]
            self.block_range = (b0, b1)
            self.row_range = (partition.row_bounds[b0][0], partition.row_bounds[b1 - 1][1])
            self.local_row_bounds = tuple((a - self.row_range[0], b - self.row_range[0])
                                          for a, b in partition.row_bounds[b0:b1])
            return
        rows = partition.rows
        if rows % granularity:
            raise ValueError(f"{rows} rows are not whole stored rows of granularity {granularity}")
        stored = rows // granularity
        if world > stored:
            raise ValueError(f"{world} ranks cannot own whole rows of a {stored}-row slice matrix")
        base, extra = divmod(stored, world)
        s0 = rank * base + min(rank, extra)
        s1 = s0 + base + (1 if rank < extra else 0)
        r0, r1 = s0 * granularity, s1 * granularity
        self.row_range = (r0, r1)
        blocks = [i for i, (a, b) in enumerate(partition.row_bounds) if a < r1 and b > r0]
        self.block_range = (blocks[0], blocks[-1] + 1)
        self.local_row_bounds = tuple((max(a, r0) - r0, min(b, r1) - r0)
                                      for a, b in partition.row_bounds[blocks[0]:blocks[-1] + 1])

    @property
    def local_rows(self) -> int:
        return self.row_range[1] - self.row_range[0]


class CudaShard:
    """Production backend: the rank's A[I_p, :] resident on its GPU (C ABI)."""

    def __init__(self, matrix, spec: ShardSpec, device=None, lam: float = 0.0, layout=None):
        from scipy import sparse
        r0, r1 = spec.row_range
        full = sparse.csr_array(matrix)
        local = sparse.csr_array(full[r0:r1, :])
        from .blockops import BlockPartition
        part = BlockPartition(spec.local_row_bounds, spec.partition.col_bounds)
        self._finish(spec, BlockOperator(local, part, device=device), full.shape[1], lam, layout)

    @classmethod
    def stacked(cls, slice_matrix, depth: int, spec: ShardSpec, device=None, lam: float = 0.0,
                layout=None) -> "CudaShard":
        """Shard of a slice-stacked operator A2 (x) I_depth: the rank's stored rows of A2."""
        from scipy import sparse
        from .blockops import BlockPartition
        if spec.granularity != depth:
            raise ValueError("a stacked shard needs ShardSpec(..., granularity=depth)")
        a2 = sparse.csr_array(slice_matrix)
        s0, s1 = spec.row_range[0] // depth, spec.row_range[1] // depth
        part = BlockPartition(spec.local_row_bounds, spec.partition.col_bounds)
        self = cls.__new__(cls)
        op = BlockOperator.stacked(sparse.csr_array(a2[s0:s1, :]), depth, part, device=device)
        self._finish(spec, op, a2.shape[1] * depth, lam, layout)
        return self

    def _finish(self, spec, op, cols, lam, layout):
        t = nat.torch()
        self.t = t
        self.spec = spec
        self.op = op
        self.dev = op.device
        self.cols = cols
        self.rows = spec.row_range[1] - spec.row_range[0]
        self.lam = lam
        self.layout = layout
        hw = (layout.height, layout.width) if (lam > 0 and layout is not None) else (0, 0)
        nbytes = int(nat.load().bsgd_epoch_workspace_bytes(op.plan, hw[0], hw[1]))
        self.ws = t.zeros((nbytes + 7) // 8, dtype=t.float64, device=self.dev)
        self.hw = hw

    # tensors
    def zeros(self, n):
        return self.t.zeros(n, dtype=self.t.float64, device=self.dev)

    def vector(self, v):
        return nat.as_f64(v, self.dev)

    def stream(self):
        return nat.stream_ptr(self.dev)

    def args(self, x_k, g, x_next, mu, cfg, f_curr, hist, counter, perm, x_true, flags):
        a = nat.EpochArgs()
        a.x_k, a.g, a.x_next = nat.ptr(x_k), nat.ptr(g), nat.ptr(x_next)
        a.x_true = nat.ptr(x_true) if x_true is not None else None
        a.perm = nat.ptr(perm) if perm is not None else None
        a.mu, a.lam = mu, cfg.lam
        a.height, a.width = self.hw
        a.depth = getattr(self.layout, "depth", 1) if self.hw[0] else 0
        a.max_inner_iters, a.tol = cfg.prox.max_inner_iters, cfg.prox.tol
        a.f_curr, a.history, a.epoch_counter = nat.ptr(f_curr), nat.ptr(hist), nat.ptr(counter)
        a.history_capacity = hist.shape[0]
        a.workspace, a.workspace_bytes = nat.ptr(self.ws), self.ws.numel() * 8
        a.flags = flags
        return a

    # compute ops used by the driver
    def grad(self, r_local, g_out):
        nat.call("bsgd_grad", self.op.plan, nat.ptr(r_local), nat.ptr(g_out), self.stream())

    def step(self, args):
        nat.call("bsgd_step", self.cols, ctypes.byref(args), self.stream())

    def forward(self, x, y_local, r_out, args):
        nat.call("bsgd_epoch_forward", self.op.plan, nat.ptr(x), nat.ptr(y_local), nat.ptr(r_out),
                 ctypes.byref(args), self.stream())

    def forward_sumsq(self, args, out1):
        nat.call("bsgd_epoch_reduce_forward", self.op.plan, ctypes.byref(args), nat.ptr(out1), self.stream())

    def tail(self, args, fnext1):
        nat.call("bsgd_epoch_tail", self.op.plan, ctypes.byref(args), nat.ptr(fnext1), self.stream())

    def dot(self, a, b, out1):
        scratch = self.t.empty(nat.SCRATCH_BYTES // 8, dtype=self.t.float64, device=self.dev)
        nat.call("bsgd_dot", a.numel(), nat.ptr(a), nat.ptr(b), nat.ptr(out1), nat.ptr(scratch), self.stream())

    def matvec(self, x, out):
        nat.call("bsgd_matvec", self.op.plan, nat.ptr(x), nat.ptr(out), self.stream())

    def rmatvec(self, w, out):
        nat.call("bsgd_rmatvec", self.op.plan, nat.ptr(w), nat.ptr(out), self.stream())


class DistributedBSGD:
    """Row-slab BSGD-TV driver (alpha = gamma = 1) over a process group.

    ``shard`` is a backend (CudaShard in production).  History rows use the
    same layout as the single-GPU path (`BSGD_H_*`), replicated on every rank.
    """

    def __init__(self, shard, y_full, cfg, x_true=None, group=None, history_capacity=1024):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.s = shard
        self.cfg = cfg
        r0, r1 = shard.spec.row_range
        y_full = np.asarray(y_full, dtype=np.float64) if not hasattr(y_full, "cpu") else y_full
        self.y = shard.vector(y_full[r0:r1])
        self.x = [shard.zeros(shard.cols), shard.zeros(shard.cols)]
        self.r = [self.y.clone(), self.y.clone()]   # r_0 = y and its lookahead y - A 0
        self.g = shard.zeros(shard.cols)
        self.xi = 0
        self.ri = 0
        self.mu = cfg.mu
        self.epoch = 0.0
        self.rng = np.random.default_rng(cfg.seed)
        self.x_true = shard.vector(x_true) if x_true is not None else None
        self.f_curr = shard.zeros(1)
        part = shard.zeros(1)
        shard.dot(self.y, self.y, part)
        self._allreduce(part)
        self.f_curr.copy_(part)
        self.hist = shard.t.zeros(history_capacity, nat.HIST_COLS, dtype=shard.t.float64, device=self.y.device)
        self.counter = shard.t.zeros(1, dtype=shard.t.int64, device=self.y.device)
        self.rows_used = 0
        self.fnext = shard.zeros(1)
        perm = None
        if cfg.lam > 0 and shard.layout is not None and not shard.layout.is_identity:
            perm = shard.t.from_numpy(shard.layout.perm.astype(np.int64)).to(self.y.device)
        self.perm = perm

    def _allreduce(self, tensor):
        if self.dist.is_initialized() and self.dist.get_world_size(self.group) > 1:
            self.dist.all_reduce(tensor, op=self.dist.ReduceOp.SUM, group=self.group)

    def epoch_step(self, monitor: bool | None = None):
        """One epoch; returns the history row index written."""
        from .solvers import schedule_pairs
        cfg = self.cfg
        s = self.s
        if monitor is None:
            monitor = cfg.monitor_decrease or cfg.enforce_decrease
        schedule_pairs(s.spec.partition.num_row_blocks, s.spec.partition.num_col_blocks, 1.0, 1.0, self.rng)
        xi, ri = self.xi, self.ri
        x_k, x_next = self.x[xi], self.x[1 - xi]
        r_k, r_ahead = self.r[ri], self.r[ri]
        flags = nat.EP_LOOKAHEAD | (nat.EP_MONITOR if monitor else 0)
        args = s.args(x_k, self.g, x_next, self.mu, cfg, self.f_curr, self.hist, self.counter, self.perm,
                      self.x_true, flags)
        s.grad(r_k, self.g)                       # local 2 A_p^T r_p
        self._allreduce(self.g)                   # g = sum_p
        s.step(args)                              # x_next = prox(x_k + mu g), stats
        s.forward(x_next, self.y, r_ahead, args)  # r_{k+2}[I_p] into the consumed r_k slot
        s.forward_sumsq(args, self.fnext)
        self._allreduce(self.fnext)               # f_next = sum_p ||r_p||^2
        s.tail(args, self.fnext)
        row = self.rows_used
        self.rows_used += 1
        self.xi, self.ri = 1 - xi, 1 - ri
        self.epoch += 1.0
        return row

    @property
    def x_current(self):
        return self.x[self.xi]

    @property
    def r_current(self):
        return self.r[self.ri]

    def history(self):
        return self.hist[: self.rows_used].cpu().numpy()


def distributed_largest_eigenvalue(shard, max_iters=50, tol=1e-10, seed=0, group=None):
    """`spectral.largest_eigenvalue` (`spectral.py:43-75`) with row-slab products."""
    import torch.distributed as dist
    t = shard.t

    def allreduce(v):
        if dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.all_reduce(v, op=dist.ReduceOp.SUM, group=group)

    rng = np.random.default_rng(seed)
    cols = shard.cols

    def fresh():
        v0 = rng.standard_normal(cols)
        v0 /= np.linalg.norm(v0)
        return shard.vector(v0)

    v = fresh()
    av = shard.zeros(shard.rows)
    atav = shard.zeros(cols)
    sc = shard.zeros(1)
    nrm = shard.zeros(1)
    est = 0.0
    for k in range(1, max_iters + 1):
        shard.matvec(v, av)
        shard.dot(av, av, sc)
        allreduce(sc)
        shard.rmatvec(av, atav)
        allreduce(atav)
        shard.dot(atav, atav, nrm)
        new, n2 = float(sc.item()), float(nrm.item())
        norm = math.sqrt(n2)
        if norm == 0.0:
            v = fresh()
            continue
        v = atav / norm
        if k > 1 and abs(new - est) <= tol * max(new, 1e-300):
            return new, True, k
        est = new
    return est, False, max_iters
