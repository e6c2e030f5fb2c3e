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
                layout=None, image_shape=None, rays=None) -> "CudaShard":
        """Shard of a slice-stacked operator A2 (x) I_depth: the rank's stored rows of A2.

        ``image_shape`` = (height, width) of A2's columns and ``rays`` =
        (num_angles, num_bins) of its angle-major rows switch on the tile-staged
        products for the shard (`BlockOperator.set_stacked_tiles`): 4 x 4 pixel
        tiles for A2^T, and 4 angles x 4 bins for the rank's rays when they are
        whole angles (else runs of 16 consecutive rays).  Results are unchanged
        bit for bit."""
        from scipy import sparse
        from .blockops import BlockPartition, grid_tiles
        if spec.granularity != depth:
            raise ValueError("a stacked shard needs ShardSpec(..., granularity=depth)")
        a2 = sparse.csr_array(slice_matrix)
        s0, s1 = spec.row_range[0] // depth, spec.row_range[1] // depth
        part = BlockPartition(spec.local_row_bounds, spec.partition.col_bounds)
        self = cls.__new__(cls)
        op = BlockOperator.stacked(sparse.csr_array(a2[s0:s1, :]), depth, part, device=device)
        if image_shape is not None:
            h, w = (int(v) for v in image_shape)
            if h * w != a2.shape[1]:
                raise ValueError("image_shape does not match the slice matrix's columns")
            op.set_stacked_tiles(True, grid_tiles(h, w))
        if rays is not None:
            na, nb = (int(v) for v in rays)
            if na * nb != a2.shape[0]:
                raise ValueError("rays does not match the slice matrix's rows")
            nloc = s1 - s0
            if s0 % nb == 0 and s1 % nb == 0:
                op.set_stacked_tiles(False, grid_tiles(nloc // nb, nb))
            else:
                op.set_stacked_tiles(False, grid_tiles(1, nloc, 1, 16))
        self._finish(spec, op, a2.shape[1] * depth, lam, layout)
        return self

    @classmethod
    def parallel_beam(cls, n: int, num_angles: int, num_bins: int, spec: ShardSpec, dtype=np.float32, device=None,
                      lam: float = 0.0, layout=None, tiles: bool = True) -> "CudaShard":
        """Row-slab shard of the Siddon parallel-beam projector generated on the
        rank's GPU: only the rank's rays are traced (`BlockOperator.from_parallel_beam`
        with an angle range), so no host CSR exists at any size (configs[3]: 1.9e9
        nonzeros over the ranks).  The rank's rows must be whole angles (configs[3]:
        each of the 8 row blocks is 180 angles x 1449 bins).  The shard's A^T is
        a blocked stream gathered in sinogram tiles like the single-GPU operator's."""
        from .blockops import BlockPartition, grid_tiles
        r0, r1 = spec.row_range
        if r0 % num_bins or r1 % num_bins:
            raise ValueError(f"rows [{r0}, {r1}) are not whole angles of {num_bins} bins")
        part = BlockPartition(spec.local_row_bounds, spec.partition.col_bounds)
        op = BlockOperator.from_parallel_beam(n, num_angles, num_bins, dtype=dtype, device=device, tiles=False,
                                              angle_range=(r0 // num_bins, r1 // num_bins), partition=part)
        if tiles:
            op.set_transposed_blocked(((r1 - r0) // num_bins, num_bins))
        self = cls.__new__(cls)
        self._finish(spec, op, n * n, lam, layout)
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

    @property
    def shape(self):
        """Global (rows, cols) of the sharded operator (`Problem` validation)."""
        return (self.spec.partition.rows, self.cols)

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

    def pair_products(self, local_rows, cols_sel, x_k, r_k, y_local, z, g_out, r_next):
        """The selected pairs' products on this rank's row blocks (`bsgd_pair_products`,
        solvers.py:274-303): z cache commit, g = 2 sum_i A_ij^T r_i over the local
        selected row blocks, r_next = y - sum_j z[j].  ``local_rows`` may be empty."""
        rs = np.asarray(local_rows, dtype=np.int64)
        cs = np.asarray(cols_sel, dtype=np.int64)
        nat.call("bsgd_pair_products", self.op.plan, rs.size, rs.ctypes.data if rs.size else None, cs.size,
                 cs.ctypes.data, nat.ptr(x_k), nat.ptr(r_k), nat.ptr(y_local), nat.ptr(z), nat.ptr(g_out),
                 nat.ptr(r_next), self.stream())

    def block_nnz_table(self):
        """nnz of this rank's (local row block, column block) blocks, (local blocks, N)."""
        return np.asarray(self.op._block_nnz, dtype=np.float64)

    def step(self, args):
        nat.call("bsgd_step", self.cols, ctypes.byref(args), self.stream())

    def forward(self, x, y_local, r_out, args):
        nat.call("bsgd_epoch_forward", self.op.plan, nat.ptr(x), nat.ptr(y_local), nat.ptr(r_out),
                 ctypes.byref(args), self.stream())

    def forward_sumsq(self, args, out1):
        nat.call("bsgd_epoch_reduce_forward", self.op.plan, ctypes.byref(args), nat.ptr(out1), self.stream())

    def tail(self, args, fnext1):
        nat.call("bsgd_epoch_tail", self.op.plan, ctypes.byref(args), nat.ptr(fnext1), self.stream())

    def prox_dims(self):
        """(depth, height, width) of the prox volume, or None without a prox."""
        if not self.hw[0]:
            return None
        return (max(1, int(getattr(self.layout, "depth", 1))), self.hw[0], self.hw[1])

    def slab_backend(self, offset, count):
        return CudaSlab(self.prox_dims(), offset, count, self.dev)

    def set_step(self, args, stats, info):
        nat.call("bsgd_epoch_set_step", self.cols, ctypes.byref(args), nat.ptr(stats), float(info["tv"]),
                 info["iterations"], info["restarts"], info["converged"], info["fell_back"], self.stream())

    def dot(self, a, b, out1):
        scratch = self.t.empty(nat.SCRATCH_BYTES // 8, dtype=self.t.float64, device=self.dev)
        nat.call("bsgd_dot", a.numel(), nat.ptr(a), nat.ptr(b), nat.ptr(out1), nat.ptr(scratch), self.stream())

    def matvec(self, x, out):
        nat.call("bsgd_matvec", self.op.plan, nat.ptr(x), nat.ptr(out), self.stream())

    def rmatvec(self, w, out):
        nat.call("bsgd_rmatvec", self.op.plan, nat.ptr(w), nat.ptr(out), self.stream())


def slice_ranges(depth: int, height: int, width: int, world: int):
    """Slices [z0, z1) of each rank for slice ownership: the slab prox's pairwise
    nodes of the slice-major (depth, height, width) volume, which must be whole
    slices (power-of-two volumes and rank counts: equal slice ranges)."""
    hw = height * width
    out = []
    for lo, n in prox_slabs(depth * hw, world, hw):
        if lo % hw or n % hw:
            raise ValueError("the pairwise slabs do not fall on whole slices")
        out.append((lo // hw, (lo + n) // hw))
    return out


class CudaSliceShard(CudaShard):
    """configs[4] by SLICES: A = A2 (x) I_D is block diagonal in the slices, so rank p
    owning slices [z0, z1) holds the stacked operator A2 (x) I_{z1-z0} of its own
    slices and its x, g, r are local -- the products need no exchange at all.
    The only collectives of an epoch are the slab prox's one-plane halos and
    scalar sums (the rank's slices are its prox slab of the slice-major volume,
    `slice_ranges`) and two small all-reduces (step statistics, ||r||^2).

    Local vectors use the interleaved order of the local operator (pixel *
    (z1 - z0) + slice - z0; rays likewise); `local_rows` / `local_cols` cut them
    from the global interleaved vectors.  The block partition is num_blocks x
    num_blocks over the local operator, so products agree with the global
    operator's to rounding (the forward products exactly)."""

    owns_slices = True

    def __init__(self, n: int, num_angles: int, num_bins: int, depth: int, rank: int, world: int,
                 num_blocks: int = 16, dtype=np.float32, device=None, lam: float = 0.0):
        import types

        from . import tv
        if not lam > 0:
            raise ValueError("slice ownership runs the slab-decomposed prox: lam must be positive")
        z0, z1 = slice_ranges(depth, n, n, world)[rank]
        dloc = z1 - z0
        op = BlockOperator.from_parallel_beam(n, num_angles, num_bins, num_blocks, num_blocks, dtype=dtype,
                                              device=device, depth=dloc)
        self.z0, self.z1, self.depth, self.n = z0, z1, depth, n
        self.rays2, self.pix2 = num_angles * num_bins, n * n
        hw = n * n
        self.slab_range = (z0 * hw, dloc * hw)
        rows_l, cols_l = op.shape
        # the global partition (the pair-order RNG advances over its M x N blocks,
        # solvers.py:176-195), with this rank's local rows
        part = make_partition(self.rays2 * depth, hw * depth, num_blocks, num_blocks)
        spec = types.SimpleNamespace(row_range=(0, rows_l), partition=part, rank=rank, world=world)
        self._finish(spec, op, cols_l, lam, tv.VolumeLayout.z_major(dloc, n, n))
        self._global_shape = (self.rays2 * depth, hw * depth)

    @property
    def shape(self):
        return self._global_shape

    def _cut(self, v, m):
        arr = v.detach().cpu().numpy() if hasattr(v, "detach") else np.asarray(v, dtype=np.float64)
        return self.vector(np.ascontiguousarray(arr.reshape(m, self.depth)[:, self.z0:self.z1]).ravel())

    def local_rows(self, y_full):
        return self._cut(y_full, self.rays2)

    def local_cols(self, x_full):
        return self._cut(x_full, self.pix2)

    def prox_dims(self):
        if not self.hw[0]:
            return None
        return (self.depth, self.n, self.n)      # the global slice-major volume

    def slab_backend(self, offset, count):
        if (offset, count) != self.slab_range:
            raise ValueError("slab does not match this rank's slices")
        be = CudaSlab(self.prox_dims(), offset, count, self.dev)
        be.interleaved = True
        return be

    def assemble_cols(self, x_local, group=None):
        """The global interleaved vector from every rank's local one (all-gather)."""
        import torch.distributed as dist
        t = self.t
        xl = x_local.reshape(self.pix2, self.z1 - self.z0)
        if dist.is_initialized() and dist.get_world_size(group) > 1:
            world = dist.get_world_size(group)
            ranges = slice_ranges(self.depth, self.n, self.n, world)
            parts = [t.empty(self.pix2 * (b - a), dtype=t.float64, device=x_local.device) for a, b in ranges]
            dist.all_gather(parts, x_local.contiguous(), group=group)
            cols = [p.reshape(self.pix2, b - a) for p, (a, b) in zip(parts, ranges)]
            return t.cat(cols, dim=1).reshape(-1)
        return xl.reshape(-1)


def ct_row_slab_shard(index: int, rank: int, world: int, device=None, group=None):
    """configs[index] (2-D CT) as this rank's row slab, generated on its GPU.

    Returns (shard, y_full, meta).  y = A x_true + noise is the single-GPU
    instance's (`problems.ct_problem_device`) bit for bit: each rank forms its
    rows of A x_true with the same kernel, the slices are all-gathered (rows
    doubles), and the seeded noise of the full length is drawn on every rank."""
    import torch.distributed as dist
    from . import problems, tv
    name, n, ang, nb, ell, noise_frac, blocks, lam, inner, epochs, dt = problems.CT_TABLE[index]
    t = nat.torch()
    rows, cols = ang * nb, n * n
    spec = ShardSpec(make_partition(rows, cols, blocks, blocks), rank, world)
    layout = tv.PixelLayout.row_major(n, n)
    shard = CudaShard.parallel_beam(n, ang, nb, spec, dtype=dt, device=device, lam=lam, layout=layout)
    x_true = problems.ellipse_phantom(n, ell, 0).ravel()
    clean_local = shard.op.matvec(x_true, charge=False)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        counts = [b - a for a, b in (ShardSpec(spec.partition, p, world).row_range for p in range(world))]
        pieces = [t.empty(c, dtype=t.float64, device=shard.dev) for c in counts]
        dist.all_gather(pieces, shard.vector(clean_local), group=group)
        clean = t.cat(pieces).cpu().numpy()
    else:
        clean = np.asarray(clean_local)
    sigma = noise_frac * float(np.max(clean))
    y = clean + np.random.default_rng(1).standard_normal(rows) * sigma
    meta = {"name": name, "height": n, "width": n, "lam": lam, "max_inner_iters": inner, "epochs": epochs,
            "x_true": x_true, "layout": layout}
    return shard, y, meta


def ct_slice_shard(rank: int, world: int, device=None, group=None, scale: float = 1.0):
    """configs[4] (3-D slice-stacked CT) as this rank's slices, generated on its GPU.

    Returns (shard, y_full, meta); y_full is the global interleaved measurement
    vector of `problems.config_device(4)` bit for bit: each rank forms its
    slices' rows of A x_true with the same kernels (the forward products of a
    slice shard are the global operator's rows exactly), the pieces are
    all-gathered and interleaved, and the seeded noise of the full length is
    drawn on every rank."""
    import torch.distributed as dist
    from . import problems
    t = nat.torch()
    n = max(16, int(round(256 * scale)))
    depth = max(2, int(round(256 * scale)))
    ang = max(8, int(round(360 * scale)))
    nb = max(9, int(round(363 * scale)) | 1)
    lam, inner, blocks, noise_frac = 0.01, 10, 16, 0.01
    shard = CudaSliceShard(n, ang, nb, depth, rank, world, num_blocks=blocks, device=device, lam=lam)
    vol = problems.ellipsoid_phantom(n, depth, 40, 0)
    x_true = np.ascontiguousarray(vol.reshape(depth, n * n).T).ravel()
    clean_l = shard.op.matvec(shard.local_cols(x_true), charge=False)
    rays = ang * nb
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        ranges = slice_ranges(depth, n, n, world)
        parts = [t.empty(rays * (b - a), dtype=t.float64, device=shard.dev) for a, b in ranges]
        dist.all_gather(parts, shard.vector(clean_l), group=group)
        clean = t.cat([p.reshape(rays, b - a) for p, (a, b) in zip(parts, ranges)], dim=1).reshape(-1).cpu().numpy()
    else:
        clean = clean_l.cpu().numpy() if hasattr(clean_l, "cpu") else np.asarray(clean_l)
    sigma = noise_frac * float(np.max(clean))
    y = clean + np.random.default_rng(1).standard_normal(clean.shape[0]) * sigma
    from . import tv
    meta = {"n": n, "depth": depth, "lam": lam, "max_inner_iters": inner, "x_true": x_true,
            "layout": tv.VolumeLayout(depth, n, n, problems.interleaved_perm(n * n, depth))}
    return shard, y, meta


SLAB_PROX_MIN_VOXELS = 1 << 22   # prox="auto" decomposes volumes from this size on


class DistributedBSGD:
    """Row-slab BSGD-TV driver over a process group.

    ``shard`` is a backend (CudaShard in production).  History rows use the
    same layout as the single-GPU path (`BSGD_H_*`), replicated on every rank.
    ``cfg.enforce_decrease`` (solvers.py:325-333) is honoured with the replicated
    prox: an epoch then reduces its f_next at once, every rank reads the Eq. 9
    flag and, while it fails, halves mu and repeats the step and the forward
    product (`_epoch_enforce`; one host read per attempt, no graph capture).
    alpha, gamma < 1 (solvers.py:186-195) run `_epoch_stochastic`: each rank commits
    the selected pairs of its own row blocks to its z cache; eager, replicated prox.
    """

    def __init__(self, shard, y_full, cfg, x_true=None, group=None, history_capacity=1024, prox: str = "auto",
                 device_decisions: bool = True):
        """``prox``: "replicated" runs the whole prox on every rank (bsgd_step);
        "slab" decomposes it over the ranks (SlabProx; needs an identity layout
        and slabs at least one halo plane thick); "auto" takes "slab" on more
        than one rank when it applies and the volume has at least
        SLAB_PROX_MIN_VOXELS voxels (configs[4]'s 256^3), "replicated" otherwise.
        ``device_decisions``: the slab prox takes its FGP decisions on the device
        (`SlabProx.run_device`, a fixed sequence with no host round trip, so the
        epoch can be captured in a CUDA graph) when the backend supports it;
        False keeps the host loop (`SlabProx.run`, only the iterations taken)."""
        import torch.distributed as dist
        self.stochastic = cfg.alpha != 1.0 or cfg.gamma != 1.0
        if self.stochastic and (getattr(shard, "owns_slices", False) or not hasattr(shard, "pair_products")):
            raise ValueError("the stochastic pair subsets (alpha, gamma < 1; solvers.py:186-195) run on row-slab "
                             "shards only")
        self.dist = dist
        self.group = group
        self.s = shard
        self.cfg = cfg
        r0, r1 = shard.spec.row_range
        y_full = np.asarray(y_full, dtype=np.float64) if not hasattr(y_full, "cpu") else y_full
        self.slices = getattr(shard, "owns_slices", False)   # configs[4] by slices: x, g, r all local
        if self.slices and (cfg.lam <= 0 or prox == "replicated"):
            raise ValueError("slice ownership needs lam > 0 and the slab prox (its g and x are local)")
        self.y = shard.local_rows(y_full) if self.slices else shard.vector(y_full[r0:r1])
        self.x = [shard.zeros(shard.cols), shard.zeros(shard.cols)]
        self.r = [self.y.clone(), self.y.clone()]   # r_0 = y and its lookahead y - A 0
        # g and, in its last slot, this rank's ||r||^2 of the previous epoch: one
        # all-reduce per epoch carries both (the previous epoch's tail runs after it)
        self._gbuf = shard.zeros(shard.cols + 1)
        self.g = self._gbuf[:shard.cols]
        self._fslot = self._gbuf[shard.cols:]
        self._pending = None        # args of the epoch whose tail waits for the next all-reduce
        self.xi = 0
        self.ri = 0
        self.mu = cfg.mu
        self.epoch = 0.0
        self.rng = np.random.default_rng(cfg.seed)
        if x_true is not None:
            self.x_true = shard.local_cols(x_true) if self.slices else shard.vector(x_true)
        else:
            self.x_true = None
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
        self.slab = None
        self.slabs = None
        self.slab_device = False
        self._graph = None
        self._graph_epochs = 0
        if prox not in ("auto", "slab", "replicated"):
            raise ValueError(f"unknown prox mode {prox!r}")
        dims = shard.prox_dims() if (cfg.lam > 0 and hasattr(shard, "prox_dims")) else None
        if dims is not None and prox != "replicated":
            comm = TorchComm(group)
            why = None
            if not shard.layout.is_identity:
                why = "slab prox needs an identity pixel layout"
            else:
                try:
                    slabs = prox_slabs(int(np.prod(dims)), comm.world, dims[1] * dims[2] if dims[0] > 1 else dims[2])
                except ValueError as e:
                    why = str(e)
            # "auto" decomposes only large volumes: the slab prox takes its FGP decisions
            # on the host (a gather and halo exchanges per pass), which costs more than
            # running a small prox redundantly on every rank (1024^2: ~0.13 ms per epoch)
            big = int(np.prod(dims)) >= SLAB_PROX_MIN_VOXELS
            if self.slices and why is None and slabs[comm.rank] != shard.slab_range:
                why = "the slice shard's slices are not this rank's prox slab"
            if self.slices and why is not None:
                raise ValueError(why)
            if why is None and (prox == "slab" or self.slices or (comm.world > 1 and big)):
                lo, n = slabs[comm.rank]
                self.slab = SlabProx(shard.slab_backend(lo, n), comm, slabs)
                self.slabs = slabs
                self.comm = comm
                # device decisions (graph-capturable) when the backend supports them
                self.slab_device = device_decisions and hasattr(self.slab.be, "decide")
            elif prox == "slab":
                raise ValueError(why or "slab prox unavailable")
        elif prox == "slab":
            raise ValueError("slab prox needs lam > 0 and a layout")
        self.prox_info = None
        if cfg.enforce_decrease and self.slab is not None:
            raise ValueError("enforce_decrease (solvers.py:325-333) needs the replicated prox: the slab prox "
                             "does not repeat a step with a halved mu")
        if self.stochastic:
            if self.slab is not None:
                raise ValueError("the stochastic pair subsets (alpha, gamma < 1) need the replicated prox")
            sp = shard.spec.partition
            # z cache of this rank's rows (solvers.py:228: zeros) and a scratch residual
            # for the monitor's / the samples' fidelity product
            self.z = shard.zeros(sp.num_col_blocks * shard.rows)
            self.r_fid = shard.zeros(shard.rows)
            # global block nnz (matvec units of the selected pairs, blockops.py:195-203)
            table = shard.t.zeros(sp.num_row_blocks, sp.num_col_blocks, dtype=shard.t.float64, device=self.y.device)
            b0, b1 = shard.spec.block_range
            table[b0:b1] += shard.t.as_tensor(shard.block_nnz_table(), dtype=shard.t.float64).to(self.y.device)
            self._allreduce(table)
            self.block_nnz = table.cpu().numpy().round().astype(np.int64)
        self.last_pairs = None

    def _allreduce(self, tensor):
        if self.dist.is_initialized() and self.dist.get_world_size(self.group) > 1:
            self.dist.all_reduce(tensor, op=self.dist.ReduceOp.SUM, group=self.group)

    def _schedule(self):
        """Draw the epoch's pairs exactly as the reference does (solvers.py:176-195); with
        alpha = gamma = 1 only the RNG advance matters."""
        from .solvers import schedule_pairs
        sp = self.s.spec.partition
        self.last_pairs = schedule_pairs(sp.num_row_blocks, sp.num_col_blocks, self.cfg.alpha, self.cfg.gamma,
                                         self.rng)
        return self.last_pairs

    def _ensure_history(self, extra: int) -> bool:
        """Grow the history table so ``extra`` more rows fit (the tail kernel skips
        rows past the capacity).  Returns True when it was reallocated, which
        voids a captured graph (it holds the old table's address)."""
        need = self.rows_used + extra
        cap = self.hist.shape[0]
        if need <= cap:
            return False
        t = self.s.t
        new = t.zeros(max(need, 2 * cap), self.hist.shape[1], dtype=self.hist.dtype, device=self.hist.device)
        new[:cap].copy_(self.hist)
        self.hist = new
        self._graph = None
        return True

    def epoch_step(self, monitor: bool | None = None):
        """One epoch; returns the history row index written."""
        self._ensure_history(1)
        pairs = self._schedule()
        if self.stochastic:
            return self._epoch_stochastic(pairs, monitor)
        return self._epoch(monitor)

    def capture(self, epochs: int = 2, monitor: bool | None = None) -> bool:
        """Capture ``epochs`` (even: the x / r rings flip every epoch) epochs,
        collectives included, into one CUDA graph for `replay`.  Needs the
        collectives warmed up by at least one eager epoch; with the slab prox
        only when its FGP decisions are on the device (``device_decisions``).  Returns
        whether a graph is ready."""
        if (self.slab is not None and not self.slab_device) or epochs < 2 or epochs % 2 or \
                not getattr(self.y, "is_cuda", False) or self.cfg.enforce_decrease or self.stochastic:
            return False
        d = self.dist
        if d.is_initialized() and d.get_world_size(self.group) > 1 and d.get_backend(self.group) != "nccl":
            return False   # gloo stages device tensors through the host: not capturable
        t = self.s.t
        saved = (self.xi, self.ri, self.rows_used, self.epoch)
        g = t.cuda.CUDAGraph()
        try:
            side = t.cuda.Stream(device=self.y.device)
            side.wait_stream(t.cuda.current_stream(self.y.device))
            with t.cuda.graph(g, stream=side):
                for _ in range(epochs):
                    self._epoch(monitor)
        except Exception:
            self._graph = None
            return False
        finally:
            self.xi, self.ri, self.rows_used, self.epoch = saved
        self._graph = g
        self._graph_epochs = epochs
        self._graph_parity = saved[:2]
        return True

    def replay(self):
        """Run the captured epochs (same arithmetic as `epoch_step`, one launch).
        When the history table is full it is grown and the graph re-captured."""
        if self.slab is None and self._pending is None:
            raise RuntimeError("the graph starts with the previous epoch's tail, which flush() / history() "
                               "already ran: take one eager epoch_step() before replaying")
        # the graph holds the x / r ring buffers of the parity it was captured at
        stale = self._graph is not None and (self.xi, self.ri) != self._graph_parity
        if self._ensure_history(self._graph_epochs) or self._graph is None or stale:
            k = self._graph_epochs
            if not self.capture(k):
                raise RuntimeError("CUDA graph re-capture failed after growing the history table")
        for _ in range(self._graph_epochs):
            self._schedule()
        self._graph.replay()
        self.rows_used += self._graph_epochs
        self.epoch += float(self._graph_epochs)

    def _epoch(self, monitor: bool | None = None):
        cfg = self.cfg
        s = self.s
        if monitor is None:
            monitor = cfg.monitor_decrease or cfg.enforce_decrease
        if cfg.enforce_decrease:
            return self._epoch_enforce()
        xi, ri = self.xi, self.ri
        x_k, x_next = self.x[xi], self.x[1 - xi]
        r_k, r_ahead = self.r[ri], self.r[ri]
        flags = nat.EP_LOOKAHEAD | (nat.EP_MONITOR if monitor else 0)
        args = s.args(x_k, self.g, x_next, self.mu, cfg, self.f_curr, self.hist, self.counter, self.perm,
                      self.x_true, flags)
        s.grad(r_k, self.g)                       # local 2 A_p^T r_p
        if self.slab is None:
            # one collective per epoch: [g | ||r_prev||^2] summed over the ranks, then
            # the previous epoch's tail (Eq. 9 test, f_curr, history row) -- it reads
            # only the statistics of its own step, which this epoch's step overwrites next
            self._allreduce(self._gbuf)
            if self._pending is not None:
                s.tail(self._pending, self._fslot)
            s.step(args)                          # x_next = prox(x_k + mu g), stats
            s.forward(x_next, self.y, r_ahead, args)  # r_{k+2}[I_p] into the consumed r_k slot
            s.forward_sumsq(args, self._fslot)    # this rank's ||r||^2, reduced with the next g
            self._pending = args
        else:
            self._slab_step(args, x_k, x_next)
            s.forward(x_next, self.y, r_ahead, args)
            s.forward_sumsq(args, self.fnext)
            self._allreduce(self.fnext)           # f_next = sum_p ||r_p||^2
            s.tail(args, self.fnext)
        row = self.rows_used
        self.rows_used += 1
        self.xi, self.ri = 1 - xi, 1 - ri
        self.epoch += 1.0
        return row

    def _epoch_stochastic(self, pairs, monitor: bool | None = None):
        """One iteration over a pair subset (alpha, gamma < 1; solvers.py:274-334): this
        rank commits the selected pairs of its own row blocks to its z cache, rebuilds
        its residual rows from the cache and contributes g = 2 sum_i A_ij^T r_i over
        them; one all-reduce gives g, the step and the prox run replicated, and the
        fidelity of x_next (the monitor's uncharged product, also the samples'
        objective) is reduced in the same epoch.  With enforce_decrease the step is
        repeated with mu halved like `_epoch_enforce`."""
        cfg, s = self.cfg, self.s
        if monitor is None:
            monitor = cfg.monitor_decrease or cfg.enforce_decrease
        sp = s.spec.partition
        b0, b1 = s.spec.block_range
        rows_sel = sorted({i for i, _ in pairs})
        cols_sel = sorted({j for _, j in pairs})
        xi, ri = self.xi, self.ri
        x_k, x_next = self.x[xi], self.x[1 - xi]
        r_k, r_next = self.r[ri], self.r[1 - ri]
        s.pair_products([i - b0 for i in rows_sel if b0 <= i < b1], cols_sel, x_k, r_k, self.y, self.z, self.g,
                        r_next)
        self._fslot.zero_()
        self._allreduce(self._gbuf)
        flags = nat.EP_MONITOR if monitor else 0
        f_before = self.f_curr.clone() if cfg.enforce_decrease else None
        row = self.rows_used
        mu, halvings = self.mu, 0
        while True:
            args = s.args(x_k, self.g, x_next, mu, cfg, self.f_curr, self.hist, self.counter, self.perm,
                          self.x_true, flags)
            s.step(args)
            s.forward(x_next, self.y, self.r_fid, args)
            s.forward_sumsq(args, self.fnext)
            self._allreduce(self.fnext)
            s.tail(args, self.fnext)
            if not cfg.enforce_decrease:
                break
            holds = float(self.hist[row, nat.H_HOLDS].item()) > 0.5
            if holds or halvings >= cfg.max_halvings:
                break
            mu *= 0.5
            halvings += 1
            self.f_curr.copy_(f_before)
            self.counter.fill_(row)
        self.mu = mu
        self.rows_used += 1
        self.xi, self.ri = 1 - xi, 1 - ri
        self.epoch += len(pairs) / (sp.num_row_blocks * sp.num_col_blocks)
        return row

    def _epoch_enforce(self):
        """One epoch with the enforced two-point decrease (solvers.py:316-334): the
        gradient is reduced once; the step, the prox and the forward product of
        x_next are repeated with mu halved until Eq. 9 holds or max_halvings is
        reached.  f_next is reduced in the epoch itself (no lagged tail) and every
        rank reads the same flag from its replicated history row, so the ranks take
        the same number of attempts.  mu stays halved for the following epochs."""
        cfg, s = self.cfg, self.s
        xi, ri = self.xi, self.ri
        x_k, x_next = self.x[xi], self.x[1 - xi]
        r_k, r_ahead = self.r[ri], self.r[ri]
        flags = nat.EP_LOOKAHEAD | nat.EP_MONITOR
        s.grad(r_k, self.g)
        self._fslot.zero_()
        self._allreduce(self._gbuf)
        f_before = self.f_curr.clone()
        row = self.rows_used
        mu, halvings = self.mu, 0
        while True:
            args = s.args(x_k, self.g, x_next, mu, cfg, self.f_curr, self.hist, self.counter, self.perm,
                          self.x_true, flags)
            s.step(args)
            s.forward(x_next, self.y, r_ahead, args)
            s.forward_sumsq(args, self.fnext)
            self._allreduce(self.fnext)
            s.tail(args, self.fnext)
            holds = float(self.hist[row, nat.H_HOLDS].item()) > 0.5
            if holds or halvings >= cfg.max_halvings:
                break
            mu *= 0.5
            halvings += 1
            self.f_curr.copy_(f_before)
            self.counter.fill_(row)
        self.mu = mu
        self.rows_used += 1
        self.xi, self.ri = 1 - xi, 1 - ri
        self.epoch += 1.0
        return row

    def _slab_step(self, args, x_k, x_next):
        """x_next = prox(x_k + mu g) with the prox decomposed over the ranks."""
        cfg = self.cfg
        comm, slabs, be = self.comm, self.slabs, self.slab.be
        if not self.slices:                       # slice ownership: g is already this rank's, complete
            comm.reduce_scatter(self.g, slabs)    # this rank's share of g = sum_p g_p
        be.step(x_k, self.g, self.mu)             # b = x_k + mu g on the slab
        if self.slab_device:                      # decisions on the device: no host round trip
            self.slab.run_device(self.mu * cfg.lam, cfg.prox.max_inner_iters, cfg.prox.tol)
            stats = be.output(False, x_next, x_k, self.g, self.x_true)
            comm.allreduce(stats)
            be.set_step_device(self.s, args, stats)
            if not self.slices:                   # the next forward product reads all of x
                comm.allgather_slabs(x_next, slabs)
            self.prox_info = None
            return
        info = self.slab.run(self.mu * cfg.lam, cfg.prox.max_inner_iters, cfg.prox.tol)
        stats = be.output(info["fell_back"], x_next, x_k, self.g, self.x_true)
        comm.allreduce(stats)
        self.s.set_step(args, stats, info)
        if not self.slices:
            comm.allgather_slabs(x_next, slabs)   # the next forward product reads all of x
        self.prox_info = info

    @property
    def x_current(self):
        return self.x[self.xi]

    @property
    def r_current(self):
        return self.r[self.ri]

    def flush(self):
        """Run the tail still waiting for the next epoch's all-reduce (history rows,
        f_curr and the Eq. 9 flag of the last epoch become current)."""
        if self._pending is not None:
            self._allreduce(self._fslot)
            self.s.tail(self._pending, self._fslot)
            self._pending = None

    def history(self):
        self.flush()
        return self.hist[: self.rows_used].cpu().numpy()


def run_solver_distributed(problem, cfg, sample_every: int = 1, group=None, *, use_graphs: bool = True,
                           chunk_epochs: int = 64, prox: str = "auto"):
    """`run_solver('bsgd', ...)` (`solvers.py:445-533`) over a process group: every
    rank passes a `Problem` whose ``op`` is its shard (`CudaShard`) and whose y,
    x_true and layout are the full ones.  Samples (epoch, relative error,
    objective, matvec units), decrease flags and the `DivergenceError` follow
    the single-GPU `solvers.run_solver` exactly; the units are charged against
    the global nonzero count.  alpha, gamma < 1 and enforce_decrease run eagerly
    with the replicated prox (see `DistributedBSGD`)."""
    import torch.distributed as dist

    from .solvers import ConvergenceTrace, DivergenceError, TraceSample
    if sample_every < 1:
        raise ValueError("sample_every must be >= 1")
    shard = problem.op
    lam = cfg.lam
    if lam > 0 and problem.layout is None:
        raise ValueError("problem layout required when lam > 0")
    if lam > 0 and shard.layout is None:
        raise ValueError("the shard was built without the pixel layout the prox needs")
    epochs = int(math.ceil(cfg.epochs - 1e-9))
    xt_norm = None
    if problem.x_true is not None:
        xt = problem.x_true
        xt_host = xt.detach().cpu().numpy() if hasattr(xt, "detach") else np.asarray(xt, dtype=np.float64)
        xt_norm = float(np.linalg.norm(xt_host))
        if xt_norm == 0.0:
            raise ValueError("reference vector is zero; relative error undefined")
    drv = DistributedBSGD(shard, problem.y, cfg, x_true=problem.x_true, group=group,
                          history_capacity=epochs + 8, prox=prox)
    nnz = shard.zeros(1)
    nnz.fill_(float(shard.op.nnz))
    drv._allreduce(nnz)
    nnz_total = int(round(float(nnz.item())))
    monitor = cfg.monitor_decrease or cfg.enforce_decrease
    trace = ConvergenceTrace()
    applied = 0                                   # nonzeros charged since the start (integer, as the reference)

    def units():
        return applied / nnz_total

    trace.append(TraceSample(0.0, 1.0 if xt_norm is not None else float("nan"), float(drv.f_curr.item()), units()))
    applied += nnz_total                          # the sample's objective evaluation is charged
    pending = []                                  # (history row, epoch, sampled, units at the sample)
    next_sample = float(sample_every)
    done = 0

    def book(ep, row=None, charged=None):
        nonlocal applied, next_sample
        # one A^T and one A product per full sweep; the selected blocks' for a pair subset
        applied += 2 * nnz_total if charged is None else charged
        sampled = ep >= next_sample - 1e-9
        u = None
        if sampled:
            u = units()
            applied += nnz_total
            next_sample = (math.floor(ep / sample_every + 1e-9) + 1) * sample_every
        # history row: epoch ep of a full-sweep run wrote row ep - 1 (rows from 0)
        pending.append((int(round(ep)) - 1 if row is None else row, ep, sampled, u))

    def drain():
        hist = drv.history()
        for row, ep, sampled, u in pending:
            h = hist[row]
            norm = math.sqrt(h[nat.H_XX]) if h[nat.H_XX] >= 0 else float("nan")
            if monitor:
                trace.decrease_flags.append(bool(h[nat.H_HOLDS] > 0.5))
            if not math.isfinite(norm) or norm > cfg.divergence_limit:
                trace.final_x = None
                pending.clear()
                return DivergenceError(f"iterate norm {norm:.3e} left the admissible region at epoch {ep:.6g}",
                                       trace)
            if sampled:
                rel = math.sqrt(max(h[nat.H_XE], 0.0)) / xt_norm if xt_norm is not None else float("nan")
                obj = float(h[nat.H_FNEXT])
                if lam > 0:
                    obj += 2.0 * lam * float(h[nat.H_TV])
                trace.append(TraceSample(ep, rel, obj, u))
        pending.clear()
        return None

    graphed = False
    if cfg.enforce_decrease:
        use_graphs = False                        # the halving loop reads a flag per attempt
    while drv.stochastic and drv.epoch < cfg.epochs - 1e-9:
        row = drv.epoch_step()                    # a pair subset: a fraction of an epoch, eager
        book(drv.epoch, row, 2 * int(sum(drv.block_nnz[i, j] for i, j in drv.last_pairs)))
        if len(pending) >= chunk_epochs:
            err = drain()
            if err is not None:
                raise err
    if drv.stochastic:
        done = epochs
    while done < epochs:
        if use_graphs and (drv.slab is None or drv.slab_device) and done >= 1 and epochs - done >= 2:
            if not graphed:
                graphed = drv.capture(2)
                if not graphed:
                    use_graphs = False
                    continue
            if drv._pending is None:              # flushed by the last drain: two eager epochs first
                for _ in range(2):                # (an even count keeps the captured ring parity)
                    drv.epoch_step()
                    done += 1
                    book(float(done))
                continue
            drv.replay()
            for _ in range(2):
                done += 1
                book(float(done))
        else:
            drv.epoch_step()
            done += 1
            book(float(done))
        if len(pending) >= chunk_epochs or done >= epochs:
            err = drain()
            if err is not None:
                raise err
    err = drain()
    if err is not None:
        raise err
    xf = drv.x_current
    if getattr(shard, "owns_slices", False):
        xf = shard.assemble_cols(xf, group)
    trace.final_x = xf.cpu().numpy().copy()
    if dist.is_initialized():
        dist.barrier(group=group)
    return trace


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


# ---------------------------------------------------------------------------
# slab-decomposed TV prox (SURVEY.md §8 e, "Prox")
# ---------------------------------------------------------------------------
#
# With the replicated prox every rank runs the whole FGP; here rank p runs it
# on its own voxels only.  Slabs are contiguous voxel ranges of the C-order
# volume chosen as nodes of numpy's pairwise recursion over the whole volume
# (`prox_slabs`), so the per-slab numpy-order sums combine in the recursion's
# order (`pw_combine`) into exactly the values np.sum gives: every restart,
# stop and fallback decision, and the result, are bit-identical to the
# single-GPU prox (tv.py:172-255; 3-D: the oracle restatement).  Per FGP
# iteration the exchange is one halo plane per neighbour for q and for c and
# one all-gather of 1 + 2 DIM doubles.  The step x_k + mu g needs only the
# rank's share of g (reduce-scatter instead of all-reduce) and the new x is
# all-gathered for the next forward product.

def _pw_split(n: int) -> int:
    n2 = n // 2
    return n2 - n2 % 8


def prox_slabs(nvox: int, world: int, halo: int):
    """Own voxel ranges (lo, count) per rank: nodes of numpy's pairwise recursion.

    Starting from the root, the largest node (leftmost on ties) is split at
    numpy's split point until there are ``world`` of them; for power-of-two
    volumes and rank counts these are equal slabs.  Raises ValueError when a
    node would have to split inside a pairwise leaf or a slab is thinner than
    one halo plane (the exchange only reaches neighbouring ranks)."""
    if world < 1:
        raise ValueError("world size must be >= 1")
    nodes = [(0, nvox)]
    while len(nodes) < world:
        k = max(range(len(nodes)), key=lambda i: (nodes[i][1], -i))
        lo, n = nodes[k]
        if n <= 128:
            raise ValueError(f"cannot split a {nvox}-voxel volume into {world} pairwise nodes")
        n2 = _pw_split(n)
        nodes[k:k + 1] = [(lo, n2), (lo + n2, n - n2)]
    if world > 1 and min(n for _, n in nodes) < halo:
        raise ValueError(f"slabs of {min(n for _, n in nodes)} voxels are thinner than the {halo}-voxel halo")
    return nodes


def pw_combine(nvox: int, slabs, values):
    """Combine per-slab numpy-order sums (one K-list per slab, slab order) into
    np.sum's values over the whole volume by walking numpy's recursion."""
    index = {tuple(s): i for i, s in enumerate(slabs)}

    def rec(lo, n):
        i = index.get((lo, n))
        if i is not None:
            return [float(v) for v in values[i]]
        if n <= 128:
            raise ValueError("slab boundary inside a pairwise leaf")
        n2 = _pw_split(n)
        a, b = rec(lo, n2), rec(lo + n2, n - n2)
        return [x + y for x, y in zip(a, b)]

    return rec(0, nvox)


def slab_program(nvox: int, slabs):
    """The postfix program of `pw_combine` for `bsgd_slab_decide`: op >= 0 pushes
    rank op's sums, -1 adds the top two (left + right), walking numpy's
    recursion from the root exactly as pw_combine does."""
    index = {tuple(s): i for i, s in enumerate(slabs)}
    prog = []

    def rec(lo, n):
        i = index.get((lo, n))
        if i is not None:
            prog.append(i)
            return
        if n <= 128:
            raise ValueError("slab boundary inside a pairwise leaf")
        n2 = _pw_split(n)
        rec(lo, n2)
        rec(lo + n2, n - n2)
        prog.append(-1)

    rec(0, nvox)
    return prog


class TorchComm:
    """Halo / gather / reduce exchanges of the slab prox over torch.distributed
    (NCCL in production, gloo in the CPU tests)."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist
        self.torch = torch
        self.dist = dist
        self.group = group
        self.active = dist.is_initialized()
        self.rank = dist.get_rank(group) if self.active else 0
        self.world = dist.get_world_size(group) if self.active else 1
        self.nccl = self.active and dist.get_backend(group) == "nccl"

    def _peer(self, r):
        return self.dist.get_global_rank(self.group, r) if self.group is not None else r

    def halo(self, bufs, n: int, h: int, lower: bool = True, upper: bool = True):
        """Fill the halos of local buffers laid out [h halo | n own | h halo]:
        ``lower`` receives the previous rank's last h own values, ``upper`` the
        next rank's first h."""
        if self.world == 1:
            return
        d = self.dist
        # gloo moves host memory only: device buffers are staged through the host
        # there (the functional multi-rank checks); NCCL sends device memory directly
        staged = not self.nccl and any(b.is_cuda for b in bufs)
        ops, back = [], []

        def send(t, peer):
            ops.append(d.P2POp(d.isend, t.cpu() if staged else t, peer, self.group))

        def recv(t, peer):
            if staged:
                tmp = self.torch.empty(t.shape, dtype=t.dtype)
                back.append((t, tmp))
                t = tmp
            ops.append(d.P2POp(d.irecv, t, peer, self.group))

        for b in bufs:
            if lower:
                if self.rank + 1 < self.world:
                    send(b[n:n + h], self._peer(self.rank + 1))
                if self.rank > 0:
                    recv(b[0:h], self._peer(self.rank - 1))
            if upper:
                if self.rank > 0:
                    send(b[h:2 * h], self._peer(self.rank - 1))
                if self.rank + 1 < self.world:
                    recv(b[n + h:n + 2 * h], self._peer(self.rank + 1))
        if ops:
            for req in d.batch_isend_irecv(ops):
                req.wait()
        for t, tmp in back:
            t.copy_(tmp)

    def gather(self, t):
        """All ranks' copies of a small tensor, as a host array [world, len]."""
        if self.world == 1:
            return t.cpu().numpy()[None, :]
        out = [self.torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t.contiguous(), group=self.group)
        return np.stack([o.cpu().numpy() for o in out])

    def gather_flat(self, t):
        """All ranks' copies of a small tensor, rank-major in one tensor on t's
        device (no host round trip: graph-capturable with NCCL)."""
        if self.world == 1:
            return t.contiguous()
        if self.nccl:
            out = self.torch.empty(self.world * t.numel(), dtype=t.dtype, device=t.device)
            self.dist.all_gather_into_tensor(out, t.contiguous(), group=self.group)
            return out
        parts = [self.torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(parts, t.contiguous(), group=self.group)
        return self.torch.cat(parts)

    def allreduce(self, t):
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)

    def reduce_scatter(self, full, slabs):
        """Sum ``full`` over ranks; at least this rank's slab ends up correct."""
        if self.world == 1:
            return
        lo, n = slabs[self.rank]
        if self.nccl and len({c for _, c in slabs}) == 1:
            out = self.torch.empty(n, dtype=full.dtype, device=full.device)
            self.dist.reduce_scatter_tensor(out, full, op=self.dist.ReduceOp.SUM, group=self.group)
            full[lo:lo + n].copy_(out)
        else:
            self.allreduce(full)

    def allgather_slabs(self, full, slabs):
        """Every rank's own slab of ``full`` into everyone's copy."""
        if self.world == 1:
            return
        lo, n = slabs[self.rank]
        if self.nccl and len({c for _, c in slabs}) == 1:
            self.dist.all_gather_into_tensor(full, full[lo:lo + n].clone(), group=self.group)
            return
        for r, (a, c) in enumerate(slabs):
            self.dist.broadcast(full[a:a + c], self._peer(r), group=self.group)


class CudaSlab:
    """The rank's slab of the prox on its GPU (bsgd_slab_* in the C ABI)."""

    def __init__(self, dims, offset: int, count: int, device=None):
        t = nat.torch()
        self.t = t
        self.dev = device if device is not None else nat.require_cuda()
        self.dims = tuple(int(v) for v in dims)
        depth, height, width = self.dims
        self.dim = 3 if depth > 1 else 2
        self.nvox = depth * height * width
        self.offset, self.count = int(offset), int(count)
        lib = nat.load()
        nbytes = int(lib.bsgd_slab_workspace_bytes(depth, height, width, count))
        self.ws = t.zeros((nbytes + 7) // 8, dtype=t.float64, device=self.dev)
        offs = (ctypes.c_int64 * nat.SLAB_SLOTS)()
        halo = ctypes.c_int64()
        nat.call("bsgd_slab_layout", depth, height, width, count, offs, ctypes.byref(halo))
        self.halo = int(halo.value)
        length = count + 2 * self.halo
        self._buf = {k: self.ws[o:o + length] for k, o in enumerate(offs[:11]) if o >= 0}
        self._sums = self.ws[offs[11]:offs[11] + 16]
        self._stats = self.ws[offs[11] + 16:offs[11] + 20]
        self.args = nat.SlabArgs(depth, height, width, offset, count, 0.0, 0, 0, nat.ptr(self.ws), self.ws.numel() * 8)
        self.parity = 0
        self.device = False   # True: FGP decisions in the workspace's control block (bsgd_slab_decide)
        self.interleaved = False   # True: step / output vectors are this rank's slices, interleaved

    def _a(self, when: int = 0):
        self.args.parity = self.parity
        flags = (nat.SLAB_DEVICE | (when << 1)) if self.device else 0
        if self.interleaved:
            flags |= nat.SLAB_INTERLEAVED
        self.args.flags = flags
        return ctypes.byref(self.args)

    def _st(self):
        return nat.stream_ptr(self.dev)

    def set_weight(self, w: float):
        self.args.weight = float(w)

    def fields(self, name: str):
        d = self.dim
        if name == "b":
            return [self._buf[0]]
        if name == "u":
            return [self._buf[10]]
        if name == "q":
            return [self._buf[7 + k] for k in range(d)]
        if name in ("d0", "d1"):   # a dual buffer by index (device decisions: parity unknown to the host)
            return [self._buf[1 + 3 * int(name[1]) + k] for k in range(d)]
        grp = self.parity if name == "p" else 1 - self.parity
        return [self._buf[1 + 3 * grp + k] for k in range(d)]

    def own(self, name: str):
        h = self.halo
        return [b[h:h + self.count] for b in self.fields(name)]

    def step(self, x_k, g, mu: float):
        nat.call("bsgd_slab_step", self._a(), nat.ptr(x_k), nat.ptr(g), float(mu), self._st())

    def init(self):
        nat.call("bsgd_slab_init", self._a(), nat.ptr(self._sums), self._st())
        return self._sums[:2]

    def candidate(self, from_p: bool, when: int = 0):
        nat.call("bsgd_slab_candidate", self._a(when), 1 if from_p else 0, self._st())

    def dual(self, beta: float, when: int = 0):
        nat.call("bsgd_slab_dual", self._a(when), float(beta), nat.ptr(self._sums), self._st())
        return self._sums[:1 + 2 * self.dim]

    def decide(self, stage: int, it: int, gathered, program, world: int, tol: float):
        when = stage if stage in (1, 2) else 0
        prog = (ctypes.c_int32 * len(program))(*program)
        nat.call("bsgd_slab_decide", self._a(when), stage, it, nat.ptr(gathered), world, prog, len(program),
                 float(tol), self._st())

    def set_step_device(self, shard, args, stats):
        nat.call("bsgd_slab_set_step", self._a(), shard.cols, ctypes.byref(args), nat.ptr(stats), self._st())

    def info(self):
        out = (ctypes.c_int32 * 4)()
        tv = ctypes.c_double()
        nat.call("bsgd_slab_info", self._a(), out, ctypes.byref(tv), self._st())
        return {"iterations": out[0], "converged": out[1], "restarts": out[2], "fell_back": out[3], "tv": tv.value}

    def finalize(self):
        nat.call("bsgd_slab_finalize", self._a(), self._st())

    def energy(self):
        nat.call("bsgd_slab_energy", self._a(), nat.ptr(self._sums), self._st())
        return self._sums[:2]

    def output(self, fell: bool, x_next, x_k, g, x_true):
        nat.call("bsgd_slab_output", self._a(), 1 if fell else 0, nat.ptr(x_next), nat.ptr(x_k), nat.ptr(g),
                 nat.ptr(x_true) if x_true is not None else None, nat.ptr(self._stats), self._st())
        return self._stats


class SlabProx:
    """Host loop of the slab-decomposed prox: the FGP of tv.py:172-255 with the
    passes on the rank's slab (``backend``) and the sums combined across ranks.

    Mirrors `fgp_kernel` (csrc/fgp.cuh) decision for decision; the scalar
    arithmetic is Python float (IEEE double), the same operations in the same
    order, so the outcome is bit-identical to the single-GPU prox."""

    def __init__(self, backend, comm, slabs):
        self.be = backend
        self.comm = comm
        self.slabs = [tuple(s) for s in slabs]
        if self.slabs[comm.rank] != (backend.offset, backend.count):
            raise ValueError("backend slab does not match this rank's slab")

    def _sums(self, t):
        return pw_combine(self.be.nvox, self.slabs, self.comm.gather(t))

    def _halo(self, name, lower=True, upper=True):
        self.comm.halo(self.be.fields(name), self.be.count, self.be.halo, lower, upper)

    def run_device(self, weight: float, max_iters: int, tol: float):
        """The same prox with every decision on the device (backend.device = True):
        a FIXED launch / collective sequence -- max_iters blocks of halo, candidate,
        halo, dual, all-gather, decide, then the restart variants that return at
        once unless a restart was decided -- with no host synchronisation, so it
        can be captured in a CUDA graph (`DistributedBSGD.capture`).  Both dual
        buffers' halos are exchanged (the host does not know which holds c).
        Bit-identical to `run`; ProxInfo afterwards from ``backend.info()``."""
        be, comm = self.be, self.comm
        if not weight > 0:
            raise ValueError("slab prox needs a positive weight")
        prog = getattr(self, "_program", None)
        if prog is None:
            prog = self._program = slab_program(be.nvox, self.slabs)
        world = comm.world
        be.device = True
        be.set_weight(weight)
        be.parity = 0
        self._halo("b")
        be.decide(0, 0, comm.gather_flat(be.init()), prog, world, tol)
        for it in range(max_iters):
            for stage, from_p in ((1, False), (2, True)):
                if not from_p:
                    self._halo("q")
                be.candidate(from_p, when=stage)
                self._halo("d0")
                self._halo("d1")
                be.decide(stage, it, comm.gather_flat(be.dual(0.0, when=stage)), prog, world, tol)
        be.finalize()
        self._halo("u", upper=False)
        be.decide(3, 0, comm.gather_flat(be.energy()), prog, world, tol)

    def run(self, weight: float, max_iters: int, tol: float):
        """Prox of the b already stored by ``backend.step``; returns ProxInfo-style fields."""
        be = self.be
        if not weight > 0:
            raise ValueError("slab prox needs a positive weight")
        be.set_weight(weight)
        be.parity = 0
        dim = be.dim
        self._halo("b")
        phi_prev, tv_b = self._sums(be.init())
        t_mom = 1.0
        iters = restarts = converged = 0
        for it in range(max_iters):
            self._halo("q")
            be.candidate(False)                       # tv.py:207-214
            self._halo("c")
            t_next = 0.5 * (1.0 + math.sqrt(1.0 + (4.0 * t_mom) * t_mom))
            beta = (t_mom - 1.0) / t_next
            vc = self._sums(be.dual(beta))            # tv.py:215-216, commit speculative
            phi = vc[0]
            if phi > phi_prev:                        # restart (tv.py:217-231)
                restarts += 1
                t_mom = 1.0
                be.candidate(True)
                self._halo("c")
                t_next = 0.5 * (1.0 + math.sqrt(1.0 + (4.0 * t_mom) * t_mom))
                beta = (t_mom - 1.0) / t_next
                vc = self._sums(be.dual(beta))
                phi = vc[0]
            be.parity ^= 1                            # p <- c
            phi_prev = phi_prev if phi_prev < phi else phi
            t_mom = t_next
            iters = it + 1
            ch2, sc2 = vc[1] + vc[2], vc[1 + dim] + vc[2 + dim]
            if dim == 3:
                ch2, sc2 = ch2 + vc[3], sc2 + vc[6]
            change, scale = math.sqrt(ch2), math.sqrt(sc2)
            if change <= tol * (1e-30 if 1e-30 > scale else scale):   # tv.py:239-248
                converged = 1
                break
        be.finalize()                                 # tv.py:250
        self._halo("u", upper=False)
        e = self._sums(be.energy())
        two_w = 2.0 * weight
        obj_out = e[0] + two_w * e[1]
        obj_b = 0.0 + two_w * tv_b
        fell = 1 if obj_out > obj_b else 0            # tv.py:251-253
        return {"iterations": iters, "converged": converged, "restarts": restarts, "fell_back": fell,
                "tv": tv_b if fell else e[1]}
