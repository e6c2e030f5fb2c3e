"""Block-partitioned sparse operator resident on a B200 (drop-in for `bsgdtv.blockops`).

Same public surface as the reference (`pkg/src/bsgdtv/blockops.py:22-278`):
`BlockPartition`, `make_partition`, `BlockOperator` and `assemble_residual`,
with the same validation and error types.  The difference is where the
arithmetic runs: construction uploads the canonical CSR once and builds the
transposed CSR on the device (`bsgd_plan_create`), and every product is an
sm_100a kernel.  Products accept numpy arrays (returned as numpy, like the
reference) or CUDA torch tensors (returned as CUDA tensors, no host copy).

The matvec-unit tally is kept exactly as the reference does: an integer
nonzero count under a lock, divided on read (`blockops.py:150-152,195-203`).
"""

from __future__ import annotations

import os
import threading
from dataclasses import dataclass

import numpy as np
from scipy import sparse

from . import _native as nat


@dataclass(frozen=True)
class BlockPartition:
    """Contiguous half-open row / column ranges (`blockops.py:22-81`)."""

    row_bounds: tuple
    col_bounds: tuple

    def __post_init__(self) -> None:
        object.__setattr__(self, "row_bounds", tuple((int(a), int(b)) for a, b in self.row_bounds))
        object.__setattr__(self, "col_bounds", tuple((int(a), int(b)) for a, b in self.col_bounds))
        for name, bounds in (("row", self.row_bounds), ("col", self.col_bounds)):
            if len(bounds) == 0:
                raise ValueError(f"empty {name} partition")
            if bounds[0][0] != 0:
                raise ValueError(f"{name} ranges must start at 0")
            for (_, b), (c, _) in zip(bounds, bounds[1:]):
                if b != c:
                    raise ValueError(f"{name} ranges must be contiguous")
            for a, b in bounds:
                if b <= a:
                    raise ValueError(f"{name} ranges must be nonempty")

    @property
    def num_row_blocks(self) -> int:
        return len(self.row_bounds)

    @property
    def num_col_blocks(self) -> int:
        return len(self.col_bounds)

    @property
    def rows(self) -> int:
        return self.row_bounds[-1][1]

    @property
    def cols(self) -> int:
        return self.col_bounds[-1][1]

    def row_range(self, i: int):
        return self.row_bounds[i]

    def col_range(self, j: int):
        return self.col_bounds[j]

    def row_slice(self, i: int) -> slice:
        a, b = self.row_bounds[i]
        return slice(a, b)

    def col_slice(self, j: int) -> slice:
        a, b = self.col_bounds[j]
        return slice(a, b)

    def row_sizes(self):
        return tuple(b - a for a, b in self.row_bounds)

    def col_sizes(self):
        return tuple(b - a for a, b in self.col_bounds)

    def row_edges(self) -> np.ndarray:
        return np.array([a for a, _ in self.row_bounds] + [self.rows], dtype=np.int64)

    def col_edges(self) -> np.ndarray:
        return np.array([a for a, _ in self.col_bounds] + [self.cols], dtype=np.int64)


def _split_even(total: int, parts: int):
    """Near-equal contiguous ranges; the first `total % parts` ranges get one extra."""
    base, extra = divmod(total, parts)
    out, start = [], 0
    for k in range(parts):
        stop = start + base + (1 if k < extra else 0)
        out.append((start, stop))
        start = stop
    return tuple(out)


def make_partition(rows: int, cols: int, num_row_blocks: int, num_col_blocks: int) -> BlockPartition:
    """M x N near-equal blocking (`blockops.py:96-109`), ValueError on M > r or N > c."""
    if rows < 1 or cols < 1:
        raise ValueError("matrix dimensions must be positive")
    if not 1 <= num_row_blocks <= rows:
        raise ValueError(f"row block count {num_row_blocks} not in [1, {rows}]")
    if not 1 <= num_col_blocks <= cols:
        raise ValueError(f"col block count {num_col_blocks} not in [1, {cols}]")
    return BlockPartition(_split_even(rows, num_row_blocks), _split_even(cols, num_col_blocks))


def grid_tiles(height: int, width: int, tile_h: int = 4, tile_w: int = 4):
    """Row grouping of a row-major height x width grid into tile_h x tile_w tiles.

    Returns (tile_ptr, tile_rows) for `BlockOperator.set_stacked_tiles`: pixels of
    one image tile (rows of A2^T), or rays of tile_h angles x tile_w bins (rows of
    an angle-major A2), share most of their columns.
    """
    if tile_h * tile_w > 16:
        raise ValueError("tiles hold at most 16 rows")
    rows, ptr = [], [0]
    for y0 in range(0, height, tile_h):
        for x0 in range(0, width, tile_w):
            ys = np.arange(y0, min(y0 + tile_h, height))
            xs = np.arange(x0, min(x0 + tile_w, width))
            rows.append((ys[:, None] * width + xs[None, :]).ravel())
            ptr.append(ptr[-1] + rows[-1].size)
    return np.asarray(ptr, dtype=np.int64), np.concatenate(rows).astype(np.int64)


def _canonical_csr(matrix, dtype=None) -> sparse.csr_array:
    """float CSR with summed duplicates and sorted indices (`blockops.py:124-126`).

    Duplicates are summed in float64, as the reference converts first and
    sums after (`csr_array(matrix, dtype=np.float64)`).  float32 input stays
    float32 only when it has no duplicates to sum or every summed value
    round-trips through float32 exactly (then the stored entries are the
    reference's float64 values); otherwise it is kept as float64.  An explicit
    ``dtype`` is honoured after the float64 summation.
    """
    csr = sparse.csr_array(matrix)
    if dtype is not None and np.dtype(dtype) not in (np.float32, np.float64):
        raise ValueError("BlockOperator values must be float32 or float64")
    if not csr.has_canonical_format:
        src = csr.dtype
        csr = csr.astype(np.float64)
        csr.sum_duplicates()
        csr.sort_indices()
        if src == np.float32 and dtype is None:
            narrow = csr.data.astype(np.float32)
            if np.array_equal(narrow.astype(np.float64), csr.data):
                csr = sparse.csr_array((narrow, csr.indices, csr.indptr), shape=csr.shape)
    want = np.dtype(dtype) if dtype is not None else (
        np.dtype(np.float32) if csr.dtype == np.float32 else np.dtype(np.float64))
    if csr.dtype != want:
        csr = csr.astype(want)
    csr.sum_duplicates()
    csr.sort_indices()
    return csr


class _Scratch:
    """Per-device reduction scratch (BSGD_SCRATCH_BYTES) and device scalars."""

    def __init__(self, device):
        t = nat.torch()
        self.buf = t.zeros(nat.SCRATCH_BYTES // 8, dtype=t.float64, device=device)
        self.scalars = t.zeros(8, dtype=t.float64, device=device)


class BlockOperator:
    """Sparse matrix with a block partition, resident on one CUDA device.

    ``device`` selects the GPU (default: the current torch device).  The host
    canonical CSR is kept (as the reference keeps its copy) for `tocsr`,
    `to_dense` and `repartition`.
    """

    def __init__(self, matrix, partition: BlockPartition | None = None, *, device=None, dtype=None):
        csr = _canonical_csr(matrix, dtype)
        if csr.nnz == 0:
            raise ValueError("matrix has no nonzeros")
        rows, cols = csr.shape
        if partition is None:
            partition = make_partition(rows, cols, 1, 1)
        if partition.rows != rows or partition.cols != cols:
            raise ValueError(
                f"partition covers {partition.rows}x{partition.cols}, matrix is {rows}x{cols}")
        self._csr = csr
        self._shape = csr.shape
        self._dtype = csr.dtype
        self._partition = partition
        self._device = nat.require_cuda(device)
        self._nnz_total = int(csr.nnz)
        self._nnz_applied = 0
        self._lock = threading.Lock()
        self._scratch = None
        indptr = np.ascontiguousarray(csr.indptr, dtype=np.int64)
        indices = np.ascontiguousarray(csr.indices, dtype=np.int32)
        values = np.ascontiguousarray(csr.data)
        rb = partition.row_edges()
        cb = partition.col_edges()
        handle = nat.c_p()
        t = nat.torch()
        with t.cuda.device(self._device):
            nat.call("bsgd_plan_create", nat.ctypes.byref(handle), self._device.index, rows, cols, csr.nnz,
                     indptr.ctypes.data, indices.ctypes.data, values.ctypes.data, values.dtype.itemsize,
                     partition.num_row_blocks, partition.num_col_blocks, rb.ctypes.data, cb.ctypes.data,
                     nat.stream_ptr(self._device))
        self._plan = handle
        self._load_block_table()

    @classmethod
    def stacked(cls, slice_matrix, depth: int, partition: BlockPartition | None = None, *, device=None,
                dtype=None) -> "BlockOperator":
        """Slice-stacked operator A = A2 (x) I_depth (configs[4], `csrc/stacked.cuh`).

        Block-diagonal with the same 2-D matrix ``slice_matrix`` on every slice,
        in the interleaved order (row r*depth + z, column c*depth + z).  Only A2
        and A2^T live on the device; ``partition`` is over the logical
        (rows2*depth) x (cols2*depth) operator.  Products run in the reference's
        block-sequential order (bit-identical to the oracle on the expanded CSR).
        """
        csr = _canonical_csr(slice_matrix, dtype)
        if csr.nnz == 0:
            raise ValueError("matrix has no nonzeros")
        if depth < 2:
            raise ValueError("depth must be >= 2 (a single slice is an ordinary BlockOperator)")
        rows2, cols2 = csr.shape
        rows, cols = rows2 * depth, cols2 * depth
        if partition is None:
            partition = make_partition(rows, cols, 1, 1)
        if partition.rows != rows or partition.cols != cols:
            raise ValueError(f"partition covers {partition.rows}x{partition.cols}, operator is {rows}x{cols}")
        self = cls.__new__(cls)
        self._device = nat.require_cuda(device)
        indptr = np.ascontiguousarray(csr.indptr, dtype=np.int64)
        indices = np.ascontiguousarray(csr.indices, dtype=np.int32)
        values = np.ascontiguousarray(csr.data)
        rb, cb = partition.row_edges(), partition.col_edges()
        handle = nat.c_p()
        t = nat.torch()
        with t.cuda.device(self._device):
            nat.call("bsgd_plan_create_stacked", nat.ctypes.byref(handle), self._device.index, depth, rows2, cols2,
                     csr.nnz, indptr.ctypes.data, indices.ctypes.data, values.ctypes.data, values.dtype.itemsize,
                     partition.num_row_blocks, partition.num_col_blocks, rb.ctypes.data, cb.ctypes.data,
                     nat.stream_ptr(self._device))
        self._init_fields(handle, (rows, cols), csr.dtype, partition, int(csr.nnz) * depth, depth=depth)
        self._slice_source = ("host", csr)
        return self

    @classmethod
    def from_parallel_beam(cls, n: int, num_angles: int, num_bins: int, num_row_blocks: int = 1,
                           num_col_blocks: int = 1, dtype=np.float32, device=None, depth: int = 1,
                           tiles: bool = True, angle_range=None,
                           partition: BlockPartition | None = None) -> "BlockOperator":
        """Siddon parallel-beam projector generated on the GPU (`bsgd_siddon_csr`).

        Same matrix as `problems.parallel_beam_matrix` (bit-identical); the host
        never holds it, so configs[3]-size problems (~2e9 nonzeros) are possible.
        ``depth`` > 1 stacks it over that many slices (configs[4]), see `stacked`;
        with ``tiles`` the stacked products are tile-staged (`set_stacked_tiles`).
        ``angle_range`` = (a0, a1) generates only the rays of angles a0 <= a < a1
        (rows (a - a0) * num_bins + bin of the result: a multi-GPU row slab,
        `parallel.CudaShard.parallel_beam`); ``partition`` then overrides the
        even num_row_blocks x num_col_blocks partition of those rows.
        """
        import math
        self = cls.__new__(cls)
        self._device = nat.require_cuda(device)
        dt = np.dtype(dtype)
        a0, a1 = (0, num_angles) if angle_range is None else (int(angle_range[0]), int(angle_range[1]))
        if not 0 <= a0 < a1 <= num_angles:
            raise ValueError(f"angle range {angle_range} outside [0, {num_angles})")
        ang = [math.pi * a / num_angles for a in range(a0, a1)]
        cs = np.array([math.cos(t) for t in ang], dtype=np.float64)
        sn = np.array([math.sin(t) for t in ang], dtype=np.float64)
        rows2, cols2 = (a1 - a0) * num_bins, n * n
        rows, cols = rows2 * depth, cols2 * depth
        if partition is None:
            partition = make_partition(rows, cols, num_row_blocks, num_col_blocks)
        elif partition.rows != rows or partition.cols != cols:
            raise ValueError(f"partition covers {partition.rows}x{partition.cols}, operator is {rows}x{cols}")
        ip, ix, vv = nat.c_p(), nat.c_p(), nat.c_p()
        nnz = nat.c_i64()
        t = nat.torch()
        with t.cuda.device(self._device):
            st = nat.stream_ptr(self._device)
            nat.call("bsgd_siddon_csr", self._device.index, n, a1 - a0, num_bins, cs.ctypes.data, sn.ctypes.data,
                     dt.itemsize, nat.ctypes.byref(ip), nat.ctypes.byref(ix), nat.ctypes.byref(vv),
                     nat.ctypes.byref(nnz), st)
            if nnz.value == 0:
                for q in (ip, ix, vv):
                    nat.load().bsgd_device_free(q)
                raise ValueError("matrix has no nonzeros")
            rb, cb = partition.row_edges(), partition.col_edges()
            handle = nat.c_p()
            if depth > 1:
                rc = nat.load().bsgd_plan_create_stacked_device(
                    nat.ctypes.byref(handle), self._device.index, depth, rows2, cols2, nnz.value, ip, ix, vv,
                    dt.itemsize, partition.num_row_blocks, partition.num_col_blocks, rb.ctypes.data, cb.ctypes.data, st)
            else:
                rc = nat.load().bsgd_plan_create_device(
                    nat.ctypes.byref(handle), self._device.index, rows, cols, nnz.value, ip, ix, vv, dt.itemsize,
                    partition.num_row_blocks, partition.num_col_blocks, rb.ctypes.data, cb.ctypes.data, st)
            if rc != nat.OK:
                for q in (ip, ix, vv):
                    nat.load().bsgd_device_free(q)
                nat.check(rc)
        self._init_fields(handle, (rows, cols), dt, partition, int(nnz.value) * depth, depth=depth)
        self._slice_source = ("siddon", (n, num_angles, num_bins, dt, a0, a1))
        if depth > 1 and tiles:
            # A2^T rows are pixels: 4 x 4 image tiles; A2 rows are rays: 4 angles x 4 bins
            self.set_stacked_tiles(True, grid_tiles(n, n))
            self.set_stacked_tiles(False, grid_tiles(a1 - a0, num_bins))
        elif depth == 1 and tiles:
            # Blocked stream for A^T gathered in sinogram tiles (8 angles x 2 bins): a
            # pixel's bins over consecutive angles and the neighbouring pixels of a warp
            # share 128-byte lines of the permuted r (configs[3] K2: CSR 6.1 ms, gather
            # tiles over 4 x 4 pixel tiles 2.9 ms, blocked 2.6 ms -- same bits as the
            # gather tiles).  BSGD_TR_GTILE=1 keeps the gather tiles (experiments).
            if os.environ.get("BSGD_TR_GTILE"):
                self.set_gather_tiles(True, grid_tiles(n, n))
            else:
                self.set_transposed_blocked((a1 - a0, num_bins))
        return self

    def set_gather_tiles(self, transposed: bool, tiles) -> None:
        """Gather-tiled products for an ordinary operator (`bsgd_plan_gather_tiles`).

        ``tiles`` = (tile_ptr, tile_rows) grouping the rows of A (``transposed``
        False) or A^T (True) into tiles of <= 16 rows that share columns
        (`grid_tiles`); None removes them.  Values agree with the CSR kernel to
        rounding.
        """
        if self.depth > 1:
            raise ValueError("stacked operators use set_stacked_tiles")
        t = nat.torch()
        with t.cuda.device(self._device):
            if tiles is None:
                nat.call("bsgd_plan_gather_tiles", self._plan, int(bool(transposed)), 0, None, None,
                         nat.stream_ptr(self._device))
                return
            ptr = np.ascontiguousarray(tiles[0], dtype=np.int64)
            rows = np.ascontiguousarray(tiles[1], dtype=np.int64)
            nat.call("bsgd_plan_gather_tiles", self._plan, int(bool(transposed)), ptr.size - 1, ptr.ctypes.data,
                     rows.ctypes.data, nat.stream_ptr(self._device))

    def set_transposed_blocked(self, grid) -> None:
        """Blocked stream for A^T (`bsgd_plan_blocked_transposed`).

        ``grid`` = (h, w) with h * w = rows of A: the grid r lives on (a sinogram's
        angles x bins); A^T's gathers then run in 16-element grid tiles (shape picked by the plan).  ``()`` builds
        the copy in A^T's own column order; None removes it.  Replaces gather
        tiles of A^T (and `set_gather_tiles(True, ...)` afterwards replaces it).  Values agree with the CSR kernel to rounding.
        """
        if self.depth > 1:
            raise ValueError("stacked operators have no blocked stream")
        h, w = (-1, -1) if grid is None else (0, 0) if len(grid) == 0 else (int(grid[0]), int(grid[1]))
        t = nat.torch()
        with t.cuda.device(self._device):
            nat.call("bsgd_plan_blocked_transposed", self._plan, h, w, nat.stream_ptr(self._device))

    def set_stacked_tiles(self, transposed: bool, tiles) -> None:
        """Tile-staged products for a stacked operator (`bsgd_plan_stacked_tiles`).

        ``tiles`` = (tile_ptr, tile_rows) grouping the stored rows of A2
        (``transposed`` False) or A2^T (True) into tiles of <= 16 rows that share
        columns (`grid_tiles`); None removes them.  Results are unchanged bit for bit.
        """
        if self.depth <= 1:
            raise ValueError("tiles apply to slice-stacked operators only")
        t = nat.torch()
        with t.cuda.device(self._device):
            if tiles is None:
                nat.call("bsgd_plan_stacked_tiles", self._plan, int(bool(transposed)), 0, None, None,
                         nat.stream_ptr(self._device))
                return
            ptr = np.ascontiguousarray(tiles[0], dtype=np.int64)
            rows = np.ascontiguousarray(tiles[1], dtype=np.int64)
            nat.call("bsgd_plan_stacked_tiles", self._plan, int(bool(transposed)), ptr.size - 1, ptr.ctypes.data,
                     rows.ctypes.data, nat.stream_ptr(self._device))

    def _init_fields(self, handle, shape, dtype, partition, nnz_total, depth=1, csr=None) -> None:
        self._plan = handle
        self._csr = csr
        self._shape = shape
        self._dtype = np.dtype(dtype)
        self._partition = partition
        self._nnz_total = nnz_total
        self._nnz_applied = 0
        self._lock = threading.Lock()
        self._scratch = None
        self._depth = depth
        self._load_block_table()

    def _load_block_table(self) -> None:
        partition = self._partition
        nb = partition.num_row_blocks * partition.num_col_blocks
        counts = np.zeros(nb, dtype=np.int64)
        for i in range(partition.num_row_blocks):
            for j in range(partition.num_col_blocks):
                out = nat.c_i64()
                nat.call("bsgd_plan_block_nnz", self._plan, i, j, nat.ctypes.byref(out))
                counts[i * partition.num_col_blocks + j] = out.value
        if int(counts.sum()) != self._nnz_total:
            raise AssertionError("blocks must partition the nonzeros")
        self._block_nnz = counts.reshape(partition.num_row_blocks, partition.num_col_blocks)

    def __del__(self):
        plan = getattr(self, "_plan", None)
        if plan is not None and nat is not None and getattr(nat, "_lib", None) is not None:
            try:
                nat.load().bsgd_plan_destroy(plan)
            except Exception:
                pass
            self._plan = None

    # --- static structure ------------------------------------------------

    @property
    def shape(self):
        return self._shape

    @property
    def nnz(self) -> int:
        return self._nnz_total

    @property
    def partition(self) -> BlockPartition:
        return self._partition

    @property
    def depth(self) -> int:
        """Slices of a stacked operator (1 for an ordinary one)."""
        return getattr(self, "_depth", 1)

    @property
    def num_row_blocks(self) -> int:
        return self._partition.num_row_blocks

    @property
    def num_col_blocks(self) -> int:
        return self._partition.num_col_blocks

    @property
    def device(self):
        return self._device

    @property
    def value_dtype(self):
        return self._dtype

    @property
    def plan(self):
        """Opaque `bsgd_plan*` handle for the C ABI."""
        return self._plan

    def kernel_info(self) -> dict:
        """The product kernels this plan runs (`bsgd_plan_kernel_info`).

        Chosen at plan creation by fixed structural rules, never by timing, so a
        given matrix always runs the same kernels (and the same arithmetic).
        """
        ki = nat.KernelInfo()
        nat.call("bsgd_plan_kernel_info", self._plan, nat.ctypes.byref(ki))
        return {"forward": nat.KERNEL_NAMES[ki.fwd_kernel], "forward_lanes": int(ki.fwd_lanes),
                "transposed": nat.KERNEL_NAMES[ki.tr_kernel], "transposed_lanes": int(ki.tr_lanes),
                "depth": int(ki.depth), "forward_order": nat.GATHER_ORDERS[ki.fwd_order],
                "transposed_order": nat.GATHER_ORDERS[ki.tr_order]}

    def set_phase_timing(self, enable: bool) -> None:
        """Record CUDA events between the phases of every eager epoch on this plan
        (`bsgd_plan_set_timing`; measurement only, never inside a graph capture)."""
        nat.call("bsgd_plan_set_timing", self._plan, int(bool(enable)))

    def phase_timing(self):
        """(milliseconds per phase summed over the recorded epochs, epochs) and reset;
        phases are `_native.TIMING_PHASES`."""
        ms = np.zeros(len(nat.TIMING_PHASES))
        n = nat.c_i64()
        nat.call("bsgd_plan_timing", self._plan, ms.ctypes.data, nat.ctypes.byref(n))
        return dict(zip(nat.TIMING_PHASES, ms.tolist())), int(n.value)

    def block(self, i: int, j: int) -> sparse.csr_array:
        """Block (i, j) with block-local indices, read back from the device copy."""
        if not (0 <= i < self.num_row_blocks and 0 <= j < self.num_col_blocks):
            raise IndexError(f"block ({i}, {j}) outside the grid")
        r0, r1 = self._partition.row_range(i)
        c0, c1 = self._partition.col_range(j)
        nz = int(self._block_nnz[i, j])
        indptr = np.zeros(r1 - r0 + 1, dtype=np.int64)
        indices = np.zeros(max(nz, 1), dtype=np.int32)
        values = np.zeros(max(nz, 1), dtype=self._dtype)
        nat.call("bsgd_plan_block_copy", self._plan, i, j, indptr.ctypes.data, indices.ctypes.data,
                 values.ctypes.data, nat.stream_ptr(self._device))
        return sparse.csr_array((values[:nz], indices[:nz], indptr), shape=(r1 - r0, c1 - c0))

    def transpose_pattern(self):
        """(indptr, indices, values) of the device-built A^T CSR (pattern checks)."""
        rows, cols = self.shape
        indptr = np.zeros(cols + 1, dtype=np.int64)
        indices = np.zeros(self.nnz, dtype=np.int32)
        values = np.zeros(self.nnz, dtype=self._dtype)
        nat.call("bsgd_plan_transpose_copy", self._plan, indptr.ctypes.data, indices.ctypes.data,
                 values.ctypes.data, nat.stream_ptr(self._device))
        return indptr, indices, values

    def block_nnz(self, i: int, j: int) -> int:
        return int(self._block_nnz[i, j])

    def to_dense(self) -> np.ndarray:
        return self.tocsr().astype(np.float64).toarray()

    def tocsr(self) -> sparse.csr_array:
        """Canonical CSR on the host (downloaded once for device-generated operators)."""
        if self._csr is None:
            rows, cols = self._shape
            indptr = np.zeros(rows + 1, dtype=np.int64)
            indices = np.zeros(self._nnz_total, dtype=np.int32)
            values = np.zeros(self._nnz_total, dtype=self._dtype)
            nat.call("bsgd_plan_csr_copy", self._plan, indptr.ctypes.data, indices.ctypes.data, values.ctypes.data,
                     nat.stream_ptr(self._device))
            self._csr = sparse.csr_array((values, indices, indptr), shape=self._shape)
        return self._csr

    def repartition(self, num_row_blocks: int, num_col_blocks: int) -> "BlockOperator":
        rows, cols = self.shape
        if self.depth > 1:
            kind, src = self._slice_source
            if kind == "host":
                return BlockOperator.stacked(src, self.depth, make_partition(rows, cols, num_row_blocks,
                                                                             num_col_blocks), device=self._device)
            n, ang, nb, dt, a0, a1 = src
            return BlockOperator.from_parallel_beam(n, ang, nb, num_row_blocks, num_col_blocks, dtype=dt,
                                                    device=self._device, depth=self.depth, angle_range=(a0, a1))
        return BlockOperator(self.tocsr(), make_partition(rows, cols, num_row_blocks, num_col_blocks),
                             device=self._device)

    # --- counter ---------------------------------------------------------

    @property
    def matvec_units(self) -> float:
        with self._lock:
            applied = self._nnz_applied
        return applied / self._nnz_total

    def _charge(self, nnz: int) -> None:
        with self._lock:
            self._nnz_applied += int(nnz)

    # --- device helpers ------------------------------------------------------

    def _scr(self) -> _Scratch:
        if self._scratch is None:
            self._scratch = _Scratch(self._device)
        return self._scratch

    def _vec(self, v, length):
        return nat.as_f64(v, self._device, length)

    def _out(self, t, like):
        return t if isinstance(like, nat.torch().Tensor) else t.cpu().numpy()

    # --- products ----------------------------------------------------------

    def block_matvec(self, i: int, j: int, x_j):
        """A_{I_i}^{J_j} @ x_j (`blockops.py:207-214`); charges nnz(block)."""
        r0, r1 = self._partition.row_range(i)
        c0, c1 = self._partition.col_range(j)
        xv = self._vec(x_j, c1 - c0)
        out = nat.torch().empty(r1 - r0, dtype=nat.torch().float64, device=self._device)
        self._charge(self._block_nnz[i, j])
        nat.call("bsgd_block_matvec", self._plan, i, j, nat.ptr(xv), nat.ptr(out), nat.stream_ptr(self._device))
        return self._out(out, x_j)

    def block_matvec_transpose(self, i: int, j: int, r_i):
        """(A_{I_i}^{J_j})^T @ r_i, no factor 2 (`blockops.py:216-223`)."""
        r0, r1 = self._partition.row_range(i)
        c0, c1 = self._partition.col_range(j)
        rv = self._vec(r_i, r1 - r0)
        out = nat.torch().empty(c1 - c0, dtype=nat.torch().float64, device=self._device)
        self._charge(self._block_nnz[i, j])
        nat.call("bsgd_block_matvec_transpose", self._plan, i, j, nat.ptr(rv), nat.ptr(out),
                 nat.stream_ptr(self._device))
        return self._out(out, r_i)

    def matvec(self, x, charge: bool = True):
        """A @ x (`blockops.py:225-244`); charges one unit unless ``charge`` is False."""
        rows, cols = self.shape
        xv = self._vec(x, cols)
        if charge:
            self._charge(self._nnz_total)
        out = nat.torch().empty(rows, dtype=nat.torch().float64, device=self._device)
        nat.call("bsgd_matvec", self._plan, nat.ptr(xv), nat.ptr(out), nat.stream_ptr(self._device))
        return self._out(out, x)

    def rmatvec(self, w, charge: bool = True):
        """A^T @ w (`blockops.py:246-261`)."""
        rows, cols = self.shape
        wv = self._vec(w, rows)
        if charge:
            self._charge(self._nnz_total)
        out = nat.torch().empty(cols, dtype=nat.torch().float64, device=self._device)
        nat.call("bsgd_rmatvec", self._plan, nat.ptr(wv), nat.ptr(out), nat.stream_ptr(self._device))
        return self._out(out, w)

    def residual_sumsq(self, x, y, charge: bool = False):
        """(y - A x, ||y - A x||^2) on the device; the squared norm stays a device scalar."""
        rows, cols = self.shape
        xv = self._vec(x, cols)
        yv = self._vec(y, rows)
        if charge:
            self._charge(self._nnz_total)
        t = nat.torch()
        r = t.empty(rows, dtype=t.float64, device=self._device)
        s = t.empty(1, dtype=t.float64, device=self._device)
        nat.call("bsgd_residual", self._plan, nat.ptr(xv), nat.ptr(yv), nat.ptr(r), nat.ptr(s),
                 nat.ptr(self._scr().buf), nat.stream_ptr(self._device))
        return r, s


def assemble_residual(y, z_cache):
    """r = y - z^0 - z^1 - ... (ascending j, `blockops.py:264-278`) on the device."""
    t = nat.torch()
    is_t = isinstance(y, t.Tensor)
    dev = y.device if is_t and y.is_cuda else nat.require_cuda()
    yv = nat.as_f64(y, dev)
    if yv.ndim != 1:
        raise ValueError("y must be a vector")
    if isinstance(z_cache, t.Tensor):
        zc = z_cache.to(device=dev, dtype=t.float64).contiguous()
    else:
        zc = t.from_numpy(np.ascontiguousarray(np.asarray(z_cache, dtype=np.float64))).to(dev)
    if zc.ndim != 2 or zc.shape[1] != yv.shape[0]:
        raise ValueError(f"z cache shape {tuple(zc.shape)} does not match y of length {yv.shape[0]}")
    out = t.empty_like(yv)
    nat.call("bsgd_assemble_residual", yv.shape[0], zc.shape[0], nat.ptr(yv), nat.ptr(zc), nat.ptr(out),
             nat.stream_ptr(dev))
    return out if is_t else out.cpu().numpy()
