"""Slab-decomposed TV prox (parallel.SlabProx), host logic on CPU.

* `prox_slabs` / `pw_combine`: slabs are nodes of numpy's pairwise recursion
  and their sums recombine to np.sum bit for bit.
* world sizes 2 and 3 over gloo: the real SlabProx loop (halo exchange,
  all-gather of the per-slab sums, restart / stop / fallback decisions) on the
  numpy stand-in backend (tests/slab_numpy.py) equals the oracle's tv_prox /
  tv_prox3 bit for bit -- image, iterations, restarts, convergence, fallback.
* DistributedBSGD with the slab prox (reduce-scatter of g, slab step, stats
  all-reduce, all-gather of x) over gloo equals the oracle's epochs.
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import REPO

# (dims, weight, max_iters, tol, seed): 2-D and 3-D, with restarts, tight and loose tol
CASES = [
    ((1, 24, 20), 0.35, 30, 1e-5, 0),
    ((1, 24, 20), 2.0, 12, 1e-12, 1),
    ((1, 32, 32), 0.05, 40, 1e-7, 2),
    ((6, 8, 10), 0.4, 25, 1e-6, 3),
    ((8, 8, 8), 1.5, 10, 1e-12, 4),
]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _volume(dims, seed):
    rng = np.random.default_rng(seed)
    v = rng.random(dims) * 2.0
    v[..., : dims[-1] // 2] += 1.0   # an edge for the TV to keep
    return v


def test_prox_slabs_are_pairwise_nodes():
    from paper_1812_01307_b200.parallel import prox_slabs, pw_combine
    assert prox_slabs(1 << 24, 8, 65536) == [(k << 21, 1 << 21) for k in range(8)]
    assert prox_slabs(1024, 3, 32) == [(0, 256), (256, 256), (512, 512)]
    with pytest.raises(ValueError):
        prox_slabs(480, 2, 300)          # thinner than a halo plane
    with pytest.raises(ValueError):
        prox_slabs(200, 4, 1)            # would split a pairwise leaf
    rng = np.random.default_rng(0)
    for n in (129, 480, 1000, 4096, 12345, 1 << 16):
        a = rng.standard_normal(n) * 10.0 ** rng.integers(-8, 8, n)
        for world in (1, 2, 3, 4, 5, 8):
            try:
                slabs = prox_slabs(n, world, 1)
            except ValueError:
                continue
            vals = [[np.sum(a[lo:lo + c]), np.sum(a[lo:lo + c] ** 2)] for lo, c in slabs]
            got = pw_combine(n, slabs, vals)
            assert got[0] == np.sum(a) and got[1] == np.sum(a ** 2), (n, world)


def _prox_worker(rank, world, port, outdir, device=False):
    import sys
    sys.path.insert(0, REPO)
    sys.path.insert(0, os.path.join(REPO, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    from paper_1812_01307_b200 import parallel
    from slab_numpy import NumpySlab, NumpySlabDevice
    comm = parallel.TorchComm()
    out = {}
    for ci, (dims, w, iters, tol, seed) in enumerate(CASES):
        nvox = int(np.prod(dims))
        halo = dims[1] * dims[2] if dims[0] > 1 else dims[2]
        slabs = parallel.prox_slabs(nvox, world, halo)
        lo, n = slabs[rank]
        be = NumpySlabDevice(dims, lo, n) if device else NumpySlab(dims, lo, n)
        vol = _volume(dims, seed).ravel()
        xk = torch.from_numpy(vol.copy())
        g = torch.zeros(nvox, dtype=torch.float64)
        be.step(xk, g, 1.0)            # b = vol on the slab
        if device:                     # fixed sequence, decisions in the backend's control block
            parallel.SlabProx(be, comm, slabs).run_device(w, iters, tol)
            info = be.info()
        else:
            info = parallel.SlabProx(be, comm, slabs).run(w, iters, tol)
        xn = torch.zeros(nvox, dtype=torch.float64)
        be.output(info["fell_back"], xn, xk, g, None)
        comm.allgather_slabs(xn, slabs)
        out[f"x{ci}"] = xn.numpy()
        out[f"info{ci}"] = np.array([info["iterations"], info["converged"], info["restarts"], info["fell_back"]])
        out[f"tv{ci}"] = info["tv"]
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), **out)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,device", [(2, False), (3, False), (2, True), (3, True)])
def test_slab_prox_gloo_matches_oracle_bit_exact(tmp_path, world, device):
    """Host-decided (SlabProx.run) and device-decided (run_device: fixed sequence,
    sums all-gathered and combined by the postfix program) slab prox over gloo."""
    from oracle import oracle as orc
    mp.spawn(_prox_worker, args=(world, _free_port(), str(tmp_path), device), nprocs=world, join=True)
    res = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    restarts = 0
    for ci, (dims, w, iters, tol, seed) in enumerate(CASES):
        vol = _volume(dims, seed)
        if dims[0] > 1:
            ref, rep = orc.tv_prox3(vol, w, iters, tol)
            tv_ref = orc.tv_value3(ref)
        else:
            ref, rep = orc.tv_prox(vol[0], w, iters, tol)
            tv_ref = orc.tv_value(ref)
        for r in range(world):
            assert np.array_equal(res[r][f"x{ci}"], ref.ravel()), (ci, r)
            got = tuple(int(v) for v in res[r][f"info{ci}"])
            assert got == (rep.iterations, int(rep.converged), rep.restarts, int(rep.fell_back)), (ci, r)
            assert float(res[r][f"tv{ci}"]) == tv_ref, (ci, r)
        restarts += rep.restarts
    assert restarts > 0   # the restart branch was exercised


class _CpuProxShard:
    """CPU stand-in for CudaShard with the slab prox (lam > 0, identity layout)."""

    def __init__(self, matrix, spec, dims, lam, device=False):
        import types
        self.device = device
        from scipy import sparse
        import torch
        from paper_1812_01307_b200 import tv
        r0, r1 = spec.row_range
        self.spec = spec
        self.t = torch
        self.a = sparse.csr_array(sparse.csr_array(matrix).astype(np.float64)[r0:r1, :])
        self.cols = matrix.shape[1]
        self.rows = r1 - r0
        self.dims = dims
        self.layout = tv.PixelLayout.row_major(dims[1], dims[2])
        self._ns = types.SimpleNamespace

    def prox_dims(self):
        return self.dims

    def slab_backend(self, offset, count):
        from slab_numpy import NumpySlab, NumpySlabDevice
        if self.device:
            be = NumpySlabDevice(self.dims, offset, count)

            def set_step_device(shard, a, stats):
                a.stats = tuple(float(v) for v in stats)
                a.tv = be.info()["tv"]

            be.set_step_device = set_step_device
            return be
        return NumpySlab(self.dims, offset, count)

    def zeros(self, n):
        return self.t.zeros(n, dtype=self.t.float64)

    def vector(self, v):
        return self.t.tensor(np.asarray(v, dtype=np.float64))

    def args(self, x_k, g, x_next, mu, cfg, f_curr, hist, counter, perm, x_true, flags):
        return self._ns(x_k=x_k, g=g, x_next=x_next, mu=mu, f_curr=f_curr, hist=hist, counter=counter,
                        flags=flags, stats=None, rsum=None)

    def grad(self, r_local, g_out):
        g_out.copy_(self.t.from_numpy(2.0 * (self.a.T @ r_local.numpy())))

    def set_step(self, a, stats, info):
        a.stats = tuple(float(v) for v in stats)

    def forward(self, x, y_local, r_out, a):
        r = y_local.numpy() - self.a @ x.numpy()
        r_out.copy_(self.t.from_numpy(r))
        a.rsum = float(r @ r)

    def forward_sumsq(self, a, out1):
        out1.fill_(a.rsum)

    def tail(self, a, fnext1):
        row = int(a.counter.item())
        a.hist[row, 0] = float(fnext1.item())
        if a.stats is not None:             # |x|^2, |x - x*|^2 (H_XX, H_XE) and TV (H_TV)
            a.hist[row, 2], a.hist[row, 3] = a.stats[0], a.stats[1]
            a.hist[row, 4] = getattr(a, "tv", 0.0)
        a.counter.fill_(row + 1)

    def dot(self, a, b, out1):
        out1.fill_(float(a.numpy() @ b.numpy()))


def _ct_case():
    from paper_1812_01307_b200 import problems
    n = 16
    a = problems.parallel_beam_matrix(n, 12, 23)
    rng = np.random.default_rng(7)
    x_true = rng.random(n * n)
    y = a @ x_true
    return a, y, x_true, (1, n, n)


def _epoch_worker(rank, world, port, outdir, epochs, device=False):
    import sys
    sys.path.insert(0, REPO)
    sys.path.insert(0, os.path.join(REPO, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1812_01307_b200 import parallel, tv
    from paper_1812_01307_b200.blockops import make_partition
    from paper_1812_01307_b200.solvers import SolverConfig
    a, y, x_true, dims = _ct_case()
    part = make_partition(a.shape[0], a.shape[1], 4, 4)
    spec = parallel.ShardSpec(part, rank, world)
    shard = _CpuProxShard(a, spec, dims, lam=0.5, device=device)
    cfg = SolverConfig(mu=2e-3, lam=0.5, epochs=epochs, monitor_decrease=False, prox=tv.ProxSettings(20, 1e-6))
    drv = parallel.DistributedBSGD(shard, y, cfg, history_capacity=epochs + 4, prox="slab")
    assert drv.slab is not None and drv.slab_device == device
    auto = parallel.DistributedBSGD(shard, y, cfg, history_capacity=4)
    assert auto.slab is None   # small image: "auto" keeps the prox replicated
    infos = []
    for _ in range(epochs):
        drv.epoch_step(monitor=False)
        info = drv.slab.be.info() if device else drv.prox_info
        infos.append([info[k] for k in ("iterations", "converged", "restarts", "fell_back")])
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), x=drv.x_current.numpy(), r=drv.r_current.numpy(),
             info=np.array(infos))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("device", [False, True])
def test_world2_gloo_epochs_with_slab_prox_match_oracle(tmp_path, device):
    from oracle import oracle as orc
    epochs = 5
    mp.spawn(_epoch_worker, args=(2, _free_port(), str(tmp_path), epochs, device), nprocs=2, join=True)
    r0, r1 = (np.load(tmp_path / f"rank{r}.npz") for r in range(2))
    assert np.array_equal(r0["x"], r1["x"]) and np.array_equal(r0["info"], r1["info"])
    a, y, x_true, dims = _ct_case()
    op = orc.OracleOperator(a, 4, 4)
    prm = orc.Params(mu=2e-3, lam=0.5, epochs=epochs, max_inner_iters=20, tol=1e-6, monitor_decrease=False)
    st = orc.init_state(op, y, prm)
    for _ in range(epochs):
        orc.epoch(st, op, y, prm, np.arange(dims[1] * dims[2]), dims[1:])
    # g is summed over ranks (and by scipy's full A^T r on each rank) rather than in
    # the oracle's ascending block order: ulp-level differences in the prox input,
    # which the FGP iterations amplify (1e-16 for three epochs, then ~5e-9 on this
    # case at world size 1 too).  The prox itself is bit-exact (tests above).
    assert np.linalg.norm(r0["x"] - st.x) / np.linalg.norm(st.x) < 1e-7
    r_full = np.concatenate([r0["r"], r1["r"]])
    assert np.linalg.norm(r_full - st.r_vec) / np.linalg.norm(st.r_vec) < 1e-7
    assert r0["info"][:, 0].max() > 1     # the prox iterated


class _CpuSliceShard(_CpuProxShard):
    """CPU stand-in for parallel.CudaSliceShard: kron(A2, I_{slices}) of this rank's
    slices (local interleaved vectors), the slab prox on its slices of the
    slice-major volume (numpy double with the interleaved step / output map)."""

    owns_slices = True

    def __init__(self, a2, n, depth, rank, world, lam):
        import types
        from scipy import sparse
        import torch
        from paper_1812_01307_b200 import parallel, tv
        from paper_1812_01307_b200.blockops import make_partition
        z0, z1 = parallel.slice_ranges(depth, n, n, world)[rank]
        self.z0, self.z1, self.depth, self.n = z0, z1, depth, n
        self.rays2, self.pix2 = a2.shape
        dl = z1 - z0
        self.a = sparse.csr_array(sparse.kron(sparse.csr_array(a2).astype(np.float64), sparse.identity(dl),
                                              format="csr"))
        self.t = torch
        self.cols, self.rows = self.pix2 * dl, self.rays2 * dl
        self.dims = (depth, n, n)
        self.layout = tv.VolumeLayout.z_major(dl, n, n)
        self.slab_range = (z0 * n * n, dl * n * n)
        self.spec = types.SimpleNamespace(row_range=(0, self.rows),
                                          partition=make_partition(self.rays2 * depth, self.pix2 * depth, 4, 4))
        self._ns = types.SimpleNamespace
        self.device = True
        self.op = types.SimpleNamespace(nnz=int(self.a.nnz))

    @property
    def shape(self):
        return (self.rays2 * self.depth, self.pix2 * self.depth)

    def _cut(self, v, m):
        return self.vector(np.ascontiguousarray(np.asarray(v).reshape(m, self.depth)[:, self.z0:self.z1]).ravel())

    def local_rows(self, y):
        return self._cut(y, self.rays2)

    def local_cols(self, x):
        return self._cut(x, self.pix2)

    def slab_backend(self, offset, count):
        be = super().slab_backend(offset, count)
        be.interleaved = True
        return be

    def assemble_cols(self, x_local, group=None):
        import torch.distributed as dist
        from paper_1812_01307_b200 import parallel
        world = dist.get_world_size(group)
        ranges = parallel.slice_ranges(self.depth, self.n, self.n, world)
        parts = [self.t.zeros(self.pix2 * (b - a), dtype=self.t.float64) for a, b in ranges]
        dist.all_gather(parts, x_local.contiguous(), group=group)
        return self.t.cat([p.reshape(self.pix2, b - a) for p, (a, b) in zip(parts, ranges)], dim=1).reshape(-1)


def _slice_case():
    from paper_1812_01307_b200 import problems
    n, depth = 8, 8
    a2 = problems.parallel_beam_matrix(n, 6, 11)
    vol = problems.ellipsoid_phantom(n, depth, 5, 0)
    x_true = np.ascontiguousarray(vol.reshape(depth, n * n).T).ravel()
    from scipy import sparse
    a = sparse.csr_array(sparse.kron(sparse.csr_array(a2), sparse.identity(depth), format="csr"))
    a.sort_indices()
    y = a @ x_true + np.random.default_rng(2).standard_normal(a.shape[0]) * 0.02
    return a2, a, y, x_true, n, depth


def _slice_worker(rank, world, port, outdir, epochs):
    import sys
    sys.path.insert(0, REPO)
    sys.path.insert(0, os.path.join(REPO, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1812_01307_b200 import problems, solvers, tv
    a2, a, y, x_true, n, depth = _slice_case()
    shard = _CpuSliceShard(a2, n, depth, rank, world, lam=0.3)
    cfg = solvers.SolverConfig(mu=0.9 / (2.0 * 60.0), lam=0.3, epochs=epochs, monitor_decrease=False,
                               prox=tv.ProxSettings(15, 1e-7))
    lay = tv.VolumeLayout(depth, n, n, problems.interleaved_perm(n * n, depth))
    tr = solvers.run_solver("bsgd", solvers.Problem(shard, y, x_true, lay), cfg, sample_every=2, group="default")
    np.savez(os.path.join(outdir, f"s{rank}.npz"), x=tr.final_x, samples=np.array([tuple(s) for s in tr.samples]))
    dist.barrier()
    dist.destroy_process_group()


def test_world2_gloo_slice_ownership_matches_oracle(tmp_path):
    """configs[4]-style slice ownership over two ranks: no product exchange, the
    slab prox on each rank's slices (device-decision choreography), against the
    oracle on the full kron(A2, I_D) with the slice-major volume view."""
    from oracle import oracle as orc
    from paper_1812_01307_b200 import problems
    epochs = 6
    mp.spawn(_slice_worker, args=(2, _free_port(), str(tmp_path), epochs), nprocs=2, join=True)
    r0, r1 = (np.load(tmp_path / f"s{r}.npz") for r in range(2))
    assert np.array_equal(r0["x"], r1["x"])
    a2, a, y, x_true, n, depth = _slice_case()
    op = orc.OracleOperator(a, 4, 4)
    prm = orc.Params(mu=0.9 / (2.0 * 60.0), lam=0.3, epochs=epochs, max_inner_iters=15, tol=1e-7,
                     monitor_decrease=False)
    ref = orc.run_bsgd(op, y, prm, x_true=x_true, perm=problems.interleaved_perm(n * n, depth), hw=(depth, n, n),
                       sample_every=2)
    assert np.linalg.norm(r0["x"] - ref.final_x) / np.linalg.norm(ref.final_x) < 1e-10
    want = np.array(ref.samples)
    assert np.array_equal(r0["samples"][:, 0], want[:, 0]) and np.array_equal(r0["samples"][:, 3], want[:, 3])
    assert np.allclose(r0["samples"][:, 1:3], want[:, 1:3], rtol=1e-10)
