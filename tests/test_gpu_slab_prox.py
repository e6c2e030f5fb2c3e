"""Slab-decomposed TV prox on the GPU (bsgd_slab_* through parallel.CudaSlab).

Ranks are emulated by host threads on the one GPU: each runs the real
parallel.SlabProx loop on its own CudaSlab, and the exchanges (halo planes,
the per-slab sums, slab gathers) are host copies between threads at barriers
(no kernel ever waits on another rank's kernel).  The result must equal the
single-GPU prox (bsgd_tv_prox / bsgd_tv_prox3) and the oracle bit for bit.
"""

import threading

import numpy as np
import pytest

from conftest import golden_cfg, golden_csr, load_golden
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


class ThreadComm:
    """parallel.TorchComm's surface over threads of one process (test double)."""

    def __init__(self, shared, rank, world):
        import torch
        self.torch = torch
        self.s = shared
        self.rank, self.world = rank, world

    def _sync(self):
        self.torch.cuda.synchronize()
        self.s["barrier"].wait()

    def _post(self, key, value):
        self.s["slots"][(self.rank, key)] = value

    def _get(self, r, key):
        return self.s["slots"][(r, key)]

    def halo(self, bufs, n, h, lower=True, upper=True):
        for k, b in enumerate(bufs):
            self._post(("halo", k), (b[h:2 * h].clone(), b[n:n + h].clone()))
        self._sync()
        for k, b in enumerate(bufs):
            if lower and self.rank > 0:
                b[0:h].copy_(self._get(self.rank - 1, ("halo", k))[1])
            if upper and self.rank + 1 < self.world:
                b[n + h:n + 2 * h].copy_(self._get(self.rank + 1, ("halo", k))[0])
        self._sync()

    def gather(self, t):
        self._post("gather", t.clone())
        self._sync()
        rows = np.stack([self._get(r, "gather").cpu().numpy() for r in range(self.world)])
        self._sync()
        return rows

    def gather_flat(self, t):
        self._post("gflat", t.clone())
        self._sync()
        out = self.torch.cat([self._get(r, "gflat") for r in range(self.world)])
        self._sync()
        return out

    def allreduce(self, t):
        self._post("reduce", t.clone())
        self._sync()
        acc = self._get(0, "reduce").clone()
        for r in range(1, self.world):
            acc += self._get(r, "reduce")
        self._sync()
        t.copy_(acc)

    def reduce_scatter(self, full, slabs):
        self.allreduce(full)

    def allgather_slabs(self, full, slabs):
        lo, n = slabs[self.rank]
        self._post("slab", full[lo:lo + n].clone())
        self._sync()
        for r, (a, c) in enumerate(slabs):
            if r != self.rank:
                full[a:a + c].copy_(self._get(r, "slab"))
        self._sync()


def run_threads(world, fn):
    shared = {"barrier": threading.Barrier(world), "slots": {}}
    out = [None] * world
    err = []

    def body(r):
        try:
            out[r] = fn(r, ThreadComm(shared, r, world))
        except BaseException as e:  # noqa: BLE001
            err.append(e)
            shared["barrier"].abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if err:
        raise err[0]
    return out


def _volume(dims, seed):
    rng = np.random.default_rng(seed)
    v = rng.random(dims) * 2.0
    v[..., : dims[-1] // 2] += 1.0
    return v


CASES = [  # dims, weight, iters, tol, world; small (general tree) and fast-path slabs
    ((1, 64, 48), 0.3, 30, 1e-6, 2),
    ((1, 64, 48), 1.0, 15, 1e-12, 4),
    ((16, 12, 10), 0.4, 20, 1e-6, 2),
    ((16, 12, 10), 1.2, 10, 1e-12, 4),
    ((1, 256, 256), 0.2, 20, 1e-6, 4),
    ((32, 32, 32), 0.5, 10, 1e-7, 4),
    ((32, 32, 32), 0.5, 10, 1e-7, 8),
]


@pytest.mark.parametrize("device", [False, True])
@pytest.mark.parametrize("dims,w,iters,tol,world", CASES)
def test_slab_prox_matches_single_gpu_bit_exact(cuda_ok, dims, w, iters, tol, world, device):
    """Host-decided (SlabProx.run) and device-decided (run_device: bsgd_slab_decide
    on all-gathered sums, a fixed launch sequence) slab prox vs the single-GPU prox."""
    import torch
    from paper_1812_01307_b200 import parallel, tv
    dev = torch.device("cuda", 0)
    vol = _volume(dims, sum(dims) + world)
    nvox = vol.size
    halo = dims[1] * dims[2] if dims[0] > 1 else dims[2]
    slabs = parallel.prox_slabs(nvox, world, halo)
    xk = torch.from_numpy(vol.ravel().copy()).to(dev)
    g = torch.zeros(nvox, dtype=torch.float64, device=dev)

    def rank(r, comm):
        lo, n = slabs[r]
        be = parallel.CudaSlab(dims, lo, n, dev)
        be.step(xk, g, 1.0)
        if device:
            parallel.SlabProx(be, comm, slabs).run_device(w, iters, tol)
            info = be.info()
        else:
            info = parallel.SlabProx(be, comm, slabs).run(w, iters, tol)
        xn = torch.zeros(nvox, dtype=torch.float64, device=dev)
        be.output(info["fell_back"], xn, xk, g, None)
        comm.allgather_slabs(xn, slabs)
        return xn.cpu().numpy(), info

    res = run_threads(world, rank)
    img = torch.from_numpy(vol if dims[0] > 1 else vol[0]).to(dev)
    ref, rinfo = tv.tv_prox(img, w, tv.ProxSettings(iters, tol), return_info=True)
    ref = ref.cpu().numpy().ravel()
    for x, info in res:
        assert np.array_equal(x, ref)
        assert (info["iterations"], bool(info["converged"]), info["restarts"], bool(info["fell_back"])) == \
            (rinfo.iterations, rinfo.converged, rinfo.restarts, rinfo.fell_back)
    if nvox <= 4096:   # and the oracle directly
        o, rep = (orc.tv_prox3(vol, w, iters, tol) if dims[0] > 1 else orc.tv_prox(vol[0], w, iters, tol))
        assert np.array_equal(res[0][0], o.ravel()) and res[0][1]["restarts"] == rep.restarts


def test_slab_prox_restart_and_fallback_paths(cuda_ok):
    """Restarting cases on two slabs, and the golden identity-fallback case
    (tv.py:251-253; a 4x4-or-smaller image, so one slab)."""
    import torch
    from paper_1812_01307_b200 import parallel
    dev = torch.device("cuda", 0)
    z = load_golden("prox")
    fb = [k for k in range(int(z["count"])) if z[f"info{k}"][3]]
    assert fb
    k = fb[0]
    w_fb, mi_fb, tol_fb = (float(v) for v in z[f"par{k}"])
    cases = [((1, 32, 32), _volume((1, 32, 32), 11), 0.05, 40, 1e-12, 2),
             ((8, 8, 8), _volume((8, 8, 8), 11), 1.0, 40, 1e-12, 2),
             ((1,) + z[f"in{k}"].shape, z[f"in{k}"][None], w_fb, int(mi_fb), tol_fb, 1)]
    restarts = fell = 0
    for dims, vol, w, iters, tol, world in cases:
        nvox = vol.size
        halo = dims[1] * dims[2] if dims[0] > 1 else dims[2]
        slabs = parallel.prox_slabs(nvox, world, halo)
        xk = torch.from_numpy(vol.ravel().copy()).to(dev)
        g = torch.zeros(nvox, dtype=torch.float64, device=dev)

        def rank(r, comm):
            be = parallel.CudaSlab(dims, *slabs[r], dev)
            be.step(xk, g, 1.0)
            info = parallel.SlabProx(be, comm, slabs).run(w, iters, tol)
            xn = torch.zeros(nvox, dtype=torch.float64, device=dev)
            be.output(info["fell_back"], xn, xk, g, None)
            comm.allgather_slabs(xn, slabs)
            return xn.cpu().numpy(), info

        x, info = run_threads(world, rank)[0]
        o, rep = orc.tv_prox3(vol, w, iters, tol) if dims[0] > 1 else orc.tv_prox(vol[0], w, iters, tol)
        assert np.array_equal(x, o.ravel())
        assert (info["iterations"], info["restarts"], bool(info["fell_back"])) == \
            (rep.iterations, rep.restarts, rep.fell_back)
        restarts += rep.restarts
        fell += int(rep.fell_back)
    assert restarts > 0 and fell == 1
    assert np.array_equal(x.reshape(z[f"out{k}"].shape), z[f"out{k}"])


def test_world1_driver_slab_prox_matches_replicated(cuda_ok):
    """DistributedBSGD at world size 1: the slab path (bsgd_slab_* + bsgd_epoch_set_step)
    gives the replicated path's iterates bit for bit."""
    from paper_1812_01307_b200 import parallel, tv
    from paper_1812_01307_b200.blockops import make_partition
    from paper_1812_01307_b200.solvers import SolverConfig
    z = load_golden("p1_ct")
    c = golden_cfg(z)
    a = golden_csr(z)
    m, n = (int(v) for v in z["mn"])
    part = make_partition(a.shape[0], a.shape[1], m, n)
    hw = tuple(int(v) for v in z["hw"])
    layout = tv.PixelLayout.row_major(*hw)
    cfg = SolverConfig(mu=c["mu"], lam=max(c["lam"], 0.05), epochs=6,
                       prox=tv.ProxSettings(c["max_inner_iters"], c["tol"]))
    runs = []
    for mode in ("replicated", "slab"):
        shard = parallel.CudaShard(a, parallel.ShardSpec(part, 0, 1), lam=cfg.lam, layout=layout)
        drv = parallel.DistributedBSGD(shard, z["y"], cfg, x_true=z["x_true"], history_capacity=16, prox=mode)
        assert (drv.slab is not None) == (mode == "slab")
        xs = []
        for _ in range(4):
            drv.epoch_step()
            xs.append(drv.x_current.cpu().numpy())
        runs.append((xs, drv.history()))
    for xa, xb in zip(runs[0][0], runs[1][0]):
        assert np.array_equal(xa, xb)
    ha, hb = runs[0][1], runs[1][1]
    assert np.array_equal(ha[:, 0], hb[:, 0]) and np.array_equal(ha[:, 1], hb[:, 1])   # f_next, holds
    assert np.array_equal(ha[:, 4:9], hb[:, 4:9])   # TV, prox iterations / restarts / converged / fell back
    assert np.allclose(ha[:, 2:4], hb[:, 2:4], rtol=1e-12)   # |x|^2, |x - x*|^2 (summation order)


SPLIT_CASES = [((1, 64, 48), 0.3, 30, 1e-6), ((1, 128, 128), 2.0, 20, 1e-12), ((16, 12, 10), 0.4, 20, 1e-6),
               ((32, 32, 32), 0.05, 40, 1e-12), ((8, 8, 8), 1.0, 40, 1e-12), ((64, 128, 128), 0.05, 10, 1e-300)]


@pytest.mark.parametrize("dims,w,iters,tol", SPLIT_CASES)
def test_split_prox_matches_fused_bit_exact(cuda_ok, monkeypatch, dims, w, iters, tol):
    """The pass-per-kernel prox with device-side decisions (chosen for large
    volumes) equals the fused cooperative kernel: image, info, dual objectives."""
    import torch
    from paper_1812_01307_b200 import tv
    dev = torch.device("cuda", 0)
    vol = _volume(dims, 3)
    img = torch.from_numpy(vol if dims[0] > 1 else vol[0]).to(dev)
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("BSGD_PROX_SPLIT", mode)
        res, info = tv.tv_prox(img, w, tv.ProxSettings(iters, tol), return_info=True)
        out[mode] = (res.cpu().numpy(), info)
    (a, ia), (b, ib) = out["0"], out["1"]
    assert np.array_equal(a, b)
    assert (ia.iterations, ia.converged, ia.restarts, ia.fell_back) == (ib.iterations, ib.converged, ib.restarts,
                                                                         ib.fell_back)
    assert ia.dual_objectives == ib.dual_objectives
    if vol.size <= 4096:
        o, rep = orc.tv_prox3(vol, w, iters, tol) if dims[0] > 1 else orc.tv_prox(vol[0], w, iters, tol)
        assert np.array_equal(b, o) and ib.restarts == rep.restarts


def test_split_prox_fallback_matches_golden(cuda_ok, monkeypatch):
    import torch
    from paper_1812_01307_b200 import tv
    monkeypatch.setenv("BSGD_PROX_SPLIT", "1")
    z = load_golden("prox")
    for k in range(int(z["count"])):
        w, mi, tol = (float(v) for v in z[f"par{k}"])
        img = torch.from_numpy(z[f"in{k}"]).cuda()
        res, info = tv.tv_prox(img, w, tv.ProxSettings(int(mi), tol), return_info=True)
        assert np.array_equal(res.cpu().numpy(), z[f"out{k}"]), k
        assert [info.iterations, int(info.converged), info.restarts, int(info.fell_back)] == list(z[f"info{k}"]), k


def test_split_prox_epochs_match_fused(cuda_ok, monkeypatch):
    """Whole epochs (prox inside bsgd_epoch, graph-replayed run_solver) with the
    split prox equal the fused prox bit for bit."""
    from paper_1812_01307_b200 import blockops, solvers, tv
    z = load_golden("p1_ct")
    c = golden_cfg(z)
    a = golden_csr(z)
    m, n = (int(v) for v in z["mn"])
    hw = tuple(int(v) for v in z["hw"])
    layout = tv.PixelLayout(*hw, z["perm"])
    cfg = solvers.SolverConfig(mu=c["mu"], lam=max(c["lam"], 0.05), epochs=6,
                               prox=tv.ProxSettings(c["max_inner_iters"], c["tol"]))
    runs = []
    for mode in ("0", "1"):
        monkeypatch.setenv("BSGD_PROX_SPLIT", mode)
        op = blockops.BlockOperator(a, blockops.make_partition(a.shape[0], a.shape[1], m, n))
        st = solvers.init_bsgd_state(op, z["y"], cfg)
        xs = []
        for _ in range(3):
            solvers.bsgd_tv_iteration(st, op, z["y"], cfg, layout=layout)
            xs.append(st.x.copy())
        tr = solvers.run_solver("bsgd", solvers.Problem(op, z["y"], z["x_true"], layout), cfg)
        runs.append((xs, tr.final_x, [(s.epoch, s.relative_error, s.objective) for s in tr.samples]))
    for xa, xb in zip(runs[0][0], runs[1][0]):
        assert np.array_equal(xa, xb)
    assert np.array_equal(runs[0][1], runs[1][1]) and runs[0][2] == runs[1][2]


def test_distributed_slab_prox_device_capture_world1_nccl(cuda_ok):
    """DistributedBSGD(prox="slab") with device decisions at world size 1 (NCCL):
    capture() succeeds (the fixed-sequence prox has no host round trip) and graph
    replays equal eager epochs, which equal the replicated-prox epochs bit for bit."""
    import torch
    import torch.distributed as dist
    from paper_1812_01307_b200 import parallel, problems, tv
    from paper_1812_01307_b200.blockops import make_partition
    from paper_1812_01307_b200.solvers import SolverConfig
    n = 32
    a = problems.parallel_beam_matrix(n, 24, 47)
    rng = np.random.default_rng(9)
    y = a @ rng.random(n * n)
    part = make_partition(a.shape[0], a.shape[1], 4, 4)
    cfg = SolverConfig(mu=5e-4, lam=2.0, epochs=10, monitor_decrease=True, prox=tv.ProxSettings(10, 1e-6))
    lay = tv.PixelLayout.row_major(n, n)
    dist.init_process_group("nccl", store=dist.HashStore(), rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        runs = []
        for mode in ("replicated", "eager", "graph"):
            shard = parallel.CudaShard(a, parallel.ShardSpec(part, 0, 1), lam=cfg.lam, layout=lay)
            drv = parallel.DistributedBSGD(shard, y, cfg, history_capacity=16,
                                           prox="replicated" if mode == "replicated" else "slab")
            assert (drv.slab is not None) == (mode != "replicated")
            drv.epoch_step()
            if mode == "graph":
                assert drv.slab_device and drv.capture(2)
                for _ in range(3):
                    drv.replay()
            else:
                for _ in range(6):
                    drv.epoch_step()
            torch.cuda.synchronize()
            runs.append((drv.x_current.cpu().numpy(), drv.r_current.cpu().numpy(), drv.history()))
    finally:
        dist.destroy_process_group()
    (x0, r0, h0), (x1, r1, h1), (x2, r2, h2) = runs
    assert np.array_equal(x0, x1) and np.array_equal(x1, x2)
    assert np.array_equal(r1, r2) and np.array_equal(h1, h2)
    assert np.array_equal(h0[:, 4:9], h1[:, 4:9])   # TV and prox iterations / restarts / converged / fell back
    assert h1[:, 5].max() > 1
