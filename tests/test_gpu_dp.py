"""GPU tests of the data-parallel C-ABI path (km_dp_*): several shards driven from one
process on one GPU (the all-reduce is an in-process sum; no kernels wait on one another).
Exact integer sums make any sharding bit-identical to one context holding all points."""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2412_02244_b200 as kmb  # noqa: E402
from paper_2412_02244_b200.dp import LibkmShard, lloyd_multi_shard  # noqa: E402


def single(P, C0, iters, tol, mode):
    n, d = P.shape
    k = C0.shape[0]
    ctx = kmb.Context(n, d, k)
    kmb.km_set_mode(ctx.handle, mode)
    C = torch.empty((k, d), dtype=torch.float32, device="cuda")
    lab = torch.empty(n, dtype=torch.int32, device="cuda")
    it, sse = kmb.km_run_ctx(ctx.handle, torch.from_numpy(P).cuda(), torch.from_numpy(C0).cuda(), iters, tol, C, lab)
    ctx.close()
    return it, sse, C.cpu().numpy(), lab.cpu().numpy()


@pytest.mark.parametrize("nshards", [2, 3])
@pytest.mark.parametrize("mode", [kmb.KM_MODE_BRUTE, kmb.KM_MODE_TILES])
@pytest.mark.parametrize("cfg,n,tol", [(2, 300_000, -1.0), (3, 200_000, -1.0), (2, 200_000, 0.0)])
def test_shards_bit_identical(nshards, mode, cfg, n, tol):
    w = synth.config(cfg, n=n)
    iters = 8 if tol < 0 else 200
    it1, sse1, C1, lab1 = single(w.points, w.init, iters, tol, mode)
    idx = np.array_split(np.arange(w.n), nshards)
    shards = [LibkmShard(torch.from_numpy(np.ascontiguousarray(w.points[i])).cuda(), w.k, mode) for i in idx]
    res = lloyd_multi_shard(shards, torch.from_numpy(w.init).cuda(), iters, tol)
    for r in res:
        assert r.iterations == it1
        np.testing.assert_array_equal(r.centroids.cpu().numpy(), C1)
    np.testing.assert_array_equal(np.concatenate([r.labels.cpu().numpy() for r in res]), lab1)
    assert res[0].sse == sse1   # Eq. 1 in fixed point: bit-identical across shardings
    for s in shards:
        s.close()


@pytest.mark.parametrize("nshards", [2, 3])
@pytest.mark.parametrize("cfg,n,k,tol", [(6, 30_000, 300, -1.0), (7, 20_000, 2600, -1.0), (6, 30_000, 100, 0.0)])
def test_shards_bit_identical_high_d(nshards, cfg, n, k, tol):
    """The high-dimensional variant (NEXT-4) sharded: the fixed point and the centring origin
    come from the all-reduced box, the running sums are exact integers, so the centroids,
    labels and iteration count equal one context holding all points."""
    w = synth.config(cfg, n=n, k=k)
    iters = 5 if tol < 0 else 100
    it1, sse1, C1, lab1 = single(w.points, w.init, iters, tol, kmb.KM_MODE_AUTO)
    idx = np.array_split(np.arange(w.n), nshards)
    shards = [LibkmShard(torch.from_numpy(np.ascontiguousarray(w.points[i])).cuda(), w.k, kmb.KM_MODE_AUTO)
              for i in idx]
    res = lloyd_multi_shard(shards, torch.from_numpy(w.init).cuda(), iters, tol)
    for r in res:
        assert r.iterations == it1
        np.testing.assert_array_equal(r.centroids.cpu().numpy(), C1)
    np.testing.assert_array_equal(np.concatenate([r.labels.cpu().numpy() for r in res]), lab1)
    assert res[0].sse == sse1   # Eq. 1 in fixed point: bit-identical across shardings
    for s in shards:
        s.close()


@pytest.mark.parametrize("d,nshards", [(100, 2), (20, 3)])
def test_shards_bit_identical_padded_width(d, nshards):
    """Padded widths (d outside the native set) sharded: box and centroids in the caller's d,
    the partial in the padded width (km_dp_partial_len); equal to one context and, for the
    labels, to the oracle."""
    import oracle
    n, k, iters = 12_000, 40, 4
    P, C0 = synth.random_instance(300 + d, n, d, k, "blobs")
    it1, sse1, C1, lab1 = single(P, C0, iters, -1.0, kmb.KM_MODE_AUTO)
    idx = np.array_split(np.arange(n), nshards)
    shards = [LibkmShard(torch.from_numpy(np.ascontiguousarray(P[i])).cuda(), k, kmb.KM_MODE_AUTO) for i in idx]
    pd = 32 if d <= 32 else 64 if d <= 64 else 128 if d <= 128 else 256
    assert shards[0].partial.numel() == k * pd + 2 * k + 1   # sums, counts, changed, Q
    res = lloyd_multi_shard(shards, torch.from_numpy(C0).cuda(), iters, -1.0)
    for r in res:
        assert r.iterations == it1 == iters
        assert tuple(r.centroids.shape) == (k, d)
        np.testing.assert_array_equal(r.centroids.cpu().numpy(), C1)
    lab = np.concatenate([r.labels.cpu().numpy() for r in res])
    np.testing.assert_array_equal(lab, lab1)
    ref = oracle.lloyd(P, C0.astype(np.float64), iters, tol=-1.0)
    np.testing.assert_array_equal(lab, ref.labels)
    assert res[0].sse == sse1   # Eq. 1 in fixed point: bit-identical across shardings
    for s in shards:
        s.close()


def _mp_worker(rank, world, port, cfg, n, iters, tol, outdir):
    import os
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist
    from paper_2412_02244_b200.dp import LibkmShard, lloyd_dp
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = synth.config(cfg, n=n)
    idx = np.array_split(np.arange(w.n), world)[rank]
    sh = LibkmShard(torch.from_numpy(np.ascontiguousarray(w.points[idx])).cuda(), w.k)
    # gloo with CUDA tensors: the all-reduce runs through host memory (no kernel waits on another)
    res = lloyd_dp(sh, torch.from_numpy(w.init).cuda(), iters, tol)
    np.save(os.path.join(outdir, f"lab{rank}.npy"), res.labels.cpu().numpy())
    np.save(os.path.join(outdir, f"C{rank}.npy"), res.centroids.cpu().numpy())
    np.save(os.path.join(outdir, f"meta{rank}.npy"), np.array([res.iterations, res.sse]))
    sh.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg,n,iters,tol", [(3, 150_000, 6, -1.0), (2, 100_000, 200, 0.0), (6, 20_000, 4, -1.0)])
def test_two_processes_libkm_equal_single(tmp_path, cfg, n, iters, tol):
    """Two processes (world size 2, gloo over CUDA tensors), each a LibkmShard on cuda:0 driven
    by dp.lloyd_dp -- the exact host orchestration bench.py --gpus N runs over NCCL: labels,
    centroids, iterations and Eq. 1 equal one context holding all points, bit for bit."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_mp_worker, args=(2, port, cfg, n, iters, tol, str(tmp_path)), nprocs=2, join=True)
    w = synth.config(cfg, n=n)
    it1, sse1, C1, lab1 = single(w.points, w.init, iters, tol, kmb.KM_MODE_AUTO)
    lab = np.concatenate([np.load(tmp_path / f"lab{r}.npy") for r in range(2)])
    np.testing.assert_array_equal(lab, lab1)
    for r in range(2):
        np.testing.assert_array_equal(np.load(tmp_path / f"C{r}.npy"), C1)
        it, sse = np.load(tmp_path / f"meta{r}.npy")
        assert int(it) == it1 and sse == sse1
