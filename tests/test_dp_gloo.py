"""Multi-process (world_size 2, gloo, CPU) tests of the data-parallel host logic
(paper_2412_02244_b200/dp.py): bbox MIN/MAX + n SUM all-reduce, one int64 SUM all-reduce
of the partials per iteration, identical refine on every rank.  The shard backend is the
test-only NumpyShard; the sharded run must equal the single-process run bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, outdir):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from dp_numpy_shard import NumpyShard
    from paper_2412_02244_b200.dp import lloyd_dp
    P, C0, iters, tol = case
    parts = np.array_split(np.arange(len(P)), world)
    sh = NumpyShard(P[parts[rank]], len(C0))
    res = lloyd_dp(sh, torch.from_numpy(C0), iters, tol, comm_device="cpu")
    np.save(os.path.join(outdir, f"lab{rank}.npy"), res.labels.numpy())
    np.save(os.path.join(outdir, f"C{rank}.npy"), res.centroids.numpy())
    np.save(os.path.join(outdir, f"meta{rank}.npy"), np.array([res.iterations, res.sse]))
    dist.destroy_process_group()


def _single(case):
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from dp_numpy_shard import NumpyShard
    from paper_2412_02244_b200.dp import lloyd_dp
    P, C0, iters, tol = case
    return lloyd_dp(NumpyShard(P, len(C0)), torch.from_numpy(C0), iters, tol, comm_device="cpu")


@pytest.mark.parametrize("seed,d,k,iters,tol", [(1, 2, 8, 6, -1.0), (2, 3, 12, 50, 0.0), (3, 2, 5, 4, -1.0),
                                               (4, 32, 6, 5, -1.0), (5, 128, 9, 30, 0.0)])
def test_dp_two_ranks_equals_single(tmp_path, seed, d, k, iters, tol):
    P, C0 = synth.random_instance(seed, 3001, d, k, "blobs")
    case = (P, C0, iters, tol)
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), case, str(tmp_path)), nprocs=world, join=True)
    ref = _single(case)
    labs = np.concatenate([np.load(tmp_path / f"lab{r}.npy") for r in range(world)])
    np.testing.assert_array_equal(labs, ref.labels.numpy())
    for r in range(world):
        np.testing.assert_array_equal(np.load(tmp_path / f"C{r}.npy"), ref.centroids.numpy())
        it, sse = np.load(tmp_path / f"meta{r}.npy")
        assert int(it) == ref.iterations
        assert sse == ref.sse   # Eq. 1 summed in fixed point: order- and sharding-independent
    if tol < 0:
        assert ref.iterations == iters


def test_dp_single_matches_oracle():
    """The orchestration with one shard is plain Lloyd (oracle mode A, within R10)."""
    import oracle
    from helpers import assert_centroids_close, assert_sse_close
    P, C0 = synth.random_instance(9, 2000, 3, 10, "uniform")
    res = _single((P, C0, 8, -1.0))
    r = oracle.lloyd(P, C0.astype(np.float64), 8, -1.0, True)
    np.testing.assert_array_equal(res.labels.numpy(), r.labels)
    assert_centroids_close(res.centroids.numpy(), r.centroids, P)
    assert_sse_close(res.sse, r.sse, rel=1e-12)
