"""World-size-2 gloo run of the multi-GPU host logic (node shards, global rho,
adjoint all-reduce) with the CPU oracle standing in for the per-rank device
compute.  The sharded forward concatenates to, and the sharded adjoint sums
to, the reference's single-process result."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT, load_golden


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, name, outdir):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from oracle import sgl_oracle as o
    from paper_1809_10786_b200.distributed import Compute, ShardedPlan, shard_bounds

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = load_golden(name)
    s, e = shard_bounds(g["points"].shape[0], rank, world)
    comp = Compute(plan=lambda B, pts, rho, **kw: o.oracle_plan(B, pts, rho=rho, **kw),
                   forward=lambda p, c: o.oracle_forward(p, c, threads=1),
                   adjoint=lambda p, v: o.oracle_adjoint(p, v, threads=1))
    sp = ShardedPlan(int(g["B"]), g["points"][s:e], compute=comp, q=int(g["q"]))
    f = sp.forward(g["coeffs"])
    a = sp.adjoint(g["values"][s:e])
    np.savez(os.path.join(outdir, f"r{rank}.npz"), f=f, a=a, rho=sp.rho, s=s, e=e)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["b8_q16", "b5_q10"])
def test_two_rank_shards_match_single_process(name, tmp_path, oracle_built):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), name, str(tmp_path)), nprocs=world, join=True)
    g = load_golden(name)
    r = [np.load(tmp_path / f"r{k}.npz") for k in range(world)]
    # rho is the all-reduce max over shards == the single-process choose_rho
    assert all(float(x["rho"]) == float(g["rho"]) for x in r)
    f = np.concatenate([x["f"] for x in r])
    assert np.max(np.abs(f - g["fwd"])) <= 1e-12 * np.max(np.abs(g["fwd"]))
    for x in r:
        assert np.max(np.abs(x["a"] - g["adj"])) <= 1e-12 * np.max(np.abs(g["adj"]))
    assert np.array_equal(r[0]["a"], r[1]["a"])


def test_shard_bounds_cover():
    from paper_1809_10786_b200.distributed import shard_bounds
    for M in (0, 1, 7, 100, 101):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(M, k, world) for k in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == M
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(e - s for s, e in spans) - min(e - s for s, e in spans) <= 1
