"""World-size-2 and -3 gloo runs of the multi-GPU host logic (node shards,
global rho, both adjoint partitions: coefficient all-reduce, and the grid
reduce-scatter -> slab 2-D FFT -> gather -> root finish) with the CPU oracle
standing in for the per-rank device compute.  The sharded forward
concatenates to, and the sharded adjoint sums to, the reference's
single-process result."""
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


def oracle_compute():
    """The CPU oracle as each rank's compute, including the grid partition's
    stage functions (spread, slab 2-D FFT + spectral box, root finish): the
    same arithmetic as the reference's adjoint (nfft.py:254-273,
    transform.py:398-429) split at the slab boundary."""
    from oracle import sgl_oracle as o
    from paper_1809_10786_b200.distributed import Compute

    def slab_fft(p, grid, a0, a1):
        g = np.fft.fft2(grid[a0:a1], axes=(1, 2))
        n1, n2 = p.n_axis[1], p.n_axis[2]
        i1 = (np.arange(n1) - n1 // 2) % p.grid[1]
        i2 = (np.arange(n2) - n2 // 2) % p.grid[2]
        return g[:, i1][:, :, i2]

    def from_packed(p, packed):
        n0 = p.n_axis[0]
        g = np.fft.fft(np.asarray(packed), axis=0)[(np.arange(n0) - n0 // 2) % p.grid[0]]
        return o.basal_adjoint(p, o._deconvolve(g / np.prod(p.grid), p.deconv))

    return Compute(plan=lambda B, pts, rho, **kw: o.oracle_plan(B, pts, rho=rho, **kw),
                   forward=lambda p, c: o.oracle_forward(p, c, threads=1),
                   adjoint=lambda p, v: o.oracle_adjoint(p, v, threads=1),
                   spread=lambda p, v: o.scatter(p.grid, p.base, p.win, np.asarray(v, complex), p.q, threads=1),
                   grid_info=lambda p: (p.grid[0], p.n_axis[1], p.n_axis[2]),
                   slab_fft=slab_fft, from_packed=from_packed)


def _worker(rank, world, port, name, outdir, partition):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from paper_1809_10786_b200.distributed import ShardedPlan, shard_bounds

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = load_golden(name)
    s, e = shard_bounds(g["points"].shape[0], rank, world)
    sp = ShardedPlan(int(g["B"]), g["points"][s:e], compute=oracle_compute(), q=int(g["q"]), partition=partition,
                     compact_k1=bool(g["compact"]))
    f = sp.forward(g["coeffs"])
    a = sp.adjoint(g["values"][s:e])
    np.savez(os.path.join(outdir, f"r{rank}.npz"), f=f, a=a, rho=sp.rho, s=s, e=e, part=sp.partition)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,world,partition", [("b8_q16", 2, "coeffs"), ("b5_q10", 2, "coeffs"),
                                                  ("b8_q16", 2, "grid"), ("b5_q10", 3, "grid"),
                                                  ("b6_q6_compact", 2, "grid")])
def test_rank_shards_match_single_process(name, world, partition, tmp_path, oracle_built):
    mp.spawn(_worker, args=(world, _free_port(), name, str(tmp_path), partition), nprocs=world, join=True)
    g = load_golden(name)
    r = [np.load(tmp_path / f"r{k}.npz") for k in range(world)]
    # rho is the all-reduce max over shards == the single-process choose_rho
    assert all(float(x["rho"]) == float(g["rho"]) for x in r)
    f = np.concatenate([x["f"] for x in r])
    assert np.max(np.abs(f - g["fwd"])) <= 1e-12 * np.max(np.abs(g["fwd"]))
    for x in r:
        assert str(x["part"]) == partition
        assert np.max(np.abs(x["a"] - g["adj"])) <= 1e-12 * np.max(np.abs(g["adj"]))
    assert all(np.array_equal(r[0]["a"], x["a"]) for x in r)


def test_partition_model_prefers_the_coefficient_allreduce_on_nvswitch():
    from paper_1809_10786_b200.distributed import partition_model
    for B in (64, 128):
        for world in (2, 4, 8):
            m = partition_model(B, world)
            assert m["choice"] == "coeffs" and m["grid"] > m["coeffs"] > 0
    # with a slow link the replicated FFT is not what dominates either way
    assert partition_model(64, 1)["choice"] == "coeffs"


def test_shard_bounds_cover():
    from paper_1809_10786_b200.distributed import shard_bounds
    for M in (0, 1, 7, 100, 101):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(M, k, world) for k in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == M
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(e - s for s, e in spans) - min(e - s for s, e in spans) <= 1
