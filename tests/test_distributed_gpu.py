"""World-size-2 runs of the multi-GPU path with the CUDA compute
(`distributed.cuda_compute`): both ranks on GPU 0 with the gloo backend (the
box has one GPU; the collectives go through host copies), node shards of one
transform, both adjoint partitions -- the coefficient all-reduce and the
north star's grid reduce-scatter over the touched planes -> slab 2-D FFT ->
all-to-all (planes to columns) -> 1-D FFT along axis 0 -> eta to the root ->
basal adjoint, through the C ABI stage entry points (sgl_adjoint_spread /
_slab_fft / sgl_plan_planes / _axis0 / _from_eta, and _from_packed for the
gather exchange).  The sharded results must equal the single-process ones and
the reference goldens."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT, load_golden

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, name, outdir, partition, backend, exchange):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from paper_1809_10786_b200.distributed import ShardedPlan, shard_bounds

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = load_golden(name)
    c = g["coeffs"] if "coeffs" in g else None
    M = g["points"].shape[0]
    s, e = shard_bounds(M, rank, world)
    # rho: the golden's (pinned to the full config's node set for the cfg subsets)
    sp = ShardedPlan(int(g["B"]), g["points"][s:e], q=int(g["q"]), partition=partition, backend=backend,
                     exchange=exchange,
                     device=0, compact_k1=bool(g["compact"]), rho=float(g["rho"]))
    f = sp.forward(c)
    a = sp.adjoint(g["values"][s:e])
    # device tensors in and out as well
    dev = torch.device("cuda", 0)
    ad = sp.adjoint(torch.as_tensor(g["values"][s:e], device=dev))
    np.savez(os.path.join(outdir, f"r{rank}.npz"), f=f, a=a, ad=ad.cpu().numpy(), rho=sp.rho, part=sp.partition)
    dist.barrier()
    dist.destroy_process_group()


def rel(x, ref):
    return float(np.max(np.abs(np.asarray(x) - ref)) / np.max(np.abs(ref)))


@pytest.mark.parametrize("name,partition,backend,exchange", [
    ("b12_q12", "grid", "auto", "alltoall"), ("b12_q12", "grid", "auto", "gather"),
    ("b12_q12", "coeffs", "auto", "alltoall"), ("cfg2_sub20k", "grid", "i8", "alltoall"),
    ("cfg2_sub20k", "coeffs", "tiled", "alltoall"), ("b6_q6_compact", "grid", "auto", "alltoall"),
    ("b6_q6_compact", "grid", "auto", "gather")])
def test_two_ranks_on_one_gpu_match_single_process(name, partition, backend, exchange, tmp_path):
    import paper_1809_10786_b200 as sgl
    g = load_golden(name)
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), name, str(tmp_path), partition, backend, exchange), nprocs=world,
             join=True)
    r = [np.load(tmp_path / f"r{k}.npz") for k in range(world)]
    assert all(str(x["part"]) == partition for x in r)
    assert all(float(x["rho"]) == float(g["rho"]) for x in r)
    p = sgl.plan(int(g["B"]), g["points"], q=int(g["q"]), rho=float(g["rho"]), backend=backend,
                 compact_k1=bool(g["compact"]))
    f1, a1 = sgl.forward(p, g["coeffs"]), sgl.adjoint(p, g["values"])
    f = np.concatenate([x["f"] for x in r])
    assert rel(f, f1) <= 1e-11 and rel(f, g["fwd"]) <= 1e-10
    for x in r:
        assert rel(x["a"], a1) <= 1e-11 and rel(x["a"], g["adj"]) <= 1e-10
        assert rel(x["ad"], x["a"]) <= 1e-12
    assert np.array_equal(r[0]["a"], r[1]["a"])


@pytest.mark.parametrize("name", ["b12_q12", "cfg2_sub20k"])
def test_single_process_multi_device_plan(name):
    """sgl_plan_create_multi (the C ABI's n_gpus): two sub-plans -- on one
    GPU here (devices [0, 0]); on a multi-GPU box, [0, 1] -- over node shards;
    forward slices and summed adjoint equal the single plan and the goldens."""
    import torch
    import paper_1809_10786_b200 as sgl
    g = load_golden(name)
    kw = dict(q=int(g["q"]), rho=float(g["rho"]))
    pm = sgl.plan(int(g["B"]), g["points"], devices=[0, 0], **kw)
    assert pm._info.n_gpus == 2 and pm.m_points == g["points"].shape[0]
    p1 = sgl.plan(int(g["B"]), g["points"], **kw)
    f, a = sgl.forward(pm, g["coeffs"]), sgl.adjoint(pm, g["values"])
    assert rel(f, sgl.forward(p1, g["coeffs"])) <= 1e-11 and rel(f, g["fwd"]) <= 1e-10
    assert rel(a, sgl.adjoint(p1, g["values"])) <= 1e-11 and rel(a, g["adj"]) <= 1e-10
    C = np.stack([g["coeffs"], 2 * g["coeffs"]])
    F = sgl.forward(pm, C)
    assert F.shape == (2, f.size) and rel(F[1], 2 * f) <= 1e-12
    dev = torch.device("cuda", 0)
    fd = sgl.forward(pm, torch.as_tensor(g["coeffs"], device=dev))
    ad = sgl.adjoint(pm, torch.as_tensor(g["values"], device=dev))
    assert rel(fd.cpu().numpy(), f) <= 1e-13 and rel(ad.cpu().numpy(), a) <= 1e-13
    f2, a2 = sgl.forward_adjoint(pm, g["coeffs"], g["values"])
    assert rel(f2, f) <= 1e-13 and rel(a2, a) <= 1e-13
    with pytest.raises(ValueError):
        sgl.plan(4, g["points"][:10], devices=[0, 99])
