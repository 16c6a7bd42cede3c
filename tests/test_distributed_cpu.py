"""World-size-2 and -3 gloo runs of the multi-GPU host logic (node shards,
global rho, both adjoint partitions: coefficient all-reduce, and the grid
reduce-scatter over the touched planes -> slab 2-D FFT -> all-to-all planes
to columns -> 1-D FFT along axis 0 -> eta gathered to the root -> basal
adjoint, or the packed planes gathered to the root) with the CPU oracle
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

    def planes(p):
        mask = np.zeros(p.grid[0], dtype=np.uint8)
        for off in range(-p.q, p.q + 1):
            mask[(p.base[0] + off) % p.grid[0]] = 1
        return mask

    def axis0(p, cols, col0):
        n0 = p.n_axis[0]
        crop2 = p.n_axis[2]
        X = np.fft.fft(np.asarray(cols), axis=0)[(np.arange(n0) - n0 // 2) % p.grid[0]]
        j = col0 + np.arange(X.shape[1])
        s = (2 * np.pi) ** 3 / np.prod(p.grid) * p.deconv[1][j // crop2] * p.deconv[2][j % crop2]
        return X * p.deconv[0][:, None] * s[None, :]

    return Compute(plan=lambda B, pts, rho, **kw: o.oracle_plan(B, pts, rho=rho, **kw),
                   forward=lambda p, c: o.oracle_forward(p, c, threads=1),
                   adjoint=lambda p, v: o.oracle_adjoint(p, v, threads=1),
                   spread=lambda p, v: o.scatter(p.grid, p.base, p.win, np.asarray(v, complex), p.q, threads=1),
                   grid_info=lambda p: (p.grid[0], p.n_axis[1], p.n_axis[2]),
                   slab_fft=slab_fft, from_packed=from_packed, planes=planes, axis0=axis0,
                   from_eta=lambda p, eta: o.basal_adjoint(p, np.asarray(eta)))


def _worker(rank, world, port, name, outdir, partition, exchange="alltoall"):
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
                     exchange=exchange, compact_k1=bool(g["compact"]))
    f = sp.forward(g["coeffs"])
    a = sp.adjoint(g["values"][s:e])
    np.savez(os.path.join(outdir, f"r{rank}.npz"), f=f, a=a, rho=sp.rho, s=s, e=e, part=sp.partition,
             pieces=np.array(sp.last_pieces or [], dtype=np.int64).reshape(-1, 4))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,world,partition,exchange", [
    ("b8_q16", 2, "coeffs", "alltoall"), ("b5_q10", 2, "coeffs", "alltoall"),
    ("b8_q16", 2, "grid", "alltoall"), ("b5_q10", 3, "grid", "alltoall"), ("b6_q6_compact", 2, "grid", "alltoall"),
    ("b8_q16", 3, "grid", "gather"), ("b6_q6_compact", 2, "grid", "gather")])
def test_rank_shards_match_single_process(name, world, partition, exchange, tmp_path, oracle_built):
    mp.spawn(_worker, args=(world, _free_port(), name, str(tmp_path), partition, exchange), nprocs=world,
             join=True)
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


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_plane_pieces_own_every_touched_plane_once(world):
    """plane_pieces / owned_planes: every touched plane has exactly one owner,
    every widened block lies inside [0, N0) and blocks of different pieces do
    not overlap (the in-place reduce-scatter writes whole blocks)."""
    from paper_1809_10786_b200.distributed import owned_planes, plane_pieces
    rng = np.random.default_rng(world)
    masks = []
    for n0 in (16, 64, 512):
        for lo, hi in ((0, n0 // 2 + 5), (n0 - 3, n0 // 2 + 7), (3, 9)):   # plain, wrapping, narrow arcs
            m = np.zeros(n0, bool)
            idx = np.arange(lo, lo + ((hi - lo) % n0)) % n0
            m[idx] = True
            masks.append(m)
        masks.append(rng.random(n0) < 0.3)
        masks.append(np.ones(n0, bool))
        masks.append(np.zeros(n0, bool))
    for m in masks:
        n0 = m.size
        pieces = plane_pieces(m, world)
        if not m.any():
            assert pieces == []
            continue
        cnt = np.zeros(n0, int)
        for k in range(world):
            for a0, a1 in owned_planes(pieces, k, world):
                cnt[a0:a1] += 1
        assert np.all(cnt[m] == 1) and cnt.max() == 1
        spans = []
        for s0, blk, ps, pe in pieces:
            assert 0 <= s0 <= ps < pe <= n0 and s0 + blk * world >= pe
            if s0 + blk * world <= n0:
                spans.append((s0, s0 + blk * world))
        if len(spans) == 2:
            assert max(spans[0][0], spans[1][0]) >= min(spans[0][1], spans[1][1])
    # the BASELINE geometry (B = 64, q = 16): half the planes plus the windows
    m = np.zeros(512, bool)
    m[:273] = True
    m[-16:] = True
    pieces = plane_pieces(m, 8)
    assert sum(pe - ps for _, _, ps, pe in pieces) == 289


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


def test_shard_indices_partition():
    """Both shard modes partition the node indices into count-balanced,
    ascending shards; radial shards are ordered shells in r."""
    import numpy as np
    from paper_1809_10786_b200.distributed import shard_indices, shard_bounds
    rng = np.random.default_rng(3)
    pts = rng.random((1001, 3)) * [7.0, 3.0, 6.0]
    for mode in ("contiguous", "radial", "theta"):
        parts = [shard_indices(pts, k, 4, mode) for k in range(4)]
        if mode != "theta":   # (theta: equal shares of weighted work)
            assert [len(x) for x in parts] == [b - a for a, b in (shard_bounds(1001, k, 4) for k in range(4))]
        assert np.array_equal(np.sort(np.concatenate(parts)), np.arange(1001))
        assert all(np.all(np.diff(x) > 0) for x in parts)
    th = [shard_indices(pts, k, 4, "theta") for k in range(4)]
    assert all(pts[th[k], 1].max() <= pts[th[k + 1], 1].min() for k in range(3))
    assert abs(len(th[0]) - 1001 / 4) < 60
    rad = [shard_indices(pts, k, 4, "radial") for k in range(4)]
    assert all(pts[rad[k], 0].max() <= pts[rad[k + 1], 0].min() for k in range(3))
    import pytest
    with pytest.raises(ValueError):
        shard_indices(pts, 0, 4, "spiral")
