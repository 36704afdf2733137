"""Multi-process (gloo, CPU) tests of the row-strip sharding host logic used by
multi-GPU runs: strip planning, the NCCL-style neighbour halo exchange through
torch.distributed, and the band schedule handed to lfe_extract_rows.  The
compute on each band is the CPU oracle here (no GPU); the GPU-side equality of
lfe_extract_rows with lfe_extract is tested in test_gpu_parity.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_1304_3992_b200 import scenes
from paper_1304_3992_b200.shard import BandShard, StripShard, plan_bands, plan_strips


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_plan_strips_covers_and_balances():
    for H in (7, 8, 100, 12000, 12001):
        for world in (1, 2, 3, 4, 8):
            if world > 1 and H // world < 7:
                with pytest.raises(ValueError):
                    plan_strips(H, world, 7)
                continue
            p = plan_strips(H, world, 7)
            assert p[0][0] == 0 and p[-1][1] == H
            assert all(a1 == b0 for (_, a1), (b0, _) in zip(p, p[1:]))
            sizes = [b - a for a, b in p]
            assert max(sizes) - min(sizes) <= 1


def test_bands_partition_each_strip():
    for world in (1, 2, 3, 8):
        for r in range(world):
            sh = StripShard(12000, 64, r, world, 7)
            bands = sh.bands()
            rows = sorted((s, s + n) for s, n, *_ in bands)
            assert rows[0][0] == 0 and rows[-1][1] == sh.rows
            assert all(a1 == b0 for (_, a1), (b0, _) in zip(rows, rows[1:]))
            # the first band never needs the exchange (it overlaps it)
            assert bands[0][5] is False


def _worker(rank, world, port, H, W, hm, q, staged=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        img = scenes.scene_c1(size=max(H, W))[:H, :W].copy()
        p = O.Params(bit_depth=8, zc_threshold=(0.01, 0.01), hybrid_median=hm)
        halo = 7 if hm else 5
        sh = StripShard(H, W, rank, world, halo)
        buf = sh.alloc(torch.uint8, "cpu")
        sh.load_owned(img)
        # staged: the host-staged variant used for gloo groups over device buffers
        # (the one-GPU N > 1 bench hook), here exercised on CPU buffers
        for w in sh.exchange(staged=staged):
            w.wait()
        # received halos equal the neighbours' boundary rows
        if sh.ha:
            assert np.array_equal(buf[:sh.ha].numpy(), img[sh.a - sh.ha:sh.a])
        if sh.hb:
            assert np.array_equal(buf[sh.ha + sh.rows:].numpy(), img[sh.b:sh.b + sh.hb])
        # run every band the way bench.py hands it to lfe_extract_rows
        out = np.zeros((sh.rows, W), np.uint8)
        B = buf.numpy()
        for s, n, ha, hb, flags, _ in sh.bands():
            r0 = sh.ha + s
            sub = np.ascontiguousarray(B[r0 - ha:r0 + n + hb])
            out[s:s + n] = O.run(sub, p)[ha:ha + n]
        q.put((rank, sh.a, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,H,hm,staged", [(2, 96, True, False), (3, 61, True, False), (2, 40, False, False),
                                               (3, 61, True, True)])
def test_gloo_strips_reproduce_whole_image(world, H, hm, staged):
    W = 72
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, H, W, hm, q, staged)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = [q.get(timeout=240) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    img = scenes.scene_c1(size=max(H, W))[:H, :W].copy()
    whole = O.run(img, O.Params(bit_depth=8, zc_threshold=(0.01, 0.01), hybrid_median=hm))
    full = np.zeros_like(whole)
    for _, a, out in got:
        full[a:a + out.shape[0]] = out
    np.testing.assert_array_equal(full, whole)


def _stats_worker(rank, world, port, H, W, q_out):
    """Each rank: partial exact sums of its OWNED rows (LoG over strip + halo,
    clamped only at the true image edges), then the SUM all-reduce."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        img = scenes.random_image(np.random.default_rng(77), H, W, 10, "mixed")
        sh = StripShard(H, W, rank, world, 2)  # LoG radius: the only halo the statistics read
        buf = sh.alloc(torch.int64, "cpu")
        sh.load_owned(img.astype(np.int64))
        for w in sh.exchange():
            w.wait()
        B = buf.numpy().astype(np.uint16)
        v = [sh.rows * W]
        rs, hi, lo = [], [], []
        for s in (0.5, 20.0):
            q, _ = O.mask_int(s, 5, 10)
            r = O.log_response(B, q)[sh.ha:sh.ha + sh.rows].astype(object)
            rs.append(int(r.sum()))
            sq = [int(x) * int(x) for x in r.ravel()]
            hi.append(sum(x >> 24 for x in sq))
            lo.append(sum(x & 0xFFFFFF for x in sq))
        I = B[sh.ha:sh.ha + sh.rows].astype(np.int64)
        v += rs + hi + lo + [int(I.sum()), int((I * I).sum())]
        t = torch.tensor(v, dtype=torch.int64)
        sh.allreduce_stats(t)
        q_out.put((rank, t.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_stats_allreduce_equals_whole_image(world):
    H, W = 61, 45
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_stats_worker, args=(r, world, port, H, W, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = [q.get(timeout=240) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    img = scenes.random_image(np.random.default_rng(77), H, W, 10, "mixed")
    for _, v in got:
        assert v[0] == H * W
        for j, s in enumerate((0.5, 20.0)):
            qm, _ = O.mask_int(s, 5, 10)
            r = O.log_response(img, qm)
            assert v[1 + j] == int(r.sum())
            assert v[3 + j] * 2**24 + v[5 + j] == sum(int(x) ** 2 for x in r.ravel())
            # and the threshold the library resolves from them equals the oracle's sigma
            assert O.global_std(v[0], v[1 + j], v[3 + j] * 2**24 + v[5 + j]) == O.std_of_response(r)


@pytest.mark.parametrize("bands,world", [(4, 1), (4, 2), (4, 3), (4, 4), (4, 8), (3, 8), (4, 6), (1, 5)])
def test_plan_bands_covers_every_band_row_once(bands, world):
    from paper_1304_3992_b200.shard import plan_bands
    H = 8192
    work = plan_bands(bands, H, world, 7)
    assert len(work) == world
    cover = {b: [] for b in range(bands)}
    for items in work:
        for b, a, e in items:
            cover[b].append((a, e))
    for b, rs in cover.items():
        rs.sort()
        assert rs[0][0] == 0 and rs[-1][1] == H
        assert all(x[1] == y[0] for x, y in zip(rs, rs[1:]))
    rows = [sum(e - a for _, a, e in items) for items in work]
    assert min(rows) > 0 and max(rows) <= 1.01 * (bands * H / world) + 7
    for items in work:  # every partial band keeps >= halo rows (one exchange suffices)
        for b, a, e in items:
            assert e - a >= 7 or (a, e) == (0, H)
    if bands % world == 0:  # whole bands, no exchange
        assert all(a == 0 and e == H for items in work for _, a, e in items)


@pytest.mark.parametrize("bands,H,world", [(1, 100, 30), (2, 40, 13), (1, 20, 3)])
def test_plan_bands_rejects_pieces_shorter_than_the_halo(bands, H, world):
    """A band piece cut on either side needs a halo of rows of its own, or one
    neighbour exchange no longer suffices (as plan_strips, which raises)."""
    from paper_1304_3992_b200.shard import plan_bands
    with pytest.raises(ValueError):
        plan_bands(bands, H, world, 7)


def test_plan_bands_short_whole_bands_are_fine():
    from paper_1304_3992_b200.shard import plan_bands
    work = plan_bands(4, 5, 4, 7)  # bands shorter than the halo, dealt out whole
    assert work == [[(0, 0, 5)], [(1, 0, 5)], [(2, 0, 5)], [(3, 0, 5)]]


def _band_worker(rank, world, port, bands, H, W, staged, q):
    """Each rank: its BandShard (whole bands + cut pieces), the halo exchange of
    the cut pieces, then every piece computed the way bench.py hands it to
    lfe_extract_bands / lfe_extract_rows -- with the oracle standing in."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(91)
        scene = np.stack([scenes.random_image(rng, H, W, 12, "mixed") for _ in range(bands)])
        p = O.Params(bit_depth=12, zc_threshold=(0.01, 0.01))
        halo = 7
        bs = BandShard(bands, H, W, rank, world, halo)
        bs.alloc(torch.int16, "cpu")  # 2-byte rows like the uint16 device buffers
        bs.load_owned(scene.astype(np.int16))
        for w in bs.exchange(staged=staged):
            w.wait()
        res = []
        for b in bs.whole:
            res.append((b, 0, O.run(scene[b], p)))
        outs = [np.zeros((e - a, W), np.uint16) for _, a, e, _, _ in bs.parts]
        for k, s, n, ha, hb, flags, need in bs.part_calls():
            b, a, e, above, below = bs.parts[k]
            B = bs.part_bufs[k].numpy().astype(np.uint16)
            r0 = (halo if above is not None else 0) + s
            sub = np.ascontiguousarray(B[r0 - ha:r0 + n + hb])
            outs[k][s:s + n] = O.run(sub, p)[ha:ha + n]
        for (b, a, e, _, _), o in zip(bs.parts, outs):
            res.append((b, a, o))
        q.put((rank, bs.owned_pixels(), res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,staged", [(2, False), (3, False), (8, False), (8, True)])
def test_gloo_band_shards_reproduce_every_band(world, staged):
    """c4's multi-GPU plan: 4 bands dealt to 2 ranks (whole bands, no exchange),
    3 ranks (bands cut mid-way), 8 ranks (every band cut between two ranks, one
    exchange per pair) -- the union of every rank's rows equals the oracle on
    each band."""
    bands, H, W = 4, 40, 56
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_band_worker, args=(r, world, port, bands, H, W, staged, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    rng = np.random.default_rng(91)
    scene = np.stack([scenes.random_image(rng, H, W, 12, "mixed") for _ in range(bands)])
    p = O.Params(bit_depth=12, zc_threshold=(0.01, 0.01))
    full = np.zeros((bands, H, W), np.uint16)
    cover = np.zeros((bands, H), np.int64)
    for _, px, res in got:
        assert px == sum(o.shape[0] * W for _, _, o in res)
        for b, a, o in res:
            full[b, a:a + o.shape[0]] = o
            cover[b, a:a + o.shape[0]] += 1
    assert (cover == 1).all()
    for b in range(bands):
        np.testing.assert_array_equal(full[b], O.run(scene[b], p))


def test_peer_strip_geometry():
    """PeerStripShard.call_args: the neighbour above's LAST LFE_PEER_ROWS = 8 rows
    (its base + (rows - 8) * pitch), the neighbour below's first row, and their flags;
    nothing on an image edge."""
    from paper_1304_3992_b200.shard import PeerStripShard
    H, W, halo = 12000, 12000, 7
    for world in (1, 2, 8):
        plan = plan_strips(H, world, halo)
        for r in range(world):
            sh = PeerStripShard(H, W, r, world, halo)
            assert (sh.a, sh.b) == plan[r]
            for k in sh.neighbours():
                a, b = plan[k]
                sh.peer[k] = (1000000 * (k + 1), 24064, b - a, 7 + k)
            da, pa, db, pb, fa, fb = sh.call_args()
            if r == 0:
                assert da == pa == fa == 0 and sh.ha == 0
            else:
                rows_above = plan[r - 1][1] - plan[r - 1][0]
                assert da == 1000000 * r + (rows_above - 8) * 24064 and pa == 24064 and fa == 7 + r - 1
            if r == world - 1:
                assert db == pb == fb == 0 and sh.hb == 0
            else:
                assert db == 1000000 * (r + 2) and fb == 7 + r + 1
