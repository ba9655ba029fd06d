"""Multi-process (gloo, CPU) tests of the row-strip driver's host logic: strip
ownership, which halo rows travel where, the exchange itself
(batch_isend_irecv), and that each rank's strip -- evaluated by the oracle
from its local rows only -- equals the whole-image result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


CASES = [  # (p, q, mode, pad, H, W, N, C)
    (3, 5, "bicubic", "replicate", 97, 40, 1, 1),
    (5, 3, "bicubic", "reflect", 61, 24, 1, 2),
    (7, 5, "bilinear", "zero", 50, 32, 2, 1),
    (4, 7, "bilinear", "replicate", 83, 16, 1, 1),
]


def _worker(rank, world, port, case, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        import paper_2203_10670_b200 as fc
        from paper_2203_10670_b200.dist import exchange, finish_exchange, strip_layout
        p, q, mode, pad, H, W, N, C = case
        pl = fc.Plan(p, q, mode, pad, C, H, W, "float32", "floor")
        lay = strip_layout(pl, rank, world)
        cfg = synth.Config("strip", N, C, H, W, "float32", "uniform", p, q, mode, pad, seed=4242)
        full = synth.make_values(cfg)
        own = synth.make_values(cfg, rows=(lay.own0, lay.own1))
        local = torch.full((N, C, max(1, lay.loc1 - lay.loc0), W), float("nan"))
        local[:, :, lay.own0 - lay.loc0:lay.own1 - lay.loc0] = torch.from_numpy(own)
        works, staged = exchange(local, lay)
        finish_exchange(works, staged)
        res = {"rank": rank, "ok": True, "msg": ""}
        if lay.loc1 > lay.loc0:
            if not np.array_equal(local.numpy(), full[:, :, lay.loc0:lay.loc1]):
                res.update(ok=False, msg="halo rows differ")
        if lay.out1 > lay.out0 and res["ok"]:
            mine = oracle.direct(local.numpy(), p, q, mode, pad, floor_extent=True, rows=(lay.out0, lay.out1),
                                 H=H, row0=lay.loc0)
            whole = oracle.direct(full, p, q, mode, pad, floor_extent=True)[:, :, lay.out0:lay.out1]
            if not np.array_equal(mine, whole):
                res.update(ok=False, msg="strip output differs")
            i0, i1 = lay.interior
            if i1 > i0:  # the interior needs only own rows
                own_only = oracle.direct(own, p, q, mode, pad, floor_extent=True, rows=(i0, i1), H=H,
                                         row0=lay.own0)
                if not np.array_equal(own_only, whole[:, :, i0 - lay.out0:i1 - lay.out0]):
                    res.update(ok=False, msg="interior differs")
        res["out"] = (lay.out0, lay.out1)
        res["sent"] = [(t.peer, t.row0, t.row1) for t in lay.sends]
        out_q.put(res)
    except Exception as e:  # report, do not hang the peers
        out_q.put({"rank": rank, "ok": False, "msg": repr(e)})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", CASES)
def test_strip_exchange_gloo(world, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    results = [q.get(timeout=180) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    for r in results:
        assert r["ok"], r
    # the strips partition the output rows
    spans = sorted(r["out"] for r in results)
    H, p, q_ = case[4], case[0], case[1]
    assert spans[0][0] == 0
    for a, b in zip(spans, spans[1:]):
        assert a[1] == b[0]
    # every halo message is at most 2 rows (bicubic reach) and goes to a neighbour
    for r in results:
        for peer, r0, r1 in r["sent"]:
            assert abs(peer - r["rank"]) == 1 and 0 < r1 - r0 <= 2


@pytest.mark.parametrize("case", CASES)
def test_peer_windows_cover_and_reproduce(case):
    """Peer transport: the windows a rank reads -- its own
    strip and whole neighbour strips -- cover every input row its output rows
    need, number at most 3, and the oracle evaluated on exactly those rows
    (the strips concatenated in row order) reproduces the whole image's rows."""
    import oracle
    import synth
    import paper_2203_10670_b200 as fc
    from paper_2203_10670_b200.dist import boundary_ranges, own_rows, peer_windows
    p, q, mode, pad, H, W, N, C = case
    pl = fc.Plan(p, q, mode, pad, C, H, W, "float32", "floor")
    cfg = synth.Config("peer", N, C, H, W, "float32", "uniform", p, q, mode, pad, seed=4343)
    full = synth.make_values(cfg)
    whole = oracle.direct(full, p, q, mode, pad, floor_extent=True)
    for world in (2, 3, 5):
        for rank in range(world):
            lay, wins = peer_windows(pl, rank, world)
            assert 1 <= len(wins) <= 3 and wins[0] == (rank, lay.own0, lay.own1)
            for peer, r0, r1 in wins:
                assert (r0, r1) == own_rows(H, peer, world)
            if lay.out1 <= lay.out0:
                continue
            rows = sorted((r0, r1) for _, r0, r1 in wins)
            lo, hi = rows[0][0], rows[-1][1]
            assert all(rows[k][1] == rows[k + 1][0] for k in range(len(rows) - 1))  # adjacent strips
            assert lo <= lay.need0 and lay.need1 <= hi
            for m0, m1 in boundary_ranges(lay):
                mine = oracle.direct(full[:, :, lo:hi], p, q, mode, pad, floor_extent=True, rows=(m0, m1), H=H,
                                     row0=lo)
                assert np.array_equal(mine, whole[:, :, m0:m1]), (world, rank, m0, m1)


def _batch_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import bench
        import synth
        res = {"rank": rank, "ok": True, "msg": "", "shares": {}}
        for name in ("C2a", "C3", "C4a"):
            cfg = synth.CONFIGS[name]
            a, b = bench.batch_share(cfg.N, rank, world)
            # every rank's images, gathered: they must tile [0, N) exactly once
            t = torch.tensor([a, b], dtype=torch.int64)
            allv = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(allv, t)
            spans = sorted(tuple(int(x) for x in v) for v in allv)
            if spans[0][0] != 0 or spans[-1][1] != cfg.N or any(s[1] != n[0] for s, n in zip(spans, spans[1:])):
                res.update(ok=False, msg=f"{name}: spans {spans}")
            # a rank's slice of the synthetic batch equals the same images of the whole batch
            if b > a:
                c1 = synth.Config(name, cfg.N, 1, 8, 8, "float32", cfg.values, cfg.p, cfg.q, cfg.mode, cfg.pad,
                                  seed=cfg.seed)
                whole = synth.make_values(c1)
                if not np.array_equal(synth.make_values(c1, a, b), whole[a:b]):
                    res.update(ok=False, msg=f"{name}: slice differs")
            res["shares"][name] = (a, b)
        out_q.put(res)
    except Exception as e:  # report, do not hang the peers
        out_q.put({"rank": rank, "ok": False, "msg": repr(e)})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 8])
def test_batch_split_partition_gloo(world):
    """bench.py --split batch: rank r scales images [rN/G, (r+1)N/G)
    -- the shares cover each config's batch exactly (C2 16, C3 64, C4 8 images)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_batch_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    results = [q.get(timeout=180) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    for r in results:
        assert r["ok"], r
    if world == 8:  # C4: one image per rank at G = 8
        assert sorted(r["shares"]["C4a"] for r in results) == [(i, i + 1) for i in range(8)]
