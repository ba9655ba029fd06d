"""GPU checks of the multi-GPU driver on the one GPU a test box has: the
row-strip runner with an NCCL process group of world size 1 (the interior /
boundary split and the run path; no peer), and every strip of a G-way split
computed by that strip's own StripRunner layout from its local rows only
(halo rows copied in as the exchange would deliver them)."""
import os
import socket

import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def pg():
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


def test_strip_runner_world1_equals_single_launch(pg):
    import paper_2203_10670_b200 as fc
    from paper_2203_10670_b200.dist import StripRunner
    cfg = synth.Config("strip1", 1, 1, 3000, 2048, "float32", "field", 3, 5, "bicubic", "replicate",
                       seed=synth.SEED_BASE + 77)
    x = synth.make_input(cfg).cuda()
    pl = fc.Plan(3, 5, "bicubic", "replicate", 1, 3000, 2048, "float32", "floor")
    sr = StripRunner(pl, 0, 1)
    local = sr.alloc_local(1, x.dtype, "cuda")
    sr.own_view(local).copy_(x)
    out = sr.alloc_out(1, x.dtype, "cuda")
    sr.run(local, out)
    torch.cuda.synchronize()
    assert torch.equal(out, pl.run(x))


@pytest.mark.parametrize("G", [2, 8])
def test_strip_layouts_reproduce_whole_image(G):
    import paper_2203_10670_b200 as fc
    from paper_2203_10670_b200.dist import strip_layout
    H, W = 2048, 1024
    cfg = synth.Config("stripG", 1, 1, H, W, "float32", "field", 3, 5, "bicubic", "replicate",
                       seed=synth.SEED_BASE + 78)
    x = synth.make_input(cfg).cuda()
    pl = fc.Plan(3, 5, "bicubic", "replicate", 1, H, W, "float32", "floor")
    whole = pl.run(x)
    parts = []
    for g in range(G):
        lay = strip_layout(pl, g, G)
        local = x[:, :, lay.loc0:lay.loc1].contiguous()  # own rows + the halo the exchange delivers
        i0, i1 = lay.interior
        out = torch.empty((1, 1, lay.out1 - lay.out0, pl.Wo), device="cuda")
        # interior first (own rows only), then the boundary rows -- as StripRunner.run does
        if i1 > i0:
            out[:, :, i0 - lay.out0:i1 - lay.out0] = pl.run_rows(local, lay.loc0, i0, i1 - i0)
        for a, b in ((lay.out0, i0), (i1, lay.out1)):
            if b > a:
                out[:, :, a - lay.out0:b - lay.out0] = pl.run_rows(local, lay.loc0, a, b - a)
        parts.append(out)
    assert torch.equal(torch.cat(parts, dim=2), whole)


def test_run_rows_segments_equals_contiguous_rows():
    """fcfs_run_rows_segments (the peer-halo launch) with three
    separate buffers standing in for a rank's strip and its neighbours' strips:
    bit-identical to the rows of the single launch (one arithmetic contract)."""
    import paper_2203_10670_b200 as fc
    from paper_2203_10670_b200._lib import FcfsError
    for (p, q, mode, pad, dtype, N, C) in [(3, 5, "bicubic", "replicate", "float32", 1, 1),
                                           (5, 3, "bicubic", "reflect", "bfloat16", 2, 3),
                                           (7, 5, "bilinear", "zero", "float16", 1, 2)]:
        H, W = 301, 257
        pl = fc.Plan(p, q, mode, pad, C, H, W, dtype, "floor")
        x = torch.from_numpy(synth.normal_f32(55, N * C * H * W).reshape(N, C, H, W)).to(getattr(torch, dtype)).cuda()
        whole = pl.run(x)
        cuts = [0, 97, 205, H]
        strips = [(x[:, :, a:b].contiguous(), a) for a, b in zip(cuts[:-1], cuts[1:])]
        for s in range(3):
            o0, o1, n0, n1 = pl.strip_rows(cuts[s], cuts[s + 1])
            wins = [strips[s]] + [strips[k] for k in (s - 1, s + 1) if 0 <= k < 3]
            got = pl.run_rows_segments(wins, o0, o1 - o0)
            assert torch.equal(got.view(torch.uint8), whole[:, :, o0:o1].contiguous().view(torch.uint8)), (p, q, s)
        # a needed row in no window / overlapping windows
        o0, o1, n0, n1 = pl.strip_rows(97, 205)
        with pytest.raises(FcfsError) as e:
            pl.run_rows_segments([strips[1]], o0, o1 - o0)
        assert e.value.name == "FCFS_E_SHAPE"
        with pytest.raises(FcfsError) as e:
            pl.run_rows_segments([strips[1], (x[:, :, 90:100].contiguous(), 90)], o0, o1 - o0)
        assert e.value.name == "FCFS_E_ARG"


def test_run_rows_segments_fused_against_oracle(monkeypatch):
    """The peer-halo boundary launch runs the fused kernel --
    its producer copies each input row from the window holding it -- on three
    windows (own strip + both neighbours' strips): every output row checked
    against the oracle's direct evaluator on exactly those rows (row0 = the
    first window row), and bitwise equal to the reference kernel's segment
    reads (FCFS_SEGMENTS_REFERENCE) and to the single launch."""
    import numpy as np
    import oracle
    import paper_2203_10670_b200 as fc
    from helpers import compare
    for (p, q, mode, pad, dtype, N, C) in [(3, 5, "bicubic", "replicate", "float32", 1, 1),
                                           (5, 3, "bicubic", "reflect", "bfloat16", 2, 3),
                                           (7, 5, "bilinear", "zero", "float16", 1, 2),
                                           (4, 7, "bilinear", "reflect", "float32", 1, 2)]:
        H, W = 301, 256
        pl = fc.Plan(p, q, mode, pad, C, H, W, dtype, "floor")
        xv = synth.normal_f32(57, N * C * H * W).reshape(N, C, H, W)
        x = torch.from_numpy(xv).to(getattr(torch, dtype)).cuda()
        xr = x.float().cpu().numpy()
        whole = pl.run(x)
        cuts = [0, 97, 205, H]
        strips = [(x[:, :, a:b].contiguous(), a) for a, b in zip(cuts[:-1], cuts[1:])]
        for s in range(3):
            o0, o1, n0, n1 = pl.strip_rows(cuts[s], cuts[s + 1])
            wins = [strips[s]] + [strips[k] for k in (s - 1, s + 1) if 0 <= k < 3]
            got = pl.run_rows_segments(wins, o0, o1 - o0)
            torch.cuda.synchronize()
            assert fc.last_launch() == {"kernel": "fused_separable", "segments": len(wins)}, fc.last_launch()
            lo = min(r0 for _, r0 in wins)
            hi = max(r0 + t.shape[2] for t, r0 in wins)
            ref = oracle.direct(xr[:, :, lo:hi], p, q, mode, pad, floor_extent=True, rows=(o0, o1), H=H, row0=lo)
            compare(got, ref, dtype, mode, float(xr.max() - xr.min()), f"segments {p}/{q} strip {s}",
                    x_absmax=float(np.abs(xr).max()))
            monkeypatch.setenv("FCFS_SEGMENTS_REFERENCE", "1")
            got_ref = pl.run_rows_segments(wins, o0, o1 - o0)
            torch.cuda.synchronize()
            monkeypatch.delenv("FCFS_SEGMENTS_REFERENCE")
            assert fc.last_launch()["kernel"] == "reference"
            assert torch.equal(got.view(torch.uint8), got_ref.view(torch.uint8)), (p, q, s)
            assert torch.equal(got.view(torch.uint8), whole[:, :, o0:o1].contiguous().view(torch.uint8)), (p, q, s)


def test_strip_runner_peer_transport_world1(pg):
    """The symmetric-memory setup and run path of the peer transport on one GPU
    (world 1: no neighbours, every row interior) equals the single launch."""
    import paper_2203_10670_b200 as fc
    from paper_2203_10670_b200.dist import StripRunner
    try:
        import torch.distributed._symmetric_memory  # noqa: F401
    except Exception as e:  # pragma: no cover
        pytest.skip(f"symmetric memory unavailable: {e}")
    pl = fc.Plan(3, 5, "bicubic", "replicate", 1, 600, 512, "float32", "floor")
    x = torch.from_numpy(synth.normal_f32(56, 600 * 512).reshape(1, 1, 600, 512)).cuda()
    sr = StripRunner(pl, 0, 1, transport="peer")
    local = sr.setup_peer(1, torch.float32, torch.device("cuda", 0))
    local.copy_(x)
    out = sr.alloc_out(1, torch.float32, torch.device("cuda", 0))
    sr.run_peer(out)
    torch.cuda.synchronize()
    assert torch.equal(out, pl.run(x))
