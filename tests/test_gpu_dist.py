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
