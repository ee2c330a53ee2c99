"""The column-block pipeline through its real
multi-process plumbing on one GPU (VERDICT r1 "Next round" item 4):
  - two processes (ranks 0 and 1 of G = 2), each with its own context; receive
    buffers exported and imported through CUDA IPC (nw_cblock_ipc_export/import),
    the handles exchanged over a gloo group, entries stored with .sys scope; the two
    ranks' kernels share the GPU by time-slicing;
  - the dist context's own path (nw_score_only on a ctx with an NCCL communicator,
    NW_OPT_DIST_PIPELINE = 1 at world 1): IPC buffers, tags, the all-reduce.
Scores are compared with the oracle."""
import os

import numpy as np
import pytest

import nwgen
import oracle
import paper_2412_21103_b200 as nwb
from paper_2412_21103_b200 import dist as nwdist

pytestmark = pytest.mark.gpu

CASES = [(3000, 9000, 0, "h16"), (2800, 6000, 500, "d16"), (2500, 4000, 700, "int32")]
SC = {"h16": nwgen.PAPER_DNA, "d16": nwgen.PAPER_DNA, "int32": nwgen.Scoring(match=2, mismatch=-4, gap=-1)}
PAIR_FORM = {"h16": 0, "d16": 1, "int32": 0}  # NW_OPT_PAIR_FORM: 1 = the difference form


def _rank_worker(m, n, w, form, out_dir):
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
    ctx.set_option("cblock_warps_per_sm", 2)  # both ranks' warps resident on the one GPU
    ctx.set_option("pair_form", PAIR_FORM[form])
    h = nwb.nw_cblock_ipc_export(ctx, m)
    hs = [None] * world
    dist.all_gather_object(hs, h)
    nwb.nw_cblock_ipc_import(ctx, hs[(rank + 1) % world])
    dist.barrier()  # every receive buffer exists (zeroed) before any rank writes
    a, b = nwgen.random_pair(4242 + m, m, n)
    da = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda()
    db = torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
    res = []
    for _ in range(2):  # two calls: per-call tags, buffers not re-zeroed
        part = torch.zeros(1, dtype=torch.int64, device="cuda")
        nwb.nw_score_only_cblock_rank_dev(ctx, da, db, SC[form], rank, world, w, None, None, part)
        ctx.sync()
        t = part.cpu()
        dist.all_reduce(t)
        res.append(int(t.item()))
        dist.barrier()
    with open(os.path.join(out_dir, f"r{rank}"), "w") as f:
        f.write(" ".join(map(str, res)))
    ctx.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("m,n,w,form", CASES)
def test_two_process_ipc_pipeline(tmp_path, m, n, w, form):
    nwdist.launch(2, _rank_worker, (m, n, w, form, str(tmp_path)))
    a, b = nwgen.random_pair(4242 + m, m, n)
    want = oracle.score(a, b, SC[form])
    for r in range(2):
        got = [int(x) for x in open(os.path.join(tmp_path, f"r{r}")).read().split()]
        assert got == [want, want]


@pytest.mark.parametrize("form", ["h16", "d16", "int32"])
def test_dist_ctx_pipeline_world1(form):
    import torch
    c = nwb.Context(0)
    c.set_option("pair_form", PAIR_FORM[form])
    c.set_dist(0, 1, nwb.nw_dist_unique_id())
    c.set_option("dist_pipeline", 1)
    for m, n in [(5000, 3000), (700, 12000), (1, 9)]:
        a, b = nwgen.random_pair(77 + m, m, n)
        want = oracle.score(a, b, SC[form])
        assert nwb.nw_score_only(c, a, b, SC[form]) == want
        d = torch.zeros(1, dtype=torch.int64, device="cuda")
        nwb.nw_score_only_dev(c, torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda(),
                              torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda(), SC[form], d)
        c.sync()
        assert int(d.item()) == want
    c.close()
