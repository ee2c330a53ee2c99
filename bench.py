"""GCUPS benchmark of the B200 NW hot path (BASELINE.json metric).

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                [--workload c3|c1|c2|c4|c5|...]

Default workload = C3 (BASELINE.json configs[2]), the configuration the metric's
1/2/4/8-GPU scaling is quoted on: all 2,096,128 pairs of 2,048 DNA sequences of
500-2,000 bp, score-only. One step = one nw_align_batch_dev call on inputs
resident in HBM: encode, the all-pairs batch fill and, with N ranks, the gather
of every rank's scores (each rank aligns its cost-balanced range).
--gpus N without a torchrun environment spawns the N ranks itself (one process
per GPU, NCCL); under torchrun the environment's ranks are used.

value   : GCUPS = m*n cells / device time per step (CUDA events on the context
          stream, per step, L2 flushed between steps), whole job over N ranks.
e2e     : the same metric through the host-pointer C ABI (nw_align_pair +
          nw_traceback on host buffers, H2D of the residues and D2H of the score
          and path inside the timed region).
roofline: the fill kernel's integer-op rate vs the issue-limited lane-op peak
          (DESIGN.md §5).
cpu_baseline: the oracle (plain C, 1 core) on a bounded sample of the workload.
--impl reference: the oracle timed on the host as the reference arm.
Multi-GPU: C3/C4 shard pairs across ranks (dist context) and gather every
score on every rank: "scaling": "strong" (the total work is fixed). C1/C2 are one
pair with no exchange step: N independent replicas, weak scaling.
check   : after the timed loop, a sample of the timed outputs is compared with the
          oracle (outside the timed region).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import nwgen  # noqa: E402

L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2
ALU_ISSUE_LANES_PER_CLK_PER_SM = 128  # 4 SMSPs x 32 lanes x 1 warp-instr/clk (tools/peaks_int.cu)
ALU_PIPE_LANES_PER_CLK_PER_SM = 64    # VIMNMX3/VIADDMNMX/IADD3/PRMT/SHF: the half-rate ALU pipe (measured)
SM_COUNT = 148
SM_MAX_MHZ = 1965.0
# SURVEY.md §8(d) algorithmic op floors per cell, by the arithmetic form of the fill:
# int32 with directions 6, int32 score-only 3, two 16-bit cells per register (H' half
# rows, C3; and the same with a moving per-strip base, C5: PRMT + IADD + VIMNMX3.U16x2 per
# two cells) 1.5, the packed difference form (the C5 checkpoint pass: PRMT + VIMNMX3.U16x2
# + 2 IADD per two cells) 2, packed with decision flags (C4) 2 (SURVEY's "u16x2 + direction")
OPS_PER_CELL = {"dirs": 6, "score": 3, "u16": 1.5, "h16": 1.5, "d16": 2, "d16dir": 2}
FORM = {"c1": "dirs", "c2": "dirs", "c1p": "dirs", "c2p": "dirs", "c1co": "dirs", "c2co": "dirs",
        "c3": "u16", "c4": "d16dir", "c5": "h16", "c5tb": "d16", "msa": "u16"}
WORKLOADS = {
    "c1": "C1: single DNA pair 1,000 x 1,000, +1/-1/-1, score + full traceback",
    "c2": "C2: single DNA pair 20,000 x 20,000, +1/-1/-1, score + 2-bit packed traceback",
    "c3": "C3: all-pairs of 2,048 DNA sequences of 500-2,000 bp (2,096,128 pairs), score-only",
    "c4": "C4: 100,000 protein pairs of 100-1,000 residues, BLOSUM62, g=-5, score + traceback",
    "c5": "C5: single DNA pair 1,000,000 x 1,000,000, score-only (linear memory)",
    "c1p": "C1 with the paper's per-cell kernel (Code 1, corrected; ablation baseline, NEXT #4)",
    "c5tb": "C5 with the full canonical traceback: checkpointed refill within half the free "
            "HBM for directions (SURVEY.md 8(f) NEXT #3)",
    "c1co": "C1 co-optimal alignments: exact count + the first 256 in depth-first pi order (NEXT #2)",
    "c2co": "C2 co-optimal alignments: exact count + the first 256 in depth-first pi order (NEXT #2)",
    "msa": "center-star MSA of the C3 set (2,048 DNA sequences of 500-2,000 bp): all-pairs "
           "scores, center, 2,047 alignments with traceback, union-gap merge (SURVEY.md 8(f) NEXT #1)",
}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))
        except Exception:
            return {}
    return {}


def cpu_oracle_sample(workload: str, budget_s: float = 15.0):
    """Time the oracle (as it stands) on a bounded sample of the workload."""
    import oracle
    if workload in ("c1", "c2", "c1p", "c2p", "c5tb", "c1co", "c2co"):
        a, b = (nwgen.config_c1() if workload in ("c1", "c1p", "c1co") else
                nwgen.config_c5() if workload == "c5tb" else nwgen.config_c2())
        # full pair if it fits the budget (~0.06 GCUPS single-core full+dirs), else a prefix
        side = len(a)
        est = side * side / 0.06e9
        if est > budget_s:
            side = int((budget_s * 0.06e9) ** 0.5)
        a, b = a[:side], b[:side]
        t0 = time.perf_counter()
        oracle.align(a, b, nwgen.PAPER_DNA)
        dt = time.perf_counter() - t0
        cells = len(a) * len(b)
        return {"value": cells / dt / 1e9, "unit": "GCUPS", "cores": 1, "kind": "oracle",
                "sample": f"{len(a)}x{len(b)} prefix of the {workload.upper()} pair, fill with "
                          f"full direction matrix + traceback, {dt:.2f} s"}
    if workload == "c5":
        a, b = nwgen.config_c5()
        side = int((budget_s * 0.4e9) ** 0.5)
        t0 = time.perf_counter()
        oracle.score(a[:side], b[:side], nwgen.PAPER_DNA)
        dt = time.perf_counter() - t0
        return {"value": side * side / dt / 1e9, "unit": "GCUPS", "cores": 1, "kind": "oracle",
                "sample": f"{side}x{side} prefix of the C5 pair, two-row score-only, {dt:.2f} s"}
    cores = len(os.sched_getaffinity(0))
    if workload == "c3":
        ss = nwgen.config_c3()
        pairs = nwgen.all_pairs(ss.nseq)
        rng = np.random.Generator(np.random.PCG64(0))
        lens = ss.lengths()
        idx = rng.permutation(len(pairs))
        cells_per = lens[pairs[idx, 0]] * lens[pairs[idx, 1]]
        target = budget_s * 0.5e9 * cores
        k = int(np.searchsorted(np.cumsum(cells_per), target)) + 1
        sub = pairs[idx[:k]]
        t0 = time.perf_counter()
        oracle.batch_score(ss.residues, ss.offs, sub, nwgen.PAPER_DNA, nthreads=cores)
        dt = time.perf_counter() - t0
        cells = int(cells_per[:k].sum())
        return {"value": cells / dt / 1e9, "unit": "GCUPS", "cores": cores, "kind": "oracle",
                "sample": f"{k} random pairs of C3 ({cells:.3e} cells), score-only, {dt:.2f} s"}
    if workload == "c4":
        ss = nwgen.config_c4(2000)
        t0 = time.perf_counter()
        cells = 0
        for k in range(2000):
            a, b = ss.seq(2 * k), ss.seq(2 * k + 1)
            oracle.align(a, b, nwgen.PROTEIN_BLOSUM62)
            cells += len(a) * len(b)
            if time.perf_counter() - t0 > budget_s:
                break
        dt = time.perf_counter() - t0
        return {"value": cells / dt / 1e9, "unit": "GCUPS", "cores": 1, "kind": "oracle",
                "sample": f"{k + 1} C4 pairs ({cells:.3e} cells), fill + traceback, 1 core, {dt:.2f} s"}
    if workload == "msa":
        from oracle import msa as omsa
        ss = nwgen.config_c3()
        nsub = 48
        seqs = [ss.seq(k) for k in range(nsub)]
        lens = np.array([len(x) for x in seqs], dtype=np.int64)
        t0 = time.perf_counter()
        c, rows = omsa.msa(seqs, nwgen.PAPER_DNA)
        dt = time.perf_counter() - t0
        cells = int((np.sum(lens) ** 2 - np.sum(lens ** 2)) // 2 + lens[c] * (lens.sum() - lens[c]))
        return {"value": cells / dt / 1e9, "unit": "GCUPS", "cores": 1, "kind": "oracle",
                "sample": f"center-star MSA of the first {nsub} C3 sequences ({cells:.3e} cells: "
                          f"all pairs + center alignments), 1 core, {dt:.2f} s"}
    raise ValueError(workload)


# ----------------------------------------------------------------------------- ours

def _pinned(torch, arr):
    """A page-locked host copy of a numpy array (numpy view of a pinned torch tensor)."""
    arr = np.ascontiguousarray(arr)
    t = torch.empty(arr.nbytes, dtype=torch.uint8, pin_memory=True)
    v = t.numpy().view(arr.dtype).reshape(arr.shape)
    v[...] = arr
    _PINNED.append(t)  # keeps the page-locked memory alive
    return v


_PINNED = []


class PairWorkload:
    """C1/C2 (fill + traceback) and C5 (score-only) single-pair steps."""

    def __init__(self, ctx, torch, workload: str, rank: int):
        import paper_2412_21103_b200 as nwb
        self.nwb, self.ctx, self.torch = nwb, ctx, torch
        self.workload = workload
        self.percell = workload in ("c1p", "c2p")
        self.linear = workload == "c5tb"
        self.coopt = workload in ("c1co", "c2co")
        gen = {"c1": nwgen.config_c1, "c2": nwgen.config_c2, "c5": nwgen.config_c5,
               "c1p": nwgen.config_c1, "c2p": nwgen.config_c2, "c5tb": nwgen.config_c5,
               "c1co": nwgen.config_c1, "c2co": nwgen.config_c2}[workload]
        a, b = gen()
        self.a, self.b = a, b
        self.m, self.n = len(a), len(b)
        self.dirs = workload not in ("c5", "c5tb")
        self.sc = nwgen.PAPER_DNA
        self.da = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda()
        self.db = torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
        self.d_score = torch.zeros(1, dtype=torch.int64, device="cuda")
        self.d_ops = torch.zeros(self.m + self.n, dtype=torch.uint8, device="cuda")
        self.d_len = torch.zeros(1, dtype=torch.int64, device="cuda")
        self.cells = self.m * self.n

    def step(self):
        if self.coopt:  # host-pointer API (synchronous)
            self.nwb.nw_cooptimal(self.ctx, self.a, self.b, self.sc, 256)
        elif self.linear:  # host-pointer API (it synchronises per segment); inputs 2 MB
            self.nwb.nw_align_pair_linear(self.ctx, self.a, self.b, self.sc)
        elif self.percell:
            self.nwb.nw_align_pair_percell_dev(self.ctx, self.da, self.db, self.sc, self.d_score,
                                               self.d_ops, self.d_len)
        elif self.dirs:
            tb = self.nwb.nw_align_pair_dev(self.ctx, self.da, self.db, self.sc, self.d_score)
            self.nwb.nw_traceback_dev(self.ctx, tb, self.d_ops, self.d_len)
            tb.free()
        else:
            self.nwb.nw_score_only_dev(self.ctx, self.da, self.db, self.sc, self.d_score)

    def step_host(self):
        """The same step through the host-pointer ABI (e2e)."""
        if self.coopt:
            cnt, sat, paths = self.nwb.nw_cooptimal(self.ctx, self.a, self.b, self.sc, 256)
            return 8 + 8 * 257 + sum(len(p) for p in paths)
        if self.linear:
            score, ops = self.nwb.nw_align_pair_linear(self.ctx, self.a, self.b, self.sc)
            return 8 + 8 + len(ops)
        if self.percell:
            score, ops = self.nwb.nw_align_pair_percell(self.ctx, self.a, self.b, self.sc)
            return 8 + 8 + len(ops)
        if self.dirs:
            score, tb = self.nwb.nw_align_pair(self.ctx, self.a, self.b, self.sc)
            ops = self.nwb.nw_traceback(self.ctx, tb)
            tb.free()
            return 8 + 8 + len(ops)
        self.nwb.nw_score_only(self.ctx, self.a, self.b, self.sc)
        return 8

    @property
    def h2d_bytes(self):
        return self.m + self.n

    def check(self):
        """The last timed step's outputs vs the oracle (outside the timed region)."""
        import oracle
        if self.coopt or self.linear:
            return {"against": "none", "what": "not checked here (see tests/)"}
        got = int(self.d_score.item())
        if self.workload == "c5":  # oracle score of the seeded pair: tools/oracle_digests.py
            dp = os.path.join(ROOT, "tests", "golden", "digests.json")
            want = json.load(open(dp)).get("c5", {}).get("score") if os.path.exists(dp) else None
            return {"against": "oracle (tests/golden/digests.json)", "what": "score", "sample": 1,
                    "mismatches": None if want is None else int(got != want)}
        ws, wops = oracle.align(self.a, self.b, self.sc)
        ln = int(self.d_len.item())
        ops = self.d_ops[:ln].cpu().numpy()
        return {"against": "oracle", "what": "score and path", "sample": 1,
                "mismatches": int(got != ws or ops.tolist() != wops.tolist())}


class BatchWorkload:
    """C3 (all pairs, score-only) and C4 (protein pairs, traceback). With N ranks the
    context is a dist context (include/nw.h): every rank passes the full inputs,
    aligns its cost-balanced range and receives every rank's outputs."""

    def __init__(self, ctx, torch, workload: str, rank: int, world: int):
        import paper_2412_21103_b200 as nwb
        self.nwb, self.ctx, self.torch = nwb, ctx, torch
        self.workload, self.rank, self.world = workload, rank, world
        if workload == "c3":
            ss = nwgen.config_c3()
            pairs = nwgen.all_pairs(ss.nseq)
            self.sc = nwgen.PAPER_DNA
            self.flags = nwb.NW_SCORE_ONLY
            self.h_pairs = None  # implicit all pairs
        else:
            ss = nwgen.config_c4()
            pairs = nwgen.consecutive_pairs(ss.nseq // 2)
            self.sc = nwgen.PROTEIN_BLOSUM62
            self.flags = nwb.NW_TRACEBACK
            self.h_pairs = pairs
        lens = ss.lengths().astype(np.int64)
        self.all_pairs = pairs
        self.total_cells = self.cells = int((lens[pairs[:, 0]] * lens[pairs[:, 1]]).sum())
        self.npairs = len(pairs)
        if world > 1:
            from paper_2412_21103_b200 import dist as nwdist
            b = nwdist.partition(ss.offs, self.h_pairs, world)
            self.range = (int(b[rank]), int(b[rank + 1]))
        self.ss = ss
        self.d_seqs = torch.from_numpy(ss.residues).cuda()
        self.d_offs = torch.from_numpy(ss.offs).cuda()
        self.d_pairs = None if self.h_pairs is None else torch.from_numpy(self.h_pairs).cuda()
        self.d_scores = torch.zeros(max(self.npairs, 1), dtype=torch.int32, device="cuda")
        if self.flags:
            oo = nwb.nw_batch_ops_offsets(ss.offs, self.h_pairs)
            self.oo = oo
            self.d_ops_off = torch.from_numpy(oo).cuda()
            self.d_ops = torch.zeros(int(oo[-1]) + 1, dtype=torch.uint8, device="cuda")
            self.d_ops_len = torch.zeros(self.npairs, dtype=torch.int32, device="cuda")
        else:
            self.d_ops_off = self.d_ops = self.d_ops_len = None
        # e2e: the host ABI reads its inputs from, and writes its outputs to, page-locked
        # host memory (the copies inside the timed region then run at DMA speed)
        self.h_res = _pinned(torch, ss.residues)
        self.h_offs = _pinned(torch, ss.offs)
        self.h_pairs_pin = None if self.h_pairs is None else _pinned(torch, self.h_pairs)
        if self.flags:
            self.h_out = (_pinned(torch, np.empty(self.npairs, np.int32)),
                          _pinned(torch, np.empty(int(oo[-1]) + 1, np.uint8)),
                          _pinned(torch, np.empty(self.npairs + 1, np.int64)),
                          _pinned(torch, np.empty(max(self.npairs, 1), np.int32)))
        else:
            self.h_out = _pinned(torch, np.empty(self.npairs, np.int32))

    def step(self):
        self.nwb.nw_align_batch_dev(self.ctx, self.d_seqs, self.d_offs, self.ss.offs, self.d_pairs,
                                    self.h_pairs, self.npairs, self.sc, self.flags, self.d_scores,
                                    self.d_ops_off, self.d_ops, self.d_ops_len)

    def step_host(self):
        r = self.nwb.nw_align_batch(self.ctx, self.h_res, self.h_offs, self.h_pairs_pin, self.sc,
                                    self.flags, out=self.h_out)
        if self.flags:
            scores, ops, ops_off, ops_len = r
            return scores.nbytes + ops.nbytes + ops_len.nbytes
        return r.nbytes

    def check(self, k: int = 48):
        """Compare a seeded sample of the last timed step's outputs (every rank's, as
        gathered) with the oracle: scores, and paths with NW_TRACEBACK."""
        import oracle
        rng = np.random.Generator(np.random.PCG64(12345))
        idx = np.sort(rng.choice(self.npairs, size=min(k, self.npairs), replace=False))
        scores = self.d_scores.cpu().numpy()
        pairs = self.all_pairs[idx]
        bad = 0
        if self.flags:
            ops, ln = self.d_ops.cpu().numpy(), self.d_ops_len.cpu().numpy()
            for i, (p, q) in zip(idx, pairs):
                ws, wops = oracle.align(self.ss.seq(p), self.ss.seq(q), self.sc)
                got = ops[self.oo[i]:self.oo[i] + ln[i]]
                bad += int(scores[i] != ws or got.tolist() != wops.tolist())
            what = "scores and paths"
        else:
            want = oracle.batch_score(self.ss.residues, self.ss.offs, pairs, self.sc)
            bad = int((scores[idx] != want).sum())
            what = "scores"
        return {"against": "oracle", "what": what, "sample": int(len(idx)), "mismatches": bad}

    @property
    def h2d_bytes(self):
        return self.ss.residues.nbytes + self.ss.offs.nbytes + (
            0 if self.h_pairs is None else self.h_pairs.nbytes)


class MsaWorkload:
    """Center-star MSA of the C3 set (NEXT #1): one nw_msa_center_star_dev call per step."""

    def __init__(self, ctx, torch, workload: str, rank: int):
        import paper_2412_21103_b200 as nwb
        self.nwb, self.ctx, self.torch = nwb, ctx, torch
        self.ss = nwgen.config_c3()
        self.sc = nwgen.PAPER_DNA
        self.d_seqs = torch.from_numpy(self.ss.residues).cuda()
        self.d_offs = torch.from_numpy(self.ss.offs).cuda()
        lens = self.ss.lengths().astype(np.int64)
        h = nwb.nw_msa_center_star_dev(ctx, self.d_seqs, self.d_offs, self.ss.offs, self.sc)
        self.center, self.width = h.center, h.width
        h.free()
        self.cells_pairs = int((lens.sum() ** 2 - (lens ** 2).sum()) // 2)
        self.cells_center = int(lens[self.center] * (lens.sum() - lens[self.center]))
        self.cells = self.total_cells = self.cells_pairs + self.cells_center

    def step(self):
        self.nwb.nw_msa_center_star_dev(self.ctx, self.d_seqs, self.d_offs, self.ss.offs,
                                        self.sc).free()

    def step_host(self):
        h = self.nwb.nw_msa_center_star(self.ctx, self.ss.residues, self.ss.offs, self.sc)
        rows = h.rows_array()
        h.free()
        return rows.nbytes

    @property
    def h2d_bytes(self):
        return self.ss.residues.nbytes + self.ss.offs.nbytes


def run_ours(args):
    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2412_21103_b200 as nwb
    stream = torch.cuda.current_stream()
    ctx = nwb.Context(local, stream.cuda_stream)
    wl = args.workload
    sharded = wl in ("c3", "c4", "c5") and world > 1
    if sharded:  # the library's own NCCL communicator (nw_ctx_set_dist), id shared by rank 0
        # (C3/C4: pair ranges + gather; C5: the column-block pipeline across the GPUs)
        from paper_2412_21103_b200 import dist as nwdist
        nwdist.init_dist_context(ctx)
    if wl in ("c1", "c2", "c5", "c1p", "c2p", "c5tb", "c1co", "c2co"):
        W = PairWorkload(ctx, torch, wl, rank)
    elif wl == "msa":
        W = MsaWorkload(ctx, torch, wl, rank)
    else:
        W = BatchWorkload(ctx, torch, wl, rank, world)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device="cuda")

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    for _ in range(args.warmup):
        W.step()
    torch.cuda.synchronize()
    ctx.set_timing(True)
    ctx.kernel_time(0)
    ctx.kernel_time(1)
    launches0 = ctx.launches()
    clocks = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    evs = []
    for _ in range(args.steps):
        flush.zero_()  # L2 flush between timed steps (outside the events)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        W.step()
        e1.record(stream)
        evs.append((e0, e1))
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    launches = ctx.launches() - launches0
    step_ms = [a.elapsed_time(b) for a, b in evs]
    fill_ms, fill_n = ctx.kernel_time(0)
    tb_ms, tb_n = ctx.kernel_time(1)
    ctx.set_timing(False)
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    if wl == "c5" and sharded:
        cells_all = W.cells          # one pair, its column blocks pipelined across the ranks
    elif sharded or wl in ("c3", "c4"):
        cells_all = W.total_cells    # one batch split over the ranks, gathered on every rank
    else:
        cells_all = W.cells * world  # replicas: every rank aligns its own pair / set
    value = cells_all / (ms_per_step / 1e3) / 1e9
    # ---- e2e through the host-pointer ABI
    torch.cuda.synchronize()
    barrier()
    e2e_steps = max(1, min(args.steps, 5 if wl in ("c3", "c4", "msa") else 2 if wl in ("c5tb", "c2co") else args.steps))
    d2h = 0
    for _ in range(min(args.warmup, 2)):  # untimed warm-up of the host path (buffer growth)
        W.step_host()
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        d2h = W.step_host()
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": cells_all / e2e_s / 1e9, "unit": "GCUPS", "h2d_bytes_per_step": W.h2d_bytes,
           "d2h_bytes_per_step": d2h}
    # ---- roofline of the dominant kernel (the fill)
    fill_avg_ms = fill_ms / max(fill_n, 1)
    fill_launches_per_step = fill_n / max(args.steps, 1)
    mode = FORM[wl]
    if wl == "c5" and sharded:  # the column-block pipeline across ranks runs the difference form
        mode = "d16"
    ops = OPS_PER_CELL[mode]
    # the step's cells over the fill time of the whole step (C4 fills in two launches:
    # the pairs kept in their orientation, then the transposed ones)
    fill_step_ms = fill_ms / max(args.steps, 1)
    achieved = W.cells * ops / (fill_step_ms / 1e3) / 1e12 if fill_n else None
    if wl == "c5tb":  # one score-only pass + the direction refills of every segment
        fill_avg_ms = fill_ms / max(args.steps, 1)
        ops = f"{OPS_PER_CELL['d16']} (checkpoint pass; refill ops not counted: a lower bound)"
        achieved = W.cells * OPS_PER_CELL["d16"] / (fill_avg_ms / 1e3) / 1e12 if fill_n else None
    if wl == "msa":  # two batch launches per step: all pairs score-only, center pairs + dirs
        ops = f"{OPS_PER_CELL['u16']} (all pairs) / {OPS_PER_CELL['d16dir']} (center alignments)"
        fill_step_ms = fill_ms / max(args.steps, 1)
        achieved = (W.cells_pairs * OPS_PER_CELL["u16"] + W.cells_center * OPS_PER_CELL["d16dir"]) / (
            fill_step_ms / 1e3) / 1e12 if fill_n else None
        fill_avg_ms = fill_step_ms
    peak_issue = ALU_ISSUE_LANES_PER_CLK_PER_SM * SM_COUNT * SM_MAX_MHZ * 1e6 / 1e12
    peak = ALU_PIPE_LANES_PER_CLK_PER_SM * SM_COUNT * SM_MAX_MHZ * 1e6 / 1e12
    # DRAM traffic per launch of the dominant kernel, from one ncu metric pass of this
    # workload (tools/traffic.py -> profiles/r02_traffic_<wl>.json; cold cache, serialised)
    kname = ("k_percell_fill" if wl in ("c1p", "c2p") else
             "k_fill_pair" if wl in ("c1", "c2", "c5", "c5tb") else "k_batch")
    traffic, tinfo = None, {}
    tp = os.path.join(ROOT, "profiles", f"r02_traffic_{wl}.json")
    if os.path.exists(tp):
        tinfo = json.load(open(tp)).get("kernels", {})
        fills = [v for k, v in tinfo.items() if k.startswith(kname + "<")]
        if fills:
            traffic = sum(v["dram_read_bytes_per_launch"] + v["dram_write_bytes_per_launch"]
                          for v in fills) / len(fills)
    hbm = load_peaks().get("hbm_gbs")
    walk = None  # the traceback kernels' HBM rate: ncu bytes over their live event time
    tbk = {k: v for k, v in tinfo.items() if k.startswith(("k_tb_", "k_batch_walk"))}
    if tbk and tb_n:
        rd = sum(v["dram_read_bytes_per_launch"] for v in tbk.values())
        wr = sum(v["dram_write_bytes_per_launch"] for v in tbk.values())
        t_ms = tb_ms / max(args.steps, 1)
        walk = {"kernels": sorted(tbk), "bound": "hbm latency (dependent loads along the paths)",
                "ms_per_step": t_ms, "dram_read_bytes_per_step": rd, "dram_write_bytes_per_step": wr,
                "readback_GBps": rd / (t_ms / 1e3) / 1e9, "peak_GBps": hbm,
                "readback_frac": (rd / (t_ms / 1e3) / 1e9) / hbm if hbm else None,
                "bytes_source": os.path.relpath(tp, ROOT)}
    dirs_write = None  # the fill's direction writes: algorithmic bytes (2 bits per cell) over the fill time
    if mode in ("dirs", "d16dir") and fill_n and wl not in ("c1co", "c2co"):
        b = W.cells / 4 * (1.29 if mode == "d16dir" else 1.0)
        dirs_write = {"algorithmic_bytes_per_step": b, "GBps": b / (fill_step_ms / 1e3) / 1e9,
                      "peak_GBps": hbm, "note": "2 bits per cell" + (
                          " over the 1.29x padded sweep (DESIGN.md §3.9)" if mode == "d16dir" else "")}
    roofline = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Tops/s (int32 lane-ops)",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "peak_issue": peak_issue, "frac_issue": (achieved / peak_issue) if achieved else None,
                "kernel": kname,
                **({"kernel_ms_is": "both k_batch launches of one step"} if wl == "msa" else {}),
                "ops_per_cell": ops, "kernel_ms_per_launch": fill_avg_ms,
                "kernel_launches_per_step": fill_launches_per_step,
                "kernel_share_of_step": (fill_ms / total_ms) if total_ms else None,
                "traceback_ms_per_step": tb_ms / max(args.steps, 1),
                "peak_source": ("tools/peaks_int.cu (profiles/r02_peaks_int.json): the ALU pipe's 64 "
                                "lane-ops/clk/SM for the 3-input / add-max / packed-16-bit ops the fills issue "
                                "(VIMNMX3, VIADDMNMX, IADD3, PRMT, SHF) x 148 SMs x 1965 MHz; peak_issue: the "
                                "128 lane-ops/clk/SM warp-issue limit (2-input VIMNMX). MEASURED_PEAKS.json "
                                "has no INT32 entry"),
                "form": mode,
                **({"traceback_readback": walk} if walk else {}),
                **({"direction_write": dirs_write} if dirs_write else {})}
    out = {
        "metric": "GCUPS (cell updates/s)", "value": value, "unit": "GCUPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong" if (wl in ("c3", "c4") or (wl == "c5" and sharded)) else "weak",
        "vs_baseline": None,
        # arithmetic of the fill kernel in use: int32 strips, or two 16-bit cells per register
        "dtype": "int32" if wl in ("c1", "c2", "c1p", "c2p", "c5tb", "c1co", "c2co") else "u16x2",
        **({"msa": {"center": W.center, "width": W.width}} if wl == "msa" else {}),
        "data": "synthetic (nwgen seeded, SURVEY.md §8(d) recipe)",
        "config": {"workload": WORKLOADS[wl], "cells_per_step": cells_all,
                   "parallelism": (f"pairs-sharded{world} (cost-balanced ranges, NCCL in-place broadcasts)"
                                   if wl in ("c3", "c4") else
                                   f"column-blocks{world} (peer-memory pipeline, CUDA IPC + NVLink)"
                                   if (wl == "c5" and sharded) else f"replicas{world}"),
                   "l2": "flushed between steps (256 MB write)"},
        "e2e": e2e, "gpu_launches": launches, "clocks": clk, "roofline": roofline,
    }
    if rank == 0 and hasattr(W, "check") and not args.no_check:
        out["check"] = W.check()  # a sample of the timed outputs vs the oracle (untimed)
    if rank == 0 and world == 1 and not args.no_cpu:
        out["cpu_baseline"] = cpu_oracle_sample(wl)
    if rank == 0:
        print(json.dumps(out))
    ctx.close()
    if world > 1:
        torch.distributed.destroy_process_group()


def run_reference(args):
    """The reference arm = the oracle on the host cores (no GPU work)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    wl = args.workload
    steps = []
    budget = max(2.0, 150.0 / max(1, args.steps + args.warmup))
    samples = None
    for k in range(args.warmup + args.steps):
        r = cpu_oracle_sample(wl, budget_s=budget)
        if k >= args.warmup:
            steps.append(r["value"])
            samples = r
    value = statistics.median(steps)
    out = {"impl": "reference", "metric": "GCUPS (cell updates/s)", "value": value, "unit": "GCUPS",
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": None, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "int64", "data": "synthetic (nwgen seeded)",
           "config": {"workload": WORKLOADS[wl], "parallelism": "host cores"},
           "cpu_baseline": {"value": value, "unit": "GCUPS", "cores": samples["cores"],
                            "kind": "oracle", "sample": samples["sample"]},
           "e2e": {"value": value, "unit": "GCUPS", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-check", action="store_true", help="skip the oracle spot check")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # no torchrun environment: one process per GPU, spawned here (rank 0 prints)
        import torch
        if torch.cuda.device_count() < args.gpus:
            raise SystemExit(f"bench.py --gpus {args.gpus}: only {torch.cuda.device_count()} CUDA "
                             "device(s) visible (one process per GPU)")
        from paper_2412_21103_b200 import dist as nwdist
        nwdist.launch(args.gpus, run_ours, (args,))
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
