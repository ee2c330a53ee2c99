"""Thin ctypes binding of include/nw.h (argument marshalling only).

Every step of the hot path runs in libnw_b200.so's CUDA kernels; this module
converts Python/numpy/torch arguments to the C ABI and back. If the shared
library is missing or has no CUDA device, calls raise -- there is no CPU path.

Names follow the C ABI: nw_score_only, nw_align_pair, nw_traceback,
nw_align_batch (+ the _dev variants on device pointers / torch CUDA tensors).
"""
from __future__ import annotations

import contextlib
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NW_LIB_PATH") or os.path.join(_HERE, "libnw_b200.so")  # experiments only

NW_OK, NW_E_INVAL, NW_E_ALPHABET, NW_E_OVERFLOW, NW_E_NOMEM, NW_E_CUDA, NW_E_TRUNC, \
    NW_E_STATE, NW_E_DEADLOCK, NW_E_COMM = range(10)
NW_DIAG, NW_UP, NW_LEFT = 1, 2, 3
NW_SCORE_ONLY, NW_TRACEBACK = 0, 1
# nw_ctx_set_option (include/nw.h): tuning / test options, 0 = the measured default
OPTIONS = {"rows_per_lane": 0, "d16_force": 1, "d16_kr": 2, "no_d16": 3, "tall_kr8": 4,
           "poll_ns": 5, "tb_step": 6, "tb_band": 7, "batch_kr16": 8, "batch_no_transpose": 9,
           "batch_tb_budget": 10, "host_plan": 11, "linear_int32": 12, "cblock_warps_per_sm": 13,
           "host_profile": 14, "watchdog_polls": 15, "test_withhold": 16,
           "dist_virtual_world": 17, "dist_virtual_rank": 18,
           "dist_pipeline": 19, "d16_chains": 20, "batch_u16_kr": 21, "batch_bnd_global": 22,
           "pair_form": 23, "h16_rebase": 24, "h16_kr": 25, "batch_mix_w": 26, "batch_mix_w24": 27}


class NWError(RuntimeError):
    def __init__(self, status: int, message: str, bad_pos: int = -1):
        super().__init__(f"[{status}] {message}")
        self.status = status
        self.bad_pos = bad_pos


class _Scoring(ctypes.Structure):
    _fields_ = [("match", ctypes.c_int32), ("mismatch", ctypes.c_int32), ("gap", ctypes.c_int32),
                ("subst", ctypes.POINTER(ctypes.c_int32)), ("alphabet", ctypes.c_char_p),
                ("K", ctypes.c_int32), ("tie", ctypes.c_uint8 * 3)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libnw_b200.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i64, i32, u32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32
    P = ctypes.POINTER
    sig = {
        "nw_ctx_create": ([ctypes.c_int, vp, P(vp)], ctypes.c_int),
        "nw_ctx_destroy": ([vp], None),
        "nw_strerror": ([ctypes.c_int], ctypes.c_char_p),
        "nw_last_error": ([vp], ctypes.c_char_p),
        "nw_last_bad_pos": ([vp], i64),
        "nw_ctx_sync": ([vp], ctypes.c_int),
        "nw_ctx_set_option": ([vp, i32, i64], ctypes.c_int),
        "nw_dist_unique_id": ([vp], ctypes.c_int),
        "nw_ctx_set_dist": ([vp, i32, i32, vp], ctypes.c_int),
        "nw_ctx_dist_info": ([vp, P(i32), P(i32)], ctypes.c_int),
        "nw_batch_partition": ([vp, i32, vp, i64, i32, vp], ctypes.c_int),
        "nw_ctx_get_option": ([vp, i32], i64),
        "nw_ctx_launches": ([vp], i64),
        "nw_ctx_set_timing": ([vp, ctypes.c_int], ctypes.c_int),
        "nw_ctx_kernel_time": ([vp, ctypes.c_int, P(ctypes.c_double), P(i64)], ctypes.c_int),
        "nw_score_only": ([vp, vp, i64, vp, i64, P(_Scoring), P(i64)], ctypes.c_int),
        "nw_score_only_dev": ([vp, vp, i64, vp, i64, P(_Scoring), vp], ctypes.c_int),
        "nw_align_pair": ([vp, vp, i64, vp, i64, P(_Scoring), P(i64), P(vp)], ctypes.c_int),
        "nw_align_pair_dev": ([vp, vp, i64, vp, i64, P(_Scoring), vp, P(vp)], ctypes.c_int),
        "nw_traceback": ([vp, vp, vp, i64, P(i64)], ctypes.c_int),
        "nw_traceback_dev": ([vp, vp, vp, i64, vp], ctypes.c_int),
        "nw_tb_free": ([vp], None),
        "nw_align_batch": ([vp, vp, vp, i32, vp, i64, P(_Scoring), u32, vp, vp, vp, vp],
                           ctypes.c_int),
        "nw_align_batch_dev": ([vp, vp, vp, vp, i32, vp, vp, i64, P(_Scoring), u32, vp, vp, vp,
                                vp], ctypes.c_int),
        "nw_batch_ops_offsets": ([vp, i32, vp, i64, vp], ctypes.c_int),
        "nw_score_only_cblock": ([vp, vp, i64, vp, i64, P(_Scoring), i32, i32, P(i64)],
                                 ctypes.c_int),
        "nw_cblock_recv_bytes": ([i64], i64),
        "nw_score_only_cblock_rank_dev": ([vp, vp, i64, vp, i64, P(_Scoring), i32, i32, i32, vp,
                                           vp, vp], ctypes.c_int),
        "nw_cblock_ipc_export": ([vp, i64, vp], ctypes.c_int),
        "nw_cblock_ipc_import": ([vp, vp], ctypes.c_int),
        "nw_msa_center_star": ([vp, vp, vp, i32, P(_Scoring), P(vp)], ctypes.c_int),
        "nw_msa_center_star_dev": ([vp, vp, vp, vp, i32, P(_Scoring), P(vp)], ctypes.c_int),
        "nw_msa_info": ([vp, P(i32), P(i64)], ctypes.c_int),
        "nw_msa_rows": ([vp, vp, vp, i64], ctypes.c_int),
        "nw_msa_rows_dev": ([vp], vp),
        "nw_msa_free": ([vp], None),
        "nw_align_pair_percell": ([vp, vp, i64, vp, i64, P(_Scoring), P(i64), vp, i64, P(i64)],
                                  ctypes.c_int),
        "nw_align_pair_percell_dev": ([vp, vp, i64, vp, i64, P(_Scoring), vp, vp, vp], ctypes.c_int),
        "nw_align_pair_linear": ([vp, vp, i64, vp, i64, P(_Scoring), i64, P(i64), vp, i64, P(i64)],
                                 ctypes.c_int),
        "nw_cooptimal": ([vp, vp, i64, vp, i64, P(_Scoring), i32, P(ctypes.c_uint64), P(i32), vp,
                          i64, vp, P(i32)], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        if os.environ.get("NW_LIB_PATH") and not hasattr(L, name):
            continue  # experiment builds of older sources may lack newer entry points
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


EXPORTED = ("nw_ctx_create", "nw_ctx_destroy", "nw_strerror", "nw_last_error", "nw_last_bad_pos",
            "nw_ctx_sync", "nw_ctx_set_option", "nw_ctx_get_option",
            "nw_dist_unique_id", "nw_ctx_set_dist", "nw_ctx_dist_info", "nw_batch_partition", "nw_ctx_launches", "nw_ctx_set_timing", "nw_ctx_kernel_time", "nw_score_only", "nw_score_only_dev",
            "nw_align_pair", "nw_align_pair_dev", "nw_traceback", "nw_traceback_dev",
            "nw_tb_free", "nw_align_batch", "nw_align_batch_dev", "nw_batch_ops_offsets",
            "nw_score_only_cblock", "nw_cblock_recv_bytes", "nw_score_only_cblock_rank_dev",
            "nw_cblock_ipc_export", "nw_cblock_ipc_import",
            "nw_msa_center_star", "nw_msa_center_star_dev", "nw_msa_info", "nw_msa_rows",
            "nw_msa_rows_dev", "nw_msa_free", "nw_align_pair_percell", "nw_align_pair_percell_dev",
            "nw_align_pair_linear", "nw_cooptimal")


def _scoring(sc) -> tuple[_Scoring, object]:
    """nw_scoring from any object with match/mismatch/gap/alphabet/subst/tie."""
    s = _Scoring()
    s.match, s.mismatch, s.gap = int(sc.match), int(sc.mismatch), int(sc.gap)
    keep = None
    if getattr(sc, "subst", None) is not None:
        keep = np.ascontiguousarray(np.asarray(sc.subst, dtype=np.int32))
        s.subst = keep.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    alpha = sc.alphabet.encode() if isinstance(sc.alphabet, str) else bytes(sc.alphabet)
    s.alphabet = alpha
    s.K = len(alpha)
    tie = tuple(getattr(sc, "tie", (1, 2, 3)))
    s.tie = (ctypes.c_uint8 * 3)(*tie)
    return s, (keep, alpha)


def _host_bytes(x) -> np.ndarray:
    if isinstance(x, (bytes, bytearray, memoryview)):
        return np.frombuffer(bytes(x), dtype=np.uint8)
    return np.ascontiguousarray(x, dtype=np.uint8)


def _ptr(x) -> int | None:
    """Address of a numpy array or torch tensor (host or device)."""
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        return x.data_ptr() if x.numel() else None
    return x.ctypes.data if x.size else None


class Context:
    """nw_ctx on one CUDA device; stream = a cudaStream_t handle (int) or None."""

    def __init__(self, device: int = 0, stream: int | None = None):
        self._h = ctypes.c_void_p()
        st = lib().nw_ctx_create(device, stream, ctypes.byref(self._h))
        if st != NW_OK:
            raise NWError(st, f"nw_ctx_create(device={device}): {lib().nw_strerror(st).decode()}")
        self.device = device

    def _check(self, st: int):
        if st != NW_OK:
            msg = lib().nw_last_error(self._h).decode(errors="replace")
            bad = lib().nw_last_bad_pos(self._h) if st == NW_E_ALPHABET else -1
            raise NWError(st, msg, bad)

    @property
    def handle(self):
        return self._h

    def launches(self) -> int:
        return int(lib().nw_ctx_launches(self._h))

    def set_timing(self, enable: bool = True):
        self._check(lib().nw_ctx_set_timing(self._h, int(enable)))

    def kernel_time(self, kernel_class: int) -> tuple[float, int]:
        """(summed event ms, launches) of class 0 = fill, 1 = traceback; resets."""
        ms, n = ctypes.c_double(), ctypes.c_int64()
        self._check(lib().nw_ctx_kernel_time(self._h, kernel_class, ctypes.byref(ms),
                                             ctypes.byref(n)))
        return ms.value, n.value

    def sync(self):
        self._check(lib().nw_ctx_sync(self._h))

    def set_option(self, name: str, value: int):
        """nw_ctx_set_option by name (OPTIONS); 0 restores the default."""
        self._check(lib().nw_ctx_set_option(self._h, OPTIONS[name], int(value)))

    def set_dist(self, rank: int, world: int, uid: bytes):
        """nw_ctx_set_dist: join the `world`-rank NCCL communicator named by uid
        (from nw_dist_unique_id on rank 0). Collective."""
        if len(uid) != 128:
            raise ValueError("uid must be 128 bytes")
        buf = ctypes.create_string_buffer(bytes(uid), 128)
        self._check(lib().nw_ctx_set_dist(self._h, int(rank), int(world), buf))

    def dist_info(self) -> tuple[int, int]:
        r, w = ctypes.c_int32(), ctypes.c_int32()
        self._check(lib().nw_ctx_dist_info(self._h, ctypes.byref(r), ctypes.byref(w)))
        return r.value, w.value

    def get_option(self, name: str) -> int:
        return int(lib().nw_ctx_get_option(self._h, OPTIONS[name]))

    @contextlib.contextmanager
    def options(self, **kw):
        """Set options for the duration of a with-block, then restore them."""
        old = {k: self.get_option(k) for k in kw}
        try:
            for k, v in kw.items():
                self.set_option(k, v)
            yield self
        finally:
            for k, v in old.items():
                self.set_option(k, v)

    def close(self):
        if self._h:
            lib().nw_ctx_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


class Traceback:
    """nw_tb handle: 2-bit packed directions resident on the device."""

    def __init__(self, ctx: Context, h: ctypes.c_void_p, m: int, n: int):
        self.ctx, self._h, self.m, self.n = ctx, h, m, n

    def free(self):
        if self._h:
            lib().nw_tb_free(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def nw_dist_unique_id() -> bytes:
    """128-byte NCCL id for Context.set_dist (no GPU needed)."""
    buf = ctypes.create_string_buffer(128)
    st = lib().nw_dist_unique_id(buf)
    if st != NW_OK:
        raise NWError(st, "nw_dist_unique_id: NCCL unavailable")
    return buf.raw


def nw_batch_partition(offs, pairs, world: int) -> np.ndarray:
    """bounds[0..world] of the dist batch partition (see include/nw.h)."""
    offs = np.ascontiguousarray(offs, dtype=np.int64)
    nseq = len(offs) - 1
    if pairs is None:
        npairs = nseq * (nseq - 1) // 2
    else:
        pairs = np.ascontiguousarray(pairs, dtype=np.int32).reshape(-1, 2)
        npairs = len(pairs)
    out = np.zeros(world + 1, dtype=np.int64)
    st = lib().nw_batch_partition(offs.ctypes.data, nseq, _ptr(pairs), npairs, world, out.ctypes.data)
    if st != NW_OK:
        raise NWError(st, "nw_batch_partition")
    return out


def nw_score_only(ctx: Context, a, b, sc) -> int:
    a, b = _host_bytes(a), _host_bytes(b)
    s, keep = _scoring(sc)
    out = ctypes.c_int64()
    ctx._check(lib().nw_score_only(ctx.handle, _ptr(a), len(a), _ptr(b), len(b), ctypes.byref(s),
                                   ctypes.byref(out)))
    return out.value


def nw_score_only_dev(ctx: Context, d_a, d_b, sc, d_score) -> None:
    """d_a, d_b: uint8 CUDA tensors; d_score: int64 CUDA tensor (1 element). Async."""
    s, keep = _scoring(sc)
    ctx._check(lib().nw_score_only_dev(ctx.handle, _ptr(d_a), d_a.numel(), _ptr(d_b), d_b.numel(),
                                       ctypes.byref(s), _ptr(d_score)))


def nw_align_pair(ctx: Context, a, b, sc) -> tuple[int, Traceback]:
    a, b = _host_bytes(a), _host_bytes(b)
    s, keep = _scoring(sc)
    out = ctypes.c_int64()
    tb = ctypes.c_void_p()
    ctx._check(lib().nw_align_pair(ctx.handle, _ptr(a), len(a), _ptr(b), len(b), ctypes.byref(s),
                                   ctypes.byref(out), ctypes.byref(tb)))
    return out.value, Traceback(ctx, tb, len(a), len(b))


def nw_align_pair_dev(ctx: Context, d_a, d_b, sc, d_score) -> Traceback:
    s, keep = _scoring(sc)
    tb = ctypes.c_void_p()
    ctx._check(lib().nw_align_pair_dev(ctx.handle, _ptr(d_a), d_a.numel(), _ptr(d_b), d_b.numel(),
                                       ctypes.byref(s), _ptr(d_score), ctypes.byref(tb)))
    return Traceback(ctx, tb, d_a.numel(), d_b.numel())


def nw_traceback(ctx: Context, tb: Traceback) -> np.ndarray:
    """Forward-order P:90 codes of the path (uint8 array)."""
    cap = tb.m + tb.n
    ops = np.empty(max(cap, 1), dtype=np.uint8)
    ln = ctypes.c_int64()
    ctx._check(lib().nw_traceback(ctx.handle, tb._h, ops.ctypes.data, cap, ctypes.byref(ln)))
    return ops[:ln.value].copy()


def nw_traceback_dev(ctx: Context, tb: Traceback, d_ops, d_len) -> None:
    """d_ops: uint8 CUDA tensor with >= m+n elements; d_len: int64 CUDA tensor. Async."""
    ctx._check(lib().nw_traceback_dev(ctx.handle, tb._h, _ptr(d_ops), d_ops.numel(), _ptr(d_len)))


def nw_batch_ops_offsets(offs: np.ndarray, pairs: np.ndarray | None) -> np.ndarray:
    offs = np.ascontiguousarray(offs, dtype=np.int64)
    nseq = len(offs) - 1
    if pairs is None:
        npairs = nseq * (nseq - 1) // 2
    else:
        pairs = np.ascontiguousarray(pairs, dtype=np.int32).reshape(-1, 2)
        npairs = len(pairs)
    out = np.empty(npairs + 1, dtype=np.int64)
    st = lib().nw_batch_ops_offsets(offs.ctypes.data, nseq, _ptr(pairs), npairs, out.ctypes.data)
    if st != NW_OK:
        raise NWError(st, "nw_batch_ops_offsets")
    return out


def batch_paths(ops: np.ndarray, ops_off: np.ndarray, ops_len: np.ndarray) -> list:
    """Per-pair forward op arrays from nw_align_batch's flat traceback output."""
    return [ops[ops_off[k]:ops_off[k] + ops_len[k]] for k in range(len(ops_len))]


def nw_align_batch(ctx: Context, seqs, offs, pairs, sc, flags: int = NW_SCORE_ONLY, out=None):
    """Host batch. Returns scores (int32[npairs]); with NW_TRACEBACK returns
    (scores, ops, ops_off, ops_len): pair k's path is ops[ops_off[k]:ops_off[k]+ops_len[k]]
    (see batch_paths). `out` = caller-owned output arrays to fill instead of fresh ones
    (scores, or (scores, ops, ops_off, ops_len) with NW_TRACEBACK), e.g. page-locked
    buffers so the library's copies run at DMA speed."""
    seqs = _host_bytes(seqs)
    offs = np.ascontiguousarray(offs, dtype=np.int64)
    nseq = len(offs) - 1
    if pairs is None:
        npairs = nseq * (nseq - 1) // 2
    else:
        pairs = np.ascontiguousarray(pairs, dtype=np.int32).reshape(-1, 2)
        npairs = len(pairs)
    s, keep = _scoring(sc)
    tbk = bool(flags & NW_TRACEBACK)
    if out is not None:
        scores, ops, ops_off, ops_len = (out, None, None, None) if not tbk else out
        if tbk:
            tot = int(nw_batch_ops_offsets(offs, pairs)[-1])
            if (len(scores) < npairs or len(ops_off) < npairs + 1 or len(ops) < max(tot, 1)
                    or len(ops_len) < max(npairs, 1)):
                raise ValueError("nw_align_batch: out buffers too small")
        elif len(scores) < npairs:
            raise ValueError("nw_align_batch: out buffer too small")
    else:
        scores = np.empty(npairs, dtype=np.int32)
        ops_off = np.empty(npairs + 1, dtype=np.int64) if tbk else None
        if tbk:
            tot = int(nw_batch_ops_offsets(offs, pairs)[-1])
            ops = np.empty(max(tot, 1), dtype=np.uint8)
            ops_len = np.empty(max(npairs, 1), dtype=np.int32)
        else:
            ops = ops_len = None
    ctx._check(lib().nw_align_batch(ctx.handle, _ptr(seqs), offs.ctypes.data, nseq, _ptr(pairs),
                                    npairs, ctypes.byref(s), flags, _ptr(scores), _ptr(ops_off),
                                    _ptr(ops), _ptr(ops_len)))
    if not tbk:
        return scores
    return scores, ops, ops_off, ops_len[:npairs]


def nw_align_batch_dev(ctx: Context, d_seqs, d_offs, h_offs, d_pairs, h_pairs, npairs: int, sc,
                       flags: int, d_scores, d_ops_off=None, d_ops=None, d_ops_len=None) -> None:
    """Device batch (torch CUDA tensors; h_offs/h_pairs numpy host copies). Async."""
    h_offs = np.ascontiguousarray(h_offs, dtype=np.int64)
    if h_pairs is not None:
        h_pairs = np.ascontiguousarray(h_pairs, dtype=np.int32)
    s, keep = _scoring(sc)
    ctx._check(lib().nw_align_batch_dev(ctx.handle, _ptr(d_seqs), _ptr(d_offs), h_offs.ctypes.data,
                                        len(h_offs) - 1, _ptr(d_pairs), _ptr(h_pairs), npairs,
                                        ctypes.byref(s), flags, _ptr(d_scores), _ptr(d_ops_off),
                                        _ptr(d_ops), _ptr(d_ops_len)))


def nw_score_only_cblock(ctx: Context, a, b, sc, ranks: int, block_cols: int = 0) -> int:
    """H(m, n) through the column-block wavefront over `ranks` virtual ranks (a10)."""
    a, b = _host_bytes(a), _host_bytes(b)
    s, keep = _scoring(sc)
    out = ctypes.c_int64()
    ctx._check(lib().nw_score_only_cblock(ctx.handle, _ptr(a), len(a), _ptr(b), len(b),
                                          ctypes.byref(s), ranks, block_cols, ctypes.byref(out)))
    return out.value


def nw_cblock_recv_bytes(m: int) -> int:
    """Bytes of one rank's receive buffer for the column-block pipeline."""
    return int(lib().nw_cblock_recv_bytes(m))


def nw_cblock_ipc_export(ctx: Context, m: int) -> bytes:
    """Allocate this context's receive buffer for m rows; its 64-byte CUDA IPC handle."""
    buf = ctypes.create_string_buffer(64)
    ctx._check(lib().nw_cblock_ipc_export(ctx.handle, int(m), buf))
    return buf.raw


def nw_cblock_ipc_import(ctx: Context, handle: bytes) -> None:
    """Open the next rank's receive buffer (its nw_cblock_ipc_export handle)."""
    ctx._check(lib().nw_cblock_ipc_import(ctx.handle, ctypes.create_string_buffer(bytes(handle), 64)))


def nw_score_only_cblock_rank_dev(ctx: Context, d_a, d_b, sc, rank: int, ranks: int,
                                  block_cols: int, recv_self, recv_next, d_score) -> None:
    """One rank of the column-block pipeline (see include/nw.h). recv_self = None: the
    context's exported/imported IPC buffers. Async."""
    s, keep = _scoring(sc)
    nxt = None if recv_next is None else _ptr(recv_next)
    ctx._check(lib().nw_score_only_cblock_rank_dev(ctx.handle, _ptr(d_a), d_a.numel(), _ptr(d_b),
                                                   d_b.numel(), ctypes.byref(s), rank, ranks,
                                                   block_cols, None if recv_self is None else _ptr(recv_self), nxt,
                                                   _ptr(d_score)))


class Msa:
    """nw_msa handle: center-star alignment rows resident on the device."""

    def __init__(self, ctx: Context, h: ctypes.c_void_p, nseq: int):
        self.ctx, self._h, self.nseq = ctx, h, nseq
        c, w = ctypes.c_int32(0), ctypes.c_int64(0)
        ctx._check(lib().nw_msa_info(h, ctypes.byref(c), ctypes.byref(w)))
        self.center, self.width = c.value, w.value

    def rows_array(self) -> np.ndarray:
        """(nseq, width) uint8 gapped rows ('-' = gap), input order."""
        out = np.empty((self.nseq, max(self.width, 1)), dtype=np.uint8)
        self.ctx._check(lib().nw_msa_rows(self.ctx.handle, self._h, out.ctypes.data, out.shape[1]))
        return out[:, :self.width]

    def rows(self) -> list[str]:
        return [r.tobytes().decode() for r in self.rows_array()]

    def rows_dev_ptr(self) -> int:
        return lib().nw_msa_rows_dev(self._h)

    def free(self):
        if self._h:
            lib().nw_msa_free(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def nw_msa_center_star(ctx: Context, seqs, offs, sc) -> Msa:
    """Center-star MSA of the sequences seqs[offs[k]:offs[k+1]] (host inputs)."""
    seqs = _host_bytes(seqs)
    offs = np.ascontiguousarray(offs, dtype=np.int64)
    s, keep = _scoring(sc)
    h = ctypes.c_void_p()
    ctx._check(lib().nw_msa_center_star(ctx.handle, _ptr(seqs), offs.ctypes.data, len(offs) - 1,
                                        ctypes.byref(s), ctypes.byref(h)))
    return Msa(ctx, h, len(offs) - 1)


def nw_msa_center_star_dev(ctx: Context, d_seqs, d_offs, h_offs, sc) -> Msa:
    """Device-input variant (torch CUDA tensors; h_offs the numpy host copy of d_offs)."""
    h_offs = np.ascontiguousarray(h_offs, dtype=np.int64)
    s, keep = _scoring(sc)
    h = ctypes.c_void_p()
    ctx._check(lib().nw_msa_center_star_dev(ctx.handle, _ptr(d_seqs), _ptr(d_offs),
                                            h_offs.ctypes.data, len(h_offs) - 1, ctypes.byref(s),
                                            ctypes.byref(h)))
    return Msa(ctx, h, len(h_offs) - 1)


def nw_align_pair_percell(ctx: Context, a, b, sc) -> tuple[int, np.ndarray]:
    """The paper's per-cell kernel (ablation baseline, NEXT #4): (score, forward ops)."""
    a, b = _host_bytes(a), _host_bytes(b)
    s, keep = _scoring(sc)
    score, ln = ctypes.c_int64(0), ctypes.c_int64(0)
    ops = np.empty(max(len(a) + len(b), 1), dtype=np.uint8)
    ctx._check(lib().nw_align_pair_percell(ctx.handle, _ptr(a), len(a), _ptr(b), len(b),
                                           ctypes.byref(s), ctypes.byref(score), ops.ctypes.data,
                                           len(ops), ctypes.byref(ln)))
    return score.value, ops[:ln.value].copy()


def nw_align_pair_percell_dev(ctx: Context, d_a, d_b, sc, d_score, d_ops, d_len) -> None:
    """Device variant of nw_align_pair_percell (torch CUDA tensors). Async."""
    s, keep = _scoring(sc)
    ctx._check(lib().nw_align_pair_percell_dev(ctx.handle, _ptr(d_a), d_a.numel(), _ptr(d_b),
                                               d_b.numel(), ctypes.byref(s), _ptr(d_score),
                                               _ptr(d_ops), _ptr(d_len)))


def nw_align_pair_linear(ctx: Context, a, b, sc, dirs_budget: int = 0) -> tuple[int, np.ndarray]:
    """Score + canonical traceback with at most ~dirs_budget bytes of directions on
    the device (checkpointed refill, NEXT #3). Returns (score, forward ops)."""
    a, b = _host_bytes(a), _host_bytes(b)
    s, keep = _scoring(sc)
    score, ln = ctypes.c_int64(0), ctypes.c_int64(0)
    ops = np.empty(max(len(a) + len(b), 1), dtype=np.uint8)
    ctx._check(lib().nw_align_pair_linear(ctx.handle, _ptr(a), len(a), _ptr(b), len(b),
                                          ctypes.byref(s), dirs_budget, ctypes.byref(score),
                                          ops.ctypes.data, len(ops), ctypes.byref(ln)))
    return score.value, ops[:ln.value].copy()


def nw_cooptimal(ctx: Context, a, b, sc, cap: int = 0):
    """(count, saturated, paths): the number of optimal alignments (saturating
    uint64) and, with cap > 0, the first cap of them in depth-first pi order."""
    a, b = _host_bytes(a), _host_bytes(b)
    s, keep = _scoring(sc)
    cnt, sat, nf = ctypes.c_uint64(0), ctypes.c_int32(0), ctypes.c_int32(0)
    ops_cap = cap * (len(a) + len(b))
    ops = np.empty(max(ops_cap, 1), dtype=np.uint8)
    off = np.zeros(cap + 1, dtype=np.int64)
    ctx._check(lib().nw_cooptimal(ctx.handle, _ptr(a), len(a), _ptr(b), len(b), ctypes.byref(s),
                                  cap, ctypes.byref(cnt), ctypes.byref(sat), ops.ctypes.data,
                                  ops_cap, off.ctypes.data, ctypes.byref(nf)))
    paths = [ops[off[k]:off[k + 1]].copy() for k in range(nf.value)] if cap else []
    return cnt.value, bool(sat.value), paths
