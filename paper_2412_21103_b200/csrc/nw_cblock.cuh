// nw_cblock.cuh -- column-block wavefront for one giant pair across ranks
// (DESIGN.md §3.7). Score-only, DNA-size alphabets.
//
// The (m+1) x (n+1) grid of Eq. 1 is cut into strips of R = 32*KR
// rows (as in nw_fill.cuh) and column blocks of W columns; block b belongs to
// rank b % G (block-cyclic). A task (s, b) sweeps strip s over block b. It needs
//   - the strip above's bottom row over the block's columns: from task (s-1, b)
//     on the same rank, through the rank's tagged 64-bit ring (indexed by global
//     column);
//   - the left boundary column: the right column of task (s, b-1), written by
//     the previous rank into this rank's receive buffer as tagged 64-bit entries
//     (one store per value: a single-copy-atomic store carries its own validity,
//     so the same protocol works over NVLink peer memory; real ranks use .sys
//     scope, virtual ranks on one device .gpu);
// and produces the next strip's top row and its own right column for rank
// (b+1) % G. Each rank claims its tasks in (k, s) order (k = b / G) with an
// atomic ticket; every wait is on a task earlier in the order (k, s, rank), so
// the pipeline cannot deadlock as long as every rank's warps are resident.
//
// Two arithmetic forms:
//   k_fill_cblock_d16  the packed difference form of nw_fill_d16.cuh (two cells per
//                      register, s - 2g >= 0): V travels down the ring, U(i, c_b)
//                      crosses the block edge (no corner: the form has no diagonal
//                      term), and H(m,n) = g(m+n) + sum_i U(i,n) is summed by the
//                      owner of the last block.
//   k_fill_cblock      int32 H' (any s - 2g): H' travels down; the left message is
//                      the corner H'(top-1, c_b) plus R rows.
// Tags: seq(b, s) = base + b*S + s + 1 (mod 2^32), base = epoch * (nblocks*S + 1):
// every call of a context gets a fresh epoch, so buffers are zeroed once when
// allocated and never between calls (no barrier across ranks per call). A ring
// entry written by task (s, b) carries seq(b, s); the message task (s, b) sends to
// block b+1 carries seq(b+1, s) - the tag its consumer (s, b+1) expects.
#pragma once
#include "nw_fill.cuh"
#include "nw_fill16.cuh"
#include "nw_fill_d16.cuh"
#include "nw_fill_h16.cuh"

namespace nwk {

struct CBlockArgs {
  const uint8_t* a;      // row codes (padded)
  const uint8_t* b;      // column codes (padded)
  const int8_t* prof;    // K x K s - 2g
  int K, m, n;
  int W;                 // block width (columns)
  int G;                 // ranks
  int S;                 // strips
  int nblocks;
  // per-rank state (indexed by rank for virtual ranks; real ranks pass their own at index 0)
  unsigned long long* bnd;   // [ranks][2][n + 1 + 64] tagged top/bottom rows (column-indexed)
  long long bstride;
  unsigned long long* const* recv_tab;  // [G]: rank r's receive buffer [2][rstride] (tagged
                                        // left columns, block-slot k % 2, S messages); peer
                                        // pointers for real ranks (only own and next used)
  long long rstride;         // entries per slot
  long long mstride;         // entries per message (d16: R, int32: R + 1)
  unsigned tag_base;         // epoch * (nblocks * S + 1)
  int* ticket;               // [ranks]
  int* hm;                   // d16: sum of U(i, n) (the last block's owner); int32: H'(m, n)
  int* err;
  long long watchdog;        // re-polls before *err is raised
  const uint16_t* sel;       // h16: selector table aligned with b (nw_fill16.cuh)
  int reb_groups;            // h16: rebase period in 8-step groups (power of two)
  int rank0;                 // first rank handled by this launch (real ranks: own rank)
  int nranks_here;           // ranks handled by this launch (virtual: G, real: 1)
};

template <bool SYS>
__device__ __forceinline__ unsigned long long cb_ld(const unsigned long long* p) {
  unsigned long long v;
  if (SYS) asm volatile("ld.relaxed.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  else asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
template <bool SYS>
__device__ __forceinline__ void cb_st(unsigned long long* p, unsigned v, unsigned tag) {
  unsigned long long e;
  asm("mov.b64 %0, {%1, %2};" : "=l"(e) : "r"(v), "r"(tag));
  if (SYS) asm volatile("st.relaxed.sys.global.b64 [%0], %1;" ::"l"(p), "l"(e) : "memory");
  else asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(e) : "memory");
}

// Task (k, s) of this warp's rank -> block, column range, sequence numbers, message pointers.
struct CBTask {
  int k, s, blk, c0, c1, w;
  unsigned seq;                    // seq(blk, s): ring tag written, and message tag expected
  const unsigned long long* lin;   // left message (null: block 0, the grid border)
  unsigned long long* rout;        // right message to block blk + 1 (null: last block)
  unsigned rtag;                   // seq(blk + 1, s)
};

__device__ __forceinline__ bool cb_next_task(const CBlockArgs& A, int lr, int rank, int lane,
                                             const unsigned long long* recv_me, CBTask& T) {
  const int G = A.G;
  const int kmax = (A.nblocks - rank + G - 1) / G;  // blocks k*G + rank < nblocks
  const long long ntask = (long long)kmax * A.S;
  long long task = 0;
  if (lane == 0) task = atomicAdd(A.ticket + lr, 1);
  task = __shfl_sync(FULL, task, 0);
  if (task >= ntask) return false;
  T.k = (int)(task / A.S);
  T.s = (int)(task % A.S);
  T.blk = T.k * G + rank;
  T.c0 = T.blk * A.W;                       // columns c0+1 .. c1 (global, 1-based)
  T.c1 = min(A.n, T.c0 + A.W);
  T.w = T.c1 - T.c0;
  T.seq = A.tag_base + (unsigned)T.blk * (unsigned)A.S + (unsigned)T.s + 1u;
  T.lin = T.blk == 0 ? nullptr : recv_me + (size_t)(T.k & 1) * A.rstride + (size_t)T.s * A.mstride;
  T.rout = nullptr;
  T.rtag = 0;
  if (T.blk + 1 < A.nblocks) {
    const int rn = (T.blk + 1) % G, kn = (T.blk + 1) / G;
    T.rout = A.recv_tab[rn] + (size_t)(kn & 1) * A.rstride + (size_t)T.s * A.mstride;
    T.rtag = T.seq + (unsigned)A.S;
  }
  return true;
}

// Poll `cnt` consecutive message entries from e0 until all carry `tag`.
template <bool SYS, int CNT>
__device__ __forceinline__ void cb_recv(const CBlockArgs& A, const unsigned long long* p, unsigned tag,
                                        unsigned (&v)[CNT], int lane) {
  unsigned long long e[CNT];
  for (long long it = 0;; ++it) {
    bool ok = true;
#pragma unroll
    for (int r = 0; r < CNT; ++r) {
      e[r] = cb_ld<SYS>(p + r);
      ok = ok && (unsigned)(e[r] >> 32) == tag;
    }
    if (__all_sync(FULL, ok)) break;
    if (it > A.watchdog) {
      if (lane == 0) atomicExch(A.err, 8);
      break;
    }
  }
#pragma unroll
  for (int r = 0; r < CNT; ++r) v[r] = (unsigned)e[r];
}

// ---------------------------------------------------------------- difference form
// One 8-step group of the packed difference-form sweep over a block (cf. d16_group in
// nw_fill_d16.cuh, local columns 1..w): masked U keeps the left boundary B until each
// half reaches local column 1; at local column w each half's U goes to the next block.
template <int KR, bool SYS, bool MASKED>
__device__ __forceinline__ void cb_d16_group(D16State<KR>& st, const StripCtx& C, int t0, int rows_lo,
                                             int rows_hi, const uint32_t (&Bv)[KR / 2], bool last,
                                             unsigned long long* rout, unsigned rtag) {
  constexpr int H = KR / 2;
  const int lane = C.lane, w = C.n;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int t = t0 + q;
    const int jT = t - 2 * lane + 1;
    const uint32_t bT = st.bc_nxt;
    st.bc_nxt = __ldg(C.b + jT);
    const uint32_t xT = bT * 17u;
    const uint32_t sel = xT + (st.xT_prev << 8) + (128u + (196u << 8));
    st.xT_prev = xT;
    const int recv = __shfl_up_sync(FULL, (int)st.vlast, 1);
    const int bval = __shfl_sync(FULL, st.chunk_cur, q);
    const uint32_t upsrc = (lane == 0) ? ((uint32_t)bval << 16) : (uint32_t)recv;
    uint32_t vup = prmt2(upsrc, st.vlast, 0x5432u);
    uint32_t mask = 0xffffffffu;
    if (MASKED) mask = (jT >= 1 ? 0x0000ffffu : 0u) | (jT >= 2 ? 0xffff0000u : 0u);
#pragma unroll
    for (int k = 0; k < H; ++k) {
      const uint32_t sp = prmt2(st.PA[k], st.PB[k], sel);
      const uint32_t ul = st.Up[k];
      const uint32_t z = __vimax3_u16x2(sp, vup, ul);
      uint32_t un = z - vup;
      const uint32_t vn = z - ul;
      if (MASKED) un = (un & mask) | (Bv[k] & ~mask);  // U(i, c0): the left boundary
      st.Up[k] = un;
      vup = vn;
    }
    st.vlast = vup;
    const int jB = jT - 1;
    if (lane == 31 && (!MASKED || (jB >= 1 && jB <= w)))
      cb_st<false>(static_cast<unsigned long long*>(C.bnd_out) + jB, vup >> 16, C.tag_out);
    if (MASKED) {
      if (jT == w) {  // low halves reached the block's last column
#pragma unroll
        for (int k = 0; k < H; ++k) {
          if (rout) cb_st<SYS>(rout + lane * KR + k, st.Up[k] & 0xffffu, rtag);
          if (last && k < rows_lo) st.usum += (int)(st.Up[k] & 0xffffu);
        }
      }
      if (jB == w) {
#pragma unroll
        for (int k = 0; k < H; ++k) {
          if (rout) cb_st<SYS>(rout + lane * KR + H + k, st.Up[k] >> 16, rtag);
          if (last && k < rows_hi) st.usum += (int)(st.Up[k] >> 16);
        }
      }
    }
  }
}

template <int KR, bool SYS>
__global__ void __launch_bounds__(32) k_fill_cblock_d16(CBlockArgs A) {
  constexpr int H = KR / 2, R = 32 * KR;
  const int lane = threadIdx.x;
  const int lr = blockIdx.x % A.nranks_here;  // warp -> rank (virtual ranks round-robin)
  const int rank = A.rank0 + lr;
  unsigned long long* ring = A.bnd + (size_t)lr * 2 * A.bstride;
  const unsigned long long* recv_me = A.recv_tab[rank];
  CBTask T;
  while (cb_next_task(A, lr, rank, lane, recv_me, T)) {
    const int s = T.s;
    // left boundary U(s*R + r, c0) of this lane's rows, packed (row k | row k+H << 16)
    uint32_t Bv[H];
    if (T.lin) {
      unsigned lo[H], hi[H];
      cb_recv<SYS, H>(A, T.lin + lane * KR, T.seq, lo, lane);
      cb_recv<SYS, H>(A, T.lin + lane * KR + H, T.seq, hi, lane);
#pragma unroll
      for (int k = 0; k < H; ++k) Bv[k] = (lo[k] & 0xffffu) | (hi[k] << 16);
    } else {
#pragma unroll
      for (int k = 0; k < H; ++k) Bv[k] = 0;
    }
    const int ia0 = s * R + lane * KR;
    D16State<KR> st;
#pragma unroll
    for (int k = 0; k < H; ++k) {
      const int a0 = A.a[ia0 + k], a1 = A.a[ia0 + k + H];
      uint32_t w0 = 0, w1 = 0;
      for (int c = 0; c < A.K; ++c) {
        w0 |= ((uint32_t)(uint8_t)A.prof[a0 * A.K + c]) << (8 * c);
        w1 |= ((uint32_t)(uint8_t)A.prof[a1 * A.K + c]) << (8 * c);
      }
      st.PA[k] = w0;
      st.PB[k] = w1;
      st.Up[k] = Bv[k];
    }
    const bool last = T.c1 == A.n;
    const int rows_lo = max(0, min(H, A.m - ia0));
    const int rows_hi = max(0, min(H, A.m - ia0 - H));
    st.vlast = 0;
    st.xT_prev = 0;
    st.usum = 0;
    st.chunk_cur = st.chunk_nxt = 0;
    StripCtx C;
    C.b = A.b + T.c0;
    st.bc_nxt = __ldg(C.b - 2 * lane);
    C.sprof = nullptr;
    C.bnd_in = (s > 0) ? ring + (size_t)(s & 1) * A.bstride + T.c0 : nullptr;
    C.bnd_out = ring + (size_t)((s + 1) & 1) * A.bstride + T.c0;
    C.tag_in = T.seq - 1u;  // the strip above wrote seq(blk, s - 1)
    C.dir_base = nullptr;
    C.err = A.err;
    C.poll_ns = 0;
    C.watchdog = A.watchdog;
    C.hm = A.hm;
    C.tag_out = T.seq;     // ring tag this task writes
    C.n = T.w;
    C.s = s;
    C.lane = lane;
    if (s > 0) st.chunk_nxt = chunk_verify<true>(C, 0, chunk_issue<true>(C, 0));
    const int ngrp = (T.w + 63 + 7) / 8;
#pragma unroll 1
    for (int g = 0; g < ngrp; ++g) {
      const int t0 = g * 8;
      st.chunk_cur = st.chunk_nxt;
      const bool more = s > 0 && t0 + 8 < T.w;
      unsigned long long raw = 0;
      if (more) raw = chunk_issue<true>(C, t0 + 8);
      const bool masked = t0 < 64 || t0 + 7 >= T.w - 1;
      if (masked) cb_d16_group<KR, SYS, true>(st, C, t0, rows_lo, rows_hi, Bv, last, T.rout, T.rtag);
      else cb_d16_group<KR, SYS, false>(st, C, t0, rows_lo, rows_hi, Bv, last, T.rout, T.rtag);
      if (more) st.chunk_nxt = chunk_verify<true>(C, t0 + 8, raw);
    }
    if (last) {
      int tot = st.usum;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(FULL, tot, o);
      if (lane == 0) atomicAdd(A.hm, tot);
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------- packed H' form
template <int KR, typename St>
__device__ __forceinline__ void h16_rebase_cb(St& st) {
  constexpr int H = KR / 2;
  uint32_t mn = st.up0_prev;
#pragma unroll
  for (int k = 0; k < H; ++k) mn = __vminu2(mn, st.Hp[k]);
  int d = (int)min(mn & 0xffffu, mn >> 16);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) d = min(d, __shfl_xor_sync(FULL, d, o));
  const uint32_t dd = (uint32_t)d * 0x00010001u;
#pragma unroll
  for (int k = 0; k < H; ++k) st.Hp[k] -= dd;
  st.up0_prev -= dd;
  st.base += d;
}

// The packed H' sweep with a moving per-strip base of nw_fill_h16.cuh over a block:
// the task's values are kept relative to a warp-uniform base B, which starts at the
// corner H'(top-1, c0) (every cell of the task is >= it) and moves up every `reb`
// groups; the ring rows and the left messages carry ABSOLUTE H' (corner + R rows, as
// the int32 form). Halves left of local column 1 hold the left boundary column; rows
// past m have an all-zero profile, so they repeat row m and the last strip's bottom
// row at column n is H'(m, n) (nw_fill16.cuh).
template <int KR>
struct CbH16State {
  uint32_t PA[KR / 2], PB[KR / 2];
  uint32_t Hp[KR / 2];
  uint32_t up0_prev;
  int chunk_cur, chunk_nxt;
  int base;
  uint32_t sel_nxt[8];
  uint32_t bot7;  // lane 31: absolute bottom-row H' of the previous group's last step
};

template <int KR, bool SYS, bool MASKED>
__device__ __forceinline__ void cb_h16_group(CbH16State<KR>& st, const StripCtx& C, const uint16_t* sel,
                                             int t0, const uint32_t (&Bv)[KR / 2], int c0, bool hm_strip,
                                             unsigned long long* rout, unsigned rtag, int* hm) {
  constexpr int H = KR / 2;
  const int lane = C.lane, w = C.n;
  uint32_t scur[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) scur[q] = st.sel_nxt[q];
  const uint16_t* sp16 = sel + (t0 + 8 - 2 * lane);
#pragma unroll
  for (int q = 0; q < 8; ++q) st.sel_nxt[q] = __ldg(sp16 + q);
  uint32_t bot[8];
  const int jc = t0 + 1 + lane;
  const int crel = (lane < 8 && jc <= w) ? st.chunk_cur - st.base : 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int t = t0 + q;
    const uint32_t s = scur[q];
    const int recv = __shfl_up_sync(FULL, (int)st.Hp[H - 1], 1);
    const int bval = __shfl_sync(FULL, crel, q);
    const uint32_t upsrc = (lane == 0) ? ((uint32_t)bval << 16) : (uint32_t)recv;
    uint32_t up = prmt2(upsrc, st.Hp[H - 1], 0x5432u);
    uint32_t diag = st.up0_prev;
    st.up0_prev = up;
    const int jT = t - 2 * lane + 1;  // local column of the low halves
    uint32_t mask = 0xffffffffu;
    if (MASKED) mask = (jT >= 1 ? 0x0000ffffu : 0u) | (jT >= 2 ? 0xffff0000u : 0u);
#pragma unroll
    for (int k = 0; k < H; ++k) {
      const uint32_t sp = prmt2(st.PA[k], st.PB[k], s);
      const uint32_t left = st.Hp[k];
      uint32_t h = __vimax3_u16x2(diag + sp, left, up);
      if (MASKED) h = (h & mask) | (Bv[k] & ~mask);  // H'(i, c0): the left boundary column
      diag = left;
      up = h;
      st.Hp[k] = h;
    }
    const int jB = jT - 1;
    bot[q] = st.Hp[H - 1] >> 16;  // lane 31's bottom row at local column jB
    if (q == 6 && lane == 31) {
      // local columns t0-63 .. t0-56 = the consumer's chunk [8c+1, 8c+8], published together
      // (as nw_fill_h16.cuh; ring entries one slot up, 16-byte aligned pairs when c0 is even)
      const unsigned long long tg = (unsigned long long)C.tag_out << 32;
      const unsigned bb = (unsigned)st.base;
      const unsigned long long e[8] = {tg | st.bot7, tg | (bot[0] + bb), tg | (bot[1] + bb), tg | (bot[2] + bb),
                                       tg | (bot[3] + bb), tg | (bot[4] + bb), tg | (bot[5] + bb), tg | (bot[6] + bb)};
      unsigned long long* p = static_cast<unsigned long long*>(C.bnd_out) + (t0 - 63);
      const int j0 = t0 - 63;
      if ((c0 & 1) == 0 && (!MASKED || (j0 >= 1 && j0 + 7 <= w))) {
#pragma unroll
        for (int u = 0; u < 8; u += 2)
          asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};" ::"l"(p + u), "l"(e[u]), "l"(e[u + 1]) : "memory");
      } else {
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (j0 + u >= 1 && j0 + u <= w) st_relaxed_u64(p + u, e[u]);
      }
    }
    if (MASKED && hm_strip && lane == 31 && jB == w) *hm = (int)bot[q] + st.base;  // H'(m, n)
    if (MASKED && rout) {  // the right column (local column w) -> the next block's rank
      if (jT == w) {
#pragma unroll
        for (int k = 0; k < H; ++k) cb_st<SYS>(rout + 1 + lane * KR + k, (st.Hp[k] & 0xffffu) + st.base, rtag);
        if (lane == 0) cb_st<SYS>(rout, (unsigned)(bval + st.base), rtag);  // corner H'(top-1, c1)
      }
      if (jB == w) {
#pragma unroll
        for (int k = 0; k < H; ++k) cb_st<SYS>(rout + 1 + lane * KR + H + k, (st.Hp[k] >> 16) + st.base, rtag);
      }
    }
  }
  st.bot7 = bot[7] + (unsigned)st.base;  // local column t0-55: published with the next chunk
}

template <int KR, bool SYS>
__global__ void __launch_bounds__(32) k_fill_cblock_h16(CBlockArgs A) {
  constexpr int H = KR / 2, R = 32 * KR;
  const int lane = threadIdx.x;
  const int lr = blockIdx.x % A.nranks_here;
  const int rank = A.rank0 + lr;
  unsigned long long* ring = A.bnd + (size_t)lr * 2 * A.bstride;
  const unsigned long long* recv_me = A.recv_tab[rank];
  CBTask T;
  while (cb_next_task(A, lr, rank, lane, recv_me, T)) {
    const int s = T.s;
    const int ia0 = s * R + lane * KR;
    // left boundary column (absolute): corner + R rows; lane l reads entries l*KR .. l*KR+KR
    // (entry 0 of lane 0 is the corner H'(top-1, c0)); the grid border is 0
    unsigned v[KR + 1];
    if (T.lin) {
      cb_recv<SYS, KR + 1>(A, T.lin + lane * KR, T.seq, v, lane);
    } else {
#pragma unroll
      for (int r = 0; r <= KR; ++r) v[r] = 0;
    }
    CbH16State<KR> st;
    st.base = __shfl_sync(FULL, (int)v[0], 0);  // the corner: every cell of the task is >= it
    uint32_t Bv[H];
#pragma unroll
    for (int k = 0; k < H; ++k) {
      Bv[k] = (v[1 + k] - (unsigned)st.base) | ((v[1 + H + k] - (unsigned)st.base) << 16);
      const int a0 = A.a[ia0 + k], a1 = A.a[ia0 + k + H];
      uint32_t w0 = 0, w1 = 0;
      for (int c = 0; c < A.K; ++c) {
        w0 |= ((uint32_t)(uint8_t)A.prof[a0 * A.K + c]) << (8 * c);
        w1 |= ((uint32_t)(uint8_t)A.prof[a1 * A.K + c]) << (8 * c);
      }
      st.PA[k] = (ia0 + k < A.m) ? w0 : 0u;  // rows past m repeat row m (zero profile)
      st.PB[k] = (ia0 + k + H < A.m) ? w1 : 0u;
      st.Hp[k] = Bv[k];
    }
    st.up0_prev = 0;  // lane 0's first diag: the corner, relative 0
    st.chunk_cur = st.chunk_nxt = 0;
    const uint16_t* sel = A.sel + T.c0;  // selector table entries of the block's columns
#pragma unroll
    for (int q = 0; q < 8; ++q) st.sel_nxt[q] = __ldg(sel + (q - 2 * lane));
    StripCtx C;
    C.b = A.b + T.c0;
    C.sprof = nullptr;
    C.bnd_in = (s > 0) ? ring + (size_t)(s & 1) * A.bstride + T.c0 + 1 : nullptr;  // column j at index j+1
    C.bnd_out = ring + (size_t)((s + 1) & 1) * A.bstride + T.c0 + 1;
    C.tag_in = T.seq - 1u;
    C.tag_out = T.seq;
    C.dir_base = nullptr;
    C.err = A.err;
    C.poll_ns = 0;
    C.watchdog = A.watchdog;
    C.hm = A.hm;
    C.n = T.w;
    C.s = s;
    C.lane = lane;
    st.bot7 = 0;
    const bool hm_strip = s == A.S - 1 && T.c1 == A.n;
    if (s > 0) st.chunk_nxt = chunk_verify<true>(C, 0, chunk_issue<true>(C, 0));
    const int ngrp = (T.w + 63 + 7) / 8;
    const int rmask = A.reb_groups - 1;
#pragma unroll 1
    for (int g = 0; g < ngrp; ++g) {
      const int t0 = g * 8;
      if ((g & rmask) == 0 && g >= 8) h16_rebase_cb<KR>(st);
      st.chunk_cur = st.chunk_nxt;
      const bool more = s > 0 && t0 + 8 < T.w;
      unsigned long long raw = 0;
      if (more) raw = chunk_issue<true>(C, t0 + 8);
      const bool masked = t0 < 64 || t0 + 7 >= T.w - 1;
      if (masked) cb_h16_group<KR, SYS, true>(st, C, sel, t0, Bv, T.c0, hm_strip, T.rout, T.rtag, A.hm);
      else cb_h16_group<KR, SYS, false>(st, C, sel, t0, Bv, T.c0, hm_strip, T.rout, T.rtag, A.hm);
      if (more) st.chunk_nxt = chunk_verify<true>(C, t0 + 8, raw);
    }
    if (lane == 31) {  // the last step's ring entry (local column 8 ngrp - 63), if inside the block
      const int jl = 8 * ngrp - 63;
      if (jl >= 1 && jl <= T.w)
        st_relaxed_u64(static_cast<unsigned long long*>(C.bnd_out) + jl, ((unsigned long long)T.seq << 32) | st.bot7);
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------- int32 form
template <int KR, bool SYS>
__global__ void __launch_bounds__(32) k_fill_cblock(CBlockArgs A) {
  constexpr int R = 32 * KR;
  const int lane = threadIdx.x;
  const int lr = blockIdx.x % A.nranks_here;
  const int rank = A.rank0 + lr;
  unsigned long long* bnd = A.bnd + (size_t)lr * 2 * A.bstride;
  const unsigned long long* recv_me = A.recv_tab[rank];
  CBTask T;
  while (cb_next_task(A, lr, rank, lane, recv_me, T)) {
    const int s = T.s, c0 = T.c0, c1 = T.c1, w = T.w;
    const int ia0 = s * R + lane * KR;
    // ---- left boundary column: corner + R rows (from rank (blk-1) % G), or the grid border
    int B[KR];
    int corner = 0;
    if (!T.lin) {
#pragma unroll
      for (int r = 0; r < KR; ++r) B[r] = 0;
    } else {
      unsigned v[KR + 1];  // lane l: entries l*KR .. l*KR+KR (its diag corner and its KR rows)
      cb_recv<SYS, KR + 1>(A, T.lin + lane * KR, T.seq, v, lane);
      corner = (int)v[0];
#pragma unroll
      for (int r = 0; r < KR; ++r) B[r] = (int)v[r + 1];
    }
    uint32_t P[KR];
#pragma unroll
    for (int r = 0; r < KR; ++r) {
      const int ac = A.a[ia0 + r];
      uint32_t pw = 0;
      for (int c = 0; c < A.K; ++c) pw |= ((uint32_t)(uint8_t)A.prof[ac * A.K + c]) << (8 * c);
      P[r] = pw;
    }
    int Hl[KR];
#pragma unroll
    for (int r = 0; r < KR; ++r) Hl[r] = B[r];
    // diag of the lane's top row at its first column: H'(top-1, c0) = corner for lane 0;
    // lanes > 0 receive lane-1's masked bottom value B (= H'(top-1, c0)) one step earlier
    int diag = (lane == 0) ? corner : 0;
    int send = B[KR - 1];
    const unsigned long long* top_in = (s > 0) ? bnd + (size_t)(s & 1) * A.bstride : nullptr;
    unsigned long long* bot_out = bnd + (size_t)((s + 1) & 1) * A.bstride;
    const int hm_here = (A.m - 1) / R == s && c1 == A.n;
    const int hm_lane = ((A.m - 1) % R) / KR, hm_r = (A.m - 1) % KR;
    int chunk = 0;
    const int nsteps = w + 31;
    for (int t0 = 0; t0 < nsteps; t0 += 32) {
      // top boundary row for lane 0's columns c0+t0+1 .. +32 (tagged; strip 0: H'(0,j) = 0)
      if (s > 0) {
        const int jj = c0 + t0 + 1 + lane;
        const bool need = jj <= c1;
        unsigned long long v = need ? cb_ld<false>(top_in + jj) : 0ull;
        bool ok = !need || (unsigned)(v >> 32) == T.seq - 1u;
        for (long long it = 0; !__all_sync(FULL, ok); ++it) {
          if (!ok) { v = cb_ld<false>(top_in + jj); ok = (unsigned)(v >> 32) == T.seq - 1u; }
          if (it > A.watchdog) { if (lane == 0) atomicExch(A.err, 8); break; }
        }
        chunk = (int)(unsigned)v;
      }
#pragma unroll 4
      for (int q = 0; q < 32; ++q) {
        const int t = t0 + q;
        const int jl = t - lane + 1;      // local column 1..w
        const int j = c0 + jl;            // global column
        const uint32_t bc = A.b[j - 1];   // padded: local jl in [-30, w+32]
        const uint32_t sel = bc * 0x1111u + 0x8880u;
        const int recv = __shfl_up_sync(FULL, send, 1);
        const int bval = __shfl_sync(FULL, chunk, q);
        const int up = (lane == 0) ? bval : recv;
        const bool on = jl >= 1 && jl <= w;
        int hd = diag, hu = up;
#pragma unroll
        for (int r = 0; r < KR; ++r) {
          const int Sc = prmt(P[r], sel);
          int h = max(max(hd + Sc, Hl[r]), hu);
          h = (jl >= 1) ? h : B[r];       // left border until the lane reaches the block
          hd = Hl[r];
          hu = h;
          Hl[r] = h;
        }
        diag = up;
        send = Hl[KR - 1];
        if (lane == 31 && on) cb_st<false>(bot_out + j, (unsigned)send, T.seq);
        if (jl == w) {
          // this lane's right column -> next rank (rows lane*KR+1 .. +KR of the message);
          // lane 0 also sends the corner H'(top-1, c1) = the top row it just used
          if (T.rout) {
#pragma unroll
            for (int r = 0; r < KR; ++r) cb_st<SYS>(T.rout + lane * KR + r + 1, (unsigned)Hl[r], T.rtag);
            if (lane == 0) cb_st<SYS>(T.rout, (unsigned)up, T.rtag);
          }
          if (hm_here && lane == hm_lane) {
#pragma unroll
            for (int r = 0; r < KR; ++r)
              if (r == hm_r) *A.hm = Hl[r];
          }
        }
      }
    }
    __syncwarp();
  }
}

}  // namespace nwk
