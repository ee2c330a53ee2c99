// nw_fill_h16.cuh -- score-only single-pair sweep in the shifted form H' with two
// cells per register and a moving per-strip base.
//
// Same recurrence as nw_fill.cuh (Eq. 1, reading R1, in the shifted form
// H' = H - g(i+j) >= 0 of DESIGN.md §3.1) and the same packed half-row layout as
// nw_fill16.cuh: lane l owns KR = 2h rows, packed register k holds row k (low half)
// and row k+h (high half, one column behind), lanes skewed by two steps, and per two
// cells the update is one PRMT (both profile bytes), one 32-bit add (diag + s', no
// carry crosses the halves) and one VIMNMX3.U16x2 -- one dependent link per packed
// row instead of the two of the difference form (nw_fill_d16.cuh: VIMNMX3 then IADD).
//
// H' itself grows without bound (up to min(m,n) * max(s')), so a strip keeps its
// values relative to a warp-uniform base B (int32): every register holds H' - B.
// Every `reb` 8-step groups the warp takes the minimum live value (a warp min of the
// lanes' minima) and moves B up by it. H' is non-decreasing down a column and along a
// row, and every live value of the strip lies between H'(top-1, jT0 - 64) and
// H'(bottom, jT0) (jT0 = lane 0's column), so with S = max(s') the relative values
// stay below S * (R + 65 + 8 * reb) + S, which the host keeps <= 65535 (h16_ok). The
// strips still exchange ABSOLUTE H' through the tagged 64-bit entries of nw_fill.cuh:
// lane 31 adds B when it publishes, lane 0's chunk subtracts B when it is taken.
// Border values (column 0, H'(i,0) = 0) are only present while B = 0: they are the
// live minimum until every half of the warp has left column 0.
#pragma once
#include "nw_fill.cuh"
#include "nw_fill16.cuh"

namespace nwk {

template <int KR>
struct H16State {
  uint32_t PA[KR / 2], PB[KR / 2];  // profile words of rows k and k+h (s' bytes per code)
  uint32_t Hp[KR / 2];              // H' - B of packed row k at the previous step
  uint32_t up0_prev;                // up(0) of the previous step (diag of packed 0)
  int chunk_cur, chunk_nxt;         // boundary H' (absolute) of 8 columns, lane q < 8: column t0+1+q
  int base;                         // B (warp-uniform)
  uint4 sel_nxt;                    // selector entries of the next group: 8 x u16 in one 16-byte load
  uint32_t acc[KR / 2], accp[KR / 2];  // DIRS: decision flags of this / the previous 8-step group
  uint32_t bot7;                    // lane 31: absolute bottom-row H' of the previous group's last step
};

// 8 steps (t0 % 8 == 0). MASKED groups hold a half outside [1, n] or the cell (m, n).
template <int KR, bool MASKED, bool DIRS = false, int PI = 123>
__device__ __forceinline__ void h16_group(H16State<KR>& st, const StripCtx& C, const uint16_t* sel,
                                          int t0) {
  using T = Tie<PI>;
  constexpr int H = KR / 2;
  const int lane = C.lane, n = C.n;
  // selectors of this group (prefetched one group ahead: a lone warp otherwise waits
  // for the first of them every group, ncu) and the loads of the next group's;
  // entry jT - 1 holds the codes of columns jT (low half) and jT - 1 (high half)
  // One 16-byte load per lane and group from the lane's shifted copy of the table
  // (FillArgs::sel4: copy k = lane % 4 is shifted by 2k entries, so the lane's 8 entries
  // start 16-byte aligned); odd entries are the high halves, moved down by an IMAD.HI
  // (FMA pipe; PRMT reads only the low 16 bits of its selector).
  const uint4 wcur = st.sel_nxt;
  st.sel_nxt = __ldg(reinterpret_cast<const uint4*>(sel + (t0 + 8 - 2 * lane)));
  const uint32_t scur[8] = {wcur.x, __umulhi(wcur.x, 65536u), wcur.y, __umulhi(wcur.y, 65536u),
                            wcur.z, __umulhi(wcur.z, 65536u), wcur.w, __umulhi(wcur.w, 65536u)};
  uint32_t bot[8];
  // lane 0 takes the boundary values relative to B (columns beyond n: 0, never read
  // by a cell inside the grid, and small enough to keep every half in range)
  const int jc = t0 + 1 + lane;
  const int crel = (lane < 8 && jc <= n) ? st.chunk_cur - st.base : 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int t = t0 + q;
    const uint32_t s = scur[q];
    const int recv = __shfl_up_sync(FULL, (int)st.Hp[H - 1], 1);
    const int bval = __shfl_sync(FULL, crel, q);
    // up(0): low = lane l-1's bottom row at jT (its packed h-1 high half, one step old;
    // for lane 0 the boundary row), high = own packed h-1 low half of the previous step
    const uint32_t upsrc = (lane == 0) ? ((uint32_t)bval << 16) : (uint32_t)recv;
    uint32_t up = prmt2(upsrc, st.Hp[H - 1], 0x5432u);
    uint32_t diag = st.up0_prev;
    st.up0_prev = up;
    const int jT = t - 2 * lane + 1;
    uint32_t mask = 0xffffffffu;
    if (MASKED) mask = (jT >= 1 ? 0x0000ffffu : 0u) | (jT >= 2 ? 0xffff0000u : 0u);
#pragma unroll
    for (int k = 0; k < H; ++k) {
      const uint32_t sp = prmt2(st.PA[k], st.PB[k], s);
      const uint32_t left = st.Hp[k];
      const uint32_t cd = diag + sp;
      uint32_t h = __vimax3_u16x2(cd, left, up);
      if (DIRS) {
        // P:90 decision for the tie order pi = (X, Y, Z): nbX = [c_X < H'], nbY = [c_Y < H'],
        // per half min(H' - c, 1) (H' >= c: no borrow between halves); two IMADs put step q
        // of the group at bits (2(7-q)+1, 2(7-q)) = (nbX, nbY) of each half, the int32
        // sweep's order (nw_fill.cuh)
        const uint32_t cX = T::X == 1 ? cd : (T::X == 2 ? up : left);
        const uint32_t cY = T::Y == 1 ? cd : (T::Y == 2 ? up : left);
        const uint32_t m = __vminu2(h - cX, 0x00010001u) * 2u + __vminu2(h - cY, 0x00010001u);
        st.acc[k] = (q == 0 ? 0u : st.acc[k] * 4u) + m;
      }
      if (MASKED) h &= mask;  // border column H'(i, 0) = 0 until each half starts (B = 0 then)
      diag = left;
      up = h;
      st.Hp[k] = h;
    }
    // lane 31's bottom row at jB = jT - 1 (relative), kept for the group's one vector store
    // (a global store every step sat in the MIO queue ahead of the next step's shuffle:
    // +40-60 cycles per step, tools/h16_step.cu)
    bot[q] = st.Hp[H - 1] >> 16;
    if (q == 6 && lane == 31) {
      // columns t0-63 .. t0-56 = the consumer's chunk [8c+1, 8c+8] (c = t0/8 - 8), complete
      // now: publish them together, so the next strip's chunk is valid at once (entries
      // sit one slot up: column j at ring index j+1, 16-byte aligned for j = 8c+1)
      const unsigned long long tg = (unsigned long long)C.tag_out << 32;
      const unsigned b = (unsigned)st.base;
      const unsigned long long e[8] = {tg | st.bot7, tg | (bot[0] + b), tg | (bot[1] + b), tg | (bot[2] + b),
                                       tg | (bot[3] + b), tg | (bot[4] + b), tg | (bot[5] + b), tg | (bot[6] + b)};
      unsigned long long* p = static_cast<unsigned long long*>(C.bnd_out) + (t0 - 63);
      const int j0 = t0 - 63;
      if (C.out_aligned && (!MASKED || (j0 >= 1 && j0 + 7 <= n))) {
#pragma unroll
        for (int u = 0; u < 8; u += 2)
          asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};" ::"l"(p + u), "l"(e[u]), "l"(e[u + 1]) : "memory");
      } else {
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (j0 + u >= 1 && j0 + u <= n) st_relaxed_u64(p + u, e[u]);
      }
    }
    if (MASKED && C.hm_lane == lane && C.hm_t == t) {  // H'(m, n), absolute
      const int hk = C.hm_r >= H ? C.hm_r - H : C.hm_r;
      uint32_t w = 0;
#pragma unroll
      for (int k = 0; k < H; ++k) w = (k == hk) ? st.Hp[k] : w;  // selects: Hp stays in registers
      *C.hm = (int)(C.hm_r >= H ? (w >> 16) : (w & 0xffffu)) + st.base;
    }
  }
  if (DIRS) {
    // Store the flags in the int32 sweep's layout (nw_fill.cuh: halfword ((s*G + g)*KR +
    // r)*32 + l, int32 step t = j - 1 + l, so the traceback kernels read either fill):
    // here the low half of lane l is at int32 step t0 + q - l, the high half at
    // t0 + q - l - 1. With l' = l (low) or l + 1 (high) = 8a + d, int32 group
    // g = t0/8 - a - 1 is complete after this group: its 8 steps are the previous
    // group's steps d..7 and this group's steps 0..d-1, i.e. bits 16-2d.. of
    // (prev << 16 | cur). Groups outside [0, G) are not stored.
    const int G = (int)C.wpl;
    const int glo = (t0 >> 3) - (lane >> 3) - 1, dlo = lane & 7;
    const int ghi = (t0 >> 3) - ((lane + 1) >> 3) - 1, dhi = (lane + 1) & 7;
    uint16_t* d = C.dir_base;
#pragma unroll
    for (int k = 0; k < H; ++k) {
      const uint32_t xlo = prmt2(st.acc[k], st.accp[k], 0x5410u);  // prev low << 16 | cur low
      const uint32_t xhi = prmt2(st.acc[k], st.accp[k], 0x7632u);  // prev high << 16 | cur high
      if (glo >= 0 && glo < G) d[((long long)glo * KR + k) * 32] = (uint16_t)(xlo >> (16 - 2 * dlo));
      if (ghi >= 0 && ghi < G) d[((long long)ghi * KR + k + H) * 32] = (uint16_t)(xhi >> (16 - 2 * dhi));
      st.accp[k] = st.acc[k];
    }
  }
  st.bot7 = bot[7] + (unsigned)st.base;  // column t0-55: published with the next group's chunk
}

// Moves B up by the warp's minimum live relative value (all halves of Hp and up0_prev).
template <int KR>
__device__ __forceinline__ void h16_rebase(H16State<KR>& st) {
  constexpr int H = KR / 2;
  uint32_t mn = st.up0_prev;
#pragma unroll
  for (int k = 0; k < H; ++k) mn = __vminu2(mn, st.Hp[k]);
  int d = (int)min(mn & 0xffffu, mn >> 16);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) d = min(d, __shfl_xor_sync(FULL, d, o));
  const uint32_t dd = (uint32_t)d * 0x00010001u;  // every half >= d: no borrow crosses
#pragma unroll
  for (int k = 0; k < H; ++k) st.Hp[k] -= dd;
  st.up0_prev -= dd;
  st.base += d;
}

// One strip, score-only, MULTIWARP (tagged 64-bit entries). A.sel4: four shifted copies
// of the selector table of nw_fill16.cuh aligned with b; A.reb_groups: rebase period in 8-step groups
// (a power of two).
// DIRS: also the P:90 decision bits for the tie order PI, stored in the int32 sweep's
// layout (A.dirs, A.wpl groups per strip), so the strip traceback reads them unchanged.
template <int KR, bool DIRS = false, int PI = 123>
__device__ __forceinline__ void strip_sweep_h16(const FillArgs& A, int s, int lane) {
  static_assert(KR % 2 == 0 && KR <= 32, "KR must be even");
  constexpr int H = KR / 2;
  constexpr int R = 32 * KR;
  const int n = A.n;
  const int ia0 = s * R + lane * KR;
  H16State<KR> st;
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
    st.Hp[k] = 0;
    st.acc[k] = 0;
    st.accp[k] = 0;
  }
  st.up0_prev = 0;
  st.base = 0;
  st.chunk_cur = st.chunk_nxt = 0;
  // the lane's copy of the selector table (entry i of copy k holds sel[i - 2k])
  const uint16_t* sel = A.sel4 + (lane & 3) * A.sel4_stride + 2 * (lane & 3);
  st.sel_nxt = __ldg(reinterpret_cast<const uint4*>(sel - 2 * lane));  // group 0
  StripCtx C;
  C.tag_in = (unsigned)s;
  C.tag_out = (unsigned)s + 1;
  C.b = A.b;
  C.sprof = nullptr;
  char* bnd = static_cast<char*>(A.bnd);
  // entries one slot up (column j at index j + 1): the chunk-aligned publication of
  // h16_group stores 16-byte-aligned pairs
  C.bnd_in = (s > 0) ? bnd + 8 * (size_t)((s % A.nslots) * A.bstride + 1) : nullptr;
  C.bnd_out = bnd + 8 * (size_t)(((s + 1) % A.nslots) * A.bstride + 1);
  C.out_aligned = 1;
  if (A.ckpt != nullptr) {  // checkpointed traceback pass: every ck_every-th
    // strip leaves its bottom row (absolute H', tagged s + 1, column j at index j: the refills'
    // layout) in a kept slot, which the next strip reads instead of the ring
    if ((s + 1) % A.ck_every == 0) {
      C.bnd_out = A.ckpt + (long long)((s + 1) / A.ck_every - 1) * A.ck_stride;
      C.out_aligned = 0;
    }
    if (s > 0 && s % A.ck_every == 0) C.bnd_in = A.ckpt + (long long)(s / A.ck_every - 1) * A.ck_stride;
  }
  if (s == 0 && A.top_row != nullptr) {  // a refill segment's strip 0: the checkpoint row above
    C.bnd_in = A.top_row;                 // (absolute H', column j at index j; tag top_tag)
    C.tag_in = A.top_tag;
  }
  if (s + 1 == A.withhold) C.bnd_out = static_cast<char*>(A.sink) + 8;
  st.bot7 = 0;
  C.dir_base = DIRS ? A.dirs + (long long)s * A.wpl * (KR * 32) + lane : nullptr;
  C.wpl = A.wpl;
  C.err = A.err;
  C.poll_ns = A.poll_ns;
  C.watchdog = A.watchdog;
  C.hm = A.hm;
  C.n = n;
  C.s = s;
  C.lane = lane;
  // where H'(m, n) lives: row rr of this strip -> lane, packed row, half; column n
  C.hm_lane = -1;
  C.hm_r = 0;
  C.hm_t = 0;
  if ((A.m - 1) / R == s) {
    const int rr = (A.m - 1) % R;
    C.hm_lane = rr / KR;
    C.hm_r = rr % KR;  // packed row hm_r % h, high half iff hm_r >= h
    C.hm_t = n - 1 + 2 * C.hm_lane + (C.hm_r >= H ? 1 : 0);
  }
  const bool has_top = C.bnd_in != nullptr;
  if (has_top) st.chunk_nxt = chunk_verify<true>(C, 0, chunk_issue<true>(C, 0));
  const int ngrp = (n + 63 + 7) / 8;  // last lane's high half reaches column n at t = n + 62
  const int rmask = A.reb_groups - 1;  // power of two
#pragma unroll 1
  for (int g = 0; g < ngrp; ++g) {
    const int t0 = g * 8;
    if ((g & rmask) == 0 && g > 0) h16_rebase<KR>(st);
#ifdef NW_TRACE
    if (A.trace && lane == 0 && (g & 255) == 0 && (g >> 8) < 256) {
      unsigned long long ts;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts));
      A.trace[(size_t)s * 256 + (g >> 8)] = ts;
    }
#endif
    st.chunk_cur = st.chunk_nxt;
    const bool more = has_top && t0 + 8 < n;
    unsigned long long raw = 0;
    if (more) raw = chunk_issue<true>(C, t0 + 8);
    const bool masked = t0 < 64 || t0 + 7 >= n - 1;
    if (masked) h16_group<KR, true, DIRS, PI>(st, C, sel, t0);
    else h16_group<KR, false, DIRS, PI>(st, C, sel, t0);
    if (more) st.chunk_nxt = chunk_verify<true>(C, t0 + 8, raw);
  }
  if (lane == 31) {  // the last step's bottom-row entry (column 8 ngrp - 63), if inside the grid
    const int jl = 8 * ngrp - 63;
    if (jl >= 1 && jl <= n)
      st_relaxed_u64(static_cast<unsigned long long*>(C.bnd_out) + jl,
                     ((unsigned long long)C.tag_out << 32) | st.bot7);
  }
  if (DIRS) {  // the last int32 group of lane 31's high half (l + 1 = 32: d = 0, a = 4)
    const int G = (int)A.wpl;
    const int ghi = ngrp - ((lane + 1) >> 3) - 1;
    const int glo = ngrp - (lane >> 3) - 1;
#pragma unroll
    for (int k = 0; k < H; ++k) {
      if (ghi < G && ((lane + 1) & 7) == 0) C.dir_base[((long long)ghi * KR + k + H) * 32] = (uint16_t)(st.accp[k] >> 16);
      if (glo < G && (lane & 7) == 0) C.dir_base[((long long)glo * KR + k) * 32] = (uint16_t)(st.accp[k] & 0xffffu);
    }
  }
  __syncwarp();
}

}  // namespace nwk
