// nw_fill_d16.cuh -- score-only sweep in difference form, two cells per register
// (DESIGN.md §3.8).
//
// Eq. 1 (reading R1) rewritten on the differences of neighbouring
// cells: with u(i,j) = H(i,j) - H(i-1,j), v(i,j) = H(i,j) - H(i,j-1) and the
// shifted U = u - g, V = v - g (both >= 0 because H(i,j) >= H(i-1,j) + g and
// H(i,j) >= H(i,j-1) + g),
//
//     Z(i,j) = max(s(a_i,b_j) - 2g,  V(i-1,j),  U(i,j-1))     (= H(i,j) - H(i-1,j-1) - 2g)
//     U(i,j) = Z(i,j) - V(i-1,j)       V(i,j) = Z(i,j) - U(i,j-1)
//
// with borders U(i,0) = 0 (from H(i,0) = i*g) and V(0,j) = 0, and
//     H(m,n) = g*(m+n) + sum_{i=1..m} U(i,n).
// Every U, V, Z lies in [0, max(s - 2g)], whatever the sequence lengths, so two
// cells share a 32-bit register at any size (C5 included): rows k and k+h of a
// lane are the low and high halves, the high half one column behind (as in
// nw_fill16.cuh), and per two cells the update is one PRMT (profile bytes), one
// VIMNMX3.U16x2 and two 32-bit IADDs (Z >= V_up and Z >= U_left half by half, so
// no borrow crosses the halves). Requires s - 2g >= 0 for every pair of symbols.
//
// Between strips only V of the bottom row travels (no diagonal term exists in
// this form). MULTIWARP strips use the tagged 64-bit entries of nw_fill.cuh.
#pragma once
#include "nw_fill.cuh"
#include "nw_fill16.cuh"

namespace nwk {

template <int KR>
struct D16State {
  uint32_t Up[KR / 2];  // U of packed row k at the previous column (U_left)
  uint32_t PA[KR / 2], PB[KR / 2];
  uint32_t vlast;       // V of packed h-1 from the previous step (its halves feed up(0))
  uint32_t xT_prev;     // 17 * code at the previous step's jT
  uint32_t bc_nxt;
  int chunk_cur, chunk_nxt;
  int usum;             // sum of U(i, n) over this lane's rows (<= m)
};

// 8 steps (t0 % 8 == 0). MASKED groups hold a half outside [1, n] or the column n.
template <int KR, bool MULTIWARP, bool MASKED>
__device__ __forceinline__ void d16_group(D16State<KR>& st, const StripCtx& C, int t0,
                                          int rows_lo, int rows_hi) {
  constexpr int H = KR / 2;
  const int lane = C.lane, n = C.n;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int t = t0 + q;
    const int jT = t - 2 * lane + 1;
    const uint32_t bT = st.bc_nxt;
    st.bc_nxt = __ldg(C.b + jT);  // next step's code (padding covers [-63, n + 95])
    const uint32_t xT = bT * 17u;
    const uint32_t sel = xT + (st.xT_prev << 8) + (128u + (196u << 8));
    st.xT_prev = xT;
    const int recv = __shfl_up_sync(FULL, (int)st.vlast, 1);
    const int bval = __shfl_sync(FULL, st.chunk_cur, q);
    // V_up(0): low = bottom row of lane l-1 at jT (its vlast high half; boundary row
    // for lane 0), high = this lane's packed h-1 low half at jB (previous step)
    const uint32_t upsrc = (lane == 0) ? ((uint32_t)bval << 16) : (uint32_t)recv;
    uint32_t vup = prmt2(upsrc, st.vlast, 0x5432u);
    uint32_t mask = 0xffffffffu;
    if (MASKED) mask = (jT >= 1 ? 0x0000ffffu : 0u) | (jT >= 2 ? 0xffff0000u : 0u);
#pragma unroll
    for (int k = 0; k < H; ++k) {
      const uint32_t sp = prmt2(st.PA[k], st.PB[k], sel);
      const uint32_t ul = st.Up[k];
      const uint32_t z = __vimax3_u16x2(sp, vup, ul);
      uint32_t un = z - vup;  // per half Z - V_up >= 0: no borrow between halves
      const uint32_t vn = z - ul;
      if (MASKED) un &= mask;  // U(i, 0) = 0 until each half reaches column 1
      st.Up[k] = un;
      vup = vn;
    }
    st.vlast = vup;
    const int jB = jT - 1;
    if (lane == 31 && (!MASKED || (jB >= 1 && jB <= n))) {
      const int vb = (int)(vup >> 16);  // bottom row V at jB
      if (MULTIWARP) {
        unsigned long long v;
        asm("mov.b64 %0, {%1, %2};" : "=l"(v) : "r"(vb), "r"(C.s + 1));
        st_relaxed_u64(static_cast<unsigned long long*>(C.bnd_out) + (t0 - 62) + q, v);
      } else {
        static_cast<int*>(C.bnd_out)[(t0 - 62) + q] = vb;
      }
    }
    if (MASKED) {
      // H(m,n) = g(m+n) + sum_i U(i,n): collect this lane's U at column n
      if (jT == n) {
#pragma unroll
        for (int k = 0; k < H; ++k)
          if (k < rows_lo) st.usum += (int)(st.Up[k] & 0xffffu);
      }
      if (jB == n) {
#pragma unroll
        for (int k = 0; k < H; ++k)
          if (k < rows_hi) st.usum += (int)(st.Up[k] >> 16);
      }
    }
  }
}

// One strip, score-only, difference form. Adds this strip's sum of U(i, n) to
// *A.hm (atomic for MULTIWARP; the batch kernel's warp owns its accumulator).
template <int KR, bool MULTIWARP>
__device__ __forceinline__ void strip_sweep_d16(const FillArgs& A, int s, int lane) {
  static_assert(KR % 2 == 0 && KR <= 32, "KR must be even");
  constexpr int H = KR / 2;
  constexpr int R = 32 * KR;
  const int n = A.n;
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
    st.Up[k] = 0;
  }
  // rows of this lane inside the grid: low half rows ia0 .. ia0+H-1, high ia0+H ..
  const int rows_lo = max(0, min(H, A.m - ia0));
  const int rows_hi = max(0, min(H, A.m - ia0 - H));
  st.vlast = 0;
  st.xT_prev = 0;
  st.usum = 0;
  st.chunk_cur = st.chunk_nxt = 0;
  st.bc_nxt = __ldg(A.b - 2 * lane);  // code at jT - 1 for step 0
  StripCtx C;
  C.tag_in = (unsigned)s;
  C.b = A.b;
  C.sprof = nullptr;
  const size_t esz = MULTIWARP ? 8 : 4;
  char* bnd = static_cast<char*>(A.bnd);
  C.bnd_in = (s > 0) ? bnd + esz * (size_t)((s % A.nslots) * A.bstride) : nullptr;
  C.bnd_out = bnd + esz * (size_t)(((s + 1) % A.nslots) * A.bstride);
  if (MULTIWARP && A.ckpt != nullptr) {  // checkpointed traceback pass:
    // every ck_every-th strip hands its bottom row's V over through a kept slot
    if ((s + 1) % A.ck_every == 0) C.bnd_out = A.ckpt + (long long)((s + 1) / A.ck_every - 1) * A.ck_stride;
    if (s > 0 && s % A.ck_every == 0) C.bnd_in = A.ckpt + (long long)(s / A.ck_every - 1) * A.ck_stride;
  }
  if (MULTIWARP && s + 1 == A.withhold) C.bnd_out = A.sink;
  C.dir_base = nullptr;
  C.err = A.err;
  C.poll_ns = A.poll_ns;
  C.watchdog = A.watchdog;
  C.hm = A.hm;
  C.n = n;
  C.s = s;
  C.lane = lane;
  if (s > 0) st.chunk_nxt = chunk_verify<MULTIWARP>(C, 0, chunk_issue<MULTIWARP>(C, 0));
  const int ngrp = (n + 63 + 7) / 8;  // last lane's high half reaches column n at t = n + 62
#pragma unroll 1
  for (int g = 0; g < ngrp; ++g) {
    const int t0 = g * 8;
    st.chunk_cur = st.chunk_nxt;
    const bool more = s > 0 && t0 + 8 < n;
    unsigned long long raw = 0;
    if (more) raw = chunk_issue<MULTIWARP>(C, t0 + 8);
    const bool masked = t0 < 64 || t0 + 7 >= n - 1;
    if (masked) d16_group<KR, MULTIWARP, true>(st, C, t0, rows_lo, rows_hi);
    else d16_group<KR, MULTIWARP, false>(st, C, t0, rows_lo, rows_hi);
    if (more) st.chunk_nxt = chunk_verify<MULTIWARP>(C, t0 + 8, raw);
  }
  // strip total of U(i, n)
  int tot = st.usum;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(FULL, tot, o);
  if (lane == 0) {
    if (MULTIWARP) atomicAdd(A.hm, tot);
    else *A.hm += tot;
  }
  __syncwarp();
}

// ---------------------------------------------------------------------------
// Two independent chains per lane (score-only, KR % 4 == 0). The sweep above runs
// one dependent chain through the lane's KR/2 packed registers per step (one
// VIMNMX3.U16x2 + one IADD per link): on C5 (KR 28: 14 links of ~10 cycles) a
// warp's step is bound by that chain, not by issue (ncu: 'wait' 44%, issue 48%).
// Here the lane's rows form four groups of Q = KR/4 rows, G0..G3 top to bottom,
// held in two register sets, each column-skewed so that within a step the two
// sets only read values the other produced in the previous step:
//   set A: low half = G0 rows at column jT,     high half = G2 rows at column jT-2
//   set B: low half = G1 rows at column jT-1,   high half = G3 rows at column jT-3
// so A's G2 half takes its top input (G1's bottom row at jT-2) and B takes G0's
// and G2's bottom rows (at jT-1, jT-3) from the previous step, and each step runs
// two chains of Q links that interleave. Lanes are skewed by 4 steps (lane l-1's
// G3 bottom row reaches column jT one step before lane l's G0 needs it). Same
// recurrence and arithmetic as d16_group, cell by cell.
template <int KR>
struct D16x2State {
  uint32_t UA[KR / 4], UB[KR / 4];    // U_left of the packed rows of sets A and B
  uint32_t PA0[KR / 4], PA2[KR / 4];  // profile words of G0 / G2 rows (set A low / high)
  uint32_t PB1[KR / 4], PB3[KR / 4];  // profile words of G1 / G3 rows (set B low / high)
  uint32_t vlastA, vlastB;            // V of each set's last packed row, previous step
  uint32_t x1, x2, x3;                // 17 * code at columns jT-1, jT-2, jT-3
  uint32_t bc_nxt;
  int chunk_cur, chunk_nxt;
  int usum;
};

template <int KR, bool MULTIWARP, bool MASKED>
__device__ __forceinline__ void d16x2_group(D16x2State<KR>& st, const StripCtx& C, int t0,
                                            const int (&rows)[4]) {
  constexpr int Q = KR / 4;
  const int lane = C.lane, n = C.n;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int t = t0 + q;
    const int jT = t - 4 * lane + 1;
    const uint32_t x0 = st.bc_nxt * 17u;
    st.bc_nxt = __ldg(C.b + jT);  // next step's code (padding covers [-127, n + 127])
    constexpr uint32_t CS = 128u + (196u << 8);
    const uint32_t selA = x0 + (st.x2 << 8) + CS;     // low: code at jT, high: at jT-2
    const uint32_t selB = st.x1 + (st.x3 << 8) + CS;  // low: at jT-1,  high: at jT-3
    st.x3 = st.x2;
    st.x2 = st.x1;
    st.x1 = x0;
    const int recv = __shfl_up_sync(FULL, (int)st.vlastB, 1);
    const int bval = __shfl_sync(FULL, st.chunk_cur, q);
    // A: low = lane above's G3 bottom row at jT (boundary row for lane 0), high = own
    // G1 bottom row at jT-2 (set B's low half, previous step). B: G0 / G2 bottom rows.
    const uint32_t upsrc = (lane == 0) ? ((uint32_t)bval << 16) : (uint32_t)recv;
    uint32_t vA = prmt2(upsrc, st.vlastB, 0x5432u);
    uint32_t vB = st.vlastA;
    uint32_t mA = 0xffffffffu, mB = 0xffffffffu;
    if (MASKED) {
      mA = (jT >= 1 ? 0x0000ffffu : 0u) | (jT >= 3 ? 0xffff0000u : 0u);
      mB = (jT >= 2 ? 0x0000ffffu : 0u) | (jT >= 4 ? 0xffff0000u : 0u);
    }
#pragma unroll
    for (int k = 0; k < Q; ++k) {
      const uint32_t spA = prmt2(st.PA0[k], st.PA2[k], selA);
      const uint32_t spB = prmt2(st.PB1[k], st.PB3[k], selB);
      const uint32_t ulA = st.UA[k], ulB = st.UB[k];
      const uint32_t zA = __vimax3_u16x2(spA, vA, ulA);
      const uint32_t zB = __vimax3_u16x2(spB, vB, ulB);
      uint32_t uA = zA - vA, uB = zB - vB;  // per half Z - V_up >= 0: no borrow across halves
      if (MASKED) { uA &= mA; uB &= mB; }
      vA = zA - ulA;
      vB = zB - ulB;
      st.UA[k] = uA;
      st.UB[k] = uB;
    }
    st.vlastA = vA;
    st.vlastB = vB;
    const int jb = jT - 3;  // bottom row (G3) column
    if (lane == 31 && (!MASKED || (jb >= 1 && jb <= n))) {
      const int vb = (int)(vB >> 16);
      if (MULTIWARP) {
        unsigned long long v;
        asm("mov.b64 %0, {%1, %2};" : "=l"(v) : "r"(vb), "r"(C.s + 1));
        st_relaxed_u64(static_cast<unsigned long long*>(C.bnd_out) + (t0 - 126) + q, v);
      } else {
        static_cast<int*>(C.bnd_out)[(t0 - 126) + q] = vb;
      }
    }
    if (MASKED) {  // H(m,n) = g(m+n) + sum_i U(i,n): each group's U at column n
      if (jT == n) {
#pragma unroll
        for (int k = 0; k < Q; ++k) if (k < rows[0]) st.usum += (int)(st.UA[k] & 0xffffu);
      }
      if (jT - 1 == n) {
#pragma unroll
        for (int k = 0; k < Q; ++k) if (k < rows[1]) st.usum += (int)(st.UB[k] & 0xffffu);
      }
      if (jT - 2 == n) {
#pragma unroll
        for (int k = 0; k < Q; ++k) if (k < rows[2]) st.usum += (int)(st.UA[k] >> 16);
      }
      if (jT - 3 == n) {
#pragma unroll
        for (int k = 0; k < Q; ++k) if (k < rows[3]) st.usum += (int)(st.UB[k] >> 16);
      }
    }
  }
}

template <int KR, bool MULTIWARP>
__device__ __forceinline__ void strip_sweep_d16x2(const FillArgs& A, int s, int lane) {
  static_assert(KR % 4 == 0 && KR <= 32, "KR must be a multiple of 4");
  constexpr int Q = KR / 4;
  constexpr int R = 32 * KR;
  const int n = A.n;
  const int ia0 = s * R + lane * KR;
  D16x2State<KR> st;
  auto word = [&](int row) {
    const int ac = A.a[row];
    uint32_t w = 0;
    for (int c = 0; c < A.K; ++c) w |= ((uint32_t)(uint8_t)A.prof[ac * A.K + c]) << (8 * c);
    return w;
  };
#pragma unroll
  for (int k = 0; k < Q; ++k) {
    st.PA0[k] = word(ia0 + k);
    st.PB1[k] = word(ia0 + Q + k);
    st.PA2[k] = word(ia0 + 2 * Q + k);
    st.PB3[k] = word(ia0 + 3 * Q + k);
    st.UA[k] = 0;
    st.UB[k] = 0;
  }
  int rows[4];
#pragma unroll
  for (int g = 0; g < 4; ++g) rows[g] = max(0, min(Q, A.m - ia0 - g * Q));
  st.vlastA = st.vlastB = 0;
  st.x1 = st.x2 = st.x3 = 0;
  st.usum = 0;
  st.chunk_cur = st.chunk_nxt = 0;
  st.bc_nxt = __ldg(A.b - 4 * lane);  // code at jT - 1 for step 0
  StripCtx C;
  C.tag_in = (unsigned)s;
  C.b = A.b;
  C.sprof = nullptr;
  const size_t esz = MULTIWARP ? 8 : 4;
  char* bnd = static_cast<char*>(A.bnd);
  C.bnd_in = (s > 0) ? bnd + esz * (size_t)((s % A.nslots) * A.bstride) : nullptr;
  C.bnd_out = bnd + esz * (size_t)(((s + 1) % A.nslots) * A.bstride);
  if (MULTIWARP && s + 1 == A.withhold) C.bnd_out = A.sink;
  C.dir_base = nullptr;
  C.err = A.err;
  C.poll_ns = A.poll_ns;
  C.watchdog = A.watchdog;
  C.hm = A.hm;
  C.n = n;
  C.s = s;
  C.lane = lane;
  if (s > 0) st.chunk_nxt = chunk_verify<MULTIWARP>(C, 0, chunk_issue<MULTIWARP>(C, 0));
  const int ngrp = (n + 127 + 7) / 8;  // lane 31's G3 reaches column n at t = n + 126
#pragma unroll 1
  for (int g = 0; g < ngrp; ++g) {
    const int t0 = g * 8;
    st.chunk_cur = st.chunk_nxt;
    const bool more = s > 0 && t0 + 8 < n;
    unsigned long long raw = 0;
    if (more) raw = chunk_issue<MULTIWARP>(C, t0 + 8);
    const bool masked = t0 < 128 || t0 + 7 >= n - 1;
    if (masked) d16x2_group<KR, MULTIWARP, true>(st, C, t0, rows);
    else d16x2_group<KR, MULTIWARP, false>(st, C, t0, rows);
    if (more) st.chunk_nxt = chunk_verify<MULTIWARP>(C, t0 + 8, raw);
  }
  int tot = st.usum;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(FULL, tot, o);
  if (lane == 0) {
    if (MULTIWARP) atomicAdd(A.hm, tot);
    else *A.hm += tot;
  }
  __syncwarp();
}

}  // namespace nwk
