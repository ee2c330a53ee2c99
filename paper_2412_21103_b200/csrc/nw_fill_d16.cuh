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

}  // namespace nwk
