// nw_fill_d16dir.cuh -- difference-form packed sweep WITH decision bits, for the
// batch kernel's traceback mode.
//
// Difference form of Eq. 1 as in nw_fill_d16.cuh (Z = max(s-2g, V_up, U_left),
// U = Z - V_up, V = Z - U_left), two cells per register (rows k and k+h of a
// lane, the high half one column behind). The P:90 decision needs no extra
// comparisons: each candidate is maximal exactly when its difference to Z is 0,
//     D maximal <=> Z - (s-2g) == 0,   U maximal <=> U == 0,   L maximal <=> V == 0,
// so the bits for the tie order pi = (X, Y, Z) are nbX = [q_X != 0], nbY = [q_Y != 0]
// (code X if !nbX, else Y if !nbY, else Z). Both halves at once: min(q, 1) per half
// (VIMNMX.U16x2, one ALU-pipe cycle) gives nb in bit 0 of each half, and two IMADs on
// the FMA pipe pack them: m = 2 min(q_Y, 1) + min(q_X, 1), acc = 4 acc + m. Over the
// 8 steps of a group acc fills each half exactly (16 bits), so nothing carries from
// the low half into the high half. Per packed register and 8 steps one 32-bit word:
//   low half = the low cell (row k), high half = the high cell (row k+h); step q's
//   nbX at bit 2(7-q) of its half and nbY at bit 2(7-q)+1.
// Word index ((s*G + g)*32 + lane)*H + k, G = 8-step groups per strip: a lane's H words
// of a group are contiguous, stored as 16-byte vectors, so the traceback walk, which
// moves up through a lane's rows and left through a group's steps, finds them in one
// load (round 1: ((s*G + g)*H + k)*32 + lane, one 4-byte word per load).
// (Round 1 used q + 0x7fff7fff, a sign-replicating PRMT and a LOP3 per register and
// step, all on the ALU pipe, which that kernel saturated while the FMA pipe idled.)
#pragma once
#include "nw_fill_d16.cuh"

namespace nwk {

template <int KR>
struct D16DirState {
  uint32_t Up[KR / 2];
  uint32_t PA[KR / 2], PB[KR / 2];  // register profile (PROFREG)
  uint32_t acc[KR / 2];             // flags of the current 8-step group
  uint32_t vlast;
  uint32_t xT_prev, bc_prev, bc_nxt;
  int usum;
};

// MASKED groups hold the cell column n (the score's sum of U) or columns outside [1, n];
// HEAD groups (t0 < 64) hold halves left of column 1: their s' is forced to 0 (selector
// override / zero profile words), which keeps U = V = Z = 0 there with no mask (the
// other inputs are 0 by induction).
template <int KR, bool PROFREG, int PI, bool MASKED, bool HEAD = MASKED>
__device__ __forceinline__ void d16dir_group(D16DirState<KR>& st, const FillArgs& A, int lane,
                                             int t0, const int* bnd_in, int* bnd_out,
                                             uint32_t* dir_base, const int8_t* sprof,
                                             int rows_lo, int rows_hi, int chunk) {
  constexpr int H = KR / 2;
  constexpr int R = 32 * KR;
  using T = Tie<PI>;
  const int n = A.n;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int t = t0 + q;
    const int jT = t - 2 * lane + 1;
    const uint32_t bT = st.bc_nxt;
    st.bc_nxt = __ldg(A.b + jT);
    uint32_t sel = 0;
    uint2 lo8 = make_uint2(0, 0), hi8 = make_uint2(0, 0);
    if (PROFREG) {
      const uint32_t xT = bT * 17u;
      sel = xT + (st.xT_prev << 8) + (128u + (196u << 8));
      st.xT_prev = xT;
    } else {
      // s' of the lane's low rows for b_jT and of its high rows for b_jB (previous code)
      if constexpr (H == 8) {
        lo8 = *reinterpret_cast<const uint2*>(sprof + bT * R + lane * KR);
        hi8 = *reinterpret_cast<const uint2*>(sprof + st.bc_prev * R + lane * KR + H);
      } else {
        static_assert(H == 4, "packed traceback sweep: 8 or 16 rows per lane");
        lo8.x = *reinterpret_cast<const uint32_t*>(sprof + bT * R + lane * KR);
        hi8.x = *reinterpret_cast<const uint32_t*>(sprof + st.bc_prev * R + lane * KR + H);
      }
      st.bc_prev = bT;
    }
    if (HEAD) {  // halves left of column 1: s' = 0 (low half iff jT < 1, high half iff jT < 2)
      if (PROFREG) {
        if (jT < 2) sel = (jT < 1) ? 0xcc88u : ((sel & 0xffu) | 0xcc00u);
      } else {
        if (jT < 1) lo8 = make_uint2(0, 0);
        if (jT < 2) hi8 = make_uint2(0, 0);
      }
    }
    const int recv = __shfl_up_sync(FULL, (int)st.vlast, 1);
    const int bval = __shfl_sync(FULL, chunk, (t & 31));
    const uint32_t upsrc = (lane == 0) ? ((uint32_t)bval << 16) : (uint32_t)recv;
    uint32_t vup = prmt2(upsrc, st.vlast, 0x5432u);
#pragma unroll
    for (int k = 0; k < H; ++k) {
      uint32_t sp;
      if (PROFREG) {
        sp = prmt2(st.PA[k], st.PB[k], sel);
      } else {
        // byte k of lo8 into the low half, byte k of hi8 into the high half (zero-extended)
        const uint32_t b = (uint32_t)(k & 3);
        const uint32_t s2 = b | ((b | 8u) << 4) | ((4u + b) << 8) | ((12u + b) << 12);
        sp = prmt2(k < 4 ? lo8.x : lo8.y, k < 4 ? hi8.x : hi8.y, s2);
      }
      const uint32_t ul = st.Up[k];
      const uint32_t z = __vimax3_u16x2(sp, vup, ul);
      uint32_t un = z - vup;
      const uint32_t vn = z - ul;
      const uint32_t dd = z - sp;
      // q_X, q_Y in {D: dd, U: un, L: vn}; flag = [q == 0] per half (top bit of each half)
      const uint32_t qX = T::X == 1 ? dd : (T::X == 2 ? un : vn);
      const uint32_t qY = T::Y == 1 ? dd : (T::Y == 2 ? un : vn);
      // nb per half = min(q, 1); m = 2 nbY + nbX (bits 0-1 and 16-17); acc = 4 acc + m,
      // the word restarting every 8-step group
      const uint32_t m = __vminu2(qY, 0x00010001u) * 2u + __vminu2(qX, 0x00010001u);
      st.acc[k] = (q == 0 ? 0u : st.acc[k] * 4u) + m;
      st.Up[k] = un;
      vup = vn;
    }
    st.vlast = vup;
    const int jB = jT - 1;
    // (past column n the row has >= 64 entries of slack: only the head needs the check)
    if (lane == 31 && (!HEAD || (jB >= 1 && jB <= n))) bnd_out[(t0 - 62) + q] = (int)(vup >> 16);
    if (MASKED) {
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
  uint32_t* d = dir_base + (long long)(t0 >> 3) * (H * 32);
  static_assert(H % 4 == 0, "flag words are stored as 16-byte vectors");
#pragma unroll
  for (int k = 0; k < H; k += 4)
    *reinterpret_cast<uint4*>(d + k) = make_uint4(st.acc[k], st.acc[k + 1], st.acc[k + 2], st.acc[k + 3]);
}

// One strip of one pair inside the batch kernel (single warp, sequential strips).
// Adds sum U(i, n) of this strip to *A.hm.
template <int KR, bool PROFREG, int PI>
__device__ __forceinline__ void strip_sweep_d16dir(const FillArgs& A, int s, int lane,
                                                   int8_t* sprof) {
  constexpr int H = KR / 2;
  constexpr int R = 32 * KR;
  const int n = A.n;
  const int ia0 = s * R + lane * KR;
  D16DirState<KR> st;
  if (PROFREG) {
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
    }
  } else {
    for (int c = 0; c < A.K; ++c) {
#pragma unroll
      for (int r = 0; r < KR; ++r) sprof[c * R + lane * KR + r] = A.prof[A.a[ia0 + r] * A.K + c];
    }
    __syncwarp();
  }
#pragma unroll
  for (int k = 0; k < H; ++k) {
    st.Up[k] = 0;
    st.acc[k] = 0;
  }
  const int rows_lo = max(0, min(H, A.m - ia0));
  const int rows_hi = max(0, min(H, A.m - ia0 - H));
  st.vlast = 0;
  st.xT_prev = 0;
  st.bc_prev = 0;
  st.usum = 0;
  st.bc_nxt = __ldg(A.b - 2 * lane);
  const int* bnd_in = (s > 0) ? static_cast<const int*>(A.bnd) + (size_t)(s % A.nslots) * A.bstride : nullptr;
  int* bnd_out = static_cast<int*>(A.bnd) + (size_t)((s + 1) % A.nslots) * A.bstride;
  uint32_t* dir_base = reinterpret_cast<uint32_t*>(A.dirs) + (long long)s * A.wpl * (H * 32) + lane * H;
  const int ngrp = (n + 63 + 7) / 8;
  int chunk = 0;
#pragma unroll 1
  for (int g = 0; g < ngrp; ++g) {
    const int t0 = g * 8;
    if ((t0 & 31) == 0) {  // boundary V values for lane 0's columns t0+1 .. t0+32
      const int jj = t0 + 1 + lane;
      chunk = (s > 0 && jj <= n) ? bnd_in[jj] : 0;
    }
    const bool masked = t0 < 64 || t0 + 7 >= n - 1;  // (one masked variant: a third, tail-only
    if (masked)                                       //  one cost more in code size than it saved)
      d16dir_group<KR, PROFREG, PI, true>(st, A, lane, t0, bnd_in, bnd_out, dir_base, sprof,
                                          rows_lo, rows_hi, chunk);
    else
      d16dir_group<KR, PROFREG, PI, false>(st, A, lane, t0, bnd_in, bnd_out, dir_base, sprof,
                                           rows_lo, rows_hi, chunk);
  }
  int tot = st.usum;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(FULL, tot, o);
  if (lane == 0) *A.hm += tot;
  __syncwarp();
}

}  // namespace nwk
