// nw_fill16.cuh -- packed u16x2 score-only sweep.
//
// Same recurrence as nw_fill.cuh (Eq. 1, in the shifted form
// H' = H - g(i+j) with H' >= 0), two cells per 32-bit register: lane l owns
// KR = 2h rows; packed register k holds row k in its low half and row k+h in
// its high half, and the high ("bottom") half runs one column behind the low
// ("top") half:
//
//   step t, lane l:  low half at column jT = t - 2l + 1,  high half at jB = jT - 1
//
// so the two halves of every register are independent cells and one DPX
// instruction updates both:
//   up(k)   = packed k-1 of this step (k >= 1); for k = 0 the low half is the
//             bottom row of lane l-1 (shuffled, one step old) and the high half
//             is this lane's packed h-1 low half of the previous step
//   left(k) = packed k of the previous step, diag(k) = up(k) of the previous step
//   H'      = VIMNMX.U16x2(VIADDMNMX.U16x2(diag, s', left), up)
// Lanes are therefore skewed by two steps. Valid when s' = s - 2g >= 0 and
// min(m,n) * max(s') <= 65535 (the host checks; otherwise the int32 sweep runs).
#pragma once
#include "nw_fill.cuh"

namespace nwk {

__device__ __forceinline__ uint32_t prmt2(uint32_t x, uint32_t y, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(x), "r"(y), "r"(sel));
  return d;
}

struct U16State {
  uint32_t up0_prev;  // up(0) of the previous step (diag of packed 0)
  uint32_t send;      // packed h-1 (its high half = this lane's bottom row at jB)
  int chunk;          // boundary values, lane q holds column t0+1+q
};

// One 32-step block (t0 % 32 == 0). BORDER blocks (t0 < 64) hold halves left of
// column 1 (and, for n < 64, right of column n). A half at column <= 0 must stay 0
// (H'(i, 0) = 0): its inputs there (left, up, diag) are 0 by induction, so it is
// enough that its s' is 0, which the selector override gives (nibble 8 / 12 = sign
// replication of byte 0 of PA / PB, s' >= 0 -> 0x00) -- 2 instructions per step
// instead of a mask on every packed register. Past column n nothing needs masking:
// the cells there are never read, and the boundary row has >= 64 entries of slack.
template <int KR, bool BORDER>
__device__ __forceinline__ void u16_block(U16State& st, uint32_t (&PA)[KR / 2],
                                          uint32_t (&PB)[KR / 2], uint32_t (&Hp)[KR / 2],
                                          const FillArgs& A, int lane, int t0, int* bnd_out) {
  constexpr int H = KR / 2;
  const int n = A.n;
  // s' selector of step t: nibbles (bT, bT|8, 4+bB, 12+bB) -> byte bT of PA zero-extended
  // into the low half, byte bB of PB into the high half (s' >= 0: sign replication =
  // 0x00); (c | (c|8)<<4) = 17c + 128 and (4+c | (12+c)<<4) = 17c + 196 for c < 4. Read
  // from the host-built table A.sel (one 16-bit load per step, no ALU work): entry
  // jT - 1 holds (17 b[jT-1] + 128) | (17 b[jT-2] + 196) << 8, bB = b at column jT - 1.
  const uint16_t* sp16 = A.sel + (t0 - 2 * lane);
  int* op = bnd_out + (t0 - 62);             // lane 31's bottom row column jB = t - 62
#pragma unroll 8
  for (int q = 0; q < 32; ++q) {
    const int t = t0 + q;
    uint32_t sel = __ldg(sp16 + q);
    const int recv = __shfl_up_sync(FULL, (int)st.send, 1);
    const int bval = __shfl_sync(FULL, st.chunk, q);
    // up(0): low = lane l-1's bottom row at jT (its packed h-1 high half),
    //        high = own packed h-1 low half from the previous step
    const uint32_t upsrc = (lane == 0) ? ((uint32_t)bval << 16) : (uint32_t)recv;
    uint32_t up = prmt2(upsrc, Hp[H - 1], 0x5432u);
    uint32_t diag = st.up0_prev;
    st.up0_prev = up;
    const int jT = t - 2 * lane + 1;
    if (BORDER) {  // low half left of column 1 iff jT < 1, high half iff jB = jT - 1 < 1
      if (jT < 2) sel = (jT < 1) ? 0xcc88u : ((sel & 0xffu) | 0xcc00u);
    }
#pragma unroll
    for (int k = 0; k < H; ++k) {
      const uint32_t sp = prmt2(PA[k], PB[k], sel);
      const uint32_t left = Hp[k];
      // diag + s' as a plain 32-bit add (both halves < 2^16 - max s': no carry crosses),
      // which ptxas may issue on the FMA pipe, then one 3-input max on the ALU pipe:
      // 4 ALU-pipe cycles per two cells instead of 5 (PRMT 2 + VIADDMNMX 2 + VIMNMX 1)
      const uint32_t h = __vimax3_u16x2(diag + sp, left, up);
      diag = left;
      up = h;
      Hp[k] = h;
    }
    st.send = Hp[H - 1];
    const int jB = jT - 1;
    if (lane == 31 && (!BORDER || (jB >= 1 && jB <= n + 31))) op[q] = (int)(st.send >> 16);
  }
}

// One strip, score-only, packed. Same FillArgs / boundary conventions as
// strip_sweep<..., MULTIWARP = false> (the batch kernel's per-warp strips). Rows past
// m get an all-zero profile (s' = 0): such a row repeats the row above exactly
// (H'(i+1, j) = max(H'(i, j-1), H'(i, j), H'(i+1, j-1)) = H'(i, j), H' being
// non-decreasing along a row), so the last strip's bottom row is H'(m, .) and H'(m, n)
// is read from the boundary row after the sweep (no per-step capture).
template <int KR>
__device__ __forceinline__ void strip_sweep_u16(const FillArgs& A, int s, int lane) {
  static_assert(KR % 2 == 0 && KR <= 32, "KR must be even");
  constexpr int H = KR / 2;
  constexpr int R = 32 * KR;
  const int n = A.n;
  const int ia0 = s * R + lane * KR;
  // profiles: PA[k] bytes = s'(a_{k}, c), PB[k] bytes = s'(a_{k+h}, c), c < K <= 4
  uint32_t PA[H], PB[H], Hp[H];
#pragma unroll
  for (int k = 0; k < H; ++k) {
    const int a0 = A.a[ia0 + k], a1 = A.a[ia0 + k + H];
    uint32_t w0 = 0, w1 = 0;
    for (int c = 0; c < A.K; ++c) {
      w0 |= ((uint32_t)(uint8_t)A.prof[a0 * A.K + c]) << (8 * c);
      w1 |= ((uint32_t)(uint8_t)A.prof[a1 * A.K + c]) << (8 * c);
    }
    PA[k] = (ia0 + k < A.m) ? w0 : 0u;
    PB[k] = (ia0 + k + H < A.m) ? w1 : 0u;
    Hp[k] = 0;
  }
  const int* bnd_in = (s > 0) ? static_cast<const int*>(A.bnd) + (size_t)(s % A.nslots) * A.bstride : nullptr;
  int* bnd_out = static_cast<int*>(A.bnd) + (size_t)((s + 1) % A.nslots) * A.bstride;
  U16State st;
  st.up0_prev = 0;
  st.send = 0;
  st.chunk = 0;
  // boundary values H'(top-1, jT) for lane 0's columns t0+1 .. t0+32 (lane q: t0+1+q),
  // fetched one block ahead; strip 0's top row is H'(0, j) = 0
  int chunk_nxt = 0;
  if (s > 0) chunk_nxt = (lane + 1 <= n) ? bnd_in[lane + 1] : 0;
  const int nsteps = n + 63;  // last lane's high half reaches column n at t = n + 62
  for (int t0 = 0; t0 < nsteps; t0 += 32) {
    // orders this block's boundary loads (columns >= t0+33) before lane 31's later stores
    // to the same row (62 columns behind, in a later block): with the row in shared
    // memory (one slot) that is a write-after-read within the warp (racecheck)
    __syncwarp();
    st.chunk = chunk_nxt;
    if (s > 0) {
      const int jj = t0 + 33 + lane;
      chunk_nxt = (jj <= n) ? bnd_in[jj] : 0;
    }
    if (t0 < 64) u16_block<KR, true>(st, PA, PB, Hp, A, lane, t0, bnd_out);
    else u16_block<KR, false>(st, PA, PB, Hp, A, lane, t0, bnd_out);
  }
  __syncwarp();
  if (s == A.nstrips - 1 && lane == 0) *A.hm = bnd_out[n];  // H'(m, n): the bottom row at n
  __syncwarp();
}

}  // namespace nwk
