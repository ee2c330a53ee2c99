// nw_fill.cuh -- the anti-diagonal wavefront fill of the NW grid on sm_100a.
//
// Computes Eq. 1 of PAPER.md (additive reading R1) over the
// (m+1) x (n+1) grid of Sec. 2.1 with the borders of Sec. 2.2, in the
// shifted form H'(i,j) = H(i,j) - g*(i+j):
//
//     H'(i,j) = max(H'(i-1,j-1) + s(a_i,b_j) - 2g,  H'(i-1,j),  H'(i,j-1))
//     H'(i,0) = H'(0,j) = 0,      H(m,n) = H'(m,n) + g*(m+n)
//
// which has the same argmax as Eq. 1 (the shift adds the same g*(i+j) to all
// three candidates) and needs no gap add on the up/left chains.
//
// Work decomposition: a warp owns a strip of R = 32*KR rows;
// lane l owns rows [l*KR, l*KR+KR) of it and sweeps the columns, lane l running
// one column behind lane l-1 (the anti-diagonal skew), so at step t lane l
// computes column j = t - l + 1 for its KR rows. The bottom cell of lane l-1 at
// column j arrives by __shfl_sync; the strip's top row comes from the strip
// above through a boundary row in global memory guarded by a release/acquire
// progress counter (replacing the per-cell spin of P:88-92, Code 1 P:110).
//
// With directions, every cell also yields two decision bits for the tie
// order pi = (X, Y, Z):  nb1 = [c_Y < c_Z],  nb0 = [c_X < max(c_Y, c_Z)]  (the
// sign bits of two differences); the code is X if !nb0, else Y if !nb1, else Z
// -- the first maximal candidate in pi. They are packed 16 cells per 32-bit
// word: word row w of lane l in strip s covers steps [w*SPW, w*SPW+SPW), cell
// index c = (t % SPW)*KR + r, bits (31-2c, 30-2c) = (nb1, nb0).
#pragma once
#include <cstdint>

namespace nwk {

constexpr unsigned FULL = 0xffffffffu;
constexpr int PAD = 64;  // code buffers carry PAD readable bytes before and after

struct FillArgs {
  const uint8_t* a;    // row codes, a[-PAD .. m+PAD) readable
  const uint8_t* b;    // column codes, b[-PAD .. n+PAD) readable
  const int8_t* prof;  // K x K table of s(x,y) - 2g (int8)
  int K;
  int m, n;
  int nstrips;
  int nslots;          // boundary ring slots (>= 2)
  int* bnd;            // [nslots][bstride] boundary rows H'(strip top, j), j = 0..n
  long long bstride;
  int* prog;           // [nstrips] columns of strip s's bottom row published
  int* ticket;         // strip dispenser
  uint32_t* dirs;      // [nstrips][wpl][32] packed decision bits (DIRS)
  long long wpl;       // words per lane per strip
  int* hm;             // H'(m, n) output
  int* err;            // watchdog flag (NW_E_DEADLOCK)
};

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Spin until *p >= need (acquire). Watchdog: ~2^24 polls with backoff, then flag.
__device__ __forceinline__ void wait_progress(const int* p, int need, int* err) {
  if (ld_acquire(p) >= need) return;
  unsigned ns = 32;
  for (long long it = 0;; ++it) {
    if (ld_acquire(p) >= need) return;
    __nanosleep(ns);
    if (ns < 256) ns <<= 1;
    if (it > (1ll << 24)) { atomicExch(err, 8); return; }
  }
}

// PRMT in its default mode: selector nibble = byte index (bits 0-2) + sign
// replicate flag (bit 3); used to sign-extend one int8 profile byte.
__device__ __forceinline__ int prmt(uint32_t x, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, 0, %2;" : "=r"(d) : "r"(x), "r"(sel));
  return (int)d;
}

// The tie order pi as a compile-time permutation: PI = 100*X + 10*Y + Z with
// X, Y, Z the P:90 codes (1 diag, 2 up, 3 left).
template <int PI>
struct Tie {
  static constexpr int X = PI / 100, Y = (PI / 10) % 10, Z = PI % 10;
};

template <int CODE>
__device__ __forceinline__ int pick(int cD, int cU, int cL) {
  return CODE == 1 ? cD : (CODE == 2 ? cU : cL);
}

// Per-lane state of one strip sweep (kept in registers: every function below
// is force-inlined and indexes the arrays with compile-time constants only).
template <int KR>
struct LaneState {
  int Hl[KR];        // H'(row r, previous column)
  uint32_t P[KR];    // register profile (PROFREG): byte c = s(a_r, c) - 2g
  int diag;          // H'(top-1, j-1)
  int send;          // H'(bottom, j), sent to lane+1
  int chunk_cur, chunk_nxt;  // boundary-row chunks (lane q holds column 32*blk+1+q)
  uint32_t acc;      // direction accumulator
};

// Strip geometry / pointers that stay fixed during one sweep.
struct StripCtx {
  const uint8_t* b;
  const int8_t* sprof;   // shared profile [K][R] (not PROFREG)
  const int* bnd_in;     // boundary row read (strip s-1's bottom), null for s == 0
  int* bnd_out;          // boundary row written (this strip's bottom)
  uint32_t* dir_base;    // this lane's direction words
  int* prog_in;          // strip s-1's progress counter (MULTIWARP)
  int* prog_out;         // this strip's progress counter (MULTIWARP)
  int* err;
  int* hm;
  int n, s, lane;
  int hm_lane, hm_r, hm_t;  // where H'(m, n) lives in this strip (hm_lane < 0: not here)
};

template <int KR, bool PROFREG>
__device__ __forceinline__ int cell_score(const LaneState<KR>& st, int r, uint32_t sel, uint2 pw) {
  if (PROFREG) return prmt(st.P[r], sel);
  const uint32_t w = (r < 4) ? pw.x : pw.y;  // byte r of the KR-byte profile column
  const uint32_t rr = (uint32_t)(r & 3);
  return prmt(w, rr | ((rr | 8u) * 0x1110u));
}

// 32 steps of the sweep: steps t0 .. t0+31, lane column j = t - lane + 1.
// MASKED blocks contain columns outside [1, n] for some lane (first / last blocks).
template <int KR, bool DIRS, bool PROFREG, int PI, bool MULTIWARP, bool MASKED>
__device__ __forceinline__ void sweep_block(LaneState<KR>& st, const StripCtx& C, int blk) {
  constexpr int R = 32 * KR, SPW = 16 / KR, WPB = 32 / SPW;
  using T = Tie<PI>;
  const int t0 = blk * 32;
  const int lane = C.lane, n = C.n;
  // boundary chunk for the next block: wait for the producer, then load
  st.chunk_cur = st.chunk_nxt;
  if (C.s > 0) {
    const int c0 = t0 + 32;  // chunk blk+1 covers columns c0+1 .. c0+32
    if (c0 < n) {
      if (MULTIWARP) wait_progress(C.prog_in, min(n, c0 + 32), C.err);
      const int jj = c0 + 1 + lane;
      st.chunk_nxt = (jj <= n) ? (MULTIWARP ? __ldcg(C.bnd_in + jj) : C.bnd_in[jj]) : 0;
    }
  }
#pragma unroll
  for (int q = 0; q < 32; ++q) {
    const int t = t0 + q;
    const int j = t - lane + 1;  // this lane's column (1-based)
    const uint32_t bc = C.b[j - 1];  // PAD bytes make j in [-31, n+62] readable
    uint32_t sel = 0;
    uint2 pw = make_uint2(0, 0);
    if (PROFREG) {
      sel = bc * 0x1111u | 0x8880u;  // byte bc, sign-replicated into bytes 1..3
    } else if (KR == 8) {
      pw = *reinterpret_cast<const uint2*>(C.sprof + bc * R + lane * KR);
    } else {
      pw.x = *reinterpret_cast<const uint32_t*>(C.sprof + bc * R + lane * KR);
    }
    // up = H'(top-1, j): lane 0 from the boundary row (0 for strip 0), others from lane-1
    const int recv = __shfl_up_sync(FULL, st.send, 1);
    const int bval = (C.s == 0) ? 0 : __shfl_sync(FULL, st.chunk_cur, q);  // s is warp-uniform
    const int up = (lane == 0) ? bval : recv;
    int hd = st.diag, hu = up;
#pragma unroll
    for (int r = 0; r < KR; ++r) {
      const int S = cell_score<KR, PROFREG>(st, r, sel, pw);
      const int cD = hd + S, cU = hu, cL = st.Hl[r];
      int h;
      if (DIRS) {
        const int cX = pick<T::X>(cD, cU, cL);
        const int cY = pick<T::Y>(cD, cU, cL);
        const int cZ = pick<T::Z>(cD, cU, cL);
        const int m1 = max(cY, cZ);
        h = max(cX, m1);
        const int d1 = cY - cZ;  // < 0  <=>  c_Y <  c_Z           (bit nb1)
        const int d0 = cX - m1;  // < 0  <=>  c_X <  max(c_Y, c_Z)  (bit nb0)
        st.acc = __funnelshift_l((uint32_t)d1, st.acc, 1);
        st.acc = __funnelshift_l((uint32_t)d0, st.acc, 1);
      } else {
        h = __vimax3_s32(cD, cU, cL);
      }
      if (MASKED) h = (j >= 1) ? h : 0;  // border column H'(i, 0) = 0 until the lane starts
      hd = st.Hl[r];
      hu = h;
      st.Hl[r] = h;
    }
    st.diag = MASKED ? ((j >= 1) ? up : 0) : up;
    st.send = st.Hl[KR - 1];
    if (DIRS && (q % SPW) == SPW - 1) C.dir_base[((long long)blk * WPB + q / SPW) * 32] = st.acc;
    if (lane == 31 && (!MASKED || (j >= 1 && j <= n))) C.bnd_out[j] = st.send;
    if (MASKED && lane == C.hm_lane && t == C.hm_t) {
#pragma unroll
      for (int r = 0; r < KR; ++r)
        if (r == C.hm_r) *C.hm = st.Hl[r];
    }
  }
  // publish this block's bottom-row columns (lane 31 wrote up to j = t0 + 1)
  if (MULTIWARP && lane == 31) {
    const int jdone = min(n, t0 + 1);
    if (jdone >= 1) st_release(C.prog_out, jdone);
  }
}

// One strip sweep: strip s = rows [s*R, s*R+R) of the grid (0-based a index).
// PROFREG: K <= 4, the lane's KR profile words live in registers and each
// cell's score is one PRMT; otherwise the profile column for b_j is read from
// shared memory (sprof, K x R bytes per warp).
template <int KR, bool DIRS, bool PROFREG, int PI, bool MULTIWARP>
__device__ __forceinline__ void strip_sweep(const FillArgs& A, int s, int lane, int8_t* sprof) {
  constexpr int R = 32 * KR;
  const int n = A.n;
  const int ia0 = s * R + lane * KR;  // 0-based row of this lane's first cell
  LaneState<KR> st;
  if (PROFREG) {
#pragma unroll
    for (int r = 0; r < KR; ++r) {
      const int ac = A.a[ia0 + r];  // rows past m read padding: garbage rows, never used
      uint32_t w = 0;
      for (int c = 0; c < A.K; ++c) w |= ((uint32_t)(uint8_t)A.prof[ac * A.K + c]) << (8 * c);
      st.P[r] = w;
    }
  } else {
#pragma unroll
    for (int r = 0; r < KR; ++r) st.P[r] = 0;
    for (int c = 0; c < A.K; ++c) {
#pragma unroll
      for (int r = 0; r < KR; ++r) sprof[c * R + lane * KR + r] = A.prof[A.a[ia0 + r] * A.K + c];
    }
    __syncwarp();
  }
#pragma unroll
  for (int r = 0; r < KR; ++r) st.Hl[r] = 0;
  st.diag = 0;
  st.send = 0;
  st.acc = 0;
  st.chunk_cur = st.chunk_nxt = 0;
  StripCtx C;
  C.b = A.b;
  C.sprof = sprof;
  C.bnd_in = (s > 0) ? A.bnd + (long long)(s % A.nslots) * A.bstride : nullptr;
  C.bnd_out = A.bnd + (long long)((s + 1) % A.nslots) * A.bstride;
  C.dir_base = DIRS ? A.dirs + (long long)s * A.wpl * 32 + lane : nullptr;
  C.prog_in = (MULTIWARP && s > 0) ? A.prog + (s - 1) : nullptr;
  C.prog_out = MULTIWARP ? A.prog + s : nullptr;
  C.err = A.err;
  C.hm = A.hm;
  C.n = n;
  C.s = s;
  C.lane = lane;
  C.hm_lane = -1; C.hm_r = 0; C.hm_t = 0;
  if ((A.m - 1) / R == s) {
    const int rr = (A.m - 1) % R;
    C.hm_lane = rr / KR; C.hm_r = rr % KR; C.hm_t = n - 1 + C.hm_lane;
  }
  // the first boundary chunk (block 0's columns 1..32)
  if (s > 0) {
    if (MULTIWARP) wait_progress(C.prog_in, min(n, 32), C.err);
    st.chunk_nxt = (lane + 1 <= n) ? (MULTIWARP ? __ldcg(C.bnd_in + lane + 1) : C.bnd_in[lane + 1]) : 0;
  }
  const int nblk = (n + 31 + 31) / 32;  // steps 0 .. n+30
  for (int blk = 0; blk < nblk; ++blk) {
    const bool masked = blk == 0 || blk * 32 + 31 >= n - 1;
    if (masked) sweep_block<KR, DIRS, PROFREG, PI, MULTIWARP, true>(st, C, blk);
    else sweep_block<KR, DIRS, PROFREG, PI, MULTIWARP, false>(st, C, blk);
  }
  if (MULTIWARP && lane == 31) st_release(C.prog_out, n);
  __syncwarp();
}

}  // namespace nwk
