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
// column j arrives by __shfl_sync. Between strips (MULTIWARP), lane 31 of strip
// s publishes its bottom row as 64-bit entries (tag = s+1, H') that strip s+1
// polls directly: a single-copy-atomic 8-byte store carries its own validity,
// so no fence or flag is needed (replacing the per-cell spin of P:88-92,
// Code 1 P:110, which had no memory ordering at all).
//
// With directions, every cell also yields two decision bits for the tie
// order pi = (X, Y, Z):  nbX = [c_X < H'],  nbY = [c_Y < H']  (the sign bits of
// c_X - H' and c_Y - H'); the code is X if !nbX, else Y if !nbY, else Z -- the
// first maximal candidate in pi. Each lane packs one row's bits of 8 steps into
// a halfword: group g = t/8, halfword index ((s*G + g)*KR + r)*32 + lane, step
// k = t%8 at bits (15-2k, 14-2k) = (nbX, nbY); every store is 64 contiguous bytes.
#pragma once
#include <cstdint>

namespace nwk {

constexpr unsigned FULL = 0xffffffffu;
constexpr int PAD = 128;  // code buffers carry PAD readable bytes before and after (lane skews up to 4 x 31)

struct FillArgs {
  const uint8_t* a;    // row codes, a[-PAD .. m+PAD) readable
  const uint8_t* b;    // column codes, b[-PAD .. n+PAD) readable
  const int8_t* prof;  // K x K table of s(x,y) - 2g (int8)
  int K;
  int m, n;
  int nstrips;
  int nslots;          // boundary ring slots (>= 2)
  void* bnd;           // [nslots][bstride] boundary rows: MULTIWARP 64-bit (tag<<32 | H'), else int H'
  long long bstride;   // entries per slot
  int* ticket;         // strip dispenser (MULTIWARP)
  uint16_t* dirs;      // [nstrips][wpl][KR][32] decision-bit halfwords (DIRS)
  long long wpl;       // 8-step groups per strip
  int* hm;             // H'(m, n) output
  int* err;            // watchdog flag (NW_E_DEADLOCK)
  // Checkpointed traceback, MULTIWARP only; null / 0 otherwise:
  unsigned long long* ckpt;           // strips s with (s+1) % ck_every == 0 write their bottom
  int ck_every;                       //   row here (tagged, slot (s+1)/ck_every - 1) instead of
  long long ck_stride;                //   the ring; strip s+1 reads it from there
  const unsigned long long* top_row;  // tagged H' of the row above strip 0 (null: zeros),
  unsigned top_tag;                   //   tagged top_tag (the checkpoint writer's s+1)
  unsigned poll_ns = 0;               // back-off between re-polls of a boundary chunk (0: spin)
  const uint16_t* sel = nullptr;      // packed sweeps (batch): selector table aligned with b, sel[i] =
                                      //   (17 b[i] + 128) | (17 b[i-1] + 196) << 8 (prmt2 of PA/PB)
  long long watchdog = 1LL << 28;     // re-polls of a late boundary chunk before *err is raised
  unsigned long long* trace = nullptr;  // experiment builds only (NW_TRACE): per-strip timestamps
  const uint16_t* sel8 = nullptr;     // int32 MULTIWARP sweep with register profiles: 8 copies of the
  long long sel8_stride = 0;          //   per-column PRMT selector (b*0x1111 + 0x8880), copy k holding
                                      //   column code b[i - k] at entry i (16-byte-aligned lane loads)
  const uint16_t* sel4 = nullptr;     // h16 sweep: 4 copies of the selector table, copy k (stride
  long long sel4_stride = 0;          //   sel4_stride entries) holding sel[i - 2k] at entry i
  int reb_groups = 64;                // h16 single-pair sweep: rebase period (8-step groups, power of 2)
  int withhold = 0;                   // test only (NW_OPT_TEST_WITHHOLD): strip withhold-1 writes its
  void* sink = nullptr;               //   bottom row to `sink` instead, so its consumer never sees it
};

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
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

// max through inline PTX: opaque to the LLVM optimiser, which would otherwise fold the
// prefix-form maxima below back into the serial chain max(c_r, H'(r-1)) (it did:
// same SASS as the chain form).
__device__ __forceinline__ int max_opq(int a, int b) {
  int d;
  asm("max.s32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ int max3_opq(int a, int b, int c) {
  int d;
  asm("max.s32 %0, %1, %2;\n\tmax.s32 %0, %0, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

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
  uint32_t acc[KR];  // decision bits of row r for the current 8-step group (DIRS)
  int diag;          // H'(top-1, j-1)
  int send;          // H'(bottom, j): sent to lane+1
  int chunk_cur, chunk_nxt;  // boundary values for 8 columns (lane q < 8 holds column t0+1+q)
  uint32_t bc_nxt;   // prefetched column code for the next step
  uint4 selw;        // (MULTIWARP, PROFREG) the next group's 8 selectors, one 16-byte load
  const uint16_t* seltab;  // this lane's copy of A.sel8, offset so that seltab[i] is b[i]'s selector
};

// Strip geometry / pointers that stay fixed during one sweep.
struct StripCtx {
  const uint8_t* b;
  const int8_t* sprof;              // shared profile [K][R] (not PROFREG)
  const void* bnd_in;               // boundary row read (strip s-1's bottom), null for s == 0
  unsigned tag_in;                  // tag the bnd_in entries carry (strip s-1 wrote s)
  unsigned tag_out;                 // tag this sweep writes (column-block sweeps; others use s+1)
  void* bnd_out;                    // boundary row written (this strip's bottom)
  uint16_t* dir_base;               // this lane's decision-bit halfwords
  long long wpl;                    // h16 with directions: 8-step (int32) groups per strip
  int out_aligned;                  // h16: bnd_out is the ring shifted one slot (16-byte pairs), not a checkpoint row
  int* err;
  int* hm;
  unsigned poll_ns;
  long long watchdog;
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

// Boundary chunk = the strip-above's bottom-row values of 8 columns c0+1..c0+8,
// lane q < 8 holding column c0+1+q. Issued one 8-step group before it is used
// and verified (MULTIWARP: tag == s) just before, so the L2 round trip overlaps
// a whole group of steps.
template <bool MULTIWARP>
__device__ __forceinline__ unsigned long long chunk_issue(const StripCtx& C, int c0) {
  const int jj = c0 + 1 + C.lane;
  if (C.lane >= 8 || jj > C.n) return 0ull;
  if (!MULTIWARP) return (unsigned)static_cast<const int*>(C.bnd_in)[jj];
  return ld_relaxed_u64(static_cast<const unsigned long long*>(C.bnd_in) + jj);
}

template <bool MULTIWARP>
__device__ __forceinline__ int chunk_verify(const StripCtx& C, int c0, unsigned long long v) {
  if (!MULTIWARP) return (int)(unsigned)v;
  const int jj = c0 + 1 + C.lane;
  const bool need = C.lane < 8 && jj <= C.n;
  const unsigned tag = C.tag_in;  // strip s-1 writes tag (s-1)+1 (a checkpoint row: top_tag)
  bool ok = !need || (unsigned)(v >> 32) == tag;
  if (__all_sync(FULL, ok)) return (int)(unsigned)v;
  const unsigned long long* p = static_cast<const unsigned long long*>(C.bnd_in) + jj;
  // re-poll without sleeping by default: a single-pair warp is usually alone on its
  // SM sub-partition, and a sleep adds its granularity to every strip hand-off;
  // poll_ns > 0 backs off (frees issue slots for co-resident warps)
  for (long long it = 0;; ++it) {
    if (C.poll_ns) __nanosleep(C.poll_ns);
    if (!ok) {
      v = ld_relaxed_u64(p);
      ok = (unsigned)(v >> 32) == tag;
    }
    if (__all_sync(FULL, ok)) break;
    if (it > C.watchdog) {  // watchdog: report and stop waiting (results invalid)
      if (C.lane == 0) atomicExch(C.err, 8);
      break;
    }
  }
  return (int)(unsigned)v;
}

// One 8-step group of the sweep starting at t0 (t0 % 8 == 0): lane column j = t - lane + 1.
// MASKED groups contain columns outside [1, n] for some lane (or the H'(m,n) cell).
template <int KR, bool DIRS, bool PROFREG, int PI, bool MULTIWARP, bool MASKED>
__device__ __forceinline__ void sweep_group(LaneState<KR>& st, const StripCtx& C, int t0) {
  constexpr int R = 32 * KR;
  using T = Tie<PI>;
  const int lane = C.lane, n = C.n;
  constexpr bool VSEL = MULTIWARP && PROFREG && KR <= 4;  // (taller strips, e.g. the checkpointed refills: slower)
  uint4 wsel = make_uint4(0, 0, 0, 0);
  if constexpr (VSEL) {  // this group's selectors (loaded a group ahead), and the next group's
    wsel = st.selw;
    st.selw = __ldg(reinterpret_cast<const uint4*>(st.seltab + (t0 + 8 - lane)));
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int t = t0 + q;
    const int j = t - lane + 1;  // this lane's column (1-based)
    uint32_t bc = 0;
    if constexpr (!VSEL) {
      bc = st.bc_nxt;
      st.bc_nxt = __ldg(C.b + j);  // next step's b_{j+1} (PAD makes j in [-31, n+62] readable)
    }
    uint32_t sel = 0;
    uint2 pw = make_uint2(0, 0);
    if constexpr (VSEL) {
      // b[j-1]'s selector: entry q of the group's 16-byte block (odd entries: the high half,
      // moved down by an IMAD.HI; PRMT reads only the low 16 bits of its selector)
      const uint32_t w = (q >> 1) == 0 ? wsel.x : (q >> 1) == 1 ? wsel.y : (q >> 1) == 2 ? wsel.z : wsel.w;
      sel = (q & 1) ? __umulhi(w, 65536u) : w;
    } else if constexpr (PROFREG) {
      sel = bc * 0x1111u + 0x8880u;  // byte bc, sign-replicated into bytes 1..3 (bc < 8: no carry)
    } else if constexpr (KR == 8) {
      pw = *reinterpret_cast<const uint2*>(C.sprof + bc * R + lane * KR);
    } else if constexpr (KR == 4) {
      pw.x = *reinterpret_cast<const uint32_t*>(C.sprof + bc * R + lane * KR);
    } else {
      static_assert(KR == 2, "shared-memory profile: KR must be 2, 4 or 8");
      pw.x = *reinterpret_cast<const uint16_t*>(C.sprof + bc * R + lane * KR);
    }
    // Prefix form of the vertical chain: with c_r = max(cD_r, cL_r) (no dependence on the
    // lane above), H'(r) = max(c_r, H'(r-1)) = max(P_r, up) for P_r = max(c_0..c_r). The
    // P_r chain runs while the shuffle bringing `up` is in flight; once it lands, every
    // row is one independent max, so the lane-to-lane critical path per step is
    // SHFL + SEL + one max instead of SHFL + KR dependent maxima.
    int S[KR], cD[KR], P[KR];
#pragma unroll
    for (int r = 0; r < KR; ++r) {
      S[r] = cell_score<KR, PROFREG>(st, r, sel, pw);
      cD[r] = (r == 0 ? st.diag : st.Hl[r - 1]) + S[r];
      P[r] = (r == 0) ? max_opq(cD[0], st.Hl[0]) : max3_opq(cD[r], st.Hl[r], P[r - 1]);
    }
    // up = H'(top-1, j): lane 0 from the boundary row (0 for strip 0), others from lane-1
    const int recv = __shfl_up_sync(FULL, st.send, 1);
    const int bval = __shfl_sync(FULL, st.chunk_cur, q);  // strip 0: chunks hold H'(0, j) = 0
    const int up = (lane == 0) ? bval : recv;
    int hu = up;
#pragma unroll
    for (int r = 0; r < KR; ++r) {
      int h = max_opq(P[r], up);
      if (DIRS) {
        const int cU = hu, cL = st.Hl[r];
        const int cX = pick<T::X>(cD[r], cU, cL);
        const int cY = pick<T::Y>(cD[r], cU, cL);
        const int dX = cX - h;  // 0 iff X is maximal, else < 0  (bit nbX = sign)
        const int dY = cY - h;  // 0 iff Y is maximal, else < 0  (bit nbY = sign)
        st.acc[r] = __funnelshift_l((uint32_t)dX, st.acc[r], 1);
        st.acc[r] = __funnelshift_l((uint32_t)dY, st.acc[r], 1);
      }
      if (MASKED) h = (j >= 1) ? h : 0;  // border column H'(i, 0) = 0 until the lane starts
      hu = h;
      st.Hl[r] = h;
    }
    st.diag = MASKED ? ((j >= 1) ? up : 0) : up;
    st.send = st.Hl[KR - 1];
    if (lane == 31 && (!MASKED || (j >= 1 && j <= n))) {
      // lane 31's column is j = t - 30: stores step through the group's base pointers
      // (stored per step: buffering the group's 8 values for one vector store, as the
      // packed H' sweep does, made C2 slower, 1.59 -> 1.68 ms: the later publication
      // lengthens every strip hand-off; publishing per consumer chunk at the step its
      // last column completes, 1.54 -> 1.61 ms: the burst of stores costs that step more
      // than the per-step stores cost the pace, tools/experiments/exp_c2trace.py)
      if (MULTIWARP) {
        unsigned long long v;
        asm("mov.b64 %0, {%1, %2};" : "=l"(v) : "r"(st.send), "r"(C.s + 1));  // (tag << 32) | H'
        st_relaxed_u64(static_cast<unsigned long long*>(C.bnd_out) + (t0 - 30) + q, v);
      } else {
        static_cast<int*>(C.bnd_out)[(t0 - 30) + q] = st.send;
      }
    }
    if (MASKED && lane == C.hm_lane && t == C.hm_t) {
      int w = 0;
#pragma unroll
      for (int r = 0; r < KR; ++r) w = (r == C.hm_r) ? st.Hl[r] : w;  // selects: Hl stays in registers
      *C.hm = w;
    }
  }
  if (DIRS) {  // group g = t0/8: halfword (g, r, lane), step k at bits (15-2k, 14-2k) = (nbX, nbY)
    uint16_t* d = C.dir_base + (long long)(t0 >> 3) * (KR * 32);
#pragma unroll
    for (int r = 0; r < KR; ++r) d[r * 32] = (uint16_t)st.acc[r];
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
  for (int r = 0; r < KR; ++r) {
    st.Hl[r] = 0;
    st.acc[r] = 0;
  }
  st.diag = 0;
  st.send = 0;
  st.chunk_cur = st.chunk_nxt = 0;
  StripCtx C;
  C.b = A.b;
  C.sprof = sprof;
  const size_t esz = MULTIWARP ? 8 : 4;
  char* bnd = static_cast<char*>(A.bnd);
  C.bnd_in = (s > 0) ? bnd + esz * (size_t)((s % A.nslots) * A.bstride) : nullptr;
  C.bnd_out = bnd + esz * (size_t)(((s + 1) % A.nslots) * A.bstride);
  C.tag_in = (unsigned)s;
  if (MULTIWARP && s == 0 && A.top_row != nullptr) {  // a segment's strip 0: the checkpoint row
    C.bnd_in = A.top_row;
    C.tag_in = A.top_tag;
  }
  if (MULTIWARP && A.ckpt != nullptr) {  // checkpoint strips hand their row over through ckpt
    if ((s + 1) % A.ck_every == 0) C.bnd_out = A.ckpt + (long long)((s + 1) / A.ck_every - 1) * A.ck_stride;
    if (s > 0 && s % A.ck_every == 0) C.bnd_in = A.ckpt + (long long)(s / A.ck_every - 1) * A.ck_stride;
  }
  if (MULTIWARP && s + 1 == A.withhold) C.bnd_out = A.sink;
  C.dir_base = DIRS ? A.dirs + (long long)s * A.wpl * (KR * 32) + lane : nullptr;
  C.err = A.err;
  C.poll_ns = A.poll_ns;
  C.watchdog = A.watchdog;
  C.hm = A.hm;
  C.n = n;
  C.s = s;
  C.lane = lane;
  C.hm_lane = -1; C.hm_r = 0; C.hm_t = 0;
  if ((A.m - 1) / R == s) {
    const int rr = (A.m - 1) % R;
    C.hm_lane = rr / KR; C.hm_r = rr % KR; C.hm_t = n - 1 + C.hm_lane;
  }
  st.bc_nxt = __ldg(A.b - lane);  // b_{j-1} for step 0 (j = 1 - lane)
  if (MULTIWARP && PROFREG && KR <= 4) {  // lane's copy k = lane % 8 of the selector table: t0 - lane
    const int k = lane & 7;    // + k are multiples of 8 (16-byte aligned)
    st.seltab = A.sel8 + (long long)k * A.sel8_stride + k;
    st.selw = __ldg(reinterpret_cast<const uint4*>(st.seltab - lane));  // group 0
  }
  const bool has_top = C.bnd_in != nullptr;
  if (has_top) st.chunk_nxt = chunk_verify<MULTIWARP>(C, 0, chunk_issue<MULTIWARP>(C, 0));
  const int ngrp = (n + 31 + 7) / 8;  // steps 0 .. n+30 in groups of 8
#pragma unroll 1
  for (int g = 0; g < ngrp; ++g) {
    const int t0 = g * 8;
#ifdef NW_TRACE
    if (MULTIWARP && A.trace && lane == 0 && (g & 255) == 0 && (g >> 8) < 256) {
      unsigned long long ts;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts));
      A.trace[(size_t)s * 256 + (g >> 8)] = ts;
    }
#endif
    st.chunk_cur = st.chunk_nxt;
    const bool more = has_top && t0 + 8 < n;
    unsigned long long raw = 0;
    if (more) raw = chunk_issue<MULTIWARP>(C, t0 + 8);
    const bool masked = t0 < 31 || t0 + 7 >= n - 1;
    if (masked) sweep_group<KR, DIRS, PROFREG, PI, MULTIWARP, true>(st, C, t0);
    else sweep_group<KR, DIRS, PROFREG, PI, MULTIWARP, false>(st, C, t0);
    if (more) st.chunk_nxt = chunk_verify<MULTIWARP>(C, t0 + 8, raw);
  }
  __syncwarp();
}

}  // namespace nwk
