// nw_cblock.cuh -- column-block wavefront for one giant pair across ranks
// (DESIGN.md §3.7). Score-only, int32, DNA profile.
//
// The (m+1) x (n+1) grid of Eq. 1 is cut into strips of R = 32*KR
// rows (as in nw_fill.cuh) and column blocks of W columns; block b belongs to
// rank b % G (block-cyclic). A task (s, b) sweeps strip s over block b. It needs
//   - the strip above's bottom row over the block's columns: from task (s-1, b)
//     on the same rank, via the rank's tagged 64-bit boundary ring (nw_fill.cuh);
//   - the left boundary column H'(s*R .. s*R+R, c_b) (corner + R rows): the right
//     column of task (s, b-1), written by the previous rank into this rank's
//     receive buffer as tagged 64-bit entries (one store per value, tag = (k, s):
//     a single-copy-atomic store carries its own validity, so the same protocol
//     works over NVLink peer memory);
// and produces the next strip's top row and its own right column for rank
// (b+1) % G. Each rank claims its tasks in (k, s) order (k = b / G) with an
// atomic ticket; every wait is on a task earlier in the order (k, s, rank), so
// the pipeline cannot deadlock as long as every rank's warps are resident.
// Virtual ranks (one device) are warps of one launch; real ranks are one
// launch per GPU with `recv_next` pointing into the next GPU's buffer.
#pragma once
#include "nw_fill.cuh"

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
  unsigned long long* const* recv_tab;  // [G]: rank r's receive buffer [2][S][R + 1] (tagged
                                        // left columns, block-slot k % 2); peer pointers for
                                        // real ranks (only own and next are dereferenced)
  long long rstride;         // entries per slot = S * (R + 1)
  int* ticket;               // [ranks]
  int* hm;                   // H'(m, n)
  int* err;
  int rank0;                 // first rank handled by this launch (real ranks: own rank)
  int nranks_here;           // ranks handled by this launch (virtual: G, real: 1)
};

template <int KR>
__global__ void __launch_bounds__(32) k_fill_cblock(CBlockArgs A) {
  constexpr int R = 32 * KR;
  const int lane = threadIdx.x;
  // warp -> rank (virtual ranks share one launch round-robin)
  const int lr = blockIdx.x % A.nranks_here;
  const int rank = A.rank0 + lr;
  const int G = A.G;
  const int kmax = (A.nblocks - rank + G - 1) / G;  // blocks k*G + rank < nblocks
  const long long ntask = (long long)kmax * A.S;
  unsigned long long* bnd = A.bnd + (size_t)lr * 2 * A.bstride;
  const unsigned long long* recv_me = A.recv_tab[rank];
  for (;;) {
    long long task = 0;
    if (lane == 0) task = atomicAdd(A.ticket + lr, 1);
    task = __shfl_sync(FULL, task, 0);
    if (task >= ntask) break;
    const int k = (int)(task / A.S), s = (int)(task % A.S);
    const int blk = k * G + rank;
    const int c0 = blk * A.W;                       // columns c0+1 .. c1 (global, 1-based)
    const int c1 = min(A.n, c0 + A.W);
    const int w = c1 - c0;
    const int ia0 = s * R + lane * KR;
    // ---- left boundary column: corner + R rows (from rank (blk-1) % G), or the grid border
    int B[KR];
    int corner = 0;
    if (blk == 0) {
#pragma unroll
      for (int r = 0; r < KR; ++r) B[r] = 0;
    } else {
      const unsigned long long* L = recv_me + (size_t)(k & 1) * A.rstride + (size_t)s * (R + 1);
      // the block-slot k % 2 is reused every second round: the tag carries k as well
      const unsigned tag = ((unsigned)(k & 0xfff) << 20) | (unsigned)(s + 1);
      // lane l needs entries l*KR .. l*KR+KR (its diag corner and its KR rows)
      unsigned long long v[KR + 1];
      for (long long it = 0;; ++it) {
        bool ok = true;
#pragma unroll
        for (int r = 0; r <= KR; ++r) {
          v[r] = ld_relaxed_u64(L + lane * KR + r);
          ok = ok && (unsigned)(v[r] >> 32) == tag;
        }
        if (__all_sync(FULL, ok)) break;
        __nanosleep(64);
        if (it > (1ll << 24)) { if (lane == 0) atomicExch(A.err, 8); break; }
      }
      corner = (int)(unsigned)v[0];
#pragma unroll
      for (int r = 0; r < KR; ++r) B[r] = (int)(unsigned)v[r + 1];
    }
    // ---- profile (DNA, K <= 4)
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
    const unsigned top_tag = (unsigned)s;   // strip s-1 wrote tag s
    unsigned long long* rnext = nullptr;    // right column -> next rank's receive buffer
    unsigned rtag = 0;
    if (blk + 1 < A.nblocks) {
      const int rn = (blk + 1) % G;
      const int kn = (blk + 1) / G;
      rnext = A.recv_tab[rn] + (size_t)(kn & 1) * A.rstride + (size_t)s * (R + 1);
      rtag = ((unsigned)(kn & 0xfff) << 20) | (unsigned)(s + 1);
    }
    const int hm_here = (A.m - 1) / R == s && c1 == A.n;
    const int hm_lane = ((A.m - 1) % R) / KR, hm_r = (A.m - 1) % KR;
    int chunk = 0;
    const int nsteps = w + 31;
    for (int t0 = 0; t0 < nsteps; t0 += 32) {
      // top boundary row for lane 0's columns c0+t0+1 .. +32 (tagged; strip 0: H'(0,j) = 0)
      if (s > 0) {
        const int jj = c0 + t0 + 1 + lane;
        const bool need = jj <= c1;
        unsigned long long v = need ? ld_relaxed_u64(top_in + jj) : 0ull;
        bool ok = !need || (unsigned)(v >> 32) == top_tag;
        for (long long it = 0; !__all_sync(FULL, ok); ++it) {
          __nanosleep(20);
          if (!ok) { v = ld_relaxed_u64(top_in + jj); ok = (unsigned)(v >> 32) == top_tag; }
          if (it > (1ll << 26)) { if (lane == 0) atomicExch(A.err, 8); break; }
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
          const int S = prmt(P[r], sel);
          int h = max(max(hd + S, Hl[r]), hu);
          h = (jl >= 1) ? h : B[r];       // left border until the lane reaches the block
          hd = Hl[r];
          hu = h;
          Hl[r] = h;
        }
        diag = up;
        send = Hl[KR - 1];
        if (lane == 31 && on) {
          unsigned long long v;
          asm("mov.b64 %0, {%1, %2};" : "=l"(v) : "r"(send), "r"(s + 1));
          st_relaxed_u64(bot_out + j, v);
        }
        if (jl == w) {
          // this lane's right column -> next rank (rows lane*KR+1 .. +KR of the message);
          // lane 0 also sends the corner H'(top-1, c1) = the top row it just used
          if (rnext) {
#pragma unroll
            for (int r = 0; r < KR; ++r) {
              unsigned long long v;
              asm("mov.b64 %0, {%1, %2};" : "=l"(v) : "r"(Hl[r]), "r"(rtag));
              st_relaxed_u64(rnext + lane * KR + r + 1, v);
            }
            if (lane == 0) {
              unsigned long long v;
              asm("mov.b64 %0, {%1, %2};" : "=l"(v) : "r"(up), "r"(rtag));
              st_relaxed_u64(rnext, v);
            }
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
