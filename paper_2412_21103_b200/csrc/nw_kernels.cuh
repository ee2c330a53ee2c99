// nw_kernels.cuh -- the sm_100a kernels behind include/nw.h.
//
//   k_init      zero the per-call progress counters / tickets / flags
//   k_encode    residues -> alphabet codes (R10), first bad position (atomicMin)
//   k_fill_pair one pair, many warps: strips chained by tagged boundary entries
//   k_tb_chain  traceback exits: entry column of every strip (one thread)
//   k_tb_segments per-strip backtracking of Sec. 2.4, all strips at once
//   k_tb_assemble  segment offsets + forward-order codes
//   (the batch kernel walks each pair with tb_walk inside the same warp)
//   k_batch     many pairs: one warp per pair, strips in sequence,
//               optional per-pair traceback by the same warp
#pragma once
#include "nw_fill.cuh"
#include "nw_fill16.cuh"
#include "nw_cblock.cuh"
#include "nw_fill_d16.cuh"
#include "nw_fill_d16dir.cuh"
#include "nw_fill_h16.cuh"

namespace nwk {

#ifdef NW_COMMON_KERNELS  // defined in exactly one TU (nw_api.cu)
struct ZeroRanges {
  void* p[4];
  long long bytes[4];  // multiples of 16, 16-byte aligned
};

// Per-call reset: small counters, the bad-position flag and up to 4 buffers
// (tagged boundary ring, padded code buffers) that must start zeroed.
__global__ void k_init(int* ints, int nints, long long* bad, ZeroRanges zr) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  for (long long i = tid; i < nints; i += nth) ints[i] = 0;
  if (bad && tid == 0) *bad = 0x7fffffffffffffffll;
  for (int r = 0; r < 4; ++r) {
    uint4* q = static_cast<uint4*>(zr.p[r]);
    const long long n16 = zr.bytes[r] / 16;
    for (long long i = tid; i < n16; i += nth) q[i] = make_uint4(0, 0, 0, 0);
  }
}

// out[k] = lut[in[k]] (0xff marks a symbol outside the alphabet: code 0 is
// written and the smallest such position + pos_base goes to *bad).
__global__ void k_encode(const uint8_t* __restrict__ in, long long len,
                         const uint8_t* __restrict__ lut, uint8_t* __restrict__ out,
                         long long* bad, long long pos_base) {
  __shared__ uint8_t slut[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) slut[i] = lut[i];
  __syncthreads();
  long long my_bad = 0x7fffffffffffffffll;
  const long long stride = (long long)gridDim.x * blockDim.x * 4;
  for (long long base = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 4; base < len;
       base += stride) {
    if (base + 4 <= len && ((reinterpret_cast<uintptr_t>(in + base) | reinterpret_cast<uintptr_t>(out + base)) & 3) == 0) {
      const uchar4 v = *reinterpret_cast<const uchar4*>(in + base);
      uchar4 o;
      o.x = slut[v.x]; o.y = slut[v.y]; o.z = slut[v.z]; o.w = slut[v.w];
      if (o.x == 0xff) { my_bad = min(my_bad, base); o.x = 0; }
      if (o.y == 0xff) { my_bad = min(my_bad, base + 1); o.y = 0; }
      if (o.z == 0xff) { my_bad = min(my_bad, base + 2); o.z = 0; }
      if (o.w == 0xff) { my_bad = min(my_bad, base + 3); o.w = 0; }
      *reinterpret_cast<uchar4*>(out + base) = o;
    } else {
      for (long long k = base; k < base + 4 && k < len; ++k) {
        uint8_t c = slut[in[k]];
        if (c == 0xff) { my_bad = min(my_bad, k); c = 0; }
        out[k] = c;
      }
    }
  }
  if (my_bad != 0x7fffffffffffffffll)
    atomicMin(reinterpret_cast<unsigned long long*>(bad), (unsigned long long)(my_bad + pos_base));
}

// Selector table of the packed sweeps (FillArgs::sel): sel[i] = (17 c[i] + 128) |
// (17 c[i-1] + 196) << 8 over codes c[-1 .. len) (c[-1] read from the padding).
// Four shifted copies of the selector table for 16-byte-aligned per-lane loads
// (nw_fill_h16.cuh): out[k*stride + PAD + i] = sel[i - 2k] for i in [-PAD, stride - PAD),
// sel[j] = (17 b[j] + 128) | (17 b[j-1] + 196) << 8, b = codes (readable on [-PAD, n + PAD));
// entries whose codes fall outside that range are 0 (never used inside the grid).
__global__ void k_sel16x4(const uint8_t* __restrict__ b, long long n, uint16_t* __restrict__ out,
                          long long stride) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < 4 * stride;
       e += (long long)gridDim.x * blockDim.x) {
    const long long k = e / stride, j = (e % stride) - PAD - 2 * k;
    out[e] = (j - 1 >= -PAD && j < n + PAD) ? (uint16_t)((17u * b[j] + 128u) | ((17u * b[j - 1] + 196u) << 8)) : 0;
  }
}

// Eight shifted copies of the int32 sweep's per-column PRMT selector (b * 0x1111 + 0x8880:
// byte b of the profile word, sign-replicated): out[k*stride + PAD + i] = sel(b[i - k]) for
// i - k in [-PAD, n + PAD), else 0 (nw_fill.cuh, FillArgs::sel8).
__global__ void k_sel8x8(const uint8_t* __restrict__ b, long long n, uint16_t* __restrict__ out,
                         long long stride) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < 8 * stride;
       e += (long long)gridDim.x * blockDim.x) {
    const long long k = e / stride, j = (e % stride) - PAD - k;
    out[e] = (j >= -PAD && j < n + PAD) ? (uint16_t)(b[j] * 0x1111u + 0x8880u) : 0;
  }
}

__global__ void k_sel16(const uint8_t* __restrict__ codes, long long len, uint16_t* __restrict__ sel) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < len;
       i += (long long)gridDim.x * blockDim.x)
    sel[i] = (uint16_t)((17u * codes[i] + 128u) | ((17u * codes[i - 1] + 196u) << 8));
}

#endif  // NW_COMMON_KERNELS

// One pair, one strip per warp at a time; strips handed out in order by an
// atomic ticket so every awaited producer is already resident (no deadlock).
// D16 (score-only, K <= 4, s - 2g >= 0): the packed difference-form sweep of
// nw_fill_d16.cuh (KR rows per lane, two per register) instead of strip_sweep.
// D16: 0 = int32 strip_sweep, 1 = packed difference form (one chain per lane),
// 2 = packed difference form with two chains per lane (strip_sweep_d16x2),
// 3 = packed H' with a moving per-strip base (strip_sweep_h16, nw_fill_h16.cuh).
template <int KR, bool DIRS, bool PROFREG, int PI, int D16 = 0>
__global__ void __launch_bounds__(32) k_fill_pair(FillArgs A) {
  extern __shared__ __align__(16) int8_t smem[];
  const int lane = threadIdx.x & 31;
  for (;;) {
    int s = 0;
    if (lane == 0) s = atomicAdd(A.ticket, 1);
    s = __shfl_sync(FULL, s, 0);
    if (s >= A.nstrips) break;
    if constexpr (D16 == 3) strip_sweep_h16<KR, DIRS, PI>(A, s, lane);
    else if constexpr (D16 == 2) strip_sweep_d16x2<KR, true>(A, s, lane);
    else if constexpr (D16 == 1) strip_sweep_d16<KR, true>(A, s, lane);
    else strip_sweep<KR, DIRS, PROFREG, PI, true>(A, s, lane, smem);
  }
}

// Decode the decision bits of interior cell (i, j) (1-based) -> P:90 code
// (layout in nw_fill.cuh: halfword ((s*G + g)*KR + r)*32 + l, step k = t%8 at
// bits (15-2k, 14-2k) = (nbX, nbY); code X if !nbX, else Y if !nbY, else Z).
template <int KR>
__device__ __forceinline__ int tb_decode(uint32_t hw, int k, int X, int Y, int Z) {
  const uint32_t f = (hw >> (14 - 2 * k)) & 3u;
  return !(f & 2u) ? X : (!(f & 1u) ? Y : Z);
}

template <int KR>
__device__ __forceinline__ long long tb_index(long long G, int i, int j, int& k) {
  constexpr int R = 32 * KR;
  const int ia = i - 1;
  const int s = ia / R, l = (ia % R) / KR, r = ia % KR;
  const int t = (j - 1) + l;
  k = t & 7;
  return (((long long)s * G + (t >> 3)) * KR + r) * 32 + l;
}

// Walk from (m, n) to (0, 0); rev[k] = k-th code from the end.
// Border cells follow R7: column 0 -> vertical, row 0 -> horizontal.
template <int KR>
__device__ long long tb_walk(const uint16_t* dirs, long long G, int m, int n, int X, int Y,
                             int Z, uint8_t* rev) {
  int i = m, j = n;
  long long k = 0;
  while (i > 0 && j > 0) {
    int kk;
    const long long idx = tb_index<KR>(G, i, j, kk);
    // L1-cached: consecutive steps mostly stay in one 128-byte line (rows r, r+1 of a
    // group); the lines were written by this warp before __syncwarp, so L1 holds no stale copy
    const int code = tb_decode<KR>(__ldca(dirs + idx), kk, X, Y, Z);
    rev[k++] = (uint8_t)code;
    i -= (code != 3);
    j -= (code != 2);
  }
  while (i > 0) { rev[k++] = 2; --i; }
  while (j > 0) { rev[k++] = 3; --j; }
  return k;
}

// ---- single-pair traceback split at strip boundaries ----
// cs[s] = column where the path enters strip s: at row m for the last strip
// (cs[S-1] = n), else on strip s's bottom row R*(s+1). The fill stores only the
// decision bits; the entries are recovered after it in two launches:
//   k_tb_spec   exits of sampled entries in a band around the diagonal, in parallel
//   k_tb_chain  the bottom-up chain: cs[s-1] = exit of strip s from cs[s], read off
//               the samples whenever the two samples bracketing cs[s] agree,
//               else walked exactly.
// Traceback paths cannot cross (each cell has one predecessor, moves are unit
// up/left/diagonal), so exits are monotone in the entry column and a path that
// enters between two sampled entries with the same exit leaves there too.

// Walk strip s's decision bits from (i, j) until the path reaches row i_stop; the
// column there is the strip's exit. Column 0 is the border (the path goes straight up).
template <int KR>
__device__ __forceinline__ int strip_exit_walk(const uint16_t* __restrict__ dirs, long long G,
                                               int i, int j, int i_stop, int X, int Y, int Z) {
  constexpr int R = 32 * KR;
  const uint16_t* base = dirs + (long long)((i - 1) / R) * G * (KR * 32);  // one strip
  while (i > i_stop && j > 0) {
    const unsigned ia = (unsigned)(i - 1);
    const int l = (int)((ia % R) / KR), r = (int)(ia % KR);
    const int t = j - 1 + l;
    // L1-cached: consecutive steps mostly stay in one 128-byte line
    const uint32_t f = (uint32_t)__ldca(base + ((long long)(t >> 3) * KR + r) * 32 + l) >>
                       (14 - 2 * (t & 7));
    const int code = !(f & 2u) ? X : (!(f & 1u) ? Y : Z);
    i -= (code != 3);
    j -= (code != 2);
  }
  return i > i_stop ? 0 : j;
}

// Sample q of strip s enters at column min(q*step, n) of row R*(s+1); strip s
// holds samples q0(s) .. q0(s)+nb-1, centred on the column the diagonal of the
// (m+1)x(n+1) grid crosses that row at.
struct TbBand {
  int m, n, step, lstep, nb, nq;  // step = 1 << lstep; nq = ceil(n/step) + 1 samples per row
  float ratio;                    // n / m
  __device__ int q0(int s, int R) const {
    const int cc = __float2int_rd(__fmul_rn((float)(R * (s + 1)), ratio));
    const int q = (cc >> lstep) - nb / 2;
    const int qmax = nq > nb ? nq - nb : 0;
    return q < 0 ? 0 : (q > qmax ? qmax : q);
  }
  __host__ __device__ int col(int q) const { return q * step < n ? q * step : n; }
};

// Copy ng decision groups of one strip (GS halfwords each) into shared memory,
// group g at word g * (GS/2 + 1): the pad puts the same (r, l) of consecutive
// groups in consecutive banks. Threads tid of nth cooperate.
template <int KR>
__device__ __forceinline__ void stage_groups(const uint16_t* __restrict__ src_hw, int ng,
                                             uint32_t* w32, int tid, int nth) {
  constexpr int GS = KR * 32, GW = GS / 2 + 1, U4 = GS / 8;
  const uint4* src = reinterpret_cast<const uint4*>(src_hw);
  const int n16 = ng * U4;
  int w = tid;
  for (; w + 7 * nth < n16; w += 8 * nth) {  // 8 loads in flight per thread
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcg(src + w + u * nth);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      uint32_t* d = w32 + ((w + u * nth) / U4) * GW + ((w + u * nth) % U4) * 4;
      d[0] = v[u].x; d[1] = v[u].y; d[2] = v[u].z; d[3] = v[u].w;
    }
  }
  for (; w < n16; w += nth) {
    const uint4 v = __ldcg(src + w);
    uint32_t* d = w32 + (w / U4) * GW + (w % U4) * 4;
    d[0] = v.x; d[1] = v.y; d[2] = v.z; d[3] = v.w;
  }
}

// Walk strip s (decision bits at base) from (i, j) up to row i_stop through the
// staged groups g_lo .. g_lo+ng-1. Returns false, with (i, j) where it stopped,
// when the path leaves the window.
template <int KR>
__device__ __forceinline__ bool walk_window(const uint32_t* w32, int g_lo, int ng, int& i, int& j,
                                            int i_stop, int X, int Y, int Z) {
  constexpr int R = 32 * KR, GW = KR * 16 + 1;
  while (i > i_stop && j > 0) {
    const unsigned ia = (unsigned)(i - 1);
    const int l = (int)((ia % R) / KR), r = (int)(ia % KR);
    const int t = j - 1 + l;
    const int g = (t >> 3) - g_lo;
    if ((unsigned)g >= (unsigned)ng) return false;
    const int x = r * 32 + l;  // halfword within the group
    const uint32_t f = w32[g * GW + (x >> 1)] >> ((x & 1) * 16 + 14 - 2 * (t & 7));
    const int code = !(f & 2u) ? X : (!(f & 1u) ? Y : Z);
    i -= (code != 3);
    j -= (code != 2);
  }
  return true;
}

// spec[s*nb + k] = exit column of strip s (s < S-1) entered at sample q0(s)+k, or
// -1 when that walk leaves its window (entries far off the path walk long gaps;
// the chain then walks the strip exactly). One warp per 32 samples: the warp
// stages its samples' columns plus left_cols to their left and each lane walks one.
template <int KR>
__global__ void __launch_bounds__(32) k_tb_spec(const uint16_t* __restrict__ dirs, long long G,
                                               TbBand B, int X, int Y, int Z, int* spec,
                                               int left_cols) {
  constexpr int R = 32 * KR, GS = KR * 32;
  extern __shared__ __align__(16) uint32_t w32[];
  const int lane = threadIdx.x;
  const int tiles = B.nb / 32;
  const int s = blockIdx.x / tiles, tile = blockIdx.x % tiles;
  const int qt = B.q0(s, R) + tile * 32;  // first sample of this warp
  if (qt >= B.nq) return;
  const int c_hi = B.col(min(qt + 31, B.nq - 1));
  const int c_lo = max(0, B.col(qt) - left_cols);
  const int g_lo = max(0, c_lo - 1) >> 3;  // groups of t = j - 1 + l, j in [c_lo, c_hi]
  const int ng = (int)min((long long)((c_hi + 30) >> 3), G - 1) - g_lo + 1;
  const uint16_t* base = dirs + (long long)s * G * GS;
  stage_groups<KR>(base + (long long)g_lo * GS, ng, w32, lane, 32);
  __syncwarp();
  const int q = qt + lane;
  if (q >= B.nq) return;
  int i = R * (s + 1), j = B.col(q);
  const bool in = walk_window<KR>(w32, g_lo, ng, i, j, R * s, X, Y, Z);
  spec[(long long)s * B.nb + tile * 32 + lane] = (!in) ? -1 : (i == R * s ? j : 0);
}

// The chain, one CTA of 1024 threads: all threads stage CH strips' samples in
// shared memory, then warp 0 chains through them. A strip whose bracket is
// unresolved (or outside the band) is walked exactly: warp 0 posts the strip and
// entry e, the whole CTA stages the strip's decision bits for columns
// [e - left_cols, e], and thread 0 walks them; a path that leaves the window on
// the left (a long gap) gets the next window staged, from where it stopped. The
// last strip (entered at (m, n)) is always walked exactly.
template <int KR>
__global__ void __launch_bounds__(1024) k_tb_chain(const uint16_t* __restrict__ dirs, long long G,
                                                   TbBand B, int S, int X, int Y, int Z,
                                                   const int* __restrict__ spec, int* cs,
                                                   int* nslow, int CH, int left_cols) {
  constexpr int R = 32 * KR, GS = KR * 32;
  extern __shared__ __align__(16) uint32_t sm[];
  __shared__ int cmd[4];  // {0 = chunk done | 1 = walk, strip, entry}; walk state (i, j, done)
  int* spc = reinterpret_cast<int*>(sm);
  uint32_t* w32 = sm + (long long)CH * B.nb;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nth = blockDim.x;
  // Exact exit of strip s entered at row i0, column cmd[2]; every thread calls it
  // after the barrier that published cmd. Returns the exit (all threads).
  auto exact = [&](int s, int i0) -> int {
    const int i_stop = R * s;
    int i = i0, j = cmd[2];
    __syncthreads();  // cmd[2..3] are rewritten below
    while (i > i_stop && j > 0) {
      const int c_lo = max(0, j - left_cols);
      const int g_lo = max(0, c_lo - 1) >> 3;  // groups of t = j' - 1 + l, j' in [c_lo, j]
      const int ng = (int)min((long long)((j + 30) >> 3), G - 1) - g_lo + 1;
      stage_groups<KR>(dirs + ((long long)s * G + g_lo) * GS, ng, w32, tid, nth);
      __syncthreads();
      if (tid == 0) {
        walk_window<KR>(w32, g_lo, ng, i, j, i_stop, X, Y, Z);
        cmd[2] = i; cmd[3] = j;
      }
      __syncthreads();
      i = cmd[2]; j = cmd[3];
      __syncthreads();
    }
    return (i > i_stop) ? 0 : j;  // j == 0: the path reached the left border and stays there
  };
  int e = B.n, slow = 1;
  if (tid == 0) { cs[S - 1] = e; cmd[2] = e; }
  __syncthreads();
  if (S >= 2) {
    e = exact(S - 1, B.m);
    if (tid == 0) cs[S - 2] = e;
  }
  for (int s_hi = S - 2; s_hi >= 1; s_hi -= CH) {
    const int s_lo = max(1, s_hi - CH + 1);
    {
      const int4* src = reinterpret_cast<const int4*>(spec + (long long)s_lo * B.nb);
      int4* dst = reinterpret_cast<int4*>(spc);
      const int n16 = (s_hi - s_lo + 1) * B.nb / 4;
      for (int w = tid; w < n16; w += blockDim.x) dst[w] = __ldcg(src + w);
    }
    __syncthreads();
    int s = s_hi;
    for (;;) {
      if (warp == 0) {  // chain through resolved brackets; stop at an unresolved one
        for (; s >= s_lo; --s) {
          const int q0 = B.q0(s, R);
          const int qa = e >> B.lstep;
          const int ka = qa - q0;
          const bool on = B.col(qa) == e;  // e is a sample itself
          int x = -1;
          if (ka >= 0 && ka < B.nb && (on || (ka + 1 < B.nb && qa + 1 < B.nq))) {
            const int* row = spc + (s - s_lo) * B.nb;
            const int xa = row[ka], xb = on ? xa : row[ka + 1];
            if (xa == xb) x = xa;  // -1 stays -1: a sample left its window
          }
          if (x < 0) break;
          e = x;
          if (lane == 0) cs[s - 1] = e;
        }
        if (lane == 0) { cmd[0] = s >= s_lo; cmd[1] = s; cmd[2] = e; }
      }
      __syncthreads();
      if (!cmd[0]) break;
      s = cmd[1];
      e = exact(s, R * (s + 1));
      ++slow;
      if (tid == 0) cs[s - 1] = e;
      --s;
    }
    e = cmd[2];  // every thread carries the chain's entry into the next chunk
    __syncthreads();
  }
  if (tid == 0) *nslow = slow;
}

// One warp per strip: walk from the strip's entry to its top boundary row (the
// last row of the strip above), codes written last-first into seg + s*segstride.
// The decision halfwords the walk can touch (columns cs[s-1] .. cs[s]) are
// staged in shared memory when they fit, so each step is a shared-memory read.
template <int KR>
__global__ void __launch_bounds__(32) k_tb_segments(const uint16_t* __restrict__ dirs, long long G,
                                                   int m, int n, int X, int Y, int Z,
                                                   const int* __restrict__ cs, uint8_t* seg,
                                                   long long segstride, int* seglen, int smem_hw,
                                                   int pad_top, int* exit_col) {
  constexpr int R = 32 * KR;
  constexpr int GS = KR * 32;  // halfwords per (strip, group)
  extern __shared__ __align__(16) uint16_t sh[];
  const int s = blockIdx.x, lane = threadIdx.x;
  const int S = gridDim.x;
  int i = (s == S - 1) ? m : R * (s + 1);
  int j = cs[s];
  const int i_stop = R * s;
  const int j_lo = (s > 0) ? cs[s - 1] : 0;
  // groups g holding steps t = j' - 1 + l for j' in [j_lo, j], l in [0, 31]
  const long long g_lo = max(0, j_lo - 1) >> 3;
  const long long g_hi = (long long)(j + 30) >> 3;
  const long long ng = g_hi - g_lo + 1;
  const bool staged = ng * GS <= smem_hw;
  const uint16_t* base = dirs + (long long)s * G * GS;
  if (staged) {
    const uint4* src = reinterpret_cast<const uint4*>(base + g_lo * GS);
    uint4* dst = reinterpret_cast<uint4*>(sh);
    const long long n16 = ng * GS / 8;
    for (long long q = lane; q < n16; q += 32) dst[q] = __ldcg(src + q);
  }
  __syncwarp();
  if (lane != 0) return;
  uint8_t* out = seg + (long long)s * segstride;
  int k = 0;
  while (i > i_stop) {
    if (j == 0) { out[k++] = 2; --i; continue; }  // border column: vertical (R7)
    const int ia = i - 1;
    const int l = (ia % R) / KR, r = ia % KR;
    const int t = (j - 1) + l;
    const long long g = t >> 3;
    const long long off = (g * KR + r) * 32 + l;
    const uint32_t hw = staged ? sh[off - g_lo * GS] : __ldcg(base + off);
    const int code = tb_decode<KR>(hw, t & 7, X, Y, Z);
    out[k++] = (uint8_t)code;
    i -= (code != 3);
    j -= (code != 2);
  }
  if (s == 0) {
    if (exit_col) *exit_col = j;  // a segment of a checkpointed traceback stops at its top row
    if (pad_top)
      while (j > 0) { out[k++] = 3; --j; }  // row 0: horizontal (R7)
  }
  seglen[s] = k;
}

#ifdef NW_COMMON_KERNELS
// out[off_s + p] = seg[s][seglen[s] - 1 - p]: forward order, one block per strip;
// off_s = sum of seglen[0 .. s) (the strips above come first), summed by the
// block itself; the last block also writes the total length.
__global__ void __launch_bounds__(256) k_tb_assemble(const uint8_t* __restrict__ seg,
                                                     long long segstride,
                                                     const int* __restrict__ seglen,
                                                     uint8_t* __restrict__ out, long long* total) {
  __shared__ long long wsum[8];
  const int s = blockIdx.x, tid = threadIdx.x;
  long long acc = 0;
  for (int k = tid; k < s; k += blockDim.x) acc += seglen[k];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((tid & 31) == 0) wsum[tid >> 5] = acc;
  __syncthreads();
  long long off = 0;
#pragma unroll
  for (int w = 0; w < 8; ++w) off += wsum[w];
  const int L = seglen[s];
  if (s == gridDim.x - 1 && tid == 0) *total = off + L;
  const uint8_t* src = seg + (long long)s * segstride;
  uint8_t* dst = out + off;
  for (int p = tid; p < L; p += blockDim.x) dst[p] = src[L - 1 - p];
}

#endif  // NW_COMMON_KERNELS



struct BatchArgs {
  const uint8_t* codes;    // concatenated codes, padded (PAD before, >= R + PAD after)
  const long long* offs;   // nseq + 1
  int nseq;
  const int* pairs;        // explicit (p, q) pairs, or null = all p<q
  const int* order;        // explicit mode: task -> pair index (LPT order), or null
  const int* perm;         // implicit mode: rank -> sequence (length-descending)
  long long npairs;
  const int8_t* prof;
  int K;
  int g;
  int* ticket;
  int* scores;             // per pair, pair order
  const uint16_t* sel16;   // selector table aligned with codes (FillArgs::sel; packed sweeps)
  // per-warp scratch
  int* wbnd;               // [nwarps][2][bstride]
  long long bstride;
  int* whm;                // [nwarps]
  uint16_t* wdirs;         // [nwarps][dstride] (TRACEBACK)
  long long dstride;
  // traceback outputs
  const long long* ops_off;
  uint8_t* ops;
  int* ops_len;
  int X, Y, Z;
  int* err;
  int transpose_ok;        // score-only, s symmetric: a pair may be filled transposed
  int mix_w16 = 1100;      // PACKED 4: relative cost (x1000) of a 512-row strip cell vs a 1,024-row one
  int mix_w24 = 1040;      // PACKED 4: the same for a 768-row strip cell
  // Two-phase traceback (the packed sweep, PACKED == 3): the fill
  // keeps every pair's decision words at tdirs + tdir_off[task] (32-bit words) and
  // k_batch_walk walks them after the fill, one thread per pair.
  uint32_t* tdirs;
  const long long* tdir_off;
  long long task0, task1;  // tasks [task0, task1) of this launch (a wave)
  int transposed;          // this fill launch sweeps its pairs transposed (b on the rows;
                           // the kernel's tie order is the mirrored one)
  long long ntr0;          // the walk: tasks >= ntr0 were filled transposed
  // Distributed all-pairs (nw_ctx_set_dist, implicit mode): this rank's tasks are the
  // rank-space tasks [tbase + task0, tbase + task1); compact = scores go to scores[task]
  // (rank-space order, gathered and scattered to pair order by k_rs_scatter).
  long long tbase = 0;
  int compact = 0;
  int bnd_smem = 0;           // packed H' sweep: the boundary row in shared memory (one slot
  int bnd_smem_off = 0;       //   of bstride ints per warp at this byte offset)
};

// flat rank-space index k -> (p', q'), p' < q', lexicographic over N items
__device__ __forceinline__ void unrank_pair(long long k, int N, int& p, int& q) {
  const double NN = 2.0 * N - 1.0;
  long long pp = (long long)((NN - sqrt(NN * NN - 8.0 * (double)k)) * 0.5);
  if (pp < 0) pp = 0;
  if (pp > N - 2) pp = N - 2;
  auto off = [N](long long x) { return x * N - x * (x + 1) / 2; };
  while (pp > 0 && off(pp) > k) --pp;
  while (pp + 1 <= N - 2 && off(pp + 1) <= k) ++pp;
  p = (int)pp;
  q = (int)(k - off(pp) + pp + 1);
}

// Task -> pair (p, q) and its output index: explicit pairs in the host's LPT order,
// or the flat rank-space index over sequences sorted by length, mapped back to the
// lexicographic p < q index.
__device__ __forceinline__ void task_pair(const BatchArgs& B, long long task, int& p, int& q,
                                          long long& outk) {
  if (B.pairs) {
    outk = B.order ? B.order[task] : task;
    p = B.pairs[2 * outk];
    q = B.pairs[2 * outk + 1];
  } else {
    int pr, qr;
    unrank_pair(B.tbase + task, B.nseq, pr, qr);
    const int x = B.perm[pr], y = B.perm[qr];
    p = min(x, y);
    q = max(x, y);
    outk = B.compact ? task : (long long)p * B.nseq - (long long)p * (p + 1) / 2 + (q - p - 1);
  }
}

// PACKED (s - 2g >= 0), KR16 rows per lane, two per register:
// 1 = the H' half-row sweep of nw_fill16.cuh (score-only, K <= 4, every H' < 2^16),
// 2 = the difference-form sweep of nw_fill_d16.cuh (score-only, K <= 4, any length),
// 3 = the difference-form sweep with decision flags of nw_fill_d16dir.cuh (DIRS),
// 4 = as 1, each pair at 32, 24 or 16 rows per lane (whichever sweeps less weighted area).
template <int KR16, bool COHERENT>
__device__ __forceinline__ void walk_lanes(const BatchArgs& B, long long task, bool act, int lane);

// The mixed-height H' sweep (PACKED 4: three sweeps, 124 registers unbounded) is held to 96
// registers (5 CTAs per SM instead of 4, no spills): C3 298 -> 291 ms (6 CTAs: 80 registers
// with spills, 338 ms)
template <int KR, bool DIRS, bool PROFREG, int PI, int PACKED = 0, int KR16 = 16>
__global__ void __launch_bounds__(128, (PACKED == 4 ? 5 : 1)) k_batch(BatchArgs B) {
  constexpr int R = 32 * KR;
  extern __shared__ __align__(16) int8_t smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const long long gw = (long long)blockIdx.x * (blockDim.x >> 5) + wib;
  constexpr int RSP = PACKED ? 32 * KR16 : R;  // strip height (shared-profile rows)
  int8_t* sprof = smem + (PROFREG ? 0 : wib * (B.K * RSP));
  // the strips of a pair run one after another in this warp; the packed H' sweep reads
  // the row above (32 columns ahead) before overwriting it (62 columns behind), so one
  // row in shared memory suffices (bnd_smem; global scratch otherwise)
  int* bnd = ((PACKED == 1 || PACKED == 4) && B.bnd_smem)
                 ? reinterpret_cast<int*>(smem + B.bnd_smem_off) + wib * B.bstride
                 : B.wbnd + gw * 2 * B.bstride;
  uint16_t* wd = DIRS ? B.wdirs + gw * B.dstride : nullptr;
  for (;;) {
    long long task = 0;
    if (lane == 0) task = B.task0 + atomicAdd(B.ticket, 1);
    task = __shfl_sync(FULL, task, 0);
    if (task >= B.task1) break;
    int p, q;
    long long outk;
    task_pair(B, task, p, q, outk);
    long long ao = B.offs[p], bo = B.offs[q];
    int m = (int)(B.offs[p + 1] - ao), n = (int)(B.offs[q + 1] - bo);
    if (DIRS && PACKED == 3 && B.transposed && m > 0 && n > 0) {  // the host's orientation choice
      const long long to = ao; ao = bo; bo = to;
      const int tm = m; m = n; n = tm;
    }
    bool half = false;  // PACKED 4: this pair runs 512-row strips (strip_sweep_u16<16>)
    bool three = false;  // PACKED 4: 768-row strips (strip_sweep_u16<24>)
    if (PACKED == 4) {
      // the orientation and strip height (1,024, 768 or 512 rows) with the least weighted
      // swept area: strips x height x (columns + lane skew), 768/512-row cells weighted
      // mix_w24/1000, mix_w16/1000
      // (their per-cell overhead is higher); transposing needs the symmetric s
      auto cost = [&](int rows, int cols, int rs, long long w) {
        return (long long)((rows + rs - 1) / rs) * rs * (cols + 64) * w;
      };
      long long best = cost(m, n, 1024, 1000);
      int pick = 0;
      const long long c1 = cost(m, n, 512, B.mix_w16);
      if (c1 < best) { best = c1; pick = 1; }
      const long long c1b = cost(m, n, 768, B.mix_w24);
      if (c1b < best) { best = c1b; pick = 4; }
      if (B.transpose_ok) {
        const long long c2 = cost(n, m, 1024, 1000), c3 = cost(n, m, 512, B.mix_w16);
        if (c2 < best) { best = c2; pick = 2; }
        if (c3 < best) { best = c3; pick = 3; }
        const long long c3b = cost(n, m, 768, B.mix_w24);
        if (c3b < best) { best = c3b; pick = 6; }
      }
      half = pick & 1;
      three = pick >= 4;
      if (pick == 6) {
        const long long to = ao; ao = bo; bo = to;
        const int tm = m; m = n; n = tm;
      }
      if (pick == 2 || pick == 3) {
        const long long to = ao; ao = bo; bo = to;
        const int tm = m; m = n; n = tm;
      }
    } else if (!DIRS && B.transpose_ok) {
      // score-only with a symmetric s: Score(a, b) = Score(b, a) (the transpose
      // invariant of the oracle pins), so put on the rows whichever sequence wastes
      // fewer lanes of the last strip: strips x (columns + lane skew)
      constexpr int RS = PACKED ? 32 * KR16 : R, SK = PACKED ? 64 : 32;
      if ((long long)((m + RS - 1) / RS) * (n + SK) > (long long)((n + RS - 1) / RS) * (m + SK)) {
        const long long to = ao; ao = bo; bo = to;
        const int tm = m; m = n; n = tm;
      }
    }
    int hmv = 0;
    if (m > 0 && n > 0) {
      FillArgs A;
      A.a = B.codes + ao; A.b = B.codes + bo; A.prof = B.prof; A.K = B.K; A.sel = B.sel16 + bo;
      constexpr int RS = PACKED == 4 ? 1024 : PACKED ? 32 * KR16 : R;  // strip height of the sweep in use
      A.m = m; A.n = n; A.nstrips = (m + RS - 1) / RS; A.nslots = ((PACKED == 1 || PACKED == 4) && B.bnd_smem) ? 1 : 2;
      A.bnd = bnd; A.bstride = B.bstride; A.ticket = nullptr; A.ckpt = nullptr; A.ck_every = 0; A.ck_stride = 0; A.top_row = nullptr; A.top_tag = 0;
      A.dirs = PACKED == 3 ? reinterpret_cast<uint16_t*>(B.tdirs + B.tdir_off[task]) : wd;
      A.wpl = PACKED ? (n + 63 + 7) / 8 : (n + 31 + 7) / 8;  // 8-step groups per strip
      A.hm = B.whm + gw; A.err = B.err;
      if constexpr (PACKED == 1) {
        for (int s = 0; s < A.nstrips; ++s) strip_sweep_u16<KR16>(A, s, lane);
      } else if constexpr (PACKED == 4) {
        if (half) {
          A.nstrips = (m + 511) / 512;
          for (int s = 0; s < A.nstrips; ++s) strip_sweep_u16<16>(A, s, lane);
        } else if (three) {
          A.nstrips = (m + 767) / 768;
          for (int s = 0; s < A.nstrips; ++s) strip_sweep_u16<24>(A, s, lane);
        } else {
          for (int s = 0; s < A.nstrips; ++s) strip_sweep_u16<32>(A, s, lane);
        }
      } else if constexpr (PACKED == 2) {
        if (lane == 0) *A.hm = 0;  // the difference-form sweep accumulates sum U(i, n)
        __syncwarp();
        for (int s = 0; s < A.nstrips; ++s) strip_sweep_d16<KR16, false>(A, s, lane);
      } else if constexpr (PACKED == 3) {
        if (lane == 0) *A.hm = 0;
        __syncwarp();
        for (int s = 0; s < A.nstrips; ++s) strip_sweep_d16dir<KR16, PROFREG, PI>(A, s, lane, sprof);
      } else {
        for (int s = 0; s < A.nstrips; ++s)
          strip_sweep<KR, DIRS, PROFREG, PI, false>(A, s, lane, sprof);
      }
      __syncwarp();
      hmv = *(volatile int*)(B.whm + gw);
      // the int32 sweep walks its pair in-warp; the packed flags (PACKED == 3) are
      // walked by k_batch_walk, one thread per pair (an in-warp walk compiled into
      // this kernel made ptxas emit every shuffle of the sweep as a collective)
      if (DIRS && PACKED != 3) {
        uint8_t* o = B.ops + B.ops_off[outk];
        long long L = 0;
        if (lane == 0) L = tb_walk<KR>(wd, A.wpl, m, n, B.X, B.Y, B.Z, o);
        L = __shfl_sync(FULL, L, 0);
        __syncwarp();
        // reverse in place: o[0..L) holds the codes last-first
        for (long long a0 = lane; a0 < L / 2; a0 += 32) {
          const uint8_t u = o[a0], v = o[L - 1 - a0];
          o[a0] = v;
          o[L - 1 - a0] = u;
        }
        if (lane == 0) B.ops_len[outk] = (int)L;
      }
    } else if (DIRS) {
      uint8_t* o = B.ops + B.ops_off[outk];
      const int L = m + n;
      for (int a0 = lane; a0 < L; a0 += 32) o[a0] = (m > 0) ? 2 : 3;
      if (lane == 0) B.ops_len[outk] = L;
    }
    if (lane == 0) B.scores[outk] = hmv + B.g * (m + n);
    __syncwarp();
  }
}

// Phase 2 of the two-phase batch traceback: each lane walks one pair's kept
// decision words from (m, n) to (0, 0) (word and bit of cell (i, j) in
// the layout of nw_fill_d16dir.cuh), writing the codes last-first from the end of the pair's ops slot
// (capacity m + n); the warp then moves each path to the start of its slot with
// coalesced copies. Called by all 32 lanes; act = this lane has a pair (task of
// the fill's order). Pairs with m = 0 or n = 0 were written by k_batch. COHERENT:
// the words were written in this kernel (by this warp), so no read-only-path loads.
template <int KR16, bool COHERENT>
__device__ __forceinline__ void walk_lanes(const BatchArgs& B, long long task, bool act, int lane) {
  constexpr int H = KR16 / 2, RS = 32 * KR16;
  int m = 0, n = 0;
  long long outk = 0;
  if (act) {
    int p, q;
    task_pair(B, task, p, q, outk);
    m = (int)(B.offs[p + 1] - B.offs[p]);
    n = (int)(B.offs[q + 1] - B.offs[q]);
    act = m > 0 && n > 0;
  }
  // a transposed pair: walk the swept (transposed) grid with the mirrored tie order and
  // emit its vertical moves as horizontal ones and vice versa
  const bool tr = act && task >= B.ntr0;
  if (tr) { const int tm = m; m = n; n = tm; }
  const int cV = tr ? 3 : 2, cH = tr ? 2 : 3;
  const int X = tr && B.X != 1 ? 5 - B.X : B.X, Y = tr && B.Y != 1 ? 5 - B.Y : B.Y,
            Z = tr && B.Z != 1 ? 5 - B.Z : B.Z;
  uint8_t* o = nullptr;
  int pos = 0;
  if (act) {
    const uint32_t* d = B.tdirs + B.tdir_off[task];
    const long long G = (n + 63 + 7) / 8;
    o = B.ops + B.ops_off[outk];
    pos = m + n;
    int i = m, j = n;
    long long cur = -1;
    uint4 blk[H / 4];  // the lane's H flag words of one 8-step group (nw_fill_d16dir.cuh)
    while (i > 0 && j > 0) {
      const int ia = i - 1;
      const int s = ia / RS, rr = ia % RS, l = rr / KR16, r = rr % KR16;
      const int hi = r >= H;
      const int kk = hi ? r - H : r;
      const int t = hi ? j + 2 * l : j - 1 + 2 * l;
      const long long bidx = (((long long)s * G + (t >> 3)) * 32 + l) * H;
      if (bidx != cur) {  // up-moves inside the lane's rows and left-moves inside the group
                          // reuse the block: one 16-byte load per block change
        const uint4* bp = reinterpret_cast<const uint4*>(d + bidx);
#pragma unroll
        for (int v = 0; v < H / 4; ++v) blk[v] = COHERENT ? __ldcg(bp + v) : __ldg(bp + v);
        cur = bidx;
      }
      uint32_t w = 0;
#pragma unroll
      for (int v = 0; v < H / 4; ++v) {
        const uint4 b4 = blk[v];
        const int k4 = kk - 4 * v;
        w = k4 == 0 ? b4.x : k4 == 1 ? b4.y : k4 == 2 ? b4.z : k4 == 3 ? b4.w : w;
      }
      const int qq = t & 7;
      // nw_fill_d16dir.cuh layout: half hi, step qq: nbX at bit 2(7-qq), nbY at 2(7-qq)+1
      const uint32_t fx = (w >> (16 * hi + 14 - 2 * qq)) & 1u, fy = (w >> (16 * hi + 15 - 2 * qq)) & 1u;
      const int code = !fx ? X : (!fy ? Y : Z);  // nb bits: 1 = not maximal
      o[--pos] = (uint8_t)(code == 1 ? 1 : (code == 2 ? cV : cH));
      i -= (code != 3);
      j -= (code != 2);
    }
    while (i > 0) { o[--pos] = (uint8_t)cV; --i; }  // column 0: vertical (R7)
    while (j > 0) { o[--pos] = (uint8_t)cH; --j; }  // row 0: horizontal
    B.ops_len[outk] = m + n - pos;
  }
  // move each path [pos, m + n) of its slot to [0, L): increasing 32-byte chunks,
  // all lanes read a chunk before any writes it, so the overlap is safe
  unsigned pend = __ballot_sync(FULL, act && pos > 0);
  while (pend) {
    const int src_lane = __ffs(pend) - 1;
    pend &= pend - 1;
    uint8_t* ob = reinterpret_cast<uint8_t*>(__shfl_sync(FULL, reinterpret_cast<unsigned long long>(o), src_lane));
    const int sb = __shfl_sync(FULL, pos, src_lane);
    const int Lb = __shfl_sync(FULL, m + n - pos, src_lane);
    __syncwarp();
    for (int c0 = 0; c0 < Lb; c0 += 32) {
      const bool in = c0 + lane < Lb;
      const uint8_t v = in ? ob[sb + c0 + lane] : 0;
      __syncwarp();
      if (in) ob[c0 + lane] = v;
      __syncwarp();
    }
  }
}

#ifdef NW_COMMON_KERNELS  // one TU
// Distributed all-pairs: rs[t] holds the score of rank-space task t (every rank's
// range, gathered); write it to its lexicographic pair index.
__global__ void k_rs_scatter(const int* __restrict__ rs, long long P, const int* __restrict__ perm,
                             int N, int* __restrict__ scores) {
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < P;
       t += (long long)gridDim.x * blockDim.x) {
    int pr, qr;
    unrank_pair(t, N, pr, qr);
    const int x = perm[pr], y = perm[qr];
    const int p = min(x, y), q = max(x, y);
    scores[(long long)p * N - (long long)p * (p + 1) / 2 + (q - p - 1)] = rs[t];
  }
}
#endif

// The walk as its own launch after the fill: one thread per task.
template <int KR16>
__global__ void __launch_bounds__(256) k_batch_walk(BatchArgs B) {
  const long long task = B.task0 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  walk_lanes<KR16, false>(B, task, task < B.task1, threadIdx.x & 31);
}

}  // namespace nwk
