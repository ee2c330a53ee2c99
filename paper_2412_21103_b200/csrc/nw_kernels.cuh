// nw_kernels.cuh -- the sm_100a kernels behind include/nw.h.
//
//   k_init      zero the per-call progress counters / tickets / flags
//   k_encode    residues -> alphabet codes (R10), first bad position (atomicMin)
//   k_fill_pair one pair, many warps: strips chained by release/acquire counters
//   k_tb_walk   backtracking of Sec. 2.4 over the packed decision bits
//   k_reverse   reversed walk -> forward-order codes (P:90 codes 1/2/3)
//   k_batch     many pairs: one warp per pair, strips in sequence,
//               optional per-pair traceback by the same warp
#pragma once
#include "nw_fill.cuh"

namespace nwk {

#ifdef NW_COMMON_KERNELS  // defined in exactly one TU (nw_api.cu)
__global__ void k_init(int* ints, int nints, long long* bad) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nints; i += gridDim.x * blockDim.x)
    ints[i] = 0;
  if (bad && blockIdx.x == 0 && threadIdx.x == 0) *bad = 0x7fffffffffffffffll;
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

#endif  // NW_COMMON_KERNELS

// One pair, one strip per warp at a time; strips handed out in order by an
// atomic ticket so every awaited producer is already resident (no deadlock).
template <int KR, bool DIRS, bool PROFREG, int PI>
__global__ void __launch_bounds__(32) k_fill_pair(FillArgs A) {
  extern __shared__ __align__(16) int8_t smem[];
  const int lane = threadIdx.x & 31;
  for (;;) {
    int s = 0;
    if (lane == 0) s = atomicAdd(A.ticket, 1);
    s = __shfl_sync(FULL, s, 0);
    if (s >= A.nstrips) break;
    strip_sweep<KR, DIRS, PROFREG, PI, true>(A, s, lane, smem);
  }
}

// Decode the 2 decision bits of cell (i, j) (1-based, interior) -> P:90 code.
template <int KR>
__device__ __forceinline__ int tb_code(const uint32_t* dirs, long long wpl, int i, int j, int X,
                                       int Y, int Z, long long& cur_w, uint32_t& word) {
  constexpr int R = 32 * KR, SPW = 16 / KR;
  const int ia = i - 1;
  const int s = ia / R, l = (ia % R) / KR, r = ia % KR;
  const int t = (j - 1) + l;
  const long long widx = ((long long)s * wpl + t / SPW) * 32 + l;
  if (widx != cur_w) { word = __ldcg(dirs + widx); cur_w = widx; }
  const int c = (t % SPW) * KR + r;
  const uint32_t f = (word >> (30 - 2 * c)) & 3u;
  return !(f & 1u) ? X : (!(f & 2u) ? Y : Z);  // f = (nb1, nb0), nw_fill.cuh
}

// Walk from (m, n) to (0, 0); rev[k] = k-th code from the end.
// Border cells follow R7: column 0 -> vertical, row 0 -> horizontal.
template <int KR>
__device__ long long tb_walk(const uint32_t* dirs, long long wpl, int m, int n, int X, int Y,
                             int Z, uint8_t* rev) {
  int i = m, j = n;
  long long k = 0, cur_w = -1;
  uint32_t word = 0;
  while (i > 0 && j > 0) {
    const int code = tb_code<KR>(dirs, wpl, i, j, X, Y, Z, cur_w, word);
    rev[k++] = (uint8_t)code;
    i -= (code != 3);
    j -= (code != 2);
  }
  while (i > 0) { rev[k++] = 2; --i; }
  while (j > 0) { rev[k++] = 3; --j; }
  return k;
}

template <int KR>
__global__ void k_tb_walk(const uint32_t* dirs, long long wpl, int m, int n, int X, int Y, int Z,
                          uint8_t* rev, long long* len) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *len = tb_walk<KR>(dirs, wpl, m, n, X, Y, Z, rev);
}

#ifdef NW_COMMON_KERNELS
// out[p] = rev[len-1-p], p < len
__global__ void k_reverse(const uint8_t* __restrict__ rev, const long long* __restrict__ len,
                          uint8_t* __restrict__ out) {
  const long long L = *len;
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < L;
       p += (long long)gridDim.x * blockDim.x)
    out[p] = rev[L - 1 - p];
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
  // per-warp scratch
  int* wbnd;               // [nwarps][2][bstride]
  long long bstride;
  int* whm;                // [nwarps]
  uint32_t* wdirs;         // [nwarps][dstride] (TRACEBACK)
  long long dstride;
  // traceback outputs
  const long long* ops_off;
  uint8_t* ops;
  int* ops_len;
  int X, Y, Z;
  int* err;
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

template <int KR, bool DIRS, bool PROFREG, int PI>
__global__ void __launch_bounds__(128) k_batch(BatchArgs B) {
  constexpr int R = 32 * KR;
  extern __shared__ __align__(16) int8_t smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const long long gw = (long long)blockIdx.x * (blockDim.x >> 5) + wib;
  int8_t* sprof = smem + (PROFREG ? 0 : wib * (B.K * R));
  int* bnd = B.wbnd + gw * 2 * B.bstride;
  uint32_t* wd = DIRS ? B.wdirs + gw * B.dstride : nullptr;
  for (;;) {
    int task = 0;
    if (lane == 0) task = atomicAdd(B.ticket, 1);
    task = __shfl_sync(FULL, task, 0);
    if (task >= B.npairs) break;
    int p, q;
    long long outk;
    if (B.pairs) {
      outk = B.order ? B.order[task] : task;
      p = B.pairs[2 * outk];
      q = B.pairs[2 * outk + 1];
    } else {
      int pr, qr;
      unrank_pair(task, B.nseq, pr, qr);
      const int x = B.perm[pr], y = B.perm[qr];
      p = min(x, y);
      q = max(x, y);
      outk = (long long)p * B.nseq - (long long)p * (p + 1) / 2 + (q - p - 1);
    }
    const long long ao = B.offs[p], bo = B.offs[q];
    const int m = (int)(B.offs[p + 1] - ao), n = (int)(B.offs[q + 1] - bo);
    int hmv = 0;
    if (m > 0 && n > 0) {
      FillArgs A;
      A.a = B.codes + ao; A.b = B.codes + bo; A.prof = B.prof; A.K = B.K;
      A.m = m; A.n = n; A.nstrips = (m + R - 1) / R; A.nslots = 2;
      A.bnd = bnd; A.bstride = B.bstride; A.prog = nullptr; A.ticket = nullptr;
      A.dirs = wd;
      A.wpl = (long long)((n + 62) / 32) * (32 / (16 / KR));
      A.hm = B.whm + gw; A.err = B.err;
      for (int s = 0; s < A.nstrips; ++s) strip_sweep<KR, DIRS, PROFREG, PI, false>(A, s, lane, sprof);
      __syncwarp();
      hmv = *(volatile int*)(B.whm + gw);
      if (DIRS) {
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

}  // namespace nwk
