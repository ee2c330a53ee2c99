// Center-star multiple alignment on the device (
// PAPER.md P:127-131; readings DESIGN.md R20-R23, §3.10).
//
//   k_msa_rowsum   row sums of the all-pairs score vector (lexicographic p<q order)
//   k_msa_argmax   center = argmax row sum, lowest index on ties
//   k_msa_gaps     per alignment (center, k): g_k(r) = gaps opened in the center
//                  before its residue r; G(r) = max_k g_k(r) by atomicMax
//   k_msa_scan     block start columns B(r) = sum_{r' < r} (G(r') + 1), width W
//   k_msa_center   the center row: residue r at column B(r) + G(r)
//   k_msa_rows     every other row: D -> residue at the center column, U -> '-',
//                  L -> residue in the gap block, left-aligned (the union-gap
//                  merge of R22 in closed form: order-independent)
// The pairwise alignments themselves come from k_batch with NW_TRACEBACK.
// Included by nw_api.cu only.
#pragma once
#include <cstdint>

namespace nwk {

__global__ void k_msa_rowsum(const int* __restrict__ scores, int nseq, long long* rowsum) {
  __shared__ long long part[32];
  const int p = blockIdx.x;
  long long acc = 0;
  for (int q = threadIdx.x; q < nseq; q += blockDim.x) {
    if (q == p) continue;
    const int lo = min(p, q), hi = max(p, q);
    // lexicographic index of (lo, hi): lo*n - lo(lo+1)/2 + (hi - lo - 1)
    const long long k = (long long)lo * nseq - (long long)lo * (lo + 1) / 2 + (hi - lo - 1);
    acc += scores[k];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t = 0;
    for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) t += part[w];
    rowsum[p] = t;
  }
}

// (sum, index) order: larger sum wins, then the lower index.
__device__ __forceinline__ bool msa_better(long long s1, int i1, long long s2, int i2) {
  return s1 > s2 || (s1 == s2 && i1 < i2);
}

__global__ void k_msa_argmax(const long long* __restrict__ rowsum, int nseq, int* center) {
  __shared__ long long ss[32];
  __shared__ int si[32];
  long long bs = 0;
  int bi = -1;
  for (int p = threadIdx.x; p < nseq; p += blockDim.x)
    if (bi < 0 || msa_better(rowsum[p], p, bs, bi)) { bs = rowsum[p]; bi = p; }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const long long os = __shfl_xor_sync(0xffffffffu, bs, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (oi >= 0 && (bi < 0 || msa_better(os, oi, bs, bi))) { bs = os; bi = oi; }
  }
  if ((threadIdx.x & 31) == 0) { ss[threadIdx.x >> 5] = bs; si[threadIdx.x >> 5] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x + 31) / 32; ++w)
      if (si[w] >= 0 && (bi < 0 || msa_better(ss[w], si[w], bs, bi))) { bs = ss[w]; bi = si[w]; }
    *center = bi < 0 ? 0 : bi;
  }
}

// One warp per alignment, 32 ops at a time. Op codes: 1 D, 2 U (a_i vs
// '-'), 3 L ('-' vs b_j); the center is a (rows), so L opens a center gap. For
// the op at absolute index t: r = center residues consumed before t, j = other
// residues consumed before t, and a run of L ops ending before the op that
// consumes center residue r has length t_r - t_prev - 1.
__global__ void k_msa_gaps(const uint8_t* __restrict__ ops, const long long* __restrict__ ops_off,
                           const int* __restrict__ ops_len, int nal, int lc, int* G) {
  const int lane = threadIdx.x & 31;
  const int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (k >= nal) return;
  const uint8_t* o = ops + ops_off[k];
  const int len = ops_len[k];
  const unsigned lt = (1u << lane) - 1u;
  int r0 = 0;
  long long last = -1;
  for (int base = 0; base < len; base += 32) {
    const int t = base + lane;
    const bool c_use = t < len && o[t] != 3;
    const unsigned cc = __ballot_sync(0xffffffffu, c_use);
    if (c_use) {
      const unsigned before = cc & lt;
      const long long prev = before ? (long long)(base + 31 - __clz(before)) : last;
      const int g = (int)(t - prev - 1);  // L run right before center residue r
      if (g > 0) atomicMax(G + r0 + __popc(before), g);
    }
    if (cc) last = base + 31 - __clz(cc);
    r0 += __popc(cc);
  }
  const int g = (int)(len - last - 1);  // trailing run: the block after the last residue
  if (lane == 0 && g > 0) atomicMax(G + lc, g);
}

// Exclusive block starts B(r) = sum_{r' < r} (G(r') + 1) for r = 0..lc, and the
// width W = B(lc) + G(lc). One block, chunks of blockDim with a carried offset.
__global__ void k_msa_scan(const int* __restrict__ G, int lc, long long* B, long long* W) {
  __shared__ long long wsum[32];
  __shared__ long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  for (int base = 0; base <= lc; base += blockDim.x) {
    const int r = base + threadIdx.x;
    const long long v = r <= lc ? (long long)G[r] + 1 : 0;
    long long x = v;  // inclusive warp scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      long long w = lane < nw ? wsum[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      if (lane < nw) wsum[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    const long long excl = carry + (warp ? wsum[warp - 1] : 0) + x - v;
    if (r <= lc) B[r] = excl;
    __syncthreads();
    if (threadIdx.x == 0) carry += wsum[nw - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) *W = B[lc] + G[lc];
}

__global__ void k_msa_center(const uint8_t* __restrict__ cres, int lc, const int* __restrict__ G,
                             const long long* __restrict__ B, uint8_t* row) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < lc; r += gridDim.x * blockDim.x)
    row[B[r] + G[r]] = cres[r];
}

// Row of the other sequence of alignment k (one warp per alignment).
__global__ void k_msa_rows(const uint8_t* __restrict__ ops, const long long* __restrict__ ops_off,
                           const int* __restrict__ ops_len, const int* __restrict__ other,
                           const uint8_t* __restrict__ seqs, const long long* __restrict__ offs,
                           int nal, const int* __restrict__ G, const long long* __restrict__ B,
                           uint8_t* rows, long long W) {
  const int lane = threadIdx.x & 31;
  const int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (k >= nal) return;
  const uint8_t* o = ops + ops_off[k];
  const int len = ops_len[k];
  const int q = other[k];
  const uint8_t* res = seqs + offs[q];
  uint8_t* row = rows + (long long)q * W;
  const unsigned lt = (1u << lane) - 1u;
  int r0 = 0, j0 = 0;
  long long last = -1;
  for (int base = 0; base < len; base += 32) {
    const int t = base + lane;
    const int op = t < len ? o[t] : 0;
    const bool c_use = t < len && op != 3, o_use = t < len && op != 2;
    const unsigned cc = __ballot_sync(0xffffffffu, c_use);
    const unsigned oc = __ballot_sync(0xffffffffu, o_use);
    const int r = r0 + __popc(cc & lt), j = j0 + __popc(oc & lt);
    if (t < len) {
      if (op == 1) {
        row[B[r] + G[r]] = res[j];
      } else if (op == 3) {
        const unsigned before = cc & lt;
        const long long prev = before ? (long long)(base + 31 - __clz(before)) : last;
        row[B[r] + (t - prev - 1)] = res[j];
      }
    }
    if (cc) last = base + 31 - __clz(cc);
    r0 += __popc(cc);
    j0 += __popc(oc);
  }
}

}  // namespace nwk
