// Co-optimal alignments (
// readings DESIGN.md R24-R25, §3.13).
//
//   k_coopt_fill   warps sweep 32-row strips (lane = row, anti-diagonal skew,
//                  up values by shuffle, strip-to-strip rows through a 2-slot
//                  buffer + per-strip progress): H' (shifted recurrence, §3.1), the optimal-
//                  branch mask of every cell and the saturating 64-bit count
//                  N(i,j) = sum of N over the optimal predecessors (N = 1 on the
//                  borders); optionally stores the masks ((m+1) x (n+1) bytes)
//   k_coopt_enum   depth-first enumeration from (m, n) over the stored masks,
//                  branches tried in the tie order pi; the first cap paths,
//                  forward order, packed back to back
// A separate, simple path: this is an analysis feature, not the headline fill.
// Included by nw_api.cu only.
#pragma once
#include <cstdint>

namespace nwk {

__device__ __forceinline__ unsigned long long sat_add(unsigned long long x, unsigned long long y) {
  const unsigned long long r = x + y;
  return r < x ? ~0ull : r;
}

// One warp per 32-row strip (lane = row, anti-diagonal skew, up values by
// shuffle), strips handed out in order by an atomic ticket; strip s passes its
// last row (H', N) to strip s+1 through slot (s+1) % 2 of a 2-slot row buffer
// and publishes progress[s] = columns written, 32 at a time (st.release; the
// reader polls with ld.acquire before loading a 32-column chunk). Two slots
// suffice: strip s+2 overwrites column j only after strip s+1 has read it.
// Masks: each lane packs 4 columns of its row into one 32-bit store.
__device__ __forceinline__ int ld_acquire_s32(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_s32(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

struct CooptArgs {
  const uint8_t* a;               // codes
  const uint8_t* b;
  const int8_t* prof;             // K x K, s - 2g
  int K, m, n, S;
  int* ticket;
  int* progress;                  // [S] columns of strip s's last row published
  int* rowH;                      // [2][n+1]
  unsigned long long* rowN;       // [2][n+1]
  uint32_t* mask;                 // [(m+1)][stride/4] packed bytes, or null
  long long stride;               // bytes per mask row (multiple of 4, >= n+1)
  unsigned long long* count;
};

__global__ void __launch_bounds__(32) k_coopt_fill(CooptArgs A) {
  const int lane = threadIdx.x, n = A.n, m = A.m;
  const long long wpr = A.stride / 4;  // mask words per row
  for (;;) {
    int s = 0;
    if (lane == 0) s = atomicAdd(A.ticket, 1);
    s = __shfl_sync(0xffffffffu, s, 0);
    if (s >= A.S) break;
    const int i = 32 * s + lane + 1;
    const bool row_ok = i <= m;
    const int ac = row_ok ? A.a[i - 1] : 0;
    const int* inH = A.rowH + (long long)(s & 1) * (n + 1);
    const unsigned long long* inN = A.rowN + (long long)(s & 1) * (n + 1);
    int* outH = A.rowH + (long long)((s + 1) & 1) * (n + 1);
    unsigned long long* outN = A.rowN + (long long)((s + 1) & 1) * (n + 1);
    int hl = 0, hprev = 0, hup_prev = 0, cH = 0;
    unsigned long long nl = 1, nprev = 0, nup_prev = 0, cN = 1;
    uint32_t macc = 2u;  // column 0 of this row: U (R24 border)
    for (int t = 0; t < n + 31; ++t) {
      const int j = t - lane + 1;
      // lane 0's column j = t + 1 comes from chunk (t >> 5): fetch it when t % 32 == 0
      if ((t & 31) == 0 && t < n) {
        const int need = min(t + 32, n);
        if (s > 0) {
          if (lane == 0)
            while (ld_acquire_s32(A.progress + s - 1) < need) {
            }
          __syncwarp();
          const int jc = t + 1 + lane;
          cH = jc <= n ? __ldcg(inH + jc) : 0;
          cN = jc <= n ? __ldcg(inN + jc) : 1ull;
        } else {
          cH = 0; cN = 1ull;
        }
      }
      const int hs = __shfl_up_sync(0xffffffffu, hprev, 1);
      const unsigned long long ns = __shfl_up_sync(0xffffffffu, nprev, 1);
      const int hc = __shfl_sync(0xffffffffu, cH, t & 31);
      const unsigned long long nc = __shfl_sync(0xffffffffu, cN, t & 31);
      if (j >= 1 && j <= n) {
        int hu, hd;
        unsigned long long nu, nd;
        if (lane == 0) {
          hu = hc; nu = nc;
          hd = (j == 1) ? 0 : hup_prev;
          nd = (j == 1) ? 1ull : nup_prev;
        } else {
          hu = hs; nu = ns;
          hd = (j == 1) ? 0 : hup_prev;       // H'(i-1, 0) = 0
          nd = (j == 1) ? 1ull : nup_prev;    // N(i-1, 0) = 1
        }
        const int cD = hd + A.prof[ac * A.K + A.b[j - 1]], cU = hu, cL = hl;
        const int h = max(cD, max(cU, cL));
        const bool mD = cD == h, mU = cU == h, mL = cL == h;
        unsigned long long nn = mD ? nd : 0ull;
        if (mU) nn = sat_add(nn, nu);
        if (mL) nn = sat_add(nn, nl);
        macc |= (uint32_t)(mD | (mU << 1) | (mL << 2)) << (8 * (j & 3));
        if ((j & 3) == 3 || j == n) {
          if (row_ok && A.mask) A.mask[(long long)i * wpr + (j >> 2)] = macc;
          macc = 0;
        }
        if (row_ok && i == m && j == n) *A.count = nn;
        hup_prev = hu; nup_prev = nu;
        hl = h; nl = nn;
        hprev = h; nprev = nn;
        if (lane == 31) {
          outH[j] = h; outN[j] = nn;
          if ((j & 31) == 0 || j == n) st_release_s32(A.progress + s, j);  // after the data
        }
      }
    }
  }
}

// Depth-first enumeration (R25): lane 0 walks the masks (the path stack rev and
// the per-depth next-branch index trial live in shared memory when m+n fits,
// else in the global scratch), the whole warp copies each finished path out.
__global__ void __launch_bounds__(32) k_coopt_enum(const uint8_t* __restrict__ mask, int m, int n,
                                                   long long mstride, int X, int Y, int Z, int cap,
                                                   uint8_t* ops, long long ops_cap,
                                                   long long* ops_off, int* nfound, uint8_t* grev,
                                                   uint8_t* gtrial, int use_smem) {
  extern __shared__ uint8_t esm[];
  const int lane = threadIdx.x;
  const long long L = (long long)m + n + 1;
  uint8_t* rev = use_smem ? esm : grev;
  uint8_t* trial = use_smem ? esm + L : gtrial;
  const int pi[3] = {X, Y, Z};
  int found = 0;
  long long used = 0, d = 0;
  int i = m, j = n;
  if (lane == 0) { ops_off[0] = 0; trial[0] = 0; }
  for (;;) {
    int status = 0;  // 1: a path is complete (length d), 2: finished
    if (lane == 0) {
      for (;;) {
        if (i == 0 && j == 0) { status = 1; break; }
        const uint32_t mk = mask[(long long)i * mstride + j];
        int t = trial[d];
        while (t < 3 && !((mk >> (pi[t] - 1)) & 1u)) ++t;
        if (t < 3) {  // descend along branch pi[t]
          const int x = pi[t];
          trial[d] = (uint8_t)(t + 1);
          rev[d] = (uint8_t)x;
          i -= (x != 3);
          j -= (x != 2);
          ++d;
          trial[d] = 0;
          continue;
        }
        if (d == 0) { status = 2; break; }  // no untried branch anywhere: done
        --d;                                // backtrack
        const int x = rev[d];
        i += (x != 3);
        j += (x != 2);
      }
    }
    status = __shfl_sync(0xffffffffu, status, 0);
    d = __shfl_sync(0xffffffffu, d, 0);
    if (status == 2 || used + d > ops_cap) break;
    __syncwarp();  // rev visible to the warp
    for (long long k = lane; k < d; k += 32) ops[used + k] = rev[d - 1 - k];
    used += d;
    ++found;
    if (lane == 0) ops_off[found] = used;
    if (found >= cap) break;
    __syncwarp();
    if (d == 0) break;  // the empty path (m = n = 0) is the only one
    if (lane == 0) {    // step back from the origin to look for the next path
      --d;
      const int x = rev[d];
      i += (x != 3);
      j += (x != 2);
    }
  }
  if (lane == 0) *nfound = found;
}

}  // namespace nwk
