// The paper's own kernel design (PAPER.md Code 1), corrected, as an
// ablation baseline for the warp-strip fill.
//
// Kept from Code 1: one thread per interior cell, a grid-stride loop over the
// row-major (m x n) interior, a zero-initialised direction grid that doubles as
// the readiness flag ("0 = not computed"), a spin loop on the neighbours
// instead of a barrier, the full H and direction grids in memory,
// and the serial backtrack over the stored directions.
// Corrected: the additive recurrence with the gap score (readings C-1/C-2: Code 1
// multiplies and never writes the maximum), the row-major index arithmetic (C-3),
// and memory ordering: the direction is published with st.release.gpu after H,
// and the waiters poll with ld.acquire.gpu (Code 1's plain loads race).
// Waiting on the up and left neighbours suffices: the up cell's own wait on its
// left neighbour orders the diagonal before it (causality).
// Forward progress: the grid is sized to be co-resident, and every cell depends
// only on cells with smaller row-major index, i.e. on the same or earlier
// iterations of co-resident threads; lanes of one warp that wait on each other
// rely on independent thread scheduling (sm_70+).
// Included by nw_api.cu only.
#pragma once
#include <cstdint>

namespace nwk {

__device__ __forceinline__ uint32_t ld_acquire_u8(const uint8_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u8 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u8(uint8_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u8 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Borders: H(i,0) = i g, H(0,j) = j g; T(i,0) = U, T(0,j) = L, and the
// origin marked computed (4); the interior of T zeroed.
__global__ void k_percell_init(int* H, uint8_t* T, int m, int n, int g) {
  const long long W = (long long)n + 1, N = ((long long)m + 1) * W;
  for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < N;
       c += (long long)gridDim.x * blockDim.x) {
    const long long i = c / W, j = c % W;
    if (i == 0 || j == 0) {
      H[c] = (int)((i + j) * g);
      T[c] = (i == 0 && j == 0) ? 4 : (i == 0 ? 3 : 2);
    } else {
      T[c] = 0;
    }
  }
}

// s(a_i, b_j) = prof[a*K + b] + 2g (the context's profile holds s - 2g).
__global__ void k_percell_fill(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b,
                               const int8_t* __restrict__ prof, int K, int m, int n, int g,
                               int X, int Y, int Z, int* H, uint8_t* T) {
  const long long W = (long long)n + 1, cells = (long long)m * n;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < cells;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long i = idx / n + 1, j = idx % n + 1;
    const long long c = i * W + j;
    while (ld_acquire_u8(T + c - W) == 0) {
    }
    while (ld_acquire_u8(T + c - 1) == 0) {
    }
    const int s = prof[a[i - 1] * K + b[j - 1]] + 2 * g;
    const int cD = H[c - W - 1] + s, cU = H[c - W] + g, cL = H[c - 1] + g;
    const int h = max(cD, max(cU, cL));
    const int cX = X == 1 ? cD : (X == 2 ? cU : cL);
    const int cY = Y == 1 ? cD : (Y == 2 ? cU : cL);
    const int code = cX == h ? X : (cY == h ? Y : Z);  // first maximal in pi
    H[c] = h;
    st_release_u8(T + c, (uint32_t)code);
  }
}

// Serial backtrack: one thread from (m, n); ops written reversed.
__global__ void k_percell_walk(const uint8_t* __restrict__ T, int m, int n, uint8_t* rev,
                               long long* len) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const long long W = (long long)n + 1;
  long long i = m, j = n, k = 0;
  while (i > 0 || j > 0) {
    const int code = (i == 0) ? 3 : (j == 0 ? 2 : T[i * W + j]);
    rev[k++] = (uint8_t)code;
    i -= (code != 3);
    j -= (code != 2);
  }
  *len = k;
}

__global__ void k_percell_reverse(const uint8_t* __restrict__ rev, const long long* __restrict__ len,
                                  uint8_t* out) {
  const long long L = *len;
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < L;
       p += (long long)gridDim.x * blockDim.x)
    out[p] = rev[L - 1 - p];
}

__global__ void k_percell_score(const int* __restrict__ H, int m, int n, long long* score) {
  *score = H[(long long)m * (n + 1) + n];
}

}  // namespace nwk
