// Microbenchmark of the packed H' step (nw_fill_h16.cuh) without memory traffic:
// cycles per step of one warp's sweep of KR rows per lane (KR/2 packed registers:
// PRMT + IADD + VIMNMX3.U16x2 each, the shuffle of the lane above's bottom row),
// with W warps per SM sub-partition and C independent strips interleaved in one
// warp's instruction stream (C = 2: two chains, as two far-apart strips per warp).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/h16_step tools/h16_step.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t prmt2(uint32_t x, uint32_t y, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(x), "r"(y), "r"(sel));
  return d;
}

// F: feature bits added to the bare step, to find what the kernel's extra cycles are:
// 1 = selector from a global table (one LDG.U16 per step, L1-resident), 2 = lane 31
// stores its bottom value to global every step (STG.64), 4 = lane 0's boundary value
// via a SHFL.IDX per step (as the kernel's chunk), 8 = an 8-step group with the
// kernel's chunk load + tag vote
template <int KR, int C, int F = 0>
__global__ void k_step(uint32_t* out, long long* cyc, int steps, const uint16_t* tab,
                       unsigned long long* sink) {
  constexpr int H = KR / 2;
  const int lane = threadIdx.x & 31;
  uint32_t PA[C][H], PB[C][H], Hp[C][H], up0p[C], acc[C][H];
#pragma unroll
  for (int c = 0; c < C; ++c) {
#pragma unroll
    for (int k = 0; k < H; ++k) {
      PA[c][k] = 0x01030103u * (lane + k + c);
      PB[c][k] = 0x03010301u * (lane + k + 2 * c);
      Hp[c][k] = 0;
      acc[c][k] = 0;
    }
    up0p[c] = 0;
  }
  uint32_t selx = 0x2c80u + lane;
  __syncthreads();
  int chunk = lane;
  const long long t0 = clock64();
#pragma unroll 1
  for (int t = 0; t < steps; t += 8) {
    unsigned long long raw = 0;  // the next group's boundary chunk (as the kernel: one group ahead)
    if (F & 8) raw = *(volatile unsigned long long*)(sink + 4096 + ((t >> 3) & 1023) * 8 + (lane & 7));
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      uint32_t s = selx + (q << 4);
      if (F & 1) s = __ldg(tab + ((t + q - 2 * lane) & 4095));
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const int recv = __shfl_up_sync(0xffffffffu, (int)Hp[c][H - 1], 1);
        uint32_t bv = (uint32_t)(t + q);
        if (F & 4) bv = (uint32_t)__shfl_sync(0xffffffffu, chunk, q);
        const uint32_t upsrc = lane == 0 ? bv << 16 : (uint32_t)recv;
        uint32_t up = prmt2(upsrc, Hp[c][H - 1], 0x5432u);
        uint32_t diag = up0p[c];
        up0p[c] = up;
#pragma unroll
        for (int k = 0; k < H; ++k) {
          const uint32_t sp = prmt2(PA[c][k], PB[c][k], s);
          const uint32_t left = Hp[c][k];
          const uint32_t cd = diag + sp;
          const uint32_t h = __vimax3_u16x2(cd, left, up);
          if (F & 16) {  // decision flags (tie order D, U, L): nbX = [h != cD], nbY = [h != cU]
            const uint32_t m = __vminu2(h - up, 0x00010001u) * 2u + __vminu2(h - cd, 0x00010001u);
            acc[c][k] = acc[c][k] * 4u + m;
          }
          diag = left;
          up = h;
          Hp[c][k] = h;
        }
        if ((F & 2) && lane == 31) sink[((t + q) & 1023) * 4 + c] = ((unsigned long long)(t + q) << 32) | Hp[c][H - 1];
      }
    }
    if (F & 16) {  // the group's flag words, as the batch traceback sweep stores them
#pragma unroll
      for (int c = 0; c < C; ++c)
#pragma unroll
        for (int k = 0; k < H; k += 2)
          *reinterpret_cast<uint2*>(sink + 8192 + ((((t >> 3) & 255) * 32 + lane) * H + k) / 2) = make_uint2(acc[c][k], acc[c][k + 1]);
    }
    if (F & 8) {
      chunk = (int)(unsigned)raw;
      if (!__all_sync(0xffffffffu, (unsigned)(raw >> 32) != 0xdeadbeefu)) chunk ^= 1;
    }
    selx ^= 0x1111u;
  }
  const long long t1 = clock64();
  uint32_t sum = 0;
#pragma unroll
  for (int c = 0; c < C; ++c)
#pragma unroll
    for (int k = 0; k < H; ++k) sum += Hp[c][k] + acc[c][k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = sum;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int KR, int C, int F = 0>
void run(uint32_t* out, long long* cyc, int W, const uint16_t* tab, unsigned long long* sink) {
  const int steps = 1 << 15;
  k_step<KR, C, F><<<1, 128 * W>>>(out, cyc, steps, tab, sink);
  k_step<KR, C, F><<<1, 128 * W>>>(out, cyc, steps, tab, sink);
  cudaDeviceSynchronize();
  long long c = 0;
  cudaMemcpy(&c, cyc, sizeof c, cudaMemcpyDeviceToHost);
  const double cps = (double)c / steps;
  // cells per cycle per SM sub-partition: W warps x C strips x 32 lanes x KR rows per step
  printf("  \"kr%d_c%d_w%d_f%d\": {\"cycles_per_step\": %.1f, \"cells_per_cycle_smsp\": %.2f},\n", KR, C, W,
         F, cps, W * C * 32.0 * KR / cps);
}

int main() {
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, 4 * 4096);
  cudaMalloc(&cyc, 8 * 16);
  uint16_t* tab;
  unsigned long long* sink;
  cudaMalloc(&tab, 2 * 4096);
  cudaMemset(tab, 0x2c, 2 * 4096);
  cudaMalloc(&sink, 8 * 65536);
  cudaMemset(sink, 0, 8 * 65536);
  printf("{\n");
  for (int W : {1, 2}) {
    run<28, 1, 0>(out, cyc, W, tab, sink);
    run<28, 1, 1>(out, cyc, W, tab, sink);
    run<28, 1, 2>(out, cyc, W, tab, sink);
    run<28, 1, 4>(out, cyc, W, tab, sink);
    run<28, 1, 8>(out, cyc, W, tab, sink);
    run<28, 1, 15>(out, cyc, W, tab, sink);
  }
  // C2-like: lone warp, KR 4 / 6 / 8 with and without decision flags (+ per-step store)
  run<4, 1, 0>(out, cyc, 1, tab, sink);
  run<4, 1, 16>(out, cyc, 1, tab, sink);
  run<4, 1, 18>(out, cyc, 1, tab, sink);
  run<8, 1, 16>(out, cyc, 1, tab, sink);
  run<8, 1, 18>(out, cyc, 1, tab, sink);
  run<6, 1, 18>(out, cyc, 1, tab, sink);
  printf("  \"end\": 0\n}\n");
  return 0;
}
