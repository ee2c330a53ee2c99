// Step-latency microbenchmark for the wavefront skeleton:
// one warp, each step = __shfl_up_sync of the previous step's bottom value,
// a lane-0 select, and a dependent chain of KR VIMNMX3 (the vertical max chain).
// Reports cycles per step for KR = 0..8, with and without a second (E-like)
// shuffle chain, to separate the shuffle round trip from per-row cost.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o step_lat tools/step_lat.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int KR, bool TWO>
__global__ void k_step(int* out, long long* cyc, int steps, int seed) {
  const int lane = threadIdx.x;
  int h[KR > 0 ? KR : 1];
  for (int r = 0; r < (KR > 0 ? KR : 1); ++r) h[r] = seed * (lane + r);
  int send = lane, esend = lane * 3;
  const long long t0 = clock64();
  for (int t = 0; t < steps; ++t) {
    const int recv = __shfl_up_sync(0xffffffffu, send, 1);
    int up = lane == 0 ? t : recv;
#pragma unroll
    for (int r = 0; r < KR; ++r) {
      up = __vimax3_s32(up, h[r], up + r);
      h[r] = up;
    }
    send = up;
    if (TWO) {
      const int erecv = __shfl_up_sync(0xffffffffu, esend, 1);
      int e = lane == 0 ? t : erecv;
#pragma unroll
      for (int r = 0; r < KR; ++r) e = (h[r] & 1) ? e : e + r;
      esend = e;
    }
  }
  const long long t1 = clock64();
  out[lane] = send + esend;
  if (lane == 0) *cyc = t1 - t0;
}

template <int KR, bool TWO>
void run(int* out, long long* cyc) {
  const int steps = 1 << 16;
  k_step<KR, TWO><<<1, 32>>>(out, cyc, steps, 7);
  k_step<KR, TWO><<<1, 32>>>(out, cyc, steps, 7);
  cudaDeviceSynchronize();
  long long c = 0;
  cudaMemcpy(&c, cyc, sizeof c, cudaMemcpyDeviceToHost);
  printf("  \"kr%d_%s\": %.2f,\n", KR, TWO ? "two_chains" : "one_chain", (double)c / steps);
}

int main() {
  int* out;
  long long* cyc;
  cudaMalloc(&out, 128);
  cudaMalloc(&cyc, 8);
  printf("{\n");
  run<0, false>(out, cyc);
  run<1, false>(out, cyc);
  run<2, false>(out, cyc);
  run<4, false>(out, cyc);
  run<8, false>(out, cyc);
  run<2, true>(out, cyc);
  run<4, true>(out, cyc);
  run<8, true>(out, cyc);
  printf("  \"unit\": \"cycles per step\"\n}\n");
  return 0;
}
