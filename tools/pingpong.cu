// SM-to-SM hand-off latency through global memory (the fill's strip hand-off,
// DESIGN.md §3.2): CTA on SM a stores a tagged word (st.relaxed.gpu), CTA on SM b
// polls it (ld.relaxed.gpu) and answers on a second word; round-trip ns for
// every b with a = 0 and a few flag addresses (L2 homing differs by address).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pingpong tools/pingpong.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long ldr(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void str(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void k_pp(unsigned long long* ping, unsigned long long* pong, int* claim, int sa, int sb,
                     int rounds, long long* out_ns) {
  unsigned sm;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  if (threadIdx.x != 0) return;
  const bool is_a = (int)sm == sa, is_b = (int)sm == sb;
  if (!is_a && !is_b) return;
  if (atomicAdd(claim + (is_a ? 0 : 1), 1) != 0) return;  // one CTA per role
  if (is_a) {
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int r = 1; r <= rounds; ++r) {
      str(ping, r);
      long long spin = 0;
      while (ldr(pong) != (unsigned long long)r) {
        if (++spin > 20000000) { *out_ns = -1; return; }  // partner absent: give up
      }
    }
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    *out_ns = (long long)(t1 - t0);
  } else {
    for (int r = 1; r <= rounds; ++r) {
      long long spin = 0;
      while (ldr(ping) != (unsigned long long)r) {
        if (++spin > 20000000) return;
      }
      str(pong, r);
    }
  }
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const size_t span = 64ull << 20;
  char* buf;
  cudaMalloc(&buf, span);
  int* claim;
  long long* out;
  cudaMalloc(&claim, 8);
  cudaMalloc(&out, 8);
  const int rounds = 2000;
  const size_t offs[3] = {0, 1ull << 20, 37ull << 20};
  printf("{\n \"unit\": \"ns per round trip (a = SM 0)\",\n");
  for (int o = 0; o < 3; ++o) {
    printf(" \"offset_%zu\": [", offs[o]);
    for (int b = 1; b < nsm; ++b) {
      unsigned long long* ping = reinterpret_cast<unsigned long long*>(buf + offs[o]);
      unsigned long long* pong = reinterpret_cast<unsigned long long*>(buf + offs[o] + 4096);
      cudaMemset(buf + offs[o], 0, 8192);
      cudaMemset(claim, 0, 8);
      cudaMemset(out, 0, 8);
      k_pp<<<nsm * 2, 32>>>(ping, pong, claim, 0, b, rounds, out);
      cudaDeviceSynchronize();
      long long ns = 0;
      cudaMemcpy(&ns, out, 8, cudaMemcpyDeviceToHost);
      printf("%s%.0f", b > 1 ? ", " : "", (double)ns / rounds);
    }
    printf("]%s\n", o < 2 ? "," : "");
  }
  printf("}\n");
  return 0;
}
