// Integer-pipe microbenchmark for the NW roofline.
//
// Measures, on the B200 it runs on, the issue throughput (warp-instructions per
// SM per clock, and lane-ops per SM per clock) and the dependent latency (cycles)
// of the integer instructions the DP fill is built from: the DPX max-plus family
// (VIMNMX3, VIADDMNMX, VIMNMX and their U16x2 forms), VIADD.16x2, IADD3, LOP3,
// PRMT, SHF, IMAD, SEL and SHFL. The results are the denominators of the
// "bound": "alu" roofline reported by bench.py.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peaks_int tools/peaks_int.cu
// Run:   ./peaks_int > peaks_int.json
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ILP 8
#define ITERS 4096

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)

// Each op is a statement updating `a` from `a`, `b`, `c` (b, c loop-invariant
// per chain; the empty asm keeps ptxas from folding idempotent max chains).
#define OP_vimax3_s32      a = __vimax3_s32(a, b, c)
#define OP_viaddmax_s32    a = __viaddmax_s32(a, b, c)
#define OP_vimax_s32       a = (uint32_t)max((int)a, (int)b)
#define OP_vimax3_u16x2    a = __vimax3_u16x2(a, b, c)
#define OP_viaddmax_u16x2  a = __viaddmax_u16x2(a, b, c)
#define OP_vimax_u16x2     a = __vmaxu2(a, b)
#define OP_vibmax_u16x2    { bool p_, q_; a = __vibmax_u16x2(a, b, &p_, &q_); c ^= (p_ ? 1u : 0u); }
#define OP_vadd2           a = __vadd2(a, b)
#define OP_iadd3           a = a + b + c
// volatile PTX: a plain (a & b) ^ c chain was folded across statements (round 1 reported
// an impossible 453 lane-ops/clk/SM, above the 128 issue limit)
#define OP_lop3            asm volatile("lop3.b32 %0, %0, %1, %2, 0x6a;" : "+r"(a) : "r"(b), "r"(c))
#define OP_prmt            a = __byte_perm(a, b, c)
#define OP_shf             a = __funnelshift_r(a, b, c)
#define OP_imad            a = a * b + c
#define OP_shfl            a = __shfl_xor_sync(0xffffffffu, a, 1) + b
#define OP_mix_viaddmax_imad   a = __viaddmax_s32(a, b, c); a = a * b + c
#define OP_mix_viaddmax_lop3   a = __viaddmax_s32(a, b, c); asm volatile("lop3.b32 %0, %0, %1, %2, 0x6a;" : "+r"(a) : "r"(b), "r"(c))
#define OP_mix_viaddmax_prmt   a = __viaddmax_s32(a, b, c); a = __byte_perm(a, b, c)
#define OP_mix_u16x2_imad      a = __viaddmax_u16x2(a, b, c); a = a * b + c

#define DEF_KERNEL(NAME)                                                          \
  __global__ void __launch_bounds__(1024) tput_##NAME(uint32_t* out, long long* cyc, uint32_t seed) { \
    uint32_t av[ILP], bv[ILP], cv[ILP];                                           \
    _Pragma("unroll") for (int k = 0; k < ILP; ++k) {                             \
      av[k] = seed * (threadIdx.x + 7 * k + 1);                                   \
      bv[k] = seed ^ (k * 0x9e3779b9u) ^ threadIdx.x;                             \
      cv[k] = (seed + k) * 0x85ebca6bu;                                           \
    }                                                                             \
    __syncthreads();                                                              \
    long long t0 = clock64();                                                     \
    for (int it = 0; it < ITERS; ++it) {                                          \
      _Pragma("unroll") for (int k = 0; k < ILP; ++k) {                           \
        uint32_t a = av[k], b = bv[k], c = cv[k];                                 \
        OP_##NAME;                                                                \
        asm volatile("" : "+r"(a), "+r"(c));                                      \
        av[k] = a; cv[k] = c;                                                     \
      }                                                                           \
    }                                                                             \
    __syncthreads();                                                              \
    long long t1 = clock64();                                                     \
    uint32_t r = 0;                                                               \
    _Pragma("unroll") for (int k = 0; k < ILP; ++k) r ^= av[k] ^ cv[k];           \
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;                               \
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;                              \
  }                                                                               \
  __global__ void lat_##NAME(uint32_t* out, long long* cyc, uint32_t seed) {      \
    uint32_t a = seed * (threadIdx.x + 1), b = seed ^ threadIdx.x, c = seed * 3u; \
    long long t0 = clock64();                                                     \
    for (int it = 0; it < ITERS; ++it) {                                          \
      OP_##NAME;                                                                  \
      asm volatile("" : "+r"(a), "+r"(c));                                        \
    }                                                                             \
    long long t1 = clock64();                                                     \
    out[threadIdx.x] = a ^ c;                                                     \
    if (threadIdx.x == 0) cyc[0] = t1 - t0;                                       \
  }

#define OPS(X) X(vimax3_s32) X(viaddmax_s32) X(vimax_s32) X(vimax3_u16x2) X(viaddmax_u16x2) \
  X(vimax_u16x2) X(vibmax_u16x2) X(vadd2) X(iadd3) X(lop3) X(prmt) X(shf) X(imad) X(shfl) \
  X(mix_viaddmax_imad) X(mix_viaddmax_lop3) X(mix_viaddmax_prmt) X(mix_u16x2_imad)

OPS(DEF_KERNEL)

// instructions per OP_ statement (for the lane-op rate); the mixes count 2
static int ops_per_stmt(const char* n) {
  if (n[0] == 'm' && n[1] == 'i' && n[2] == 'x') return 2;
  if (!__builtin_strcmp(n, "vibmax_u16x2")) return 3;  // VIMNMX.U16x2 + SEL + LOP3
  if (!__builtin_strcmp(n, "shfl")) return 2;          // SHFL + IADD
  return 1;
}

int main() {
  int dev = 0;
  CK(cudaSetDevice(dev));
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, dev));
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  const int nsm = p.multiProcessorCount;
  uint32_t* out; long long* cyc;
  CK(cudaMalloc(&out, sizeof(uint32_t) * nsm * 1024));
  CK(cudaMalloc(&cyc, sizeof(long long) * nsm));
  long long* hc = new long long[nsm];
  printf("{\"device\": \"%s\", \"sm_count\": %d, \"cc\": \"%d.%d\", \"clock_khz_attr\": %d, "
         "\"smem_per_sm\": %zu, \"l2_bytes\": %d, \"regs_per_sm\": %d,\n \"ilp\": %d, \"iters\": %d, \"ops\": {\n",
         p.name, nsm, p.major, p.minor, clk_khz, p.sharedMemPerMultiprocessor, p.l2CacheSize,
         p.regsPerMultiprocessor, ILP, ITERS);
  bool first = true;
#define RUN(NAME) {                                                                       \
    float best_ipc = 0.f;                                                                 \
    for (int warps = 8; warps <= 32; warps *= 2) {                                        \
      tput_##NAME<<<nsm, warps * 32>>>(out, cyc, 12345u);                                 \
      CK(cudaGetLastError()); CK(cudaDeviceSynchronize());                                \
      tput_##NAME<<<nsm, warps * 32>>>(out, cyc, 12345u);                                 \
      CK(cudaDeviceSynchronize());                                                        \
      CK(cudaMemcpy(hc, cyc, sizeof(long long) * nsm, cudaMemcpyDeviceToHost));           \
      long long mx = 0; for (int s = 0; s < nsm; ++s) mx = hc[s] > mx ? hc[s] : mx;       \
      double stmts = (double)warps * ITERS * ILP;                                         \
      float ipc = (float)(stmts * ops_per_stmt(#NAME) / (double)mx);                      \
      if (ipc > best_ipc) best_ipc = ipc;                                                 \
    }                                                                                     \
    lat_##NAME<<<1, 32>>>(out, cyc, 777u);                                                \
    CK(cudaDeviceSynchronize());                                                          \
    lat_##NAME<<<1, 32>>>(out, cyc, 777u);                                                \
    CK(cudaDeviceSynchronize());                                                          \
    CK(cudaMemcpy(hc, cyc, sizeof(long long), cudaMemcpyDeviceToHost));                   \
    printf("%s  \"%s\": {\"warp_instr_per_clk_per_sm\": %.3f, \"lane_ops_per_clk_per_sm\": %.1f, " \
           "\"dep_cycles_per_stmt\": %.2f}", first ? "" : ",\n", #NAME, best_ipc, best_ipc * 32.f, \
           (double)hc[0] / ITERS);                                                        \
    first = false;                                                                        \
  }
  OPS(RUN)
  printf("\n}}\n");
  return 0;
}
