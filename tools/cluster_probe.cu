// Placement probe for thread-block clusters of one-warp CTAs (the
// cluster hand-off variants of the single-pair fill lost more the larger the
// cluster). Launches G CTAs of 32 threads in clusters of CS with a given dynamic
// shared-memory request and records, per CTA, %smid and %warpid (the warp slot; its
// low two bits are taken here as the SM sub-partition). Reports how many CTAs share
// an SM and a sub-partition, for CS = 1, 2, 4, 8.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/cluster_probe tools/cluster_probe.cu
#include <cstdio>
#include <map>
#include <vector>
#include <cuda_runtime.h>

__global__ void probe(int* out, long long spin) {
  extern __shared__ int dsm[];
  unsigned smid, warpid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  asm volatile("mov.u32 %0, %%warpid;" : "=r"(warpid));
  if (threadIdx.x == 0) {
    dsm[0] = 1;
    out[2 * blockIdx.x] = (int)smid;
    out[2 * blockIdx.x + 1] = (int)warpid;
  }
  const long long t0 = clock64();  // stay resident so all CTAs coexist
  while (clock64() - t0 < spin) {}
}

int main() {
  const int G = 160;  // ~C2's strip count at KR 4 (157)
  int* d;
  cudaMalloc(&d, 2 * G * sizeof(int));
  for (int smem_kb : {4, 100}) {
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kb * 1024);
    for (int CS : {1, 2, 4, 8}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(G);
      cfg.blockDim = dim3(32);
      cfg.dynamicSmemBytes = (size_t)smem_kb * 1024;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = CS;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaMemset(d, 0xff, 2 * G * sizeof(int));
      cudaError_t e = cudaLaunchKernelEx(&cfg, probe, d, 20000000LL);
      cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("smem %d KB CS %d: launch failed: %s\n", smem_kb, CS, cudaGetErrorString(e));
        continue;
      }
      std::vector<int> h(2 * G);
      cudaMemcpy(h.data(), d, 2 * G * sizeof(int), cudaMemcpyDeviceToHost);
      std::map<int, int> per_sm;
      std::map<std::pair<int, int>, int> per_smsp;
      int same_sm_in_cluster = 0, same_smsp_in_cluster = 0;
      for (int b = 0; b < G; ++b) {
        per_sm[h[2 * b]]++;
        per_smsp[{h[2 * b], h[2 * b + 1] & 3}]++;
        if (b % CS) {  // compare with the previous rank of the same cluster
          same_sm_in_cluster += h[2 * b] == h[2 * (b - 1)];
          same_smsp_in_cluster += h[2 * b] == h[2 * (b - 1)] && (h[2 * b + 1] & 3) == (h[2 * (b - 1) + 1] & 3);
        }
      }
      int max_sm = 0, max_smsp = 0, shared_smsp = 0;
      for (auto& kv : per_sm) max_sm = kv.second > max_sm ? kv.second : max_sm;
      for (auto& kv : per_smsp) {
        max_smsp = kv.second > max_smsp ? kv.second : max_smsp;
        shared_smsp += kv.second > 1 ? kv.second : 0;
      }
      printf("smem %3d KB CS %d: %3zu SMs used, max %d CTAs/SM, max %d CTAs/sub-partition, "
             "%d CTAs share a sub-partition; consecutive ranks on the same SM %d, same sub-partition %d\n",
             smem_kb, CS, per_sm.size(), max_sm, max_smsp, shared_smsp, same_sm_in_cluster,
             same_smsp_in_cluster);
    }
  }
  return 0;
}
