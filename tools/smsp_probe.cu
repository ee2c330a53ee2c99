// Placement probe: where do the 1-warp CTAs of a persistent single-pair launch land?
// Every CTA records (%smid, %warpid) and stays resident until all have arrived (as the
// fill's strips do), then the host histograms warps per SM sub-partition (warpid % 4).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/smsp_probe tools/smsp_probe.cu
#include <cstdio>
#include <vector>
#include <map>
#include <cuda_runtime.h>
__global__ void probe(int* rec, int* arrived, int n) {
  unsigned smid, wid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
  if (threadIdx.x == 0) {
    rec[2 * blockIdx.x] = smid;
    rec[2 * blockIdx.x + 1] = wid;
    atomicAdd(arrived, 1);
    while (atomicAdd(arrived, 0) < n) { }
  }
  __syncwarp();
}
int main(int argc, char** argv) {
  for (int n : {157, 1117, 1184, 1737, 2233}) {
    int *rec, *arr;
    cudaMalloc(&rec, 8 * n); cudaMalloc(&arr, 4); cudaMemset(arr, 0, 4);
    probe<<<n, 32>>>(rec, arr, n);
    cudaDeviceSynchronize();
    std::vector<int> h(2 * n);
    cudaMemcpy(h.data(), rec, 8 * n, cudaMemcpyDeviceToHost);
    std::map<long, int> per;  // (sm, smsp) -> warps
    std::map<int, int> persm;
    for (int i = 0; i < n; ++i) { per[(long)h[2 * i] * 4 + (h[2 * i + 1] % 4)]++; persm[h[2 * i]]++; }
    std::map<int, int> hist, hsm;
    for (auto& kv : per) hist[kv.second]++;
    for (auto& kv : persm) hsm[kv.second]++;
    printf("{\"ctas\": %d, \"smsp_used\": %zu, \"warps_per_smsp_hist\": {", n, per.size());
    bool f = true; for (auto& kv : hist) { printf("%s\"%d\": %d", f ? "" : ", ", kv.first, kv.second); f = false; }
    printf("}, \"ctas_per_sm_hist\": {"); f = true;
    for (auto& kv : hsm) { printf("%s\"%d\": %d", f ? "" : ", ", kv.first, kv.second); f = false; }
    printf("}}\n");
    cudaFree(rec); cudaFree(arr);
  }
}
