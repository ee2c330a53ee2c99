// nw_launch.cuh -- host launchers for the templated kernels, split across
// translation units (one per tie order) so the library compiles in parallel.
#pragma once
#include <cuda_runtime.h>

#include "nw_kernels.cuh"

namespace nwk {

constexpr int KR_MAX = 8;    // rows per lane: single-pair kernels pick 2, 4 or 8 per shape
constexpr int R_MAX = 32 * 32;  // tallest strip of any sweep (packed KR = 32): code padding
constexpr int KR_BATCH = 8;  // rows per lane, batch kernel

// DIRS = true launchers, one instantiation per tie order PI (nw_inst_<PI>.cu)
template <int PI>
void launch_fill_dirs(const FillArgs& A, int kr, bool profreg, int grid, size_t smem, cudaStream_t st);
template <int PI>
void launch_batch_dirs(const BatchArgs& B, bool profreg, int packed_kr, int grid, size_t smem,
                       cudaStream_t st);
// the packed H' single-pair fill with decision bits (nw_fill_h16.cuh), KR 4 or 8
template <int PI>
void launch_fill_dirs_h16(const FillArgs& A, int kr, int grid, cudaStream_t st);

template <int KR, bool DIRS, bool PROFREG, int PI, int D16 = 0>
void launch_fill_t(const FillArgs& A, int grid, size_t smem, cudaStream_t st) {
  auto k = k_fill_pair<KR, DIRS, PROFREG, PI, D16>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<<<grid, 32, smem, st>>>(A);
}

template <int KR, bool DIRS, bool PROFREG, int PI, int PACKED = 0, int KR16 = 16>
void launch_batch_t(const BatchArgs& B, int grid, size_t smem, cudaStream_t st) {
  auto k = k_batch<KR, DIRS, PROFREG, PI, PACKED, KR16>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<<<grid, 128, smem, st>>>(B);
}

#define NW_DEFINE_DIRS_LAUNCHERS(PI)                                                          \
  template <>                                                                                 \
  void launch_fill_dirs<PI>(const FillArgs& A, int kr, bool profreg, int grid, size_t smem,   \
                            cudaStream_t st) {                                                \
    if (kr == 2) {                                                                            \
      if (profreg) launch_fill_t<2, true, true, PI>(A, grid, smem, st);                       \
      else launch_fill_t<2, true, false, PI>(A, grid, smem, st);                              \
    } else if (kr == 4) {                                                                     \
      if (profreg) launch_fill_t<4, true, true, PI>(A, grid, smem, st);                       \
      else launch_fill_t<4, true, false, PI>(A, grid, smem, st);                              \
    } else if (kr == 5 && profreg) {                                                          \
      launch_fill_t<5, true, true, PI>(A, grid, smem, st);                                    \
    } else if (kr == 6 && profreg) {                                                          \
      launch_fill_t<6, true, true, PI>(A, grid, smem, st);                                    \
    } else if (kr == 10 && profreg) {                                                         \
      launch_fill_t<10, true, true, PI>(A, grid, smem, st);                                   \
    } else if (kr == 12 && profreg) {                                                         \
      launch_fill_t<12, true, true, PI>(A, grid, smem, st);                                   \
    } else {                                                                                  \
      if (profreg) launch_fill_t<8, true, true, PI>(A, grid, smem, st);                       \
      else launch_fill_t<8, true, false, PI>(A, grid, smem, st);                              \
    }                                                                                         \
  }                                                                                           \
  template <>                                                                                 \
  void launch_fill_dirs_h16<PI>(const FillArgs& A, int kr, int grid, cudaStream_t st) {       \
    if (kr == 8) launch_fill_t<8, true, true, PI, 3>(A, grid, 0, st);                         \
    else launch_fill_t<4, true, true, PI, 3>(A, grid, 0, st);                                 \
  }                                                                                           \
  template <>                                                                                 \
  void launch_batch_dirs<PI>(const BatchArgs& B, bool profreg, int packed_kr, int grid,      \
                             size_t smem, cudaStream_t st) {                                  \
    if (packed_kr == 16) {                                                                    \
      if (profreg) launch_batch_t<KR_BATCH, true, true, PI, 3, 16>(B, grid, smem, st);        \
      else launch_batch_t<KR_BATCH, true, false, PI, 3, 16>(B, grid, smem, st);               \
    } else if (packed_kr == 8) {                                                              \
      if (profreg) launch_batch_t<KR_BATCH, true, true, PI, 3, 8>(B, grid, smem, st);         \
      else launch_batch_t<KR_BATCH, true, false, PI, 3, 8>(B, grid, smem, st);                \
    } else {                                                                                  \
      if (profreg) launch_batch_t<KR_BATCH, true, true, PI>(B, grid, smem, st);               \
      else launch_batch_t<KR_BATCH, true, false, PI>(B, grid, smem, st);                      \
    }                                                                                         \
  }

}  // namespace nwk
