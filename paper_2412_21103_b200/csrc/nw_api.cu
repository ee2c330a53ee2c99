// nw_api.cu -- host side of the C ABI declared in include/nw.h.
//
// Validation, alphabet/profile tables, workspace, kernel dispatch and error
// reporting. Every step of the computation runs in the kernels of
// nw_kernels.cuh; this file only marshals. There is no CPU fallback: without
// a CUDA device every entry point returns NW_E_CUDA.
#include <cuda_runtime.h>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/nw.h"
#define NW_COMMON_KERNELS 1
#include "nw_launch.cuh"
#include "nw_msa.cuh"
#include "nw_percell.cuh"
#include "nw_coopt.cuh"
#include "nw_dist.cuh"

using namespace nwk;

namespace {

constexpr int SCORE_MAX = 31;
constexpr int GAP_MAX = 48;

}  // namespace

struct nw_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int sm_count = 0;
  char err[512] = {0};
  long long bad_pos = -1;
  long long launches = 0;
  // workspace (grow-only)
  uint8_t* d_lut = nullptr;     // 256
  int8_t* d_prof = nullptr;     // 64*64
  long long* d_bad = nullptr;   // [0] first bad residue position, [1] watchdog flag (int): sticky
  int* d_err = nullptr;         //   = (int*)(d_bad + 1); both cleared only by check_deferred
  int* d_ints = nullptr;        // small ints: [0] ticket [1] err [2] hm [5] slow traceback strips
  size_t ints_cap = 0;
  uint8_t* d_codes = nullptr;   // encoded inputs
  size_t codes_cap = 0;
  uint8_t* d_raw = nullptr;     // raw residues copied from the host
  size_t raw_cap = 0;
  unsigned long long* d_bnd = nullptr;  // 2-slot tagged boundary ring
  size_t bnd_cap = 0;
  uint8_t* d_rev = nullptr;     // reversed traceback
  size_t rev_cap = 0;
  long long* d_len = nullptr;   // traceback length
  long long* d_score = nullptr; // score staging
  uint16_t* d_sel16 = nullptr;  // batch: selector table of the packed sweeps (FillArgs::sel)
  size_t sel16_cap = 0;
  void* d_scratch = nullptr;    // batch per-warp scratch
  size_t scratch_cap = 0;
  void* d_aux = nullptr;        // batch perm/order/offs/pairs staging
  size_t aux_cap = 0;
  // host scratch of the batch planner, kept between calls (no page faults per call)
  std::vector<int> h_aux, h_bkt, h_cnt;
  std::vector<long long> h_words, h_tw, h_tdoff;
  void* d_plan = nullptr;        // device batch planner scratch (buckets, words, histogram, scan)
  size_t plan_cap = 0;
  void* h_stage = nullptr;      // page-locked staging for per-call host tables (batch order, offsets)
  size_t stage_cap = 0;
  cudaEvent_t stage_ev = nullptr;  // the last staged copy (the buffer is reused after it)
  void* d_tbdirs = nullptr;     // two-phase batch traceback: every pair's decision words
  size_t tbdirs_cap = 0;
  long long* d_tdoff = nullptr; // ... and their word offsets per task
  size_t tdoff_cap = 0;
  // kernel timing (nw_ctx_set_timing): event pairs per kernel class
  bool timing = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_open[2];
  std::vector<cudaEvent_t> ev_pool;
  // tuning / test options (nw_ctx_set_option; 0 = the measured default)
  long long opt[NW_OPT_COUNT_] = {0};
  // distributed context (nw_ctx_set_dist): one process per GPU, NCCL communicator
  int rank = 0, world = 1;
  ncclComm_t comm = nullptr;
  int* d_rs = nullptr;          // implicit dist batches: every rank-space task's score
  size_t rs_cap = 0;
  int* d_pmat = nullptr;        // implicit dist traceback batches: materialised lex pairs
  size_t pmat_cap = 0;
  std::vector<long long> h_bounds, h_oo;
  std::vector<int> h_pmat;
  // column-block pipeline (a10): per-call tags, buffers zeroed once (nw_cblock.cuh)
  unsigned cb_tag_next = 1;
  void* d_cb_ring = nullptr;    // [ranks here][2][n + 66] tagged top/bottom rows
  size_t cb_ring_cap = 0;
  void* d_cb_recv = nullptr;    // this rank's receive buffer (cudaMalloc: IPC-exportable)
  size_t cb_recv_cap = 0;
  void* cb_next = nullptr;      // the next rank's receive buffer, IPC-opened
  void* d_cb_vrecv = nullptr;   // virtual ranks' receive buffers
  size_t cb_vrecv_cap = 0;
  void* d_cb_tab = nullptr;     // receive-buffer pointer table
  size_t cb_tab_cap = 0;
  // live handles: nw_ctx_destroy releases their device memory and detaches them, so
  // a handle freed after its context only deletes its host struct
  std::vector<nw_tb*> live_tb;
  std::vector<nw_msa*> live_msa;
  // last scoring uploaded (avoid re-uploading identical tables)
  bool have_tables = false;
  uint8_t lut_h[256];
  int8_t prof_h[64 * 64];
};

struct nw_msa {
  nw_ctx* ctx;               // null once the context was destroyed
  int nseq = 0, center = 0;
  long long W = 0;           // MSA columns
  uint8_t* d_rows = nullptr; // [nseq][W] gapped rows ('-' = gap), input order
};

struct nw_tb {
  nw_ctx* ctx;        // null once the context was destroyed
  void* mem;          // one device allocation holding everything below
  uint16_t* dirs;     // [S][wpl][KR][32] decision-bit halfwords (nw_fill.cuh)
  long long wpl;      // 8-step groups per strip
  int* spec;          // [S-1][nq] + 1: exits of sampled entries (k_tb_spec)
  int* cs;            // [S] entry column per strip (traceback)
  int* seglen;        // [S]
  uint8_t* seg;       // [S][segstride] reversed per-strip path segments
  long long segstride;
  int m, n, S;
  int kr;             // rows per lane of the fill that wrote `dirs`
  int lstep, nb;      // sampled-exit spacing (log2) and samples per strip (k_tb_spec)
  uint8_t tie[3];
};

namespace {

nw_status fail(nw_ctx* c, nw_status st, const char* fmt, ...) {
  if (c) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(c->err, sizeof c->err, fmt, ap);
    va_end(ap);
  }
  return st;
}

#define CUDA_TRY(c, x)                                                                    \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess) {                                                              \
      return fail((c), e_ == cudaErrorMemoryAllocation ? NW_E_NOMEM : NW_E_CUDA,          \
                  "%s: %s (%s:%d)", #x, cudaGetErrorString(e_), __FILE__, __LINE__);      \
    }                                                                                     \
  } while (0)

#define NCCL_TRY(c, x)                                                                    \
  do {                                                                                    \
    ncclResult_t r_ = (x);                                                                \
    if (r_ != ncclSuccess)                                                                \
      return fail((c), NW_E_COMM, "%s: %s", #x, nwd::nccl().GetErrorString(r_));          \
  } while (0)

#define LAUNCHED(c) ((c)->launches++)

cudaEvent_t take_event(nw_ctx* c) {
  if (!c->ev_pool.empty()) {
    cudaEvent_t e = c->ev_pool.back();
    c->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// Brackets kernel launches of one class with events when timing is enabled.
struct KernelTimer {
  nw_ctx* c;
  int cls;
  cudaEvent_t e0 = nullptr;
  KernelTimer(nw_ctx* ctx, int k) : c(ctx), cls(k) {
    if (c->timing) {
      e0 = take_event(c);
      cudaEventRecord(e0, c->stream);
    }
  }
  ~KernelTimer() {
    if (c->timing) {
      cudaEvent_t e1 = take_event(c);
      cudaEventRecord(e1, c->stream);
      c->ev_open[cls].push_back({e0, e1});
    }
  }
};

template <class T>
nw_status grow(nw_ctx* c, T*& p, size_t& cap, size_t need_bytes) {
  if (need_bytes <= cap && p) return NW_OK;
  if (p) {
    cudaFreeAsync(p, c->stream);
    p = nullptr;
    cap = 0;
  }
  size_t bytes = std::max<size_t>(need_bytes, 256);
  bytes = bytes + bytes / 4;
  CUDA_TRY(c, cudaMallocAsync(reinterpret_cast<void**>(&p), bytes, c->stream));
  cap = bytes;
  return NW_OK;
}

// Host -> device copies of per-call tables through a page-locked staging buffer:
// an async copy from pageable memory may wait for the stream, which leaves the
// GPU idle while the host prepares the rest of the call. Waits only for the
// previous staged copy (normally long finished) before reusing the buffer.
struct StagedCopy { void* dst; const void* src; size_t bytes; };
nw_status upload_staged(nw_ctx* c, const StagedCopy* cp, int k) {
  size_t total = 0;
  for (int i = 0; i < k; ++i) total += (cp[i].bytes + 255) & ~size_t(255);
  if (total == 0) return NW_OK;
  if (c->stage_ev) CUDA_TRY(c, cudaEventSynchronize(c->stage_ev));
  else CUDA_TRY(c, cudaEventCreateWithFlags(&c->stage_ev, cudaEventDisableTiming));
  if (total > c->stage_cap) {
    if (c->h_stage) cudaFreeHost(c->h_stage);
    c->h_stage = nullptr;
    c->stage_cap = 0;
    const size_t bytes = total + total / 4;
    CUDA_TRY(c, cudaMallocHost(&c->h_stage, bytes));
    c->stage_cap = bytes;
  }
  char* h = static_cast<char*>(c->h_stage);
  for (int i = 0; i < k; ++i) {
    if (!cp[i].bytes) continue;
    memcpy(h, cp[i].src, cp[i].bytes);
    CUDA_TRY(c, cudaMemcpyAsync(cp[i].dst, h, cp[i].bytes, cudaMemcpyHostToDevice, c->stream));
    h += (cp[i].bytes + 255) & ~size_t(255);
  }
  CUDA_TRY(c, cudaEventRecord(c->stage_ev, c->stream));
  return NW_OK;
}

nw_status check_scoring(nw_ctx* c, const nw_scoring* sc) {
  if (!sc) return fail(c, NW_E_INVAL, "scoring is NULL");
  if (!sc->alphabet) return fail(c, NW_E_INVAL, "alphabet is NULL");
  if (sc->K < 1 || sc->K > 64) return fail(c, NW_E_INVAL, "K=%d outside [1,64]", sc->K);
  if (sc->gap >= 0) return fail(c, NW_E_INVAL, "gap %d must be negative", sc->gap);
  if (sc->gap < -GAP_MAX) return fail(c, NW_E_INVAL, "gap %d below -%d", sc->gap, GAP_MAX);
  int seen[4] = {0, 0, 0, 0};
  for (int t = 0; t < 3; ++t) {
    if (sc->tie[t] < 1 || sc->tie[t] > 3 || seen[sc->tie[t]])
      return fail(c, NW_E_INVAL, "tie order is not a permutation of {1,2,3}");
    seen[sc->tie[t]] = 1;
  }
  for (int x = 0; x < sc->K; ++x)
    for (int y = 0; y < x; ++y)
      if (sc->alphabet[x] == sc->alphabet[y])
        return fail(c, NW_E_INVAL, "alphabet symbol '%c' repeated", sc->alphabet[x]);
  if (sc->subst) {
    for (int k = 0; k < sc->K * sc->K; ++k)
      if (sc->subst[k] < -SCORE_MAX || sc->subst[k] > SCORE_MAX)
        return fail(c, NW_E_INVAL, "substitution score %d outside [-%d,%d]", sc->subst[k],
                    SCORE_MAX, SCORE_MAX);
  } else {
    if (sc->match <= sc->mismatch)
      return fail(c, NW_E_INVAL, "match %d must exceed mismatch %d", sc->match, sc->mismatch);
    if (sc->match > SCORE_MAX || sc->mismatch < -SCORE_MAX)
      return fail(c, NW_E_INVAL, "match/mismatch outside [-%d,%d]", SCORE_MAX, SCORE_MAX);
  }
  return NW_OK;
}

int score_of(const nw_scoring* sc, int x, int y) {
  return sc->subst ? sc->subst[x * sc->K + y] : (x == y ? sc->match : sc->mismatch);
}

// Upload the 256-entry residue -> code table and the K x K profile of
// s(x,y) - 2g (the shifted recurrence, nw_fill.cuh).
nw_status upload_tables(nw_ctx* c, const nw_scoring* sc) {
  uint8_t lut[256];
  memset(lut, 0xff, sizeof lut);
  for (int k = 0; k < sc->K; ++k) lut[(uint8_t)sc->alphabet[k]] = (uint8_t)k;
  int8_t prof[64 * 64];
  memset(prof, 0, sizeof prof);
  for (int x = 0; x < sc->K; ++x)
    for (int y = 0; y < sc->K; ++y) prof[x * sc->K + y] = (int8_t)(score_of(sc, x, y) - 2 * sc->gap);
  if (c->have_tables && !memcmp(lut, c->lut_h, sizeof lut) && !memcmp(prof, c->prof_h, sizeof prof))
    return NW_OK;
  memcpy(c->lut_h, lut, sizeof lut);
  memcpy(c->prof_h, prof, sizeof prof);
  CUDA_TRY(c, cudaMemcpyAsync(c->d_lut, c->lut_h, 256, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(c->d_prof, c->prof_h, sizeof prof, cudaMemcpyHostToDevice, c->stream));
  c->have_tables = true;
  return NW_OK;
}

// |H| <= (m+n) * max(|g|, max|s|) must leave headroom in int32 (R11);
// the shifted H' adds up to (m+n)*|g| more.
nw_status check_bounds(nw_ctx* c, const nw_scoring* sc, long long m, long long n) {
  if (m < 0 || n < 0) return fail(c, NW_E_INVAL, "negative length");
  int smax = std::abs(sc->gap);
  for (int x = 0; x < sc->K; ++x)
    for (int y = 0; y < sc->K; ++y) smax = std::max(smax, std::abs(score_of(sc, x, y)));
  const double bound = (double)(m + n) * (double)(smax + 2 * std::abs(sc->gap));
  if (bound >= (double)(1 << 30) || m > (1 << 28) || n > (1 << 28))
    return fail(c, NW_E_OVERFLOW, "m=%lld n=%lld exceed the int32 score bound", m, n);
  return NW_OK;
}

int pi_code(const uint8_t tie[3]) { return tie[0] * 100 + tie[1] * 10 + tie[2]; }

long long pad16(long long x) { return (x + 15) & ~15ll; }

// Sampled strip exits: spacing of the samples in columns (log2;
// NW_OPT_TB_STEP rounds down to a power of two) and samples per strip (a multiple of 32).
int tb_lstep(const nw_ctx* c) {
  const long long k = c->opt[NW_OPT_TB_STEP] >= 1 ? c->opt[NW_OPT_TB_STEP] : 4;
  int l = 0;
  while ((2LL << l) <= k) ++l;
  return l;
}
// Default: 256 samples (C2, profiles/r01_exp_tbband.json); 32 when a row has at most 512
// samples (n <= ~2k columns): the wide band's warps mostly stage and walk for nothing
// (C1: 93 -> 72 us of traceback, tools/experiments/exp_c1tb.py).
int tb_band(const nw_ctx* c, long long n, int lstep) {
  const long long nq = (n >> lstep) + 1;
  const long long dflt = nq <= 512 ? 32 : 256;
  const long long k = c->opt[NW_OPT_TB_BAND] >= 32 ? std::min(c->opt[NW_OPT_TB_BAND], 4096LL) : dflt;
  return (int)((k + 31) / 32 * 32);
}

// Entries per boundary-ring slot (columns 0..n plus the sweep's overhang), 16-byte multiple.
long long bnd_stride(long long n) { return (n + 1 + 64 + 1) & ~1ll; }

// ---- kernel dispatch: score-only kernels here, one TU per tie order for DIRS ----
}  // namespace
namespace nwk {
NW_DEFINE_DIRS_LAUNCHERS(123)
}  // namespace nwk
namespace {

template <int KR>
void launch_score(const FillArgs& A, bool profreg, int grid, size_t smem, cudaStream_t st) {
  if (profreg) launch_fill_t<KR, false, true, 123>(A, grid, smem, st);
  else launch_fill_t<KR, false, false, 123>(A, grid, smem, st);
}

bool dispatch_fill(bool dirs, int pi, int kr, bool profreg, const FillArgs& A, int grid,
                   size_t smem, cudaStream_t st, bool d16 = false, bool two_chains = false) {
  if (!dirs && d16 && two_chains && kr % 4 == 0 && kr >= 16) {  // two chains per lane
    if (kr == 28) launch_fill_t<28, false, true, 123, 2>(A, grid, smem, st);
    else if (kr == 32) launch_fill_t<32, false, true, 123, 2>(A, grid, smem, st);
    else if (kr == 24) launch_fill_t<24, false, true, 123, 2>(A, grid, smem, st);
    else if (kr == 20) launch_fill_t<20, false, true, 123, 2>(A, grid, smem, st);
    else launch_fill_t<16, false, true, 123, 2>(A, grid, smem, st);
    return true;
  }
  if (!dirs && d16) {  // packed difference form, KR rows per lane (2 per register)
    if (kr == 32) launch_fill_t<32, false, true, 123, 1>(A, grid, smem, st);
    else if (kr == 30) launch_fill_t<30, false, true, 123, 1>(A, grid, smem, st);
    else if (kr == 28) launch_fill_t<28, false, true, 123, 1>(A, grid, smem, st);
    else if (kr == 26) launch_fill_t<26, false, true, 123, 1>(A, grid, smem, st);
    else if (kr == 24) launch_fill_t<24, false, true, 123, 1>(A, grid, smem, st);
    else if (kr == 22) launch_fill_t<22, false, true, 123, 1>(A, grid, smem, st);
    else if (kr == 20) launch_fill_t<20, false, true, 123, 1>(A, grid, smem, st);
    else if (kr == 18) launch_fill_t<18, false, true, 123, 1>(A, grid, smem, st);
    else if (kr == 14) launch_fill_t<14, false, true, 123, 1>(A, grid, smem, st);
    else if (kr == 12) launch_fill_t<12, false, true, 123, 1>(A, grid, smem, st);
    else if (kr == 16) launch_fill_t<16, false, true, 123, 1>(A, grid, smem, st);
    else if (kr == 8) launch_fill_t<8, false, true, 123, 1>(A, grid, smem, st);
    else launch_fill_t<4, false, true, 123, 1>(A, grid, smem, st);
    return true;
  }
  if (!dirs) {
    if (kr == 2) launch_score<2>(A, profreg, grid, smem, st);
    else if (kr == 4) launch_score<4>(A, profreg, grid, smem, st);
    else if (kr == 5 && profreg) launch_fill_t<5, false, true, 123>(A, grid, smem, st);  // experiments
    else if (kr == 6 && profreg) launch_fill_t<6, false, true, 123>(A, grid, smem, st);
    else launch_score<8>(A, profreg, grid, smem, st);
    return true;
  }
  switch (pi) {
    case 123: launch_fill_dirs<123>(A, kr, profreg, grid, smem, st); return true;
    case 132: launch_fill_dirs<132>(A, kr, profreg, grid, smem, st); return true;
    case 213: launch_fill_dirs<213>(A, kr, profreg, grid, smem, st); return true;
    case 231: launch_fill_dirs<231>(A, kr, profreg, grid, smem, st); return true;
    case 312: launch_fill_dirs<312>(A, kr, profreg, grid, smem, st); return true;
    case 321: launch_fill_dirs<321>(A, kr, profreg, grid, smem, st); return true;
  }
  return false;
}

// Packed H' pair sweep with a moving base (nw_fill_h16.cuh).
template <int F>
bool dispatch_fill_h16_t(int kr, const FillArgs& A, int grid, cudaStream_t st) {
  switch (kr) {
    case 8: launch_fill_t<8, false, true, 123, F>(A, grid, 0, st); return true;
    case 12: launch_fill_t<12, false, true, 123, F>(A, grid, 0, st); return true;
    case 16: launch_fill_t<16, false, true, 123, F>(A, grid, 0, st); return true;
    case 18: launch_fill_t<18, false, true, 123, F>(A, grid, 0, st); return true;
    case 20: launch_fill_t<20, false, true, 123, F>(A, grid, 0, st); return true;
    case 22: launch_fill_t<22, false, true, 123, F>(A, grid, 0, st); return true;
    case 24: launch_fill_t<24, false, true, 123, F>(A, grid, 0, st); return true;
    case 26: launch_fill_t<26, false, true, 123, F>(A, grid, 0, st); return true;
    case 28: launch_fill_t<28, false, true, 123, F>(A, grid, 0, st); return true;
    case 30: launch_fill_t<30, false, true, 123, F>(A, grid, 0, st); return true;
    case 32: launch_fill_t<32, false, true, 123, F>(A, grid, 0, st); return true;
  }
  return false;
}
bool dispatch_fill_h16(int kr, const FillArgs& A, int grid, cudaStream_t st) {
  return dispatch_fill_h16_t<3>(kr, A, grid, st);
}

#ifdef NW_TRACE
// experiment builds only: per-strip timestamps of the h16 sweep (every 1024 groups)
unsigned long long* g_trace = nullptr;
int g_trace_strips = 0;
unsigned long long* nw_trace_buffer(int nstrips) {
  if (nstrips > g_trace_strips) {
    if (g_trace) cudaFree(g_trace);
    cudaMalloc(&g_trace, sizeof(unsigned long long) * 256 * nstrips);
    g_trace_strips = nstrips;
  }
  cudaMemset(g_trace, 0, sizeof(unsigned long long) * 256 * g_trace_strips);
  return g_trace;
}
#endif

// Packed difference form (nw_fill_d16.cuh) applies to score-only DNA-size
// alphabets with s - 2g >= 0 for every symbol pair.
bool d16_ok(const nw_ctx* c, const nw_scoring* sc) {
  if (sc->K > 4 || c->opt[NW_OPT_NO_D16]) return false;
  for (int x = 0; x < sc->K; ++x)
    for (int y = 0; y < sc->K; ++y)
      if (score_of(sc, x, y) - 2 * sc->gap < 0) return false;
  return true;
}

// Rows per lane for a single pair: the strip count m/(32 KR)
// is the number of warps that can work at once; small KR buys parallelism at the
// cost of a longer lane skew (m/KR steps). NW_OPT_ROWS_PER_LANE overrides.
int choose_kr_shape(const nw_ctx* c, long long m, long long n, bool dirs);
// KR 5 and 6 exist only with register profiles (K <= 4)
int choose_kr(const nw_ctx* c, long long m, long long n, bool dirs, int K) {
  const int k = choose_kr_shape(c, m, n, dirs);
  return (K > 4 && (k == 5 || k == 6)) ? 4 : (K > 4 && k > 8) ? 8 : k;
}
int choose_kr_shape(const nw_ctx* c, long long m, long long n, bool dirs) {
  if (c->opt[NW_OPT_ROWS_PER_LANE]) {
    const int k = (int)c->opt[NW_OPT_ROWS_PER_LANE];
    if (k == 2 || k == 4 || k == 8 || k == 5 || k == 6) return k;  // 5, 6: register profiles only
    if (k == 10 || k == 12) return dirs ? k : 8;  // direction fills only
  }
  (void)dirs;
  // Tall pairs (>= ~150 strips at KR = 8): the largest KR, the lag is amortised
  // (80k x 2k best at 8, profiles/r01_exp_fill.json). Otherwise the wavefront
  // model of DESIGN.md §3.2: time ~ c(KR) (n + 31) + L(KR) (S - 1) cycles, with
  // the measured step cost c and strip-to-strip lag L (tools/exp_lag.py: c = 75,
  // 97.5, 150 and L = 9450, 9650, 12450 cycles at KR = 2, 4, 8): C2 -> 4,
  // C1 (1k x 1k) -> 4, 2k x 80k -> 2.
  if (m >= 32LL * 8 * 150) {
    // tall: the largest KR amortises the lag; with directions and register profiles,
    // 10 or 12 rows per lane once 8 would put more than two strips per SM
    // sub-partition (the lock-step pace of DESIGN.md §3.8; NW_OPT_TALL_KR8: always 8)
    if (dirs && !c->opt[NW_OPT_TALL_KR8])
      for (int k : {8, 10, 12})
        if ((m + 32LL * k - 1) / (32LL * k) <= 8LL * c->sm_count) return k;
    return 8;
  }
  const int ks[3] = {2, 4, 8};
  const double cs[3] = {75.0, 97.5, 150.0}, L[3] = {9450.0, 9650.0, 12450.0};
  int best = 2;
  double tbest = 1e300;
  for (int i = 0; i < 3; ++i) {
    const double S = (double)((m + 32 * ks[i] - 1) / (32 * ks[i]));
    const double t = cs[i] * (double)(n + 31) + L[i] * (S - 1.0);
    if (t < tbest) { tbest = t; best = ks[i]; }
  }
  return best;
}

// Rows per lane of the packed score-only sweep for a tall pair: the
// strips advance in lock-step, so the pair runs at the pace of the most loaded SM
// sub-partition: the smallest even KR >= 16 that keeps the strip count within two
// warps per sub-partition (1M^2: KR 28 = 1,117 strips, 6.5 TCUPS, vs KR 32 = 977
// strips 6.2 and KR 26 = 1,202 strips 5.5; tools/exp_c5kr.py). NW_OPT_D16_KR overrides.
int d16_kr(const nw_ctx* c, long long m) {
  int kd = 32;
  for (int k = 16; k <= 32; k += 2)
    if ((m + 32LL * k - 1) / (32LL * k) <= 8LL * c->sm_count) { kd = k; break; }
  const long long k = c->opt[NW_OPT_D16_KR];
  return (k >= 12 && k <= 32 && k % 2 == 0) ? (int)k : kd;
}

// Rebase period (8-step groups) of the packed H' pair sweep at KR rows per lane, or 0
// when the form does not apply: every relative value must stay below 2^16, i.e.
// S (32 KR + 8 reb + 160) <= 65535 with S = max(s - 2g) (nw_fill_h16.cuh).
int h16_rebase_groups(const nw_ctx* c, const nw_scoring* sc, int kr) {
  if (!d16_ok(c, sc)) return 0;
  int smax = 0;
  for (int x = 0; x < sc->K; ++x)
    for (int y = 0; y < sc->K; ++y) smax = std::max(smax, score_of(sc, x, y) - 2 * sc->gap);
  int reb = (int)std::max(0LL, std::min(c->opt[NW_OPT_H16_REBASE], 64LL));
  if (reb == 0) reb = 64;
  while (reb & (reb - 1)) reb &= reb - 1;  // power of two
  while (reb >= 1 && (long long)smax * (32LL * kr + 8LL * reb + 160) > 65535) reb >>= 1;
  return reb;
}

// Rows per lane of the packed H' pair sweep: NW_OPT_H16_KR, else the strip-count rule
// of d16_kr (same lock-step argument).
int h16_kr(const nw_ctx* c, long long m) {
  const long long k = c->opt[NW_OPT_H16_KR];
  if (k >= 8 && k <= 32 && k % 2 == 0 && (k >= 16 || k == 8 || k == 12)) return (int)k;
  int kd = 32;
  for (int q = 16; q <= 32; q += 2)
    if ((m + 32LL * q - 1) / (32LL * q) <= 8LL * c->sm_count) { kd = q; break; }
  return kd;
}

bool dispatch_batch(bool dirs, int pi, bool profreg, bool u16, bool d16, int packed_kr,
                    const BatchArgs& B, int grid, size_t smem, cudaStream_t st, int u16_kr = 16) {
  if (!dirs) {
    if (u16 && u16_kr == 1) launch_batch_t<KR_BATCH, false, true, 123, 4, 32>(B, grid, smem, st);
    else if (u16 && u16_kr == 32) launch_batch_t<KR_BATCH, false, true, 123, 1, 32>(B, grid, smem, st);
    else if (u16 && u16_kr == 8) launch_batch_t<KR_BATCH, false, true, 123, 1, 8>(B, grid, smem, st);
    else if (u16) launch_batch_t<KR_BATCH, false, true, 123, 1>(B, grid, smem, st);
    else if (d16) launch_batch_t<KR_BATCH, false, true, 123, 2>(B, grid, smem, st);
    else if (profreg) launch_batch_t<KR_BATCH, false, true, 123>(B, grid, smem, st);
    else launch_batch_t<KR_BATCH, false, false, 123>(B, grid, smem, st);
    return true;
  }
  switch (pi) {
    case 123: launch_batch_dirs<123>(B, profreg, d16 ? packed_kr : 0, grid, smem, st); return true;
    case 132: launch_batch_dirs<132>(B, profreg, d16 ? packed_kr : 0, grid, smem, st); return true;
    case 213: launch_batch_dirs<213>(B, profreg, d16 ? packed_kr : 0, grid, smem, st); return true;
    case 231: launch_batch_dirs<231>(B, profreg, d16 ? packed_kr : 0, grid, smem, st); return true;
    case 312: launch_batch_dirs<312>(B, profreg, d16 ? packed_kr : 0, grid, smem, st); return true;
    case 321: launch_batch_dirs<321>(B, profreg, d16 ? packed_kr : 0, grid, smem, st); return true;
  }
  return false;
}

// Encode `len` device residues at `raw` into codes at `out` (PAD zero bytes
// on both sides are the caller's allocation). Positions reported + pos_base.
void launch_encode(nw_ctx* c, const uint8_t* raw, long long len, uint8_t* out, long long pos_base) {
  if (len <= 0) return;
  long long blocks = (len + 4 * 256 - 1) / (4 * 256);
  blocks = std::min<long long>(blocks, (long long)c->sm_count * 8);
  k_encode<<<(int)blocks, 256, 0, c->stream>>>(raw, len, c->d_lut, out, c->d_bad, pos_base);
  LAUNCHED(c);
}

nw_status init_small(nw_ctx* c, int nints, ZeroRanges zr = ZeroRanges{{nullptr, nullptr, nullptr, nullptr}, {0, 0, 0, 0}}) {
  nw_status st = grow(c, c->d_ints, c->ints_cap, sizeof(int) * (size_t)nints);
  if (st) return st;
  long long work = nints;
  for (int r = 0; r < 4; ++r) work = std::max(work, zr.bytes[r] / 16);
  const int blocks = (int)std::min<long long>((long long)c->sm_count * 4, (work + 255) / 256 + 1);
  k_init<<<blocks, 256, 0, c->stream>>>(c->d_ints, nints, nullptr, zr);  // error flags are sticky
  LAUNCHED(c);
  return NW_OK;
}

// Device-side core of nw_score_only / nw_align_pair on already-encoded codes.
// ca, cb: codes with PAD before and >= R + PAD after. Writes H(m,n) to d_score.
nw_status pair_core(nw_ctx* c, const uint8_t* ca, long long m, const uint8_t* cb, long long n,
                    const nw_scoring* sc, long long* d_score, nw_tb* tb, int kr,
                    unsigned long long* ckpt = nullptr, int ck_every = 0, long long ck_stride = 0,
                    const unsigned long long* top_row = nullptr, unsigned top_tag = 0,
                    int h16_reb = 0);

bool cblock_dist_applies(const nw_ctx* c, long long m, long long n, const nw_scoring* sc);
nw_status cblock_dist(nw_ctx* c, const uint8_t* a, long long m, const uint8_t* b, long long n,
                      const nw_scoring* sc, bool host, long long* d_score);

}  // namespace

// ---- kernels for tiny bookkeeping ----
namespace nwk {
// Checkpoint rows of the packed score-only pass hold V(r, j) = H'(r, j) - H'(r, j-1)
// as tagged entries j = 1..n; the refills read H'(r, j). One block
// per slot turns each row into its inclusive prefix sum (H'(r, 0) = 0), tags kept.
__global__ void __launch_bounds__(1024) k_ckpt_prefix(unsigned long long* ckpt, long long stride,
                                                      int n, int nslots) {
  if ((int)blockIdx.x >= nslots) return;
  unsigned long long* row = ckpt + (long long)blockIdx.x * stride;
  __shared__ int wsum[32];
  __shared__ int carry_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int PER = 8, TILE = 1024 * PER;
  if (tid == 0) carry_s = 0;
  __syncthreads();
  for (int base = 1; base <= n; base += TILE) {
    unsigned long long e[PER];
    int acc = 0;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int j = base + tid * PER + u;
      e[u] = j <= n ? row[j] : 0ull;
      acc += (int)(unsigned)e[u];
    }
    int x = acc;  // inclusive scan of the per-thread totals
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int w = wsum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      wsum[lane] = w;
    }
    __syncthreads();
    int run = carry_s + (warp ? wsum[warp - 1] : 0) + x - acc;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int j = base + tid * PER + u;
      run += (int)(unsigned)e[u];
      if (j <= n) row[j] = (e[u] & 0xffffffff00000000ull) | (unsigned)run;
    }
    __syncthreads();
    if (tid == 1023) carry_s = run;
    __syncthreads();
  }
}

__global__ void k_finish_score(const int* hm, long long gmn, long long* out, int m_or_n_zero) {
  *out = (m_or_n_zero ? 0 : (long long)*hm) + gmn;
}
}  // namespace nwk

namespace {

nw_status pair_core(nw_ctx* c, const uint8_t* ca, long long m, const uint8_t* cb, long long n,
                    const nw_scoring* sc, long long* d_score, nw_tb* tb, int kr,
                    unsigned long long* ckpt, int ck_every, long long ck_stride,
                    const unsigned long long* top_row, unsigned top_tag, int h16_reb) {
  const int R = 32 * kr;
  const int nstrips = (int)((m + R - 1) / R);
  const bool dirs = tb != nullptr;
  nw_status st = NW_OK;
  int* ticket = c->d_ints;
  int* errf = c->d_err;
  int* hm = c->d_ints + 2;
  const long long gmn = (long long)sc->gap * (m + n);
  if (m > 0 && n > 0) {
    FillArgs A;
    A.a = ca; A.b = cb; A.prof = c->d_prof; A.K = sc->K;
    A.m = (int)m; A.n = (int)n; A.nstrips = nstrips; A.nslots = 2;
    A.bnd = c->d_bnd; A.bstride = bnd_stride(n); A.ticket = ticket;
    A.dirs = dirs ? tb->dirs : nullptr;
    A.wpl = dirs ? tb->wpl : 0;
    A.hm = hm; A.err = errf;
    A.poll_ns = (unsigned)std::max(0LL, std::min(c->opt[NW_OPT_POLL_NS], 100000LL));
    A.ckpt = ckpt; A.ck_every = ck_every; A.ck_stride = ck_stride;
    A.top_row = top_row; A.top_tag = top_tag;
    if (c->opt[NW_OPT_WATCHDOG_POLLS] > 0) A.watchdog = c->opt[NW_OPT_WATCHDOG_POLLS];
    const long long wh = c->opt[NW_OPT_TEST_WITHHOLD];
    if (wh > 0 && wh <= nstrips && c->bnd_cap >= sizeof(unsigned long long) * 3 * (size_t)bnd_stride(n)) {
      A.withhold = (int)wh;  // test hook: that strip's bottom row goes to the ring's third slot
      A.sink = c->d_bnd + 2 * bnd_stride(n);
    }
    const bool profreg = sc->K <= 4;
    const size_t smem = profreg ? 0 : (size_t)sc->K * R;
    const bool h16 = h16_reb > 0 && !(dirs && ckpt);  // with dirs: KR 4 or 8 (the caller checks)
    const bool d16 = !dirs && (kr >= 12 || (!ckpt && c->opt[NW_OPT_D16_FORCE] && d16_ok(c, sc)));
    if (h16) {  // 4 shifted copies of the selector table over cb[-PAD, n + PAD) (FillArgs::sel4)
      const long long ls = (n + 2 * PAD + 7) & ~7LL;
      st = grow(c, c->d_sel16, c->sel16_cap, sizeof(uint16_t) * 4 * (size_t)ls);
      if (st) return st;
      const int blocks = (int)std::min<long long>((4 * ls + 255) / 256, (long long)c->sm_count * 8);
      k_sel16x4<<<std::max(blocks, 1), 256, 0, c->stream>>>(cb, n, c->d_sel16, ls);
      LAUNCHED(c);
      A.sel4 = c->d_sel16 + PAD;
      A.sel4_stride = ls;
      A.reb_groups = h16_reb;
#ifdef NW_TRACE
      A.trace = nw_trace_buffer(nstrips);
#endif
    }
#ifdef NW_TRACE
    if (!h16) A.trace = nw_trace_buffer(nstrips);
#endif
    if (!h16 && profreg && kr <= 4) {  // 8 shifted copies of the per-column selectors (FillArgs::sel8)
      const long long ls = (n + 2 * PAD + 15) & ~7LL;
      st = grow(c, c->d_sel16, c->sel16_cap, sizeof(uint16_t) * 8 * (size_t)ls);
      if (st) return st;
      const int blocks = (int)std::min<long long>((8 * ls + 255) / 256, (long long)c->sm_count * 8);
      k_sel8x8<<<std::max(blocks, 1), 256, 0, c->stream>>>(cb, n, c->d_sel16, ls);
      LAUNCHED(c);
      A.sel8 = c->d_sel16 + PAD;
      A.sel8_stride = ls;
    }
    // persistent grid: one warp per CTA, at most the resident capacity
    int per_sm = 16;
    int grid = std::min<long long>(nstrips, (long long)c->sm_count * per_sm);
    const int pi = dirs ? pi_code(sc->tie) : 123;
    bool ok;
    {
      KernelTimer kt(c, 0);
      if (h16 && dirs) {
        ok = true;
        switch (pi) {
          case 123: launch_fill_dirs_h16<123>(A, kr, grid, c->stream); break;
          case 132: launch_fill_dirs_h16<132>(A, kr, grid, c->stream); break;
          case 213: launch_fill_dirs_h16<213>(A, kr, grid, c->stream); break;
          case 231: launch_fill_dirs_h16<231>(A, kr, grid, c->stream); break;
          case 312: launch_fill_dirs_h16<312>(A, kr, grid, c->stream); break;
          case 321: launch_fill_dirs_h16<321>(A, kr, grid, c->stream); break;
          default: ok = false;
        }
      } else if (h16) ok = dispatch_fill_h16(kr, A, grid, c->stream);
      else
        ok = dispatch_fill(dirs, pi, kr, profreg, A, grid, smem, c->stream, d16,
                           c->opt[NW_OPT_D16_CHAINS] == 2 && !ckpt);
    }
    if (!ok) return fail(c, NW_E_INVAL, "bad tie order");
    LAUNCHED(c);
    CUDA_TRY(c, cudaGetLastError());
  }
  k_finish_score<<<1, 1, 0, c->stream>>>(hm, gmn, d_score, (m == 0 || n == 0) ? 1 : 0);
  LAUNCHED(c);
  CUDA_TRY(c, cudaGetLastError());
  return NW_OK;
}

// Reads (and clears) the sticky device error flags: the first bad residue
// position (atomicMin over every call since the last check) and the watchdog
// flag. A _dev call's error therefore surfaces at the next synchronising call on
// the context, even when other calls were enqueued in between.
nw_status check_deferred(nw_ctx* c) {
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  long long flags[2] = {0, 0};
  CUDA_TRY(c, cudaMemcpy(flags, c->d_bad, sizeof flags, cudaMemcpyDeviceToHost));
  const long long bad = flags[0];
  const int errf = (int)(flags[1] & 0xffffffff);
  if (bad != 0x7fffffffffffffffll || errf) {
    const long long clear[2] = {0x7fffffffffffffffll, 0};
    CUDA_TRY(c, cudaMemcpy(c->d_bad, clear, sizeof clear, cudaMemcpyHostToDevice));
  }
  if (bad != 0x7fffffffffffffffll) {
    c->bad_pos = bad;
    return fail(c, NW_E_ALPHABET, "residue at position %lld is not in the alphabet", bad);
  }
  if (errf) return fail(c, NW_E_DEADLOCK, "inter-warp dependency watchdog fired");
  if (c->comm) {
    ncclResult_t ar = ncclSuccess;
    if (nwd::nccl().CommGetAsyncError(c->comm, &ar) != ncclSuccess || ar != ncclSuccess)
      return fail(c, NW_E_COMM, "NCCL communicator error: %s", nwd::nccl().GetErrorString(ar));
  }
  return NW_OK;
}


// Stage residues into device codes (PAD | a | pad to R + PAD), after k_init
// has zeroed the code buffer and the tagged boundary ring (pair_entry).
nw_status stage_pair(nw_ctx* c, const uint8_t* a, long long m, const uint8_t* b, long long n,
                     bool host, uint8_t** ca, uint8_t** cb) {
  constexpr long long R = R_MAX;
  const long long la = pad16(PAD + m + R + PAD);
  *ca = c->d_codes + PAD;
  *cb = c->d_codes + la + PAD;
  const uint8_t *ra = a, *rb = b;
  if (host) {
    nw_status st = grow(c, c->d_raw, c->raw_cap, (size_t)(m + n + 16));
    if (st) return st;
    if (m) CUDA_TRY(c, cudaMemcpyAsync(c->d_raw, a, (size_t)m, cudaMemcpyHostToDevice, c->stream));
    if (n) CUDA_TRY(c, cudaMemcpyAsync(c->d_raw + m, b, (size_t)n, cudaMemcpyHostToDevice, c->stream));
    ra = c->d_raw;
    rb = c->d_raw + m;
  }
  launch_encode(c, ra, m, *ca, 0);
  launch_encode(c, rb, n, *cb, m);
  CUDA_TRY(c, cudaGetLastError());
  return NW_OK;
}

nw_status new_tb(nw_ctx* c, long long m, long long n, const nw_scoring* sc, int kr, nw_tb** out) {
  const int R = 32 * kr;
  nw_tb* tb = new (std::nothrow) nw_tb;
  if (!tb) return fail(c, NW_E_NOMEM, "host allocation");
  memset(tb, 0, sizeof *tb);
  tb->ctx = c;
  c->live_tb.push_back(tb);
  tb->m = (int)m;
  tb->n = (int)n;
  tb->kr = kr;
  memcpy(tb->tie, sc->tie, 3);
  const long long S = std::max<long long>((m + R - 1) / R, 1);
  tb->S = (int)S;
  tb->wpl = (n + 31 + 7) / 8;
  tb->segstride = pad16(R + n + 1);
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t b_dirs = al((size_t)S * tb->wpl * kr * 32 * sizeof(uint16_t));
  tb->lstep = tb_lstep(c);
  tb->nb = tb_band(c, n, tb->lstep);
  const size_t b_spec = al((size_t)S * tb->nb * sizeof(int));
  const size_t b_cs = al((size_t)S * sizeof(int)), b_len = b_cs;
  const size_t b_seg = al((size_t)S * tb->segstride);
  const size_t bytes = b_dirs + b_spec + b_cs + b_len + b_seg;
  if (m > 0 && n > 0) {
    cudaError_t e = cudaMallocAsync(&tb->mem, bytes, c->stream);
    if (e != cudaSuccess) {
      c->live_tb.pop_back();
      delete tb;
      return fail(c, NW_E_NOMEM, "traceback buffers of %zu bytes: %s", bytes, cudaGetErrorString(e));
    }
    char* p = static_cast<char*>(tb->mem);
    tb->dirs = reinterpret_cast<uint16_t*>(p); p += b_dirs;
    tb->spec = reinterpret_cast<int*>(p); p += b_spec;
    tb->cs = reinterpret_cast<int*>(p); p += b_cs;
    tb->seglen = reinterpret_cast<int*>(p); p += b_len;
    tb->seg = reinterpret_cast<uint8_t*>(p);
  }
  *out = tb;
  return NW_OK;
}

nw_status pair_entry(nw_ctx* c, const uint8_t* a, long long m, const uint8_t* b, long long n,
                     const nw_scoring* sc, bool host, long long* score_out, nw_tb** tb_out,
                     bool want_dirs) {
  if (!c) return NW_E_INVAL;
  if ((m > 0 && !a) || (n > 0 && !b) || !score_out) return fail(c, NW_E_INVAL, "NULL argument");
  nw_status st = check_scoring(c, sc);
  if (st) return st;
  st = check_bounds(c, sc, m, n);
  if (st) return st;
  CUDA_TRY(c, cudaSetDevice(c->device));
  if (!want_dirs && cblock_dist_applies(c, m, n, sc)) {  // C5 across the ranks of a dist ctx
    long long* d_score = host ? c->d_score : score_out;
    st = cblock_dist(c, a, m, b, n, sc, host, d_score);
    if (st) return st;
    if (host) {
      CUDA_TRY(c, cudaMemcpyAsync(score_out, c->d_score, sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
      return check_deferred(c);
    }
    return NW_OK;
  }
  st = upload_tables(c, sc);
  if (st) return st;
  // workspace: padded code buffers and the tagged 2-slot boundary ring
  constexpr long long R = R_MAX;
  const long long la = pad16(PAD + m + R + PAD), lb = pad16(PAD + n + R + PAD);
  int kr = choose_kr(c, m, n, want_dirs, sc->K);
  // packed difference form (two rows per register) for tall score-only pairs: it
  // halves the ALU work per cell but doubles the lane skew, so it only pays when
  // there are enough 512-row strips to fill the GPU (measured: 1M^2 2.4 -> 5.9
  // TCUPS; 20k^2 1.44 -> 2.14 ms, slower)
  // and 28-32 rows per lane by the strip-count rule of d16_kr.
  if (!want_dirs && d16_ok(c, sc) && m >= 32LL * 16 * 150) kr = d16_kr(c, m);
  // NW_OPT_D16_FORCE = <4|8|12..32 even> runs any score-only pair in the packed form
  if (!want_dirs && d16_ok(c, sc) && c->opt[NW_OPT_D16_FORCE]) {
    const int f = (int)std::max(4LL, std::min(c->opt[NW_OPT_D16_FORCE], 32LL));
    kr = (f >= 12 && f <= 32 && f % 2 == 0) ? f : (f >= 32 ? 32 : (f >= 16 ? 16 : (f >= 8 ? 8 : 4)));
  }
  // packed H' with a moving base: the default for tall score-only
  // pairs; NW_OPT_H16_KR forces it at any size (tests)
  int h16_reb = 0;
  const bool h16_tall = m >= 32LL * 16 * 150 && c->opt[NW_OPT_PAIR_FORM] != 1 && !c->opt[NW_OPT_D16_FORCE];
  if (!want_dirs && d16_ok(c, sc) && (h16_tall || c->opt[NW_OPT_H16_KR])) {
    const int kh = h16_kr(c, m);
    h16_reb = h16_rebase_groups(c, sc, kh);
    if (h16_reb > 0) kr = kh;
  }
  // with directions, NW_OPT_PAIR_FORM = 2: the packed H' fill writing the int32 sweep's
  // decision layout at the same rows per lane (4 or 8), so the strip traceback is
  // unchanged (C2: 1.88 vs 1.59 ms for the int32 fill, not the default)
  if (want_dirs && d16_ok(c, sc) && (kr == 4 || kr == 8) && c->opt[NW_OPT_PAIR_FORM] == 2)
    h16_reb = h16_rebase_groups(c, sc, kr);
  // tall direction fills (8+ rows per lane) with long rows take it by default: at 8 rows per
  // lane the four packed registers amortise the per-step overhead (~20% faster steps) but
  // the lane skew doubles, so the rows must be long against the strips' start lag:
  // n >= 128 x strips (checkpointed refills, 1M columns: 501 -> 411 ms; 100k x 3k: slower)
  if (want_dirs && d16_ok(c, sc) && kr >= 8 && c->opt[NW_OPT_PAIR_FORM] == 0 &&
      !c->opt[NW_OPT_ROWS_PER_LANE] && n >= 128 * ((m + 255) / 256)) {
    const int rb = h16_rebase_groups(c, sc, 8);
    if (rb > 0) { h16_reb = rb; kr = 8; }
  }
  st = grow(c, c->d_codes, c->codes_cap, (size_t)(la + lb));
  if (st) return st;
  // two ring slots (+ a sink slot for the NW_OPT_TEST_WITHHOLD hook)
  const long long bbytes = (long long)sizeof(unsigned long long) * (c->opt[NW_OPT_TEST_WITHHOLD] ? 3 : 2) *
                           bnd_stride(n);
  st = grow(c, c->d_bnd, c->bnd_cap, (size_t)bbytes);
  if (st) return st;
  // one launch zeroes ticket/err/hm, the bad-position flag, the code
  // buffers (their padding must hold valid codes) and the boundary ring (tags)
  ZeroRanges zr{{c->d_codes, c->d_bnd, nullptr, nullptr}, {la + lb, bbytes, 0, 0}};
  st = init_small(c, 8, zr);  // [0] ticket [1] err [2] hm [5] slow traceback strips
  if (st) return st;
  uint8_t *ca, *cb;
  st = stage_pair(c, a, m, b, n, host, &ca, &cb);
  if (st) return st;
  nw_tb* tb = nullptr;
  if (want_dirs) {
    st = new_tb(c, m, n, sc, kr, &tb);
    if (st) return st;
  }
  long long* d_score = host ? c->d_score : score_out;
  st = pair_core(c, ca, m, cb, n, sc, d_score, tb, kr, nullptr, 0, 0, nullptr, 0, h16_reb);
  if (st) {
    if (tb) nw_tb_free(tb);
    return st;
  }
  if (host) {
    CUDA_TRY(c, cudaMemcpyAsync(score_out, c->d_score, sizeof(long long), cudaMemcpyDeviceToHost,
                                c->stream));
    st = check_deferred(c);
    if (st) {
      if (tb) nw_tb_free(tb);
      return st;
    }
  }
  if (tb_out) *tb_out = tb;
  else if (tb) nw_tb_free(tb);
  return NW_OK;
}

}  // namespace

// ======================= exported C ABI =======================

extern "C" {

#ifdef NW_TRACE
int nw_debug_trace(unsigned long long* out, int max_strips) {
  const int k = std::min(max_strips, g_trace_strips);
  if (g_trace && k > 0) cudaMemcpy(out, g_trace, sizeof(unsigned long long) * 256 * k, cudaMemcpyDeviceToHost);
  return k;
}
#endif

const char* nw_strerror(nw_status st) {
  switch (st) {
    case NW_OK: return "ok";
    case NW_E_INVAL: return "invalid argument";
    case NW_E_ALPHABET: return "residue not in alphabet";
    case NW_E_OVERFLOW: return "input too large for int32 scores";
    case NW_E_NOMEM: return "out of memory";
    case NW_E_CUDA: return "CUDA error";
    case NW_E_TRUNC: return "ops buffer too small";
    case NW_E_STATE: return "traceback handle not valid for this context";
    case NW_E_DEADLOCK: return "dependency watchdog fired";
    case NW_E_COMM: return "communication error";
  }
  return "unknown status";
}

nw_status nw_ctx_create(int device, void* cuda_stream, nw_ctx** out) {
  if (!out) return NW_E_INVAL;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return NW_E_CUDA;
  if (device < 0 || device >= ndev) return NW_E_INVAL;
  nw_ctx* c = new (std::nothrow) nw_ctx;
  if (!c) return NW_E_NOMEM;
  c->device = device;
  c->stream = (cudaStream_t)cuda_stream;
  if (cudaSetDevice(device) != cudaSuccess ||
      cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) {
    delete c;
    return NW_E_CUDA;
  }
  if (cudaMalloc(&c->d_lut, 256) != cudaSuccess || cudaMalloc(&c->d_prof, 64 * 64) != cudaSuccess ||
      cudaMalloc(&c->d_bad, 4 * sizeof(long long)) != cudaSuccess ||
      cudaMalloc(&c->d_len, sizeof(long long)) != cudaSuccess ||
      cudaMalloc(&c->d_score, sizeof(long long)) != cudaSuccess) {
    nw_ctx_destroy(c);
    return NW_E_NOMEM;
  }
  const long long init_flags[4] = {0x7fffffffffffffffll, 0, 0, 0};
  cudaMemcpy(c->d_bad, init_flags, sizeof init_flags, cudaMemcpyHostToDevice);
  c->d_err = reinterpret_cast<int*>(c->d_bad + 1);
  // keep freed stream-ordered allocations in the pool (steady-state calls allocate nothing new)
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  *out = c;
  return NW_OK;
}

void nw_ctx_destroy(nw_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (nw_tb* tb : c->live_tb) {  // detach: a later nw_tb_free only deletes the host struct
    if (tb->mem) cudaFreeAsync(tb->mem, c->stream);
    tb->mem = nullptr;
    tb->ctx = nullptr;
  }
  for (nw_msa* h : c->live_msa) {
    if (h->d_rows) cudaFreeAsync(h->d_rows, c->stream);
    h->d_rows = nullptr;
    h->ctx = nullptr;
  }
  cudaFree(c->d_lut);
  cudaFree(c->d_prof);
  cudaFree(c->d_bad);
  cudaFree(c->d_len);
  cudaFree(c->d_score);
  if (c->d_ints) cudaFreeAsync(c->d_ints, c->stream);
  if (c->d_codes) cudaFreeAsync(c->d_codes, c->stream);
  if (c->d_raw) cudaFreeAsync(c->d_raw, c->stream);
  if (c->d_bnd) cudaFreeAsync(c->d_bnd, c->stream);
  if (c->d_rev) cudaFreeAsync(c->d_rev, c->stream);
  if (c->d_scratch) cudaFreeAsync(c->d_scratch, c->stream);
  if (c->d_sel16) cudaFreeAsync(c->d_sel16, c->stream);
  if (c->d_aux) cudaFreeAsync(c->d_aux, c->stream);
  if (c->d_plan) cudaFreeAsync(c->d_plan, c->stream);
  if (c->stage_ev) { cudaEventSynchronize(c->stage_ev); cudaEventDestroy(c->stage_ev); }
  if (c->h_stage) cudaFreeHost(c->h_stage);
  if (c->d_tbdirs) cudaFreeAsync(c->d_tbdirs, c->stream);
  if (c->d_rs) cudaFreeAsync(c->d_rs, c->stream);
  if (c->d_cb_tab) cudaFreeAsync(c->d_cb_tab, c->stream);
  cudaStreamSynchronize(c->stream);
  if (c->cb_next) cudaIpcCloseMemHandle(c->cb_next);
  if (c->d_cb_ring) cudaFree(c->d_cb_ring);
  if (c->d_cb_recv) cudaFree(c->d_cb_recv);
  if (c->d_cb_vrecv) cudaFree(c->d_cb_vrecv);
  if (c->d_pmat) cudaFreeAsync(c->d_pmat, c->stream);
  if (c->d_tdoff) cudaFreeAsync(c->d_tdoff, c->stream);
  cudaStreamSynchronize(c->stream);
  for (auto& v : c->ev_open)
    for (auto& pr : v) { cudaEventDestroy(pr.first); cudaEventDestroy(pr.second); }
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  if (c->comm) nwd::nccl().CommDestroy(c->comm);
  delete c;
}

const char* nw_last_error(const nw_ctx* c) { return c ? c->err : "no context"; }
int64_t nw_last_bad_pos(const nw_ctx* c) { return c ? c->bad_pos : -1; }
int64_t nw_ctx_launches(const nw_ctx* c) { return c ? c->launches : 0; }

nw_status nw_ctx_set_timing(nw_ctx* c, int enable) {
  if (!c) return NW_E_INVAL;
  c->timing = enable != 0;
  return NW_OK;
}

nw_status nw_ctx_kernel_time(nw_ctx* c, int cls, double* total_ms, int64_t* launches) {
  if (!c || cls < 0 || cls > 1 || !total_ms || !launches) return NW_E_INVAL;
  CUDA_TRY(c, cudaSetDevice(c->device));
  double tot = 0;
  for (auto& pr : c->ev_open[cls]) {
    CUDA_TRY(c, cudaEventSynchronize(pr.second));
    float ms = 0;
    CUDA_TRY(c, cudaEventElapsedTime(&ms, pr.first, pr.second));
    tot += ms;
    c->ev_pool.push_back(pr.first);
    c->ev_pool.push_back(pr.second);
  }
  *launches = (int64_t)c->ev_open[cls].size();
  c->ev_open[cls].clear();
  *total_ms = tot;
  return NW_OK;
}

nw_status nw_dist_unique_id(uint8_t* id) {
  if (!id) return NW_E_INVAL;
  const nwd::NcclApi& api = nwd::nccl();
  if (!api.ok) return NW_E_COMM;
  ncclUniqueId u;
  if (api.GetUniqueId(&u) != ncclSuccess) return NW_E_COMM;
  memcpy(id, &u, sizeof u);
  return NW_OK;
}

nw_status nw_ctx_set_dist(nw_ctx* c, int32_t rank, int32_t world, const uint8_t* id) {
  if (!c) return NW_E_INVAL;
  if (world < 1 || rank < 0 || rank >= world || !id)
    return fail(c, NW_E_INVAL, "rank %d / world %d / id", rank, world);
  const nwd::NcclApi& api = nwd::nccl();
  if (!api.ok) return fail(c, NW_E_COMM, "%s", api.why);
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (c->comm) {
    api.CommDestroy(c->comm);
    c->comm = nullptr;
  }
  ncclUniqueId u;
  memcpy(&u, id, sizeof u);
  ncclComm_t comm = nullptr;
  const ncclResult_t r = api.CommInitRank(&comm, world, u, rank);
  if (r != ncclSuccess) return fail(c, NW_E_COMM, "ncclCommInitRank: %s", api.GetErrorString(r));
  c->comm = comm;
  c->rank = rank;
  c->world = world;
  // a new group: the column-block buffers, their peer mapping and the tag counter start
  // afresh (identically on every rank), so stale entries of earlier calls can never match
  if (c->cb_next) cudaIpcCloseMemHandle(c->cb_next);
  c->cb_next = nullptr;
  if (c->d_cb_recv) cudaFree(c->d_cb_recv);
  c->d_cb_recv = nullptr;
  c->cb_recv_cap = 0;
  if (c->d_cb_ring) cudaFree(c->d_cb_ring);
  c->d_cb_ring = nullptr;
  c->cb_ring_cap = 0;
  if (c->d_cb_vrecv) cudaFree(c->d_cb_vrecv);
  c->d_cb_vrecv = nullptr;
  c->cb_vrecv_cap = 0;
  c->cb_tag_next = 1;
  return NW_OK;
}

nw_status nw_ctx_dist_info(const nw_ctx* c, int32_t* rank, int32_t* world) {
  if (!c || !rank || !world) return NW_E_INVAL;
  *rank = c->rank;
  *world = c->comm ? c->world : 1;
  return NW_OK;
}

nw_status nw_batch_partition(const int64_t* offs, int32_t nseq, const int32_t* pairs, int64_t npairs,
                             int32_t world, int64_t* bounds) {
  if (!offs || !bounds || nseq < 0 || npairs < 0 || world < 1) return NW_E_INVAL;
  if (!pairs && npairs != (int64_t)nseq * (nseq - 1) / 2) return NW_E_INVAL;
  for (int64_t k = 0; pairs && k < 2 * npairs; ++k)
    if (pairs[k] < 0 || pairs[k] >= nseq) return NW_E_INVAL;
  nwd::partition_bounds(reinterpret_cast<const long long*>(offs), nseq, pairs, npairs, world,
                        reinterpret_cast<long long*>(bounds));
  return NW_OK;
}

nw_status nw_ctx_set_option(nw_ctx* c, int32_t option, int64_t value) {
  if (!c) return NW_E_INVAL;
  if (option < 0 || option >= NW_OPT_COUNT_) return fail(c, NW_E_INVAL, "unknown option %d", option);
  if (value < 0) return fail(c, NW_E_INVAL, "option %d: negative value", option);
  c->opt[option] = value;
  return NW_OK;
}

int64_t nw_ctx_get_option(const nw_ctx* c, int32_t option) {
  return (c && option >= 0 && option < NW_OPT_COUNT_) ? c->opt[option] : -1;
}

nw_status nw_ctx_sync(nw_ctx* c) {
  if (!c) return NW_E_INVAL;
  CUDA_TRY(c, cudaSetDevice(c->device));
  return check_deferred(c);
}

nw_status nw_score_only(nw_ctx* c, const uint8_t* a, int64_t m, const uint8_t* b, int64_t n,
                        const nw_scoring* sc, int64_t* score) {
  return pair_entry(c, a, m, b, n, sc, true, reinterpret_cast<long long*>(score), nullptr, false);
}

nw_status nw_score_only_dev(nw_ctx* c, const uint8_t* d_a, int64_t m, const uint8_t* d_b,
                            int64_t n, const nw_scoring* sc, int64_t* d_score) {
  return pair_entry(c, d_a, m, d_b, n, sc, false, reinterpret_cast<long long*>(d_score), nullptr,
                    false);
}

nw_status nw_align_pair(nw_ctx* c, const uint8_t* a, int64_t m, const uint8_t* b, int64_t n,
                        const nw_scoring* sc, int64_t* score, nw_tb** tb) {
  return pair_entry(c, a, m, b, n, sc, true, reinterpret_cast<long long*>(score), tb, true);
}

nw_status nw_align_pair_dev(nw_ctx* c, const uint8_t* d_a, int64_t m, const uint8_t* d_b,
                            int64_t n, const nw_scoring* sc, int64_t* d_score, nw_tb** tb) {
  return pair_entry(c, d_a, m, d_b, n, sc, false, reinterpret_cast<long long*>(d_score), tb, true);
}

void nw_tb_free(nw_tb* tb) {
  if (!tb) return;
  if (nw_ctx* c = tb->ctx) {
    if (tb->mem) cudaFreeAsync(tb->mem, c->stream);
    auto& v = c->live_tb;
    v.erase(std::remove(v.begin(), v.end(), tb), v.end());
  }
  delete tb;
}

// pad_top = false, exit_col: stop at row 0 (the top of a checkpoint segment,
// DESIGN.md §3.12) instead of walking the border, and report the column reached.
static nw_status traceback_core(nw_ctx* c, const nw_tb* tb, uint8_t* d_ops, bool pad_top = true,
                                int* exit_col = nullptr) {
  const long long L = (long long)tb->m + tb->n;
  nw_status st = grow(c, c->d_rev, c->rev_cap, (size_t)std::max<long long>(L, 1));
  if (st) return st;
  (void)L;
  {
    KernelTimer kt(c, 1);
    const int S = tb->S;
    // strip entries: sampled exit walks in a band around the diagonal (in
    // parallel), then the bottom-up chain over the brackets
    const int kr = tb->kr, R = 32 * kr;
    nwk::TbBand B;
    B.m = tb->m; B.n = tb->n; B.lstep = tb->lstep; B.step = 1 << B.lstep; B.nb = tb->nb;
    B.ratio = (float)tb->n / (float)tb->m;
    B.nq = (tb->n + B.step - 1) / B.step + 1;
    const int left_cols = R + 128;  // > one strip's drift on a near-diagonal path
    const int gw_bytes = (kr * 16 + 1) * 4;
    if (S >= 2) {
      auto kspec = kr == 2 ? k_tb_spec<2> : kr == 4 ? k_tb_spec<4> : kr == 5 ? k_tb_spec<5>
                 : kr == 6 ? k_tb_spec<6> : kr == 10 ? k_tb_spec<10> : kr == 12 ? k_tb_spec<12> : k_tb_spec<8>;
      const size_t win = (size_t)((32 * B.step + left_cols + 40) / 8 + 2) * gw_bytes;
      cudaFuncSetAttribute(kspec, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)win);
      kspec<<<(S - 1) * (B.nb / 32), 32, win, c->stream>>>(tb->dirs, tb->wpl, B, tb->tie[0],
                                                          tb->tie[1], tb->tie[2], tb->spec, left_cols);
      LAUNCHED(c);
    }
    {
      auto kchain = kr == 2 ? k_tb_chain<2> : kr == 4 ? k_tb_chain<4> : kr == 5 ? k_tb_chain<5>
                  : kr == 6 ? k_tb_chain<6> : kr == 10 ? k_tb_chain<10> : kr == 12 ? k_tb_chain<12> : k_tb_chain<8>;
      // exact walks: windows of ~96 KB of decision bits left of the entry
      // a window of 2R + 256 columns left of the entry (re-staged further left
      // when a long gap leaves it): staging, not the walk, dominated at 96 KB
      const int left_exact = 2 * R + 256;
      const int win_groups = left_exact / 8 + 6;
      const int CH = std::max(1, std::min(S, (int)(64 * 1024 / (B.nb * 4))));
      const size_t smem = (size_t)CH * B.nb * 4 + (size_t)win_groups * gw_bytes;
      cudaFuncSetAttribute(kchain, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      kchain<<<1, 1024, smem, c->stream>>>(tb->dirs, tb->wpl, B, S, tb->tie[0], tb->tie[1],
                                           tb->tie[2], tb->spec, tb->cs, c->d_ints + 5, CH,
                                           left_exact);
      LAUNCHED(c);
    }
    const int smem_bytes = 96 * 1024;
    auto kseg = kr == 2 ? k_tb_segments<2> : kr == 4 ? k_tb_segments<4> : kr == 5 ? k_tb_segments<5>
              : kr == 6 ? k_tb_segments<6> : kr == 10 ? k_tb_segments<10> : kr == 12 ? k_tb_segments<12>
              : k_tb_segments<8>;
    cudaFuncSetAttribute(kseg, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    kseg<<<S, 32, smem_bytes, c->stream>>>(tb->dirs, tb->wpl, tb->m, tb->n, tb->tie[0],
                                           tb->tie[1], tb->tie[2], tb->cs, tb->seg, tb->segstride,
                                           tb->seglen, smem_bytes / 2, pad_top ? 1 : 0, exit_col);
    LAUNCHED(c);
    k_tb_assemble<<<S, 256, 0, c->stream>>>(tb->seg, tb->segstride, tb->seglen, d_ops, c->d_len);
    LAUNCHED(c);
  }
  CUDA_TRY(c, cudaGetLastError());
  return NW_OK;
}

nw_status nw_traceback(nw_ctx* c, const nw_tb* tb, uint8_t* ops, int64_t cap, int64_t* len) {
  if (!c || !tb || !len) return c ? fail(c, NW_E_INVAL, "NULL argument") : NW_E_INVAL;
  if (tb->ctx != c) return fail(c, NW_E_STATE, "traceback handle belongs to another context");
  CUDA_TRY(c, cudaSetDevice(c->device));
  const long long L = (long long)tb->m + tb->n;
  if (tb->m == 0 || tb->n == 0) {
    *len = L;
    if (cap < L) return fail(c, NW_E_TRUNC, "cap %lld < length %lld", (long long)cap, L);
    for (long long k = 0; k < L; ++k) ops[k] = tb->m > 0 ? NW_UP : NW_LEFT;
    return NW_OK;
  }
  uint8_t* d_ops = nullptr;
  CUDA_TRY(c, cudaMallocAsync(reinterpret_cast<void**>(&d_ops), (size_t)L, c->stream));
  nw_status st = traceback_core(c, tb, d_ops);
  if (st) { cudaFreeAsync(d_ops, c->stream); return st; }
  long long hl = 0;
  CUDA_TRY(c, cudaMemcpyAsync(&hl, c->d_len, sizeof hl, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  *len = hl;
  if (cap < hl) {
    cudaFreeAsync(d_ops, c->stream);
    return fail(c, NW_E_TRUNC, "cap %lld < length %lld", (long long)cap, hl);
  }
  CUDA_TRY(c, cudaMemcpyAsync(ops, d_ops, (size_t)hl, cudaMemcpyDeviceToHost, c->stream));
  cudaFreeAsync(d_ops, c->stream);
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return NW_OK;
}

nw_status nw_traceback_dev(nw_ctx* c, const nw_tb* tb, uint8_t* d_ops, int64_t cap, int64_t* d_len) {
  if (!c || !tb || !d_ops || !d_len) return c ? fail(c, NW_E_INVAL, "NULL argument") : NW_E_INVAL;
  if (tb->ctx != c) return fail(c, NW_E_STATE, "traceback handle belongs to another context");
  const long long L = (long long)tb->m + tb->n;
  if (cap < L) return fail(c, NW_E_INVAL, "cap %lld < m+n = %lld", (long long)cap, L);
  CUDA_TRY(c, cudaSetDevice(c->device));
  if (tb->m == 0 || tb->n == 0) {
    if (L) CUDA_TRY(c, cudaMemsetAsync(d_ops, tb->m > 0 ? NW_UP : NW_LEFT, (size_t)L, c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(d_len, &L, sizeof L, cudaMemcpyHostToDevice, c->stream));
    return NW_OK;
  }
  nw_status st = traceback_core(c, tb, d_ops);
  if (st) return st;
  CUDA_TRY(c, cudaMemcpyAsync(d_len, c->d_len, sizeof(long long), cudaMemcpyDeviceToDevice,
                              c->stream));
  return NW_OK;
}

}  // extern "C"

namespace {

// ---- column-block wavefront (a10) ----
// Geometry of one column-block call: arithmetic form, strip height, blocks, messages.
struct CbGeom {
  bool d16;             // packed difference form (s - 2g >= 0), else int32 H'
  bool h16;             // packed H' with a moving base: preferred over d16
  int reb;              // h16: rebase period (8-step groups)
  int KR, R, S, W, nblocks;
  long long mstride;    // entries per left-column message: R (d16) or R + 1 (int32)
  long long rstride;    // entries per receive slot: S * mstride
  size_t recv_bytes;    // one rank's receive buffer: 2 slots
};

constexpr int CB_KR32 = 8;

// Receive-buffer bound for any form and strip height (m rows in strips of >= 256 rows,
// <= R + 1 entries per strip, two slots).
long long cb_recv_bound(long long m) { return 16LL * (m + m / 256 + 1 + 1025); }

CbGeom cb_geom(const nw_ctx* c, long long m, long long n, const nw_scoring* sc, int G, int block_cols) {
  CbGeom g;
  g.d16 = d16_ok(c, sc);
  g.KR = g.d16 ? d16_kr(c, std::max(m, 1LL)) : CB_KR32;
  g.reb = (g.d16 && c->opt[NW_OPT_PAIR_FORM] != 1) ? h16_rebase_groups(c, sc, g.KR) : 0;
  g.h16 = g.reb > 0;
  if (g.h16) g.d16 = false;
  g.R = 32 * g.KR;
  g.S = (int)std::max<long long>((m + g.R - 1) / g.R, 1);
  if (block_cols > 0) g.W = block_cols;
  else if (G == 1) g.W = (int)std::max<long long>(n, 1);
  else g.W = (int)std::max<long long>(1024, ((n + 32LL * G - 1) / (32LL * G) + 1) & ~1LL);  // ~32 rounds, even
  g.nblocks = (int)std::max<long long>((n + g.W - 1) / g.W, 1);
  g.mstride = g.d16 ? g.R : g.R + 1;  // h16 and int32: corner + R rows
  g.rstride = (long long)g.S * g.mstride;
  g.recv_bytes = sizeof(unsigned long long) * 2 * (size_t)g.rstride;
  return g;
}

// Buffers the column-block kernels poll carry per-call tags (nw_cblock.cuh): they are
// zeroed once, when allocated. cudaMalloc (not the stream pool): the receive buffer of
// a real rank is exported through CUDA IPC.
nw_status grow_zeroed(nw_ctx* c, void*& p, size_t& cap, size_t need) {
  if (need <= cap && p) return NW_OK;
  if (p) {
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    cudaFree(p);
    p = nullptr;
    cap = 0;
  }
  const size_t bytes = std::max<size_t>(need, 256);
  CUDA_TRY(c, cudaMalloc(&p, bytes));
  CUDA_TRY(c, cudaMemsetAsync(p, 0, bytes, c->stream));
  cap = bytes;
  return NW_OK;
}

// Tags of one call: [base, base + nblocks*S + 1). A per-context counter, identical on
// every rank that makes the same sequence of calls; wrapping (after ~2^32 / (nblocks*S)
// calls) re-zeroes this context's buffers (rank callers must then re-synchronise).
unsigned cb_tags(nw_ctx* c, const CbGeom& g, bool* wrapped) {
  const unsigned long long span = (unsigned long long)g.nblocks * g.S + 2;
  *wrapped = (unsigned long long)c->cb_tag_next + span >= 0xffffffffull;
  if (*wrapped) c->cb_tag_next = 1;
  const unsigned base = c->cb_tag_next;
  c->cb_tag_next += (unsigned)span;
  return base;
}

// Shared body: ranks [rank0, rank0 + nhere) run in this launch; recv_tab (device, G
// entries) points at every rank's receive buffer (virtual ranks: all local; a real rank:
// its own and the next rank's). d_score receives this launch's H(m,n) share.
nw_status cblock_core(nw_ctx* c, const uint8_t* ca, long long m, const uint8_t* cb, long long n,
                      const nw_scoring* sc, const CbGeom& g, int G, int rank0, int nhere,
                      unsigned long long* const* recv_tab, long long* d_score, bool owner_adds_gap,
                      bool sys, unsigned tag_base) {
  const long long bstride = bnd_stride(n);
  nw_status st = grow_zeroed(c, c->d_cb_ring, c->cb_ring_cap, sizeof(unsigned long long) * (size_t)nhere * 2 * bstride);
  if (st) return st;
  st = init_small(c, 4 + nhere);  // [2] hm, [4..] tickets
  if (st) return st;
  const int last_owner = (g.nblocks - 1) % G;
  if (m > 0 && n > 0) {
    CBlockArgs A;
    A.a = ca; A.b = cb; A.prof = c->d_prof; A.K = sc->K; A.m = (int)m; A.n = (int)n;
    A.W = g.W; A.G = G; A.S = g.S; A.nblocks = g.nblocks;
    A.bnd = static_cast<unsigned long long*>(c->d_cb_ring);
    A.bstride = bstride;
    A.recv_tab = recv_tab;
    A.rstride = g.rstride;
    A.mstride = g.mstride;
    A.tag_base = tag_base;
    A.ticket = c->d_ints + 4;
    A.hm = c->d_ints + 2;
    A.err = c->d_err;
    A.watchdog = c->opt[NW_OPT_WATCHDOG_POLLS] > 0 ? c->opt[NW_OPT_WATCHDOG_POLLS] : (1LL << 28);
    A.rank0 = rank0;
    A.nranks_here = nhere;
    A.sel = nullptr;
    A.reb_groups = g.reb;
    if (g.h16) {  // selector table over cb[-PAD, n + PAD) (nw_fill16.cuh)
      const long long ls = n + 2 * PAD;
      st = grow(c, c->d_sel16, c->sel16_cap, sizeof(uint16_t) * (size_t)ls);
      if (st) return st;
      const int blocks = (int)std::min<long long>((ls - 1 + 255) / 256, (long long)c->sm_count * 8);
      k_sel16<<<std::max(blocks, 1), 256, 0, c->stream>>>(cb - PAD + 1, ls - 1, c->d_sel16 + 1);
      LAUNCHED(c);
      A.sel = c->d_sel16 + PAD;
    }
    // every rank's warps must be resident together (they wait on each other);
    // NW_OPT_CBLOCK_WARPS_PER_SM caps this launch's share of the GPU
    int per_sm = 8;
    if (c->opt[NW_OPT_CBLOCK_WARPS_PER_SM] > 0) per_sm = (int)std::min(c->opt[NW_OPT_CBLOCK_WARPS_PER_SM], 16LL);
    const long long want = (long long)g.S * nhere;
    const int grid = (int)std::min<long long>((long long)c->sm_count * per_sm, want);
    const int grid_r = std::max(nhere, grid - grid % nhere);
    {
      KernelTimer kt(c, 0);
      if (g.h16) {
        switch (g.KR) {
#define NW_CB_CASE(K)                                                                 \
  case K:                                                                             \
    if (sys) k_fill_cblock_h16<K, true><<<grid_r, 32, 0, c->stream>>>(A);            \
    else k_fill_cblock_h16<K, false><<<grid_r, 32, 0, c->stream>>>(A);               \
    break;
          NW_CB_CASE(16) NW_CB_CASE(18) NW_CB_CASE(20) NW_CB_CASE(22) NW_CB_CASE(24)
          NW_CB_CASE(26) NW_CB_CASE(28) NW_CB_CASE(30) NW_CB_CASE(32)
#undef NW_CB_CASE
          default: return fail(c, NW_E_INVAL, "column-block rows per lane %d", g.KR);
        }
      } else if (g.d16) {
        switch (g.KR) {
#define NW_CB_CASE(K)                                                                 \
  case K:                                                                             \
    if (sys) k_fill_cblock_d16<K, true><<<grid_r, 32, 0, c->stream>>>(A);            \
    else k_fill_cblock_d16<K, false><<<grid_r, 32, 0, c->stream>>>(A);               \
    break;
          NW_CB_CASE(16) NW_CB_CASE(18) NW_CB_CASE(20) NW_CB_CASE(22) NW_CB_CASE(24)
          NW_CB_CASE(26) NW_CB_CASE(28) NW_CB_CASE(30) NW_CB_CASE(32)
#undef NW_CB_CASE
          default: return fail(c, NW_E_INVAL, "column-block rows per lane %d", g.KR);
        }
      } else if (sys) {
        k_fill_cblock<CB_KR32, true><<<grid_r, 32, 0, c->stream>>>(A);
      } else {
        k_fill_cblock<CB_KR32, false><<<grid_r, 32, 0, c->stream>>>(A);
      }
    }
    LAUNCHED(c);
    CUDA_TRY(c, cudaGetLastError());
  }
  const bool owner = rank0 <= last_owner && last_owner < rank0 + nhere;
  // the owner of the last block reports H(m,n); other real ranks report 0
  const bool here = owner || !owner_adds_gap;
  const long long gmn = here ? (long long)sc->gap * (m + n) : 0;
  k_finish_score<<<1, 1, 0, c->stream>>>(c->d_ints + 2, gmn, d_score, (m == 0 || n == 0) ? 1 : 0);
  LAUNCHED(c);
  CUDA_TRY(c, cudaGetLastError());
  return NW_OK;
}

nw_status cblock_check(nw_ctx* c, long long m, long long n, const nw_scoring* sc, int G) {
  nw_status st = check_scoring(c, sc);
  if (st) return st;
  st = check_bounds(c, sc, m, n);
  if (st) return st;
  if (sc->K > 4) return fail(c, NW_E_INVAL, "column-block path supports K <= 4");
  if (G < 1 || G > 64) return fail(c, NW_E_INVAL, "ranks %d outside [1,64]", G);
  return NW_OK;
}

// Codes of a (device or host) pair into the context's padded code buffers.
nw_status cb_stage(nw_ctx* c, const uint8_t* a, long long m, const uint8_t* b, long long n, bool host,
                   const nw_scoring* sc, uint8_t** ca, uint8_t** cbp) {
  nw_status st = upload_tables(c, sc);
  if (st) return st;
  const long long la = pad16(PAD + m + R_MAX + PAD), lb = pad16(PAD + n + R_MAX + PAD);
  st = grow(c, c->d_codes, c->codes_cap, (size_t)(la + lb));
  if (st) return st;
  CUDA_TRY(c, cudaMemsetAsync(c->d_codes, 0, (size_t)(la + lb), c->stream));
  return stage_pair(c, a, m, b, n, host, ca, cbp);
}

// This rank's share of the pipeline on a real rank (own receive buffer + the next
// rank's, peer-mapped): async on ctx's stream.
nw_status cblock_rank(nw_ctx* c, const uint8_t* d_a, long long m, const uint8_t* d_b, long long n,
                      const nw_scoring* sc, int rank, int ranks, int block_cols, void* recv_self,
                      void* recv_next, long long* d_score) {
  const CbGeom g = cb_geom(c, m, n, sc, ranks, block_cols);
  if (g.recv_bytes > (size_t)cb_recv_bound(m)) return fail(c, NW_E_INVAL, "receive buffer bound");
  uint8_t *ca, *cb;
  nw_status st = cb_stage(c, d_a, m, d_b, n, false, sc, &ca, &cb);
  if (st) return st;
  std::vector<unsigned long long*> tab(ranks, nullptr);
  tab[rank] = static_cast<unsigned long long*>(recv_self);
  tab[(rank + 1) % ranks] = static_cast<unsigned long long*>(ranks > 1 ? recv_next : recv_self);
  st = grow(c, c->d_cb_tab, c->cb_tab_cap, sizeof(void*) * (size_t)ranks);
  if (st) return st;
  const StagedCopy cp[1] = {{c->d_cb_tab, tab.data(), sizeof(void*) * (size_t)ranks}};
  st = upload_staged(c, cp, 1);
  if (st) return st;
  bool wrapped = false;
  const unsigned base = cb_tags(c, g, &wrapped);
  if (wrapped) {
    CUDA_TRY(c, cudaMemsetAsync(recv_self, 0, g.recv_bytes, c->stream));
    if (c->d_cb_ring) CUDA_TRY(c, cudaMemsetAsync(c->d_cb_ring, 0, c->cb_ring_cap, c->stream));
  }
  return cblock_core(c, ca, m, cb, n, sc, g, ranks, rank, 1,
                     static_cast<unsigned long long* const*>(c->d_cb_tab), d_score, true, ranks > 1, base);
}

// Dist ctx: the receive buffer is allocated (zeroed) once per size and its CUDA IPC
// handle all-gathered over the communicator; the next rank's buffer is opened once.
nw_status cblock_dist_buffers(nw_ctx* c, size_t need) {
  if (need <= c->cb_recv_cap && c->d_cb_recv && (c->world == 1 || c->cb_next)) return NW_OK;
  const nwd::NcclApi& api = nwd::nccl();
  nw_status st = grow_zeroed(c, c->d_cb_recv, c->cb_recv_cap, need);
  if (st) return st;
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (c->cb_next) {
    cudaIpcCloseMemHandle(c->cb_next);
    c->cb_next = nullptr;
  }
  if (c->world == 1) return NW_OK;
  cudaIpcMemHandle_t h;
  CUDA_TRY(c, cudaIpcGetMemHandle(&h, c->d_cb_recv));
  const size_t hb = sizeof(cudaIpcMemHandle_t);
  char* d = nullptr;
  CUDA_TRY(c, cudaMallocAsync(reinterpret_cast<void**>(&d), hb * (size_t)(c->world + 1), c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(d + hb * c->world, &h, hb, cudaMemcpyHostToDevice, c->stream));
  const ncclResult_t r = api.AllGather(d + hb * c->world, d, hb, ncclUint8, c->comm, c->stream);
  if (r != ncclSuccess) {
    cudaFreeAsync(d, c->stream);
    return fail(c, NW_E_COMM, "handle all-gather: %s", api.GetErrorString(r));
  }
  std::vector<cudaIpcMemHandle_t> all(c->world);
  CUDA_TRY(c, cudaMemcpyAsync(all.data(), d, hb * (size_t)c->world, cudaMemcpyDeviceToHost, c->stream));
  cudaFreeAsync(d, c->stream);
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  CUDA_TRY(c, cudaIpcOpenMemHandle(&c->cb_next, all[(c->rank + 1) % c->world],
                                   cudaIpcMemLazyEnablePeerAccess));
  // every rank's buffer is zero before any rank's kernel can write into it
  long long* one = nullptr;
  CUDA_TRY(c, cudaMallocAsync(reinterpret_cast<void**>(&one), sizeof(long long), c->stream));
  const ncclResult_t r2 = api.AllReduce(one, one, 1, ncclInt64, ncclSum, c->comm, c->stream);
  cudaFreeAsync(one, c->stream);
  if (r2 != ncclSuccess) return fail(c, NW_E_COMM, "barrier: %s", api.GetErrorString(r2));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return NW_OK;
}

// Score-only pairs on a dist ctx take the pipeline when there are several ranks (or
// NW_OPT_DIST_PIPELINE = 1) and the pair is large (>= 2^34 cells; DNA-size alphabets).
bool cblock_dist_applies(const nw_ctx* c, long long m, long long n, const nw_scoring* sc) {
  if (!c->comm || sc->K > 4 || m <= 0 || n <= 0) return false;
  const long long mode = c->opt[NW_OPT_DIST_PIPELINE];
  if (mode == 2) return false;
  if (mode == 1) return true;
  return c->world > 1 && (double)m * (double)n >= 17179869184.0;
}

// nw_score_only(_dev) on a dist ctx with world > 1: the C5 pipeline across the ranks,
// then one all-reduce (sum of the owner's H(m,n) and everyone else's 0).
nw_status cblock_dist(nw_ctx* c, const uint8_t* a, long long m, const uint8_t* b, long long n,
                      const nw_scoring* sc, bool host, long long* d_score) {
  const CbGeom g = cb_geom(c, m, n, sc, c->world, 0);
  nw_status st = cblock_dist_buffers(c, (size_t)cb_recv_bound(m));
  if (st) return st;
  uint8_t *ca, *cb;
  st = cb_stage(c, a, m, b, n, host, sc, &ca, &cb);
  if (st) return st;
  const int G = c->world;
  std::vector<unsigned long long*> tab(G, nullptr);
  tab[(c->rank + 1) % G] = static_cast<unsigned long long*>(c->cb_next);
  tab[c->rank] = static_cast<unsigned long long*>(c->d_cb_recv);  // (G = 1: the same entry)
  st = grow(c, c->d_cb_tab, c->cb_tab_cap, sizeof(void*) * (size_t)G);
  if (st) return st;
  const StagedCopy cp[1] = {{c->d_cb_tab, tab.data(), sizeof(void*) * (size_t)G}};
  st = upload_staged(c, cp, 1);
  if (st) return st;
  bool wrapped = false;
  const unsigned base = cb_tags(c, g, &wrapped);
  if (wrapped) {  // re-zero every rank's buffers, then a barrier (rare: ~2^32 tags)
    CUDA_TRY(c, cudaMemsetAsync(c->d_cb_recv, 0, c->cb_recv_cap, c->stream));
    if (c->d_cb_ring) CUDA_TRY(c, cudaMemsetAsync(c->d_cb_ring, 0, c->cb_ring_cap, c->stream));
    NCCL_TRY(c, nwd::nccl().AllReduce(d_score, d_score, 1, ncclInt64, ncclMax, c->comm, c->stream));
  }
  st = cblock_core(c, ca, m, cb, n, sc, g, G, c->rank, 1, static_cast<unsigned long long* const*>(c->d_cb_tab),
                   d_score, true, true, base);
  if (st) return st;
  NCCL_TRY(c, nwd::nccl().AllReduce(d_score, d_score, 1, ncclInt64, ncclSum, c->comm, c->stream));
  return NW_OK;
}

}  // namespace

extern "C" {

int64_t nw_cblock_recv_bytes(int64_t m) { return cb_recv_bound(m); }

nw_status nw_score_only_cblock(nw_ctx* c, const uint8_t* a, int64_t m, const uint8_t* b,
                               int64_t n, const nw_scoring* sc, int32_t ranks,
                               int32_t block_cols, int64_t* score) {
  if (!c) return NW_E_INVAL;
  if ((m > 0 && !a) || (n > 0 && !b) || !score) return fail(c, NW_E_INVAL, "NULL argument");
  nw_status st = cblock_check(c, m, n, sc, ranks);
  if (st) return st;
  CUDA_TRY(c, cudaSetDevice(c->device));
  const CbGeom g = cb_geom(c, m, n, sc, ranks, block_cols);
  uint8_t *ca, *cb;
  st = cb_stage(c, a, m, b, n, true, sc, &ca, &cb);
  if (st) return st;
  // virtual ranks: all receive buffers in one kept allocation (zeroed once) + the table
  const size_t per = (g.recv_bytes + 255) & ~size_t(255);
  st = grow_zeroed(c, c->d_cb_vrecv, c->cb_vrecv_cap, per * (size_t)ranks);
  if (st) return st;
  std::vector<unsigned long long*> tab(ranks);
  for (int r = 0; r < ranks; ++r)
    tab[r] = reinterpret_cast<unsigned long long*>(static_cast<char*>(c->d_cb_vrecv) + (size_t)r * per);
  st = grow(c, c->d_cb_tab, c->cb_tab_cap, sizeof(void*) * (size_t)ranks);
  if (st) return st;
  const StagedCopy cp[1] = {{c->d_cb_tab, tab.data(), sizeof(void*) * (size_t)ranks}};
  st = upload_staged(c, cp, 1);
  if (st) return st;
  bool wrapped = false;
  const unsigned base = cb_tags(c, g, &wrapped);
  if (wrapped) {
    CUDA_TRY(c, cudaMemsetAsync(c->d_cb_vrecv, 0, c->cb_vrecv_cap, c->stream));
    if (c->d_cb_ring) CUDA_TRY(c, cudaMemsetAsync(c->d_cb_ring, 0, c->cb_ring_cap, c->stream));
  }
  st = cblock_core(c, ca, m, cb, n, sc, g, ranks, 0, ranks, static_cast<unsigned long long* const*>(c->d_cb_tab),
                   c->d_score, false, false, base);
  if (st) return st;
  CUDA_TRY(c, cudaMemcpyAsync(score, c->d_score, sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
  return check_deferred(c);
}

nw_status nw_score_only_cblock_rank_dev(nw_ctx* c, const uint8_t* d_a, int64_t m,
                                        const uint8_t* d_b, int64_t n, const nw_scoring* sc,
                                        int32_t rank, int32_t ranks, int32_t block_cols,
                                        void* recv_self, void* recv_next, int64_t* d_score) {
  if (!c) return NW_E_INVAL;
  if (!recv_self) {  // the buffers of nw_cblock_ipc_export / nw_cblock_ipc_import
    recv_self = c->d_cb_recv;
    recv_next = c->cb_next;
    if (!recv_self || (size_t)nw_cblock_recv_bytes(m) > c->cb_recv_cap || (ranks > 1 && !recv_next))
      return fail(c, NW_E_STATE, "no exported/imported receive buffers for m=%lld", (long long)m);
  }
  if ((m > 0 && !d_a) || (n > 0 && !d_b) || !d_score || (ranks > 1 && !recv_next))
    return fail(c, NW_E_INVAL, "NULL argument");
  nw_status st = cblock_check(c, m, n, sc, ranks);
  if (st) return st;
  if (rank < 0 || rank >= ranks) return fail(c, NW_E_INVAL, "rank %d outside [0,%d)", rank, ranks);
  CUDA_TRY(c, cudaSetDevice(c->device));
  return cblock_rank(c, d_a, m, d_b, n, sc, rank, ranks, block_cols, recv_self, recv_next,
                     reinterpret_cast<long long*>(d_score));
}

nw_status nw_cblock_ipc_export(nw_ctx* c, int64_t m, uint8_t* handle) {
  if (!c || !handle || m < 0) return c ? fail(c, NW_E_INVAL, "NULL argument") : NW_E_INVAL;
  CUDA_TRY(c, cudaSetDevice(c->device));
  nw_status st = grow_zeroed(c, c->d_cb_recv, c->cb_recv_cap, (size_t)nw_cblock_recv_bytes(m));
  if (st) return st;
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  cudaIpcMemHandle_t h;
  CUDA_TRY(c, cudaIpcGetMemHandle(&h, c->d_cb_recv));
  memcpy(handle, &h, sizeof h);
  return NW_OK;
}

nw_status nw_cblock_ipc_import(nw_ctx* c, const uint8_t* handle) {
  if (!c || !handle) return c ? fail(c, NW_E_INVAL, "NULL argument") : NW_E_INVAL;
  CUDA_TRY(c, cudaSetDevice(c->device));
  if (c->cb_next) {
    cudaIpcCloseMemHandle(c->cb_next);
    c->cb_next = nullptr;
  }
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof h);
  CUDA_TRY(c, cudaIpcOpenMemHandle(&c->cb_next, h, cudaIpcMemLazyEnablePeerAccess));
  return NW_OK;
}

nw_status nw_batch_ops_offsets(const int64_t* h_offs, int32_t nseq, const int32_t* h_pairs,
                               int64_t npairs, int64_t* ops_off) {
  if (!h_offs || !ops_off || nseq < 0 || npairs < 0) return NW_E_INVAL;
  long long acc = 0;
  ops_off[0] = 0;
  if (h_pairs) {
    for (long long k = 0; k < npairs; ++k) {
      const int p = h_pairs[2 * k], q = h_pairs[2 * k + 1];
      if (p < 0 || p >= nseq || q < 0 || q >= nseq) return NW_E_INVAL;
      acc += (h_offs[p + 1] - h_offs[p]) + (h_offs[q + 1] - h_offs[q]);
      ops_off[k + 1] = acc;
    }
  } else {
    long long k = 0;
    if (npairs != (long long)nseq * (nseq - 1) / 2) return NW_E_INVAL;
    for (int p = 0; p < nseq; ++p)
      for (int q = p + 1; q < nseq; ++q) {
        acc += (h_offs[p + 1] - h_offs[p]) + (h_offs[q + 1] - h_offs[q]);
        ops_off[++k] = acc;
      }
  }
  return NW_OK;
}

}  // extern "C"

namespace {

// Shared body of the batch entry points. All pointers device; h_offs/h_pairs host.
// ---- device batch planner (explicit pairs, two-phase traceback) ----
// The host plan of batch_core computed on the GPU: cost buckets (LPT), orientation,
// per-pair flag words, bucket starts, a scatter into task order and the word
// offsets (a CUB scan). Order within a bucket follows atomic arrival: it changes
// only the schedule, never a result (every output is indexed by the pair).
constexpr int PLAN_NB = 4096;

__global__ void k_plan_bucket(const int* __restrict__ pairs, const long long* __restrict__ offs,
                              long long np, int lrs, unsigned long long inv, int orient,
                              long long wpg, int* bkt, long long* words, int* hist) {
  __shared__ int h[2 * PLAN_NB];
  for (int i = threadIdx.x; i < 2 * PLAN_NB; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const long long RS = 1LL << lrs;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < np;
       k += (long long)gridDim.x * blockDim.x) {
    const int p = pairs[2 * k], q = pairs[2 * k + 1];
    const long long m = offs[p + 1] - offs[p], n = offs[q + 1] - offs[q];
    const long long sm_ = (m + RS - 1) >> lrs, sn_ = (n + RS - 1) >> lrs;
    const bool tr = orient && m > 0 && n > 0 && sn_ * (m + 70) < sm_ * (n + 70);
    const int q16 = (int)(((unsigned long long)(m * n) * inv) >> 32);
    const int b = (tr ? PLAN_NB : 0) + (PLAN_NB - 1) - min(PLAN_NB - 1, q16);
    bkt[k] = b;
    words[k] = (m > 0 && n > 0) ? (tr ? sn_ * ((m + 70) >> 3) : sm_ * ((n + 70) >> 3)) * wpg : 0LL;
    atomicAdd(&h[b], 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * PLAN_NB; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[i], h[i]);
}

// in place: hist -> exclusive bucket starts; small[0] = start of the transposed buckets
__global__ void __launch_bounds__(1024) k_plan_scan(int* hist, long long* small) {
  __shared__ int ws[32];
  constexpr int PER = 2 * PLAN_NB / 1024;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int v[PER], acc = 0;
#pragma unroll
  for (int u = 0; u < PER; ++u) { v[u] = hist[tid * PER + u]; acc += v[u]; }
  int x = acc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, x, o); if (lane >= o) x += y; }
  if (lane == 31) ws[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = ws[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, w, o); if (lane >= o) w += y; }
    ws[lane] = w;
  }
  __syncthreads();
  int run = (warp ? ws[warp - 1] : 0) + x - acc;
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int b = tid * PER + u;
    if (b == PLAN_NB) small[0] = run;
    hist[b] = run;
    run += v[u];
  }
}

__global__ void k_plan_scatter(const int* __restrict__ bkt, const long long* __restrict__ words,
                               long long np, int* starts, int* aux, long long* tw) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < np;
       k += (long long)gridDim.x * blockDim.x) {
    const int pos = atomicAdd(&starts[bkt[k]], 1);
    aux[pos] = (int)k;
    tw[pos] = words[k];
  }
}

__global__ void k_plan_total(const long long* tw, const long long* tdoff, long long np, long long* small) {
  small[1] = tdoff[np - 1] + tw[np - 1];
}

// Fills c->d_aux (task -> pair) and c->d_tdoff (task -> word offset); returns the
// first transposed task and the total words (one small device -> host copy).
nw_status device_plan(nw_ctx* c, const int* d_pairs, const long long* d_offs, long long npairs,
                      long long RS, long long maxlen, bool orient, long long* ntr0, long long* total) {
  int lrs = 0;
  while ((1LL << lrs) < RS) ++lrs;
  const unsigned long long inv = ((unsigned long long)(PLAN_NB - 1) << 32) /
                                 (unsigned long long)std::max(1LL, maxlen * maxlen);
  size_t cub_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, cub_bytes, (const long long*)nullptr, (long long*)nullptr,
                                (int)npairs, c->stream);
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t b_bkt = al(sizeof(int) * npairs), b_w = al(sizeof(long long) * npairs),
               b_h = al(sizeof(int) * (2 * PLAN_NB + 1)), b_small = 256, b_tw = b_w;
  nw_status st = grow(c, c->d_plan, c->plan_cap, b_bkt + b_w + b_h + b_small + b_tw + al(cub_bytes));
  if (st) return st;
  st = grow(c, c->d_aux, c->aux_cap, sizeof(int) * (size_t)npairs + 16);
  if (st) return st;
  st = grow(c, c->d_tdoff, c->tdoff_cap, sizeof(long long) * (size_t)npairs);
  if (st) return st;
  char* p = static_cast<char*>(c->d_plan);
  int* bkt = reinterpret_cast<int*>(p); p += b_bkt;
  long long* words = reinterpret_cast<long long*>(p); p += b_w;
  int* hist = reinterpret_cast<int*>(p); p += b_h;
  long long* small = reinterpret_cast<long long*>(p); p += b_small;
  long long* tw = reinterpret_cast<long long*>(p); p += b_tw;
  void* cub_tmp = p;
  CUDA_TRY(c, cudaMemsetAsync(hist, 0, sizeof(int) * 2 * PLAN_NB, c->stream));
  const int blocks = (int)std::min<long long>((npairs + 255) / 256, (long long)c->sm_count * 4);
  k_plan_bucket<<<blocks, 256, 0, c->stream>>>(d_pairs, d_offs, npairs, lrs, inv, orient ? 1 : 0,
                                                RS / 2, bkt, words, hist);
  k_plan_scan<<<1, 1024, 0, c->stream>>>(hist, small);
  k_plan_scatter<<<blocks, 256, 0, c->stream>>>(bkt, words, npairs, hist, static_cast<int*>(c->d_aux), tw);
  CUDA_TRY(c, cub::DeviceScan::ExclusiveSum(cub_tmp, cub_bytes, tw, c->d_tdoff, (int)npairs, c->stream));
  k_plan_total<<<1, 1, 0, c->stream>>>(tw, c->d_tdoff, npairs, small);
  c->launches += 5;
  CUDA_TRY(c, cudaGetLastError());
  long long h[2] = {0, 0};
  CUDA_TRY(c, cudaMemcpyAsync(h, small, sizeof h, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  *ntr0 = orient ? h[0] : npairs;
  *total = h[1];
  return NW_OK;
}

struct HostLaps {  // NW_OPT_HOST_PROFILE: host-side phase times of one call, to stderr
  bool on;
  explicit HostLaps(const nw_ctx* c) : on(c->opt[NW_OPT_HOST_PROFILE] != 0) {}
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void lap(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "  [host] %-24s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

// Implicit all-pairs on a dist context: this rank's rank-space tasks
// [tbase, tbase + ntasks), scores written compactly (d_scores[task]).
struct DistRange { long long tbase, ntasks; };

nw_status batch_core(nw_ctx* c, const uint8_t* d_codes_raw_or_codes, bool already_coded,
                     const long long* d_offs, const long long* h_offs, int nseq, const int* d_pairs,
                     const int* h_pairs, long long npairs, const nw_scoring* sc, uint32_t flags,
                     int* d_scores, const long long* d_ops_off, uint8_t* d_ops, int* d_ops_len,
                     const DistRange* dr = nullptr) {
  const long long ntasks = (dr && !h_pairs) ? dr->ntasks : npairs;
  constexpr int R = 32 * KR_BATCH;
  HostLaps hl(c);
  const bool tbk = (flags & NW_TRACEBACK) != 0;
  const long long total = h_offs[nseq];
  long long maxlen = 0;
  for (int k = 0; k < nseq; ++k) maxlen = std::max<long long>(maxlen, h_offs[k + 1] - h_offs[k]);
  nw_status st = check_bounds(c, sc, maxlen, maxlen);
  if (st) return st;
  st = init_small(c, 4);
  if (st) return st;
  // codes buffer: PAD | codes | tail: the sweeps read up to one strip of rows
  // (512 for the packed sweep) and ~94 columns past a sequence's end
  const long long lc = PAD + total + R_MAX + 2 * PAD;
  st = grow(c, c->d_codes, c->codes_cap, (size_t)lc);
  if (st) return st;
  CUDA_TRY(c, cudaMemsetAsync(c->d_codes, 0, (size_t)lc, c->stream));
  uint8_t* codes = c->d_codes + PAD;
  (void)already_coded;
  launch_encode(c, d_codes_raw_or_codes, total, codes, 0);
  hl.lap("bounds, memset, encode");
  // order: implicit all-pairs -> perm of sequences by length (descending);
  // explicit pairs -> LPT order by m*n (descending), bucketed.
  std::vector<int>& aux = c->h_aux;
  aux.clear();
  if (!h_pairs) {
    aux.resize(nseq);
    for (int k = 0; k < nseq; ++k) aux[k] = k;
    std::stable_sort(aux.begin(), aux.end(), [&](int x, int y) {
      return (h_offs[x + 1] - h_offs[x]) > (h_offs[y + 1] - h_offs[y]);
    });
  }  // explicit pairs: ordered below, once the strip height is known
  hl.lap("implicit order");

  // per-warp scratch
  const int warps_per_cta = 4;
  const bool profreg = sc->K <= 4;
  // packed score-only sweeps: the H' form when every H' fits 16 bits (measured
  // faster on C3), else the difference form (any length); both need s - 2g >= 0
  const bool packed = !tbk && profreg && d16_ok(c, sc);
  int smax = 0;
  for (int x = 0; x < sc->K; ++x)
    for (int y = 0; y < sc->K; ++y) smax = std::max(smax, score_of(sc, x, y) - 2 * sc->gap);
  const bool u16 = packed && (long long)maxlen * smax <= 65535;
  if (u16) {  // selector table of the packed H' sweep (FillArgs::sel), aligned with the codes
    st = grow(c, c->d_sel16, c->sel16_cap, sizeof(uint16_t) * (size_t)lc);
    if (st) return st;
    const int blocks = (int)std::min<long long>((lc - 1 + 255) / 256, (long long)c->sm_count * 8);
    k_sel16<<<std::max(blocks, 1), 256, 0, c->stream>>>(c->d_codes + 1, lc - 1, c->d_sel16 + 1);
    LAUNCHED(c);
  }
  bool d16 = packed && !u16;
  if (tbk && !c->opt[NW_OPT_NO_D16]) {  // traceback: difference form with decision flags
    int smin = 1 << 30;
    for (int x = 0; x < sc->K; ++x)
      for (int y = 0; y < sc->K; ++y) smin = std::min(smin, score_of(sc, x, y) - 2 * sc->gap);
    d16 = smin >= 0;
  }
  const bool packed_sweep = u16 || d16;  // two rows per register
  // packed traceback strips: 16 rows per lane, or 8 when most pairs are short
  // (a 512-row strip over a 300-row pair idles 40% of the lanes); NW_BATCH_KR16 overrides
  int packed_kr = 16;
  if (tbk && d16) {
    std::vector<long long> rl;
    rl.reserve(std::min<long long>(npairs, 4096));
    for (long long k = 0; k < npairs && k < 4096; ++k) {
      const int p = h_pairs ? h_pairs[2 * k] : (int)(k % std::max(nseq, 1));
      rl.push_back(h_offs[p + 1] - h_offs[p]);
    }
    std::nth_element(rl.begin(), rl.begin() + rl.size() / 2, rl.end());
    if (!rl.empty() && rl[rl.size() / 2] <= 768) packed_kr = 8;
    if (c->opt[NW_OPT_BATCH_KR16]) packed_kr = c->opt[NW_OPT_BATCH_KR16] == 8 ? 8 : 16;
  }
  const long long RS = packed_sweep ? 32 * (tbk && d16 ? packed_kr : 16) : R;
  // Two-phase traceback (explicit pairs, packed flags): the fill keeps
  // every pair's decision words in HBM (C4: 7.6 GB; the per-warp scratch of the
  // in-warp walk spilled to HBM anyway) and k_batch_walk walks all pairs at once,
  // one thread each, so the walk's dependent loads overlap across 100k pairs instead
  // of idling 31 lanes of a filling warp. Pairs are cut into waves whose words fit
  // the budget (half the free memory; NW_BATCH_TB_BUDGET bytes overrides).
  const bool two_phase = tbk && d16;
  bool sym = true;  // s(x, y) = s(y, x): a pair may be filled transposed
  for (int x = 0; x < sc->K; ++x)
    for (int y = 0; y < x; ++y) sym = sym && score_of(sc, x, y) == score_of(sc, y, x);
  long long ntr0 = npairs;  // explicit-pair tasks [ntr0, npairs) are filled transposed
  // the plan on the device for large explicit two-phase batches (C4: ~1.4 ms of host
  // planning, all GPU idle, becomes a few tiny kernels and one small copy); used when
  // the kept flag buffer already holds every pair's words (else the host plans waves)
  bool dev_plan = false;
  if (h_pairs && two_phase && npairs >= 4096 && c->tbdirs_cap > 0 && !c->opt[NW_OPT_HOST_PLAN]) {
    long long total = 0, nt = npairs;
    st = device_plan(c, d_pairs, d_offs, npairs, RS, maxlen,
                     sym && !c->opt[NW_OPT_BATCH_NO_TRANSPOSE], &nt, &total);
    if (st) return st;
    if ((size_t)total * 4 <= c->tbdirs_cap && !c->opt[NW_OPT_BATCH_TB_BUDGET]) {
      dev_plan = true;
      ntr0 = nt;
    }
  }
  if (h_pairs && !dev_plan) {
    // LPT order: counting sort on the cost quantised to NB levels (descending,
    // stable), O(npairs) -- a comparison sort of C4's 100k pairs took ~15 ms of host
    // time per call and left the GPU idle (tools/exp_c4.py). Two-phase traceback with
    // a symmetric s also picks each pair's orientation here: a pair is filled with b
    // on the rows when that sweeps fewer padded cells (strips x (columns + skew));
    // its flags are those of the mirrored tie order (U <-> L) on the transposed grid,
    // whose path is the pair's own with U and L exchanged (the oracle's mirror pin).
    // C4: 1.38x -> 1.29x the useful cells. Transposed tasks come after the others
    // (NB more buckets), each part in LPT order; each part is its own fill launch.
    const bool orient = two_phase && sym && !c->opt[NW_OPT_BATCH_NO_TRANSPOSE];
    // one pass: bucket (cost quantised against maxlen^2, so no max pass), orientation
    // and the pair's flag words; a second pass scatters them into LPT order
    constexpr int NB = 4096;
    const long long wpg = RS / 2;
    int lrs = 0;  // RS is a power of two: strip counts by shifts (divisions dominated this loop)
    while ((1LL << lrs) < RS) ++lrs;
    // bucket = (NB-1) - floor(cost * (NB-1) / maxlen^2) in integers (cost <= maxlen^2)
    const unsigned long long inv = ((unsigned long long)(NB - 1) << 32) /
                                   (unsigned long long)std::max(1LL, maxlen * maxlen);
    aux.resize(npairs);
    c->h_bkt.resize(npairs);
    c->h_words.resize(two_phase ? npairs : 0);
    c->h_cnt.assign(2 * NB + 1, 0);
    int* bk = c->h_bkt.data();
    int* cnt = c->h_cnt.data();
    long long* wd = c->h_words.data();
    // (an OpenMP split of these loops made the C4 step slower: the worker threads'
    // spin-wait competes with the launching thread)
    for (long long k = 0; k < npairs; ++k) {
      const int p = h_pairs[2 * k], q = h_pairs[2 * k + 1];
      const long long m = h_offs[p + 1] - h_offs[p], n = h_offs[q + 1] - h_offs[q];
      const long long sm_ = (m + RS - 1) >> lrs, sn_ = (n + RS - 1) >> lrs;
      const bool tr = orient && m > 0 && n > 0 &&  // empty pairs never: k_batch writes their gaps
                      sn_ * (m + 70) < sm_ * (n + 70);
      const int q16 = (int)(((unsigned long long)(m * n) * inv) >> 32);
      bk[k] = (tr ? NB : 0) + (NB - 1) - std::min(NB - 1, q16);
      ++cnt[bk[k] + 1];
      if (two_phase)
        wd[k] = (m > 0 && n > 0) ? (tr ? sn_ * ((m + 70) >> 3) : sm_ * ((n + 70) >> 3)) * wpg : 0LL;
    }
    for (int b = 0; b < 2 * NB; ++b) cnt[b + 1] += cnt[b];
    if (orient) ntr0 = cnt[NB];
    for (long long k = 0; k < npairs; ++k) aux[cnt[bk[k]]++] = (int)k;
  }
  hl.lap("LPT order + orientation");
  if (!dev_plan) {
    st = grow(c, c->d_aux, c->aux_cap, sizeof(int) * aux.size() + 16);
    if (st) return st;
  }
  std::vector<long long>& tdoff = c->h_tdoff;
  std::vector<long long> wave_end;
  tdoff.clear();
  if (dev_plan) wave_end.push_back(npairs);  // one wave: the kept buffer holds every pair's words
  if (two_phase && !dev_plan) {
    const long long wpg = RS / 2;  // words per (strip, 8-step group): H packed rows x 32 lanes
    auto len = [&](int s) { return h_offs[s + 1] - h_offs[s]; };
    auto words_mn = [&](long long m, long long n) {
      return (m > 0 && n > 0) ? ((m + RS - 1) / RS) * ((n + 63 + 7) / 8) * wpg : 0LL;
    };
    // words of every task in the fill's order: explicit pairs by aux (LPT), implicit
    // all-pairs in rank order over the length-sorted sequences (aux = that perm),
    // the row sequence being the lower original index as in task_pair
    std::vector<long long>& tw = c->h_tw;
    tw.resize(npairs);
    if (h_pairs) {
      const long long* wd = c->h_words.data();
      const int* ax = aux.data();
      long long* twp = tw.data();
      for (long long t = 0; t < npairs; ++t) twp[t] = wd[ax[t]];
    } else {
      long long t = 0;
      for (int pr = 0; pr < nseq; ++pr)
        for (int qr = pr + 1; qr < nseq; ++qr, ++t) {
          const int x = aux[pr], y = aux[qr];
          tw[t] = words_mn(len(std::min(x, y)), len(std::max(x, y)));
        }
    }
    long long all_words = 0;
    for (long long t = 0; t < npairs; ++t) all_words += tw[t];
    long long budget = all_words;  // one wave when the kept buffer already holds it
    if ((size_t)all_words * 4 > c->tbdirs_cap) {
      size_t free_b = 0, tot_b = 0;
      CUDA_TRY(c, cudaMemGetInfo(&free_b, &tot_b));
      budget = (long long)((free_b + c->tbdirs_cap) / 2 / 4);
    }
    if (c->opt[NW_OPT_BATCH_TB_BUDGET] > 0) budget = std::max(1LL, c->opt[NW_OPT_BATCH_TB_BUDGET] / 4);
    tdoff.resize(npairs);
    long long acc = 0, maxwave = 0;
    for (long long t = 0; t < npairs; ++t) {
      const long long words = tw[t];
      if (acc > 0 && acc + words > budget) {
        wave_end.push_back(t);
        maxwave = std::max(maxwave, acc);
        acc = 0;
      }
      tdoff[t] = acc;
      acc += words;
    }
    wave_end.push_back(npairs);
    maxwave = std::max(maxwave, acc);
    st = grow(c, c->d_tbdirs, c->tbdirs_cap, (size_t)std::max(1LL, maxwave) * 4);
    if (st) return st;
    st = grow(c, c->d_tdoff, c->tdoff_cap, sizeof(long long) * (size_t)std::max(1LL, npairs));
    if (st) return st;
  }
  if (!dev_plan) {
    const StagedCopy cp[2] = {{c->d_aux, aux.data(), sizeof(int) * aux.size()},
                              {c->d_tdoff, tdoff.data(), sizeof(long long) * tdoff.size()}};
    hl.lap("words, waves, grow");
    st = upload_staged(c, cp, 2);
    hl.lap("staged upload");
    if (st) return st;
  }
  const size_t smem_prof = profreg ? 0 : (((size_t)warps_per_cta * sc->K * RS + 15) & ~size_t(15));
  // the packed H' sweep keeps its boundary row in shared memory when 6 CTAs still fit
  // an SM (C3: 4 warps x 2,066 ints = 33 KB per CTA); its DRAM traffic is then the
  // inputs and the scores (the global per-warp rows were 533 MB of DRAM writes per C3
  // launch, evicted from L2)
  const size_t smem_bnd = ((size_t)warps_per_cta * (size_t)(maxlen + 1 + 64) * 4 + 15) & ~size_t(15);
  const bool bnd_smem = u16 && smem_prof + smem_bnd <= 37 * 1024 && !c->opt[NW_OPT_BATCH_BND_GLOBAL];
  const size_t smem = smem_prof + (bnd_smem ? smem_bnd : 0);
  // 6 x 4 warps per SM (24 warps, 72 registers each): C4 2.11 -> 2.26 TCUPS, C3 6.73 -> 6.84
  // over 4 per SM; 8 no better (tools/exp_ctas.sh, profiles/r01_exp_ctas.txt)
  int ctas_per_sm = 6;  // (8 measured equal on C3 and C4 in round 2)
  // no more warps than pairs: the int32 traceback path sizes its per-warp direction
  // scratch (~maxlen^2/4 bytes) per launched warp
  const long long nwarps = std::min<long long>((long long)c->sm_count * ctas_per_sm * warps_per_cta,
                                               (ntasks + warps_per_cta - 1) / warps_per_cta * warps_per_cta);
  const long long bstride = (maxlen + 1 + 64 + 1) & ~1LL;  // even: 8-byte vector stores of the bottom row (nw_fill.cuh)
  // direction scratch per warp, in halfwords: int32 sweep = halfword per (group,
  // row, lane); packed sweep = 32-bit word per (group, packed row, lane)
  const long long wpl = (maxlen + (packed_sweep ? 63 : 31) + 7) / 8;  // 8-step groups per strip
  const long long dstride = (!tbk || two_phase) ? 0
      : packed_sweep ? ((maxlen + RS - 1) / RS) * wpl * (RS / 64) * 32 * 2
                     : ((maxlen + R - 1) / R) * wpl * KR_BATCH * 32;
  const size_t bytes_bnd = sizeof(int) * (size_t)(nwarps * 2 * bstride);
  const size_t bytes_hm = sizeof(int) * (size_t)nwarps;
  const size_t bytes_dirs = sizeof(uint16_t) * (size_t)(nwarps * dstride);
  st = grow(c, c->d_scratch, c->scratch_cap, bytes_bnd + bytes_hm + bytes_dirs + 256);
  if (st) return st;
  BatchArgs B;
  B.codes = codes;
  B.offs = d_offs;
  B.nseq = nseq;
  B.pairs = d_pairs;
  B.order = d_pairs ? static_cast<const int*>(c->d_aux) : nullptr;
  B.perm = d_pairs ? nullptr : static_cast<const int*>(c->d_aux);
  B.npairs = npairs;
  B.prof = c->d_prof;
  B.K = sc->K;
  B.g = sc->gap;
  B.ticket = c->d_ints;
  B.err = c->d_err;
  B.scores = d_scores;
  B.sel16 = c->d_sel16 ? c->d_sel16 + PAD : nullptr;  // read by the u16 sweep only
  B.bnd_smem = bnd_smem ? 1 : 0;
  B.bnd_smem_off = (int)smem_prof;
  char* base = static_cast<char*>(c->d_scratch);
  B.wbnd = reinterpret_cast<int*>(base);
  B.bstride = bstride;
  B.whm = reinterpret_cast<int*>(base + bytes_bnd);
  B.wdirs = tbk ? reinterpret_cast<uint16_t*>(base + ((bytes_bnd + bytes_hm + 255) & ~size_t(255)))
                : nullptr;
  B.dstride = dstride;
  B.ops_off = d_ops_off;
  B.ops = d_ops;
  B.ops_len = d_ops_len;
  B.transpose_ok = (!tbk && sym && !c->opt[NW_OPT_BATCH_NO_TRANSPOSE]) ? 1 : 0;
  B.transposed = 0;
  B.ntr0 = ntr0;
  B.tdirs = two_phase ? static_cast<uint32_t*>(c->d_tbdirs) : nullptr;
  B.tdir_off = two_phase ? c->d_tdoff : nullptr;
  B.task0 = 0;
  B.task1 = ntasks;
  if (dr && !h_pairs) {
    B.tbase = dr->tbase;
    B.compact = 1;
  }
  B.X = sc->tie[0];
  B.Y = sc->tie[1];
  B.Z = sc->tie[2];
  if (tbk && bytes_bnd + bytes_hm + 256 + bytes_dirs > c->scratch_cap)
    return fail(c, NW_E_NOMEM, "batch scratch");
  const int grid = (int)(nwarps / warps_per_cta);
  const int pi = tbk ? pi_code(sc->tie) : 123;
  // packed 16-bit sweep (score-only DNA-size alphabets) when s' = s - 2g >= 0 and
  // min(m,n) * max(s') <= 65535 for every pair (bounded by the longest sequence)

  if (two_phase) {
    hl.lap("scratch, args");
    long long t0 = 0;
    bool first = true;
    for (const long long t1 : wave_end) {
      if (t1 <= t0) continue;
      // fills: the wave's normal tasks, then its transposed tasks (mirrored tie order)
      for (int part = 0; part < 2; ++part) {
        const long long a0 = part ? std::max(t0, ntr0) : t0, a1 = part ? t1 : std::min(t1, ntr0);
        if (a1 <= a0) continue;
        uint8_t tie[3];
        for (int i = 0; i < 3; ++i) tie[i] = (uint8_t)(part && sc->tie[i] != 1 ? 5 - sc->tie[i] : sc->tie[i]);
        B.task0 = a0;
        B.task1 = a1;
        B.transposed = part;
        if (!first) CUDA_TRY(c, cudaMemsetAsync(B.ticket, 0, sizeof(int), c->stream));
        first = false;
        bool ok;
        {
          KernelTimer kt(c, 0);
          ok = dispatch_batch(tbk, pi_code(tie), profreg, u16, d16, packed_kr, B, grid, smem, c->stream);
        }
        if (!ok) return fail(c, NW_E_INVAL, "bad tie order");
        LAUNCHED(c);
        CUDA_TRY(c, cudaGetLastError());
      }
      B.task0 = t0;
      B.task1 = t1;
      B.transposed = 0;
      {  // (walking every 32 pairs inside the filling warp instead was slower on C4:
         // fill + walk 12.74 vs 10.93 + 1.52 ms, profiles/r01_exp_c4_walk_inline.txt)
        KernelTimer kt(c, 1);
        const unsigned wg = (unsigned)((t1 - t0 + 255) / 256);
        if (packed_kr == 8) k_batch_walk<8><<<wg, 256, 0, c->stream>>>(B);
        else k_batch_walk<16><<<wg, 256, 0, c->stream>>>(B);
        LAUNCHED(c);
        CUDA_TRY(c, cudaGetLastError());
      }
      t0 = t1;
    }
    hl.lap("launches");
    return NW_OK;
  }
  bool ok;
  {
    KernelTimer kt(c, 0);
    // rows per lane of the packed H' sweep: more rows amortise the per-step overhead,
    // fewer waste less of a short pair's last strip; by the median sequence length
    // (C3, median ~1,250: 32 rows = 9.51 TCUPS vs 16: 9.20, 8: 7.73; profiles/r02_exp_u16kr.json)
    int u16_kr = 16;
    if (u16) {
      std::vector<long long> ls;
      ls.reserve(std::min<long long>(nseq, 4096));
      for (int k = 0; k < nseq && k < 4096; ++k) ls.push_back(h_offs[k + 1] - h_offs[k]);
      if (!ls.empty()) {
        std::nth_element(ls.begin(), ls.begin() + ls.size() / 2, ls.end());
        const long long med = ls[ls.size() / 2];
        u16_kr = med >= 1024 ? 1 : (med >= 384 ? 16 : 8);  // 1: each pair at 32 or 16 rows per lane
      }
      const long long o = c->opt[NW_OPT_BATCH_U16_KR];
      if (o == 1 || o == 8 || o == 16 || o == 32) u16_kr = (int)o;
      if (c->opt[NW_OPT_BATCH_MIX_W] > 0) B.mix_w16 = (int)std::min(c->opt[NW_OPT_BATCH_MIX_W], 100000LL);
      if (c->opt[NW_OPT_BATCH_MIX_W24] > 0) B.mix_w24 = (int)std::min(c->opt[NW_OPT_BATCH_MIX_W24], 100000LL);
    }
    ok = dispatch_batch(tbk, pi, profreg, u16, d16, packed_kr, B, grid, smem, c->stream, u16_kr);
  }
  if (!ok) return fail(c, NW_E_INVAL, "bad tie order");
  LAUNCHED(c);
  CUDA_TRY(c, cudaGetLastError());
  return NW_OK;
}

nw_status batch_check(nw_ctx* c, const long long* h_offs, int nseq, const int* h_pairs,
                      long long npairs, const nw_scoring* sc, uint32_t flags) {
  nw_status st = check_scoring(c, sc);
  if (st) return st;
  if (nseq < 0 || npairs < 0 || !h_offs) return fail(c, NW_E_INVAL, "bad batch sizes");
  if (flags & ~1u) return fail(c, NW_E_INVAL, "unknown flags 0x%x", flags);
  if (h_offs[0] != 0) return fail(c, NW_E_INVAL, "offs[0] must be 0");
  for (int k = 0; k < nseq; ++k)
    if (h_offs[k + 1] < h_offs[k]) return fail(c, NW_E_INVAL, "offs not non-decreasing");
  if (!h_pairs) {
    if (npairs != (long long)nseq * (nseq - 1) / 2)
      return fail(c, NW_E_INVAL, "pairs=NULL requires npairs = nseq*(nseq-1)/2");
  } else {
    for (long long k = 0; k < 2 * npairs; ++k)
      if (h_pairs[k] < 0 || h_pairs[k] >= nseq) return fail(c, NW_E_INVAL, "pair index out of range");
  }
  if (npairs > (1ll << 31) - 2) return fail(c, NW_E_OVERFLOW, "too many pairs");
  return NW_OK;
}


// nw_align_batch(_dev) on a dist context: every rank passes
// the same inputs, aligns the cost-balanced contiguous share partition_bounds gives
// it, and one group of in-place broadcasts (an all-gather of variable-size ranges)
// leaves every output on every rank. No index travels: the ranges follow from the
// inputs. Explicit pairs: pair-index ranges, outputs written in place (scores,
// path lengths, and the ops bytes [ops_off[lo], ops_off[hi])). Implicit all-pairs,
// score-only: ranges of k_batch's rank space (longest sequences first), scores
// gathered in rank-space order and scattered to pair order by k_rs_scatter.
// Implicit with traceback: the lexicographic pairs are materialised (explicit).
nw_status batch_dist(nw_ctx* c, const uint8_t* d_raw, const long long* d_offs, const long long* h_offs,
                     int nseq, const int* d_pairs, const int* h_pairs, long long npairs,
                     const nw_scoring* sc, uint32_t flags, int* d_scores, const long long* d_ops_off,
                     const long long* h_ops_off, uint8_t* d_ops, int* d_ops_len) {
  const nwd::NcclApi& api = nwd::nccl();
  const bool tbk = (flags & NW_TRACEBACK) != 0;
  // NW_OPT_DIST_VIRTUAL_WORLD / _RANK (test only, no communicator): run one rank's range
  // of the partition and skip the gather, so G sequential calls on one GPU replay G ranks
  const bool virt = c->comm == nullptr;
  const int G = virt ? (int)c->opt[NW_OPT_DIST_VIRTUAL_WORLD] : c->world;
  const int me = virt ? (int)std::min<long long>(c->opt[NW_OPT_DIST_VIRTUAL_RANK], G - 1) : c->rank;
  nw_status st = NW_OK;
  if (!h_pairs && tbk) {  // materialise the lexicographic pairs
    c->h_pmat.resize(2 * (size_t)npairs);
    long long k = 0;
    for (int p = 0; p < nseq; ++p)
      for (int q = p + 1; q < nseq; ++q, ++k) { c->h_pmat[2 * k] = p; c->h_pmat[2 * k + 1] = q; }
    st = grow(c, c->d_pmat, c->pmat_cap, sizeof(int) * 2 * (size_t)npairs);
    if (st) return st;
    CUDA_TRY(c, cudaMemcpyAsync(c->d_pmat, c->h_pmat.data(), sizeof(int) * 2 * (size_t)npairs,
                                cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));  // h_pmat is reused by the next call
    h_pairs = c->h_pmat.data();
    d_pairs = c->d_pmat;
  }
  std::vector<long long>& bd = c->h_bounds;
  bd.assign(G + 1, 0);
  nwd::partition_bounds(h_offs, nseq, h_pairs, npairs, G, bd.data());
  const long long lo = bd[me], hi = bd[me + 1];
  if (!h_pairs) {  // implicit, score-only
    st = grow(c, c->d_rs, c->rs_cap, sizeof(int) * (size_t)std::max(1LL, npairs));
    if (st) return st;
    const DistRange dr{lo, hi - lo};
    if (hi > lo) {
      st = batch_core(c, d_raw, false, d_offs, h_offs, nseq, nullptr, nullptr, npairs, sc, flags,
                      c->d_rs + lo, nullptr, nullptr, nullptr, &dr);
      if (st) return st;
    } else {  // no tasks here: the permutation k_rs_scatter needs still comes from batch_core
      std::vector<int> perm;
      nwd::length_perm(h_offs, nseq, perm);
      st = grow(c, c->d_aux, c->aux_cap, sizeof(int) * perm.size() + 16);
      if (st) return st;
      const StagedCopy cp[1] = {{c->d_aux, perm.data(), sizeof(int) * perm.size()}};
      st = upload_staged(c, cp, 1);
      if (st) return st;
    }
    if (!virt) NCCL_TRY(c, api.GroupStart());
    for (int g = 0; g < G && !virt; ++g)
      if (bd[g + 1] > bd[g])
        NCCL_TRY(c, api.Broadcast(c->d_rs + bd[g], c->d_rs + bd[g], (size_t)(bd[g + 1] - bd[g]),
                                  ncclInt32, g, c->comm, c->stream));
    if (!virt) NCCL_TRY(c, api.GroupEnd());
    const int blocks = (int)std::min<long long>((npairs + 255) / 256, (long long)c->sm_count * 8);
    nwk::k_rs_scatter<<<std::max(blocks, 1), 256, 0, c->stream>>>(c->d_rs, npairs, static_cast<const int*>(c->d_aux),
                                                                  nseq, d_scores);
    LAUNCHED(c);
    CUDA_TRY(c, cudaGetLastError());
    return NW_OK;
  }
  if (hi > lo) {
    st = batch_core(c, d_raw, false, d_offs, h_offs, nseq, d_pairs + 2 * lo, h_pairs + 2 * lo, hi - lo, sc,
                    flags, d_scores + lo, tbk ? d_ops_off + lo : nullptr, d_ops, tbk ? d_ops_len + lo : nullptr);
    if (st) return st;
  }
  const long long* oo = h_ops_off;
  if (tbk && !oo) {
    c->h_oo.resize(npairs + 1);
    st = nw_batch_ops_offsets(reinterpret_cast<const int64_t*>(h_offs), nseq, h_pairs, npairs,
                              reinterpret_cast<int64_t*>(c->h_oo.data()));
    if (st) return fail(c, st, "ops offsets");
    oo = c->h_oo.data();
  }
  if (virt) return NW_OK;
  NCCL_TRY(c, api.GroupStart());
  for (int g = 0; g < G; ++g) {
    const long long a = bd[g], b = bd[g + 1];
    if (b <= a) continue;
    NCCL_TRY(c, api.Broadcast(d_scores + a, d_scores + a, (size_t)(b - a), ncclInt32, g, c->comm, c->stream));
    if (tbk) {
      NCCL_TRY(c, api.Broadcast(d_ops_len + a, d_ops_len + a, (size_t)(b - a), ncclInt32, g, c->comm, c->stream));
      if (oo[b] > oo[a])
        NCCL_TRY(c, api.Broadcast(d_ops + oo[a], d_ops + oo[a], (size_t)(oo[b] - oo[a]), ncclUint8, g, c->comm,
                                  c->stream));
    }
  }
  NCCL_TRY(c, api.GroupEnd());
  return NW_OK;
}

}  // namespace

extern "C" {

nw_status nw_align_batch(nw_ctx* c, const uint8_t* seqs, const int64_t* offs, int32_t nseq,
                         const int32_t* pairs, int64_t npairs, const nw_scoring* sc,
                         uint32_t flags, int32_t* scores, int64_t* ops_off, uint8_t* ops,
                         int32_t* ops_len) {
  if (!c) return NW_E_INVAL;
  const long long* h_offs = reinterpret_cast<const long long*>(offs);
  nw_status st = batch_check(c, h_offs, nseq, pairs, npairs, sc, flags);
  if (st) return st;
  const bool tbk = flags & NW_TRACEBACK;
  if (npairs == 0) {  // nothing to align: outputs may be NULL; ops_off[0] = 0 if given
    if (tbk && ops_off) ops_off[0] = 0;
    return NW_OK;
  }
  if (!scores || (h_offs[nseq] > 0 && !seqs) || (tbk && (!ops_off || !ops || !ops_len)))
    return fail(c, NW_E_INVAL, "NULL argument");
  CUDA_TRY(c, cudaSetDevice(c->device));
  st = upload_tables(c, sc);
  if (st) return st;
  if (tbk) {
    st = nw_batch_ops_offsets(offs, nseq, pairs, npairs, ops_off);
    if (st) return fail(c, st, "ops offsets");
  }
  const long long total = h_offs[nseq];
  // device staging: raw residues, offs, pairs, scores, (ops_off, ops, ops_len)
  const size_t b_raw = (size_t)total + 16, b_offs = sizeof(long long) * (nseq + 1),
               b_pairs = pairs ? sizeof(int) * 2 * npairs : 0, b_sc = sizeof(int) * npairs,
               b_oo = tbk ? sizeof(long long) * (npairs + 1) : 0,
               b_ops = tbk ? (size_t)ops_off[npairs] + 16 : 0, b_ol = tbk ? sizeof(int) * npairs : 0;
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t need = al(b_raw) + al(b_offs) + al(b_pairs) + al(b_sc) + al(b_oo) + al(b_ops) + al(b_ol);
  char* d = nullptr;
  CUDA_TRY(c, cudaMallocAsync(reinterpret_cast<void**>(&d), need, c->stream));
  char* p = d;
  uint8_t* d_raw = reinterpret_cast<uint8_t*>(p); p += al(b_raw);
  long long* d_offs = reinterpret_cast<long long*>(p); p += al(b_offs);
  int* d_pairs = pairs ? reinterpret_cast<int*>(p) : nullptr; p += al(b_pairs);
  int* d_scores = reinterpret_cast<int*>(p); p += al(b_sc);
  long long* d_oo = tbk ? reinterpret_cast<long long*>(p) : nullptr; p += al(b_oo);
  uint8_t* d_ops = tbk ? reinterpret_cast<uint8_t*>(p) : nullptr; p += al(b_ops);
  int* d_ol = tbk ? reinterpret_cast<int*>(p) : nullptr;
  if (total) CUDA_TRY(c, cudaMemcpyAsync(d_raw, seqs, (size_t)total, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(d_offs, offs, b_offs, cudaMemcpyHostToDevice, c->stream));
  if (pairs) CUDA_TRY(c, cudaMemcpyAsync(d_pairs, pairs, b_pairs, cudaMemcpyHostToDevice, c->stream));
  if (tbk) CUDA_TRY(c, cudaMemcpyAsync(d_oo, ops_off, b_oo, cudaMemcpyHostToDevice, c->stream));
  st = (c->comm || c->opt[NW_OPT_DIST_VIRTUAL_WORLD] > 0) ? batch_dist(c, d_raw, d_offs, h_offs, nseq, d_pairs, pairs, npairs, sc, flags, d_scores,
                            d_oo, reinterpret_cast<const long long*>(ops_off), d_ops, d_ol)
               : batch_core(c, d_raw, false, d_offs, h_offs, nseq, d_pairs, pairs, npairs, sc, flags, d_scores,
                            d_oo, d_ops, d_ol);
  if (st) { cudaFreeAsync(d, c->stream); return st; }
  CUDA_TRY(c, cudaMemcpyAsync(scores, d_scores, b_sc, cudaMemcpyDeviceToHost, c->stream));
  if (tbk) {
    CUDA_TRY(c, cudaMemcpyAsync(ops, d_ops, (size_t)ops_off[npairs], cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(ops_len, d_ol, b_ol, cudaMemcpyDeviceToHost, c->stream));
  }
  cudaFreeAsync(d, c->stream);
  return check_deferred(c);
}

nw_status nw_align_batch_dev(nw_ctx* c, const uint8_t* d_seqs, const int64_t* d_offs,
                             const int64_t* h_offs, int32_t nseq, const int32_t* d_pairs,
                             const int32_t* h_pairs, int64_t npairs, const nw_scoring* sc,
                             uint32_t flags, int32_t* d_scores, const int64_t* d_ops_off,
                             uint8_t* d_ops, int32_t* d_ops_len) {
  if (!c) return NW_E_INVAL;
  const long long* ho = reinterpret_cast<const long long*>(h_offs);
  nw_status st = batch_check(c, ho, nseq, h_pairs, npairs, sc, flags);
  if (st) return st;
  const bool tbk = flags & NW_TRACEBACK;
  if (npairs == 0) return NW_OK;  // nothing to align: outputs may be NULL
  if (!d_scores || !d_offs || (ho[nseq] > 0 && !d_seqs) || (d_pairs && !h_pairs) ||
      (!d_pairs && h_pairs) || (tbk && (!d_ops_off || !d_ops || !d_ops_len)))
    return fail(c, NW_E_INVAL, "NULL argument");
  CUDA_TRY(c, cudaSetDevice(c->device));
  st = upload_tables(c, sc);
  if (st) return st;
  if (c->comm || c->opt[NW_OPT_DIST_VIRTUAL_WORLD] > 0)
    return batch_dist(c, d_seqs, reinterpret_cast<const long long*>(d_offs), ho, nseq, d_pairs, h_pairs, npairs,
                      sc, flags, d_scores, reinterpret_cast<const long long*>(d_ops_off), nullptr, d_ops,
                      d_ops_len);
  return batch_core(c, d_seqs, false, reinterpret_cast<const long long*>(d_offs), ho, nseq, d_pairs,
                    h_pairs, npairs, sc, flags, d_scores, reinterpret_cast<const long long*>(d_ops_off),
                    d_ops, d_ops_len);
}

}  // extern "C"

namespace {

// Center-star MSA (R20-R23): all-pairs scores -> center ->
// alignments (center, k) with traceback -> union-gap merge, all on the device;
// the host reads back the center index and the width (two synchronisations).
nw_status msa_core(nw_ctx* c, const uint8_t* d_seqs, const long long* d_offs,
                   const long long* h_offs, int nseq, const nw_scoring* sc, nw_msa** out) {
  const long long P = (long long)nseq * (nseq - 1) / 2;
  const int nal = nseq - 1;
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  // phase 1: scores of every pair, row sums, center
  char* w1 = nullptr;
  const size_t b_sc = al(sizeof(int) * P), b_rs = al(sizeof(long long) * nseq);
  CUDA_TRY(c, cudaMallocAsync(reinterpret_cast<void**>(&w1), b_sc + b_rs + 256, c->stream));
  int* d_sc = reinterpret_cast<int*>(w1);
  long long* d_rs = reinterpret_cast<long long*>(w1 + b_sc);
  int* d_center = reinterpret_cast<int*>(w1 + b_sc + b_rs);
  nw_status st = batch_core(c, d_seqs, false, d_offs, h_offs, nseq, nullptr, nullptr, P, sc,
                            NW_SCORE_ONLY, d_sc, nullptr, nullptr, nullptr);
  if (st) { cudaFreeAsync(w1, c->stream); return st; }
  k_msa_rowsum<<<nseq, 256, 0, c->stream>>>(d_sc, nseq, d_rs);
  LAUNCHED(c);
  k_msa_argmax<<<1, 1024, 0, c->stream>>>(d_rs, nseq, d_center);
  LAUNCHED(c);
  int center = 0;
  CUDA_TRY(c, cudaMemcpyAsync(&center, d_center, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  cudaFreeAsync(w1, c->stream);
  st = check_deferred(c);
  if (st) return st;
  // phase 2: alignments (center, k), k != center, with traceback
  std::vector<int> hp(2 * (size_t)nal), other(nal);
  for (int k = 0, a = 0; k < nseq; ++k)
    if (k != center) { hp[2 * a] = center; hp[2 * a + 1] = k; other[a] = k; ++a; }
  std::vector<long long> oo((size_t)nal + 1);
  if (nw_batch_ops_offsets(reinterpret_cast<const int64_t*>(h_offs), nseq, hp.data(), nal,
                           reinterpret_cast<int64_t*>(oo.data())))
    return fail(c, NW_E_INVAL, "msa ops offsets");
  const int lc = (int)(h_offs[center + 1] - h_offs[center]);
  const size_t b_p = al(sizeof(int) * 2 * nal), b_o = al(sizeof(int) * nal),
               b_oo = al(sizeof(long long) * (nal + 1)), b_ops = al((size_t)oo[nal] + 16),
               b_ol = al(sizeof(int) * nal), b_s2 = al(sizeof(int) * nal),
               b_G = al(sizeof(int) * (lc + 1)), b_B = al(sizeof(long long) * (lc + 1)),
               b_W = al(sizeof(long long));
  char* w2 = nullptr;
  CUDA_TRY(c, cudaMallocAsync(reinterpret_cast<void**>(&w2),
                              b_p + b_o + b_oo + b_ops + b_ol + b_s2 + b_G + b_B + b_W, c->stream));
  char* q = w2;
  int* d_pairs = reinterpret_cast<int*>(q); q += b_p;
  int* d_other = reinterpret_cast<int*>(q); q += b_o;
  long long* d_oo = reinterpret_cast<long long*>(q); q += b_oo;
  uint8_t* d_ops = reinterpret_cast<uint8_t*>(q); q += b_ops;
  int* d_ol = reinterpret_cast<int*>(q); q += b_ol;
  int* d_s2 = reinterpret_cast<int*>(q); q += b_s2;
  int* d_G = reinterpret_cast<int*>(q); q += b_G;
  long long* d_B = reinterpret_cast<long long*>(q); q += b_B;
  long long* d_W = reinterpret_cast<long long*>(q);
  auto bail = [&](nw_status e) { cudaFreeAsync(w2, c->stream); return e; };
  if (nal > 0) {
    CUDA_TRY(c, cudaMemcpyAsync(d_pairs, hp.data(), sizeof(int) * 2 * nal, cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(d_other, other.data(), sizeof(int) * nal, cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(d_oo, oo.data(), sizeof(long long) * (nal + 1), cudaMemcpyHostToDevice, c->stream));
    st = batch_core(c, d_seqs, false, d_offs, h_offs, nseq, d_pairs, hp.data(), nal, sc,
                    NW_TRACEBACK, d_s2, d_oo, d_ops, d_ol);
    if (st) return bail(st);
  }
  // phase 3: union gapping G(r), block starts B(r), width
  CUDA_TRY(c, cudaMemsetAsync(d_G, 0, sizeof(int) * (lc + 1), c->stream));
  if (nal > 0) {
    k_msa_gaps<<<(nal + 3) / 4, 128, 0, c->stream>>>(d_ops, d_oo, d_ol, nal, lc, d_G);
    LAUNCHED(c);
  }
  k_msa_scan<<<1, 1024, 0, c->stream>>>(d_G, lc, d_B, d_W);
  LAUNCHED(c);
  long long W = 0;
  CUDA_TRY(c, cudaMemcpyAsync(&W, d_W, sizeof W, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  // phase 4: rows
  nw_msa* h = new (std::nothrow) nw_msa;
  if (!h) return bail(fail(c, NW_E_NOMEM, "msa handle"));
  h->ctx = c; h->nseq = nseq; h->center = center; h->W = W;
  c->live_msa.push_back(h);
  if (W > 0 && (size_t)nseq * (size_t)W > 0) {
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&h->d_rows), (size_t)nseq * W, c->stream);
    if (e != cudaSuccess) {
      c->live_msa.pop_back();
      delete h;
      return bail(fail(c, NW_E_NOMEM, "msa rows of %lld bytes: %s", (long long)nseq * W, cudaGetErrorString(e)));
    }
    CUDA_TRY(c, cudaMemsetAsync(h->d_rows, '-', (size_t)nseq * W, c->stream));
    if (lc > 0) {
      k_msa_center<<<(lc + 255) / 256, 256, 0, c->stream>>>(d_seqs + h_offs[center], lc, d_G, d_B,
                                                            h->d_rows + (long long)center * W);
      LAUNCHED(c);
    }
    if (nal > 0) {
      k_msa_rows<<<(nal + 3) / 4, 128, 0, c->stream>>>(d_ops, d_oo, d_ol, d_other, d_seqs, d_offs,
                                                      nal, d_G, d_B, h->d_rows, W);
      LAUNCHED(c);
    }
  }
  cudaFreeAsync(w2, c->stream);
  CUDA_TRY(c, cudaGetLastError());
  *out = h;
  return NW_OK;
}

}  // namespace

extern "C" {

nw_status nw_msa_center_star(nw_ctx* c, const uint8_t* seqs, const int64_t* offs, int32_t nseq,
                             const nw_scoring* sc, nw_msa** out) {
  if (!c) return NW_E_INVAL;
  if (!out || !offs) return fail(c, NW_E_INVAL, "NULL argument");
  *out = nullptr;
  if (nseq < 2) return fail(c, NW_E_INVAL, "center star needs nseq >= 2 (S:295)");
  const long long* h_offs = reinterpret_cast<const long long*>(offs);
  const long long P = (long long)nseq * (nseq - 1) / 2;
  nw_status st = batch_check(c, h_offs, nseq, nullptr, P, sc, 0);
  if (st) return st;
  if (h_offs[nseq] > 0 && !seqs) return fail(c, NW_E_INVAL, "NULL argument");
  CUDA_TRY(c, cudaSetDevice(c->device));
  st = upload_tables(c, sc);
  if (st) return st;
  const long long total = h_offs[nseq];
  char* d = nullptr;
  const size_t b_raw = ((size_t)total + 16 + 255) & ~size_t(255);
  CUDA_TRY(c, cudaMallocAsync(reinterpret_cast<void**>(&d), b_raw + sizeof(long long) * (nseq + 1), c->stream));
  uint8_t* d_raw = reinterpret_cast<uint8_t*>(d);
  long long* d_offs = reinterpret_cast<long long*>(d + b_raw);
  if (total) CUDA_TRY(c, cudaMemcpyAsync(d_raw, seqs, (size_t)total, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(d_offs, offs, sizeof(long long) * (nseq + 1), cudaMemcpyHostToDevice, c->stream));
  st = msa_core(c, d_raw, d_offs, h_offs, nseq, sc, out);
  cudaFreeAsync(d, c->stream);
  if (!st) st = check_deferred(c);
  if (st && *out) { nw_msa_free(*out); *out = nullptr; }
  return st;
}

nw_status nw_msa_center_star_dev(nw_ctx* c, const uint8_t* d_seqs, const int64_t* d_offs,
                                 const int64_t* h_offs, int32_t nseq, const nw_scoring* sc,
                                 nw_msa** out) {
  if (!c) return NW_E_INVAL;
  if (!out || !h_offs || !d_offs) return fail(c, NW_E_INVAL, "NULL argument");
  *out = nullptr;
  if (nseq < 2) return fail(c, NW_E_INVAL, "center star needs nseq >= 2 (S:295)");
  const long long* ho = reinterpret_cast<const long long*>(h_offs);
  nw_status st = batch_check(c, ho, nseq, nullptr, (long long)nseq * (nseq - 1) / 2, sc, 0);
  if (st) return st;
  if (ho[nseq] > 0 && !d_seqs) return fail(c, NW_E_INVAL, "NULL argument");
  CUDA_TRY(c, cudaSetDevice(c->device));
  st = upload_tables(c, sc);
  if (st) return st;
  return msa_core(c, d_seqs, reinterpret_cast<const long long*>(d_offs), ho, nseq, sc, out);
}

nw_status nw_msa_info(const nw_msa* h, int32_t* center, int64_t* width) {
  if (!h || !center || !width) return NW_E_INVAL;
  *center = h->center;
  *width = h->W;
  return NW_OK;
}

const uint8_t* nw_msa_rows_dev(const nw_msa* h) { return h ? h->d_rows : nullptr; }

nw_status nw_msa_rows(nw_ctx* c, const nw_msa* h, uint8_t* rows, int64_t row_stride) {
  if (!c || !h) return c ? fail(c, NW_E_INVAL, "NULL argument") : NW_E_INVAL;
  if (h->ctx != c) return fail(c, NW_E_STATE, "msa handle belongs to another context");
  if (row_stride < h->W) return fail(c, NW_E_TRUNC, "row_stride %lld < width %lld", (long long)row_stride, h->W);
  if (h->W == 0) return NW_OK;
  if (!rows) return fail(c, NW_E_INVAL, "NULL argument");
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaMemcpy2DAsync(rows, (size_t)row_stride, h->d_rows, (size_t)h->W, (size_t)h->W,
                                (size_t)h->nseq, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return NW_OK;
}

void nw_msa_free(nw_msa* h) {
  if (!h) return;
  if (nw_ctx* c = h->ctx) {
    if (h->d_rows) cudaFreeAsync(h->d_rows, c->stream);
    auto& v = c->live_msa;
    v.erase(std::remove(v.begin(), v.end(), h), v.end());
  }
  delete h;
}

}  // extern "C"

namespace {

// The paper's per-cell kernel: full H and direction grids,
// one thread per cell with acquire/release flags, serial backtrack.
nw_status percell_entry(nw_ctx* c, const uint8_t* a, long long m, const uint8_t* b, long long n,
                        const nw_scoring* sc, bool host, long long* d_score, uint8_t* d_ops,
                        long long* d_len) {
  nw_status st = check_scoring(c, sc);
  if (st) return st;
  st = check_bounds(c, sc, m, n);
  if (st) return st;
  CUDA_TRY(c, cudaSetDevice(c->device));
  st = upload_tables(c, sc);
  if (st) return st;
  constexpr long long R = R_MAX;
  const long long la = pad16(PAD + m + R + PAD), lb = pad16(PAD + n + R + PAD);
  st = grow(c, c->d_codes, c->codes_cap, (size_t)(la + lb));
  if (st) return st;
  ZeroRanges zr{{c->d_codes, nullptr, nullptr, nullptr}, {la + lb, 0, 0, 0}};
  st = init_small(c, 8, zr);
  if (st) return st;
  uint8_t *ca, *cb;
  st = stage_pair(c, a, m, b, n, host, &ca, &cb);
  if (st) return st;
  const size_t cells = (size_t)(m + 1) * (size_t)(n + 1);
  const size_t b_H = (cells * sizeof(int) + 255) & ~size_t(255);
  char* mem = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&mem), b_H + cells + (size_t)(m + n) + 16, c->stream);
  if (e != cudaSuccess)
    return fail(c, NW_E_NOMEM, "per-cell grids of %zu bytes: %s", b_H + cells, cudaGetErrorString(e));
  int* H = reinterpret_cast<int*>(mem);
  uint8_t* T = reinterpret_cast<uint8_t*>(mem + b_H);
  uint8_t* rev = T + cells;
  k_percell_init<<<c->sm_count * 8, 256, 0, c->stream>>>(H, T, (int)m, (int)n, sc->gap);
  LAUNCHED(c);
  {
    KernelTimer kt(c, 0);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_percell_fill, 256, 0);
    const long long want = (m * n + 255) / 256;
    const int grid = (int)std::max<long long>(1, std::min<long long>(want, (long long)c->sm_count * std::max(per_sm, 1)));
    k_percell_fill<<<grid, 256, 0, c->stream>>>(ca, cb, c->d_prof, sc->K, (int)m, (int)n, sc->gap,
                                                 sc->tie[0], sc->tie[1], sc->tie[2], H, T);
    LAUNCHED(c);
  }
  k_percell_score<<<1, 1, 0, c->stream>>>(H, (int)m, (int)n, d_score);
  LAUNCHED(c);
  {
    KernelTimer kt(c, 1);
    k_percell_walk<<<1, 32, 0, c->stream>>>(T, (int)m, (int)n, rev, d_len);
    LAUNCHED(c);
    k_percell_reverse<<<c->sm_count, 256, 0, c->stream>>>(rev, d_len, d_ops);
    LAUNCHED(c);
  }
  cudaFreeAsync(mem, c->stream);
  CUDA_TRY(c, cudaGetLastError());
  return NW_OK;
}

}  // namespace

extern "C" {

nw_status nw_align_pair_percell_dev(nw_ctx* c, const uint8_t* d_a, int64_t m, const uint8_t* d_b,
                                    int64_t n, const nw_scoring* sc, int64_t* d_score,
                                    uint8_t* d_ops, int64_t* d_len) {
  if (!c) return NW_E_INVAL;
  if ((m > 0 && !d_a) || (n > 0 && !d_b) || !d_score || !d_len || (m + n > 0 && !d_ops))
    return fail(c, NW_E_INVAL, "NULL argument");
  return percell_entry(c, d_a, m, d_b, n, sc, false, reinterpret_cast<long long*>(d_score), d_ops,
                       reinterpret_cast<long long*>(d_len));
}

nw_status nw_align_pair_percell(nw_ctx* c, const uint8_t* a, int64_t m, const uint8_t* b,
                                int64_t n, const nw_scoring* sc, int64_t* score, uint8_t* ops,
                                int64_t cap, int64_t* len) {
  if (!c) return NW_E_INVAL;
  if ((m > 0 && !a) || (n > 0 && !b) || !score || !len) return fail(c, NW_E_INVAL, "NULL argument");
  CUDA_TRY(c, cudaSetDevice(c->device));
  uint8_t* d_ops = nullptr;
  CUDA_TRY(c, cudaMallocAsync(reinterpret_cast<void**>(&d_ops), (size_t)(m + n) + 16, c->stream));
  nw_status st = percell_entry(c, a, m, b, n, sc, true, c->d_score, d_ops, c->d_len);
  if (st) { cudaFreeAsync(d_ops, c->stream); return st; }
  long long hl = 0, hs = 0;
  CUDA_TRY(c, cudaMemcpyAsync(&hs, c->d_score, sizeof hs, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(&hl, c->d_len, sizeof hl, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  st = check_deferred(c);
  if (st) { cudaFreeAsync(d_ops, c->stream); return st; }
  *score = hs;
  *len = hl;
  if (cap < hl) {
    cudaFreeAsync(d_ops, c->stream);
    return fail(c, NW_E_TRUNC, "cap %lld < length %lld", (long long)cap, hl);
  }
  if (hl) CUDA_TRY(c, cudaMemcpyAsync(ops, d_ops, (size_t)hl, cudaMemcpyDeviceToHost, c->stream));
  cudaFreeAsync(d_ops, c->stream);
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return NW_OK;
}

}  // extern "C"

namespace {

// Checkpointed traceback: a score-only
// pass that keeps the H' row at every seg_rows-th row, then, bottom-up, each
// segment is refilled with directions from its checkpoint row (columns only up
// to where the path enters it) and walked to its top row. The refill makes the
// same decisions as a full fill, so the path is the canonical one.
nw_status linear_core(nw_ctx* c, const uint8_t* a, long long m, const uint8_t* b, long long n,
                      const nw_scoring* sc, long long budget, long long* score_out,
                      std::vector<uint8_t>& path) {
  constexpr long long R = R_MAX;
  const long long la = pad16(PAD + m + R + PAD), lb = pad16(PAD + n + R + PAD);
  nw_status st = grow(c, c->d_codes, c->codes_cap, (size_t)(la + lb));
  if (st) return st;
  const long long bstr = bnd_stride(n);
  const long long bbytes = (long long)sizeof(unsigned long long) * 2 * bstr;
  st = grow(c, c->d_bnd, c->bnd_cap, (size_t)bbytes);
  if (st) return st;
  ZeroRanges zr{{c->d_codes, c->d_bnd, nullptr, nullptr}, {la + lb, bbytes, 0, 0}};
  st = init_small(c, 8, zr);
  if (st) return st;
  uint8_t *ca, *cb;
  st = stage_pair(c, a, m, b, n, true, &ca, &cb);
  if (st) return st;
  // segment height: directions take (n + 38) / 4 bytes per row
  // the checkpoint pass is score-only: the packed difference form when it applies
  // (its rows carry V; k_ckpt_prefix turns them into H' for the refills)
  const bool ck_d16 = d16_ok(c, sc) && m >= 32LL * 16 * 150 && !c->opt[NW_OPT_LINEAR_INT32];
  const int kr_ck = ck_d16 ? d16_kr(c, m) : choose_kr(c, m, n, false, sc->K);
  // the packed H' form of §3.16 when it fits: its checkpoint rows already hold H'
  const int ck_reb = (ck_d16 && c->opt[NW_OPT_PAIR_FORM] != 1) ? h16_rebase_groups(c, sc, kr_ck) : 0;
  const long long Rck = 32LL * kr_ck;
  const long long rows_max = std::max<long long>(1, budget / ((n + 38) / 4 + 1));
  const long long K = std::max<long long>(1, rows_max / Rck);
  const long long seg_rows = K * Rck;
  const long long nseg = (m + seg_rows - 1) / seg_rows;
  unsigned long long* ckpt = nullptr;
  if (nseg > 1) {  // one slot per segment boundary, plus one for a last strip ending on one
    const size_t ckb = sizeof(unsigned long long) * (size_t)bstr * (size_t)nseg;
    CUDA_TRY(c, cudaMallocAsync(reinterpret_cast<void**>(&ckpt), ckb, c->stream));
    CUDA_TRY(c, cudaMemsetAsync(ckpt, 0, ckb, c->stream));
  }
  auto done = [&](nw_status e) { if (ckpt) cudaFreeAsync(ckpt, c->stream); return e; };
  st = pair_core(c, ca, m, cb, n, sc, c->d_score, nullptr, kr_ck, ckpt, (int)K, bstr, nullptr, 0, ck_reb);
  if (st) return done(st);
  if (ck_d16 && ck_reb == 0 && nseg > 1) {
    k_ckpt_prefix<<<(unsigned)nseg, 1024, 0, c->stream>>>(ckpt, bstr, (int)n, (int)nseg);
    LAUNCHED(c);
    CUDA_TRY(c, cudaGetLastError());
  }
  CUDA_TRY(c, cudaMemcpyAsync(score_out, c->d_score, sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
  st = check_deferred(c);  // synchronises; reports alphabet errors
  if (st) return done(st);
  std::vector<std::vector<uint8_t>> segs((size_t)nseg);
  long long col = n;  // where the path enters the current segment's bottom row
  uint8_t* d_ops = nullptr;
  CUDA_TRY(c, cudaMallocAsync(reinterpret_cast<void**>(&d_ops), (size_t)(seg_rows + n) + 16, c->stream));
  for (long long sg = nseg - 1; sg >= 0; --sg) {
    const long long r0 = sg * seg_rows, r1 = std::min(m, r0 + seg_rows), mm = r1 - r0;
    if (col == 0) {  // the path reached column 0: straight up to the origin (R7)
      segs[(size_t)sg].assign((size_t)r1, (uint8_t)NW_UP);
      break;
    }
    ZeroRanges zb{{c->d_bnd, nullptr, nullptr, nullptr}, {bbytes, 0, 0, 0}};
    st = init_small(c, 8, zb);  // fresh ticket, error flag and ring tags for this fill
    if (st) break;
    int kr = choose_kr(c, mm, col, true, sc->K);
    // tall refills of DNA-size pairs: the packed H' direction fill (§3.16) at 8 rows per
    // lane, its flags in the int32 layout (NW_OPT_PAIR_FORM = 1: the int32 fill)
    int rf_reb = 0;
    if (ck_d16 && kr >= 8 && c->opt[NW_OPT_PAIR_FORM] != 1 && !c->opt[NW_OPT_LINEAR_INT32] &&
        col >= 128 * ((mm + 255) / 256)) {
      rf_reb = h16_rebase_groups(c, sc, 8);
      if (rf_reb > 0) kr = 8;
    }
    nw_tb* tb = nullptr;
    st = new_tb(c, mm, col, sc, kr, &tb);
    if (st) break;
    const unsigned long long* top = sg > 0 ? ckpt + (sg - 1) * bstr : nullptr;
    // the checkpoint row above segment sg was written by strip sg*K - 1: tag sg*K
    st = pair_core(c, ca + r0, mm, cb, col, sc, c->d_score, tb, kr, nullptr, 0, 0, top,
                   (unsigned)(sg * K), rf_reb);
    int* d_exit = c->d_ints + 6;
    if (!st) st = grow(c, c->d_rev, c->rev_cap, (size_t)(mm + col));
    if (!st) st = traceback_core(c, tb, d_ops, sg == 0, d_exit);
    long long L = 0;
    int ex = 0;
    if (!st) {
      CUDA_TRY(c, cudaMemcpyAsync(&L, c->d_len, sizeof L, cudaMemcpyDeviceToHost, c->stream));
      CUDA_TRY(c, cudaMemcpyAsync(&ex, d_exit, sizeof ex, cudaMemcpyDeviceToHost, c->stream));
      CUDA_TRY(c, cudaStreamSynchronize(c->stream));
      segs[(size_t)sg].resize((size_t)L);
      if (L) CUDA_TRY(c, cudaMemcpy(segs[(size_t)sg].data(), d_ops, (size_t)L, cudaMemcpyDeviceToHost));
    }
    nw_tb_free(tb);
    if (st) break;
    st = check_deferred(c);
    if (st) break;
    col = ex;
  }
  cudaFreeAsync(d_ops, c->stream);
  if (st) return done(st);
  path.clear();
  for (auto& v : segs) path.insert(path.end(), v.begin(), v.end());
  return done(NW_OK);
}

}  // namespace

extern "C" {

nw_status nw_align_pair_linear(nw_ctx* c, const uint8_t* a, int64_t m, const uint8_t* b, int64_t n,
                               const nw_scoring* sc, int64_t dirs_budget, int64_t* score,
                               uint8_t* ops, int64_t cap, int64_t* len) {
  if (!c) return NW_E_INVAL;
  if ((m > 0 && !a) || (n > 0 && !b) || !score || !len) return fail(c, NW_E_INVAL, "NULL argument");
  nw_status st = check_scoring(c, sc);
  if (st) return st;
  st = check_bounds(c, sc, m, n);
  if (st) return st;
  CUDA_TRY(c, cudaSetDevice(c->device));
  st = upload_tables(c, sc);
  if (st) return st;
  if (dirs_budget <= 0) {  // default: half of the free device memory
    size_t fr = 0, tot = 0;
    CUDA_TRY(c, cudaMemGetInfo(&fr, &tot));
    dirs_budget = (int64_t)(fr / 2);
  }
  std::vector<uint8_t> path;
  long long sc_out = 0;
  if (m == 0 || n == 0) {
    sc_out = (long long)sc->gap * (m + n);
    path.assign((size_t)(m + n), (uint8_t)(m > 0 ? NW_UP : NW_LEFT));
  } else {
    st = linear_core(c, a, m, b, n, sc, dirs_budget, &sc_out, path);
    if (st) return st;
  }
  *score = sc_out;
  *len = (int64_t)path.size();
  if (cap < (int64_t)path.size())
    return fail(c, NW_E_TRUNC, "cap %lld < length %lld", (long long)cap, (long long)path.size());
  if (!path.empty()) {
    if (!ops) return fail(c, NW_E_INVAL, "NULL argument");
    memcpy(ops, path.data(), path.size());
  }
  return NW_OK;
}

}  // extern "C"

extern "C" {

nw_status nw_cooptimal(nw_ctx* c, const uint8_t* a, int64_t m, const uint8_t* b, int64_t n,
                       const nw_scoring* sc, int32_t cap, uint64_t* count, int32_t* saturated,
                       uint8_t* ops, int64_t ops_cap, int64_t* ops_off, int32_t* nfound) {
  if (!c) return NW_E_INVAL;
  if ((m > 0 && !a) || (n > 0 && !b) || !count || !saturated || cap < 0)
    return fail(c, NW_E_INVAL, "NULL argument or cap < 0");
  if (cap > 0 && (!ops_off || !nfound || (ops_cap > 0 && !ops)))
    return fail(c, NW_E_INVAL, "NULL argument");
  nw_status st = check_scoring(c, sc);
  if (st) return st;
  st = check_bounds(c, sc, m, n);
  if (st) return st;
  CUDA_TRY(c, cudaSetDevice(c->device));
  st = upload_tables(c, sc);
  if (st) return st;
  constexpr long long R = R_MAX;
  const long long la = pad16(PAD + m + R + PAD), lb = pad16(PAD + n + R + PAD);
  st = grow(c, c->d_codes, c->codes_cap, (size_t)(la + lb));
  if (st) return st;
  ZeroRanges zr{{c->d_codes, nullptr, nullptr, nullptr}, {la + lb, 0, 0, 0}};
  st = init_small(c, 8, zr);
  if (st) return st;
  uint8_t *ca, *cb;
  st = stage_pair(c, a, m, b, n, true, &ca, &cb);
  if (st) return st;
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const long long stride = (n + 1 + 3) & ~3ll;  // mask bytes per row
  const int S = (int)((m + 31) / 32);
  const size_t b_h = al(sizeof(int) * 2 * (n + 1)), b_n = al(sizeof(unsigned long long) * 2 * (n + 1)),
               b_c = al(sizeof(unsigned long long)), b_p = al(sizeof(int) * ((size_t)S + 1)),
               b_m = cap > 0 ? al((size_t)(m + 1) * (size_t)stride) : 0,
               b_s = cap > 0 ? al((size_t)(m + n + 1)) : 0, b_o = cap > 0 ? al((size_t)ops_cap + 1) : 0,
               b_oo = cap > 0 ? al(sizeof(long long) * ((size_t)cap + 1)) : 0, b_nf = al(sizeof(int));
  char* mem = nullptr;
  const size_t total = b_h + b_n + b_c + b_p + b_m + 2 * b_s + b_o + b_oo + b_nf;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&mem), total, c->stream);
  if (e != cudaSuccess) return fail(c, NW_E_NOMEM, "co-optimal buffers of %zu bytes: %s", total, cudaGetErrorString(e));
  char* q = mem;
  int* rowH = reinterpret_cast<int*>(q); q += b_h;
  unsigned long long* rowN = reinterpret_cast<unsigned long long*>(q); q += b_n;
  unsigned long long* d_count = reinterpret_cast<unsigned long long*>(q); q += b_c;
  int* d_prog = reinterpret_cast<int*>(q); q += b_p;
  uint8_t* d_mask = cap > 0 ? reinterpret_cast<uint8_t*>(q) : nullptr; q += b_m;
  uint8_t* d_rev = reinterpret_cast<uint8_t*>(q); q += b_s;
  uint8_t* d_trial = reinterpret_cast<uint8_t*>(q); q += b_s;
  uint8_t* d_ops = reinterpret_cast<uint8_t*>(q); q += b_o;
  long long* d_oo = reinterpret_cast<long long*>(q); q += b_oo;
  int* d_nf = reinterpret_cast<int*>(q);
  CUDA_TRY(c, cudaMemsetAsync(d_prog, 0, b_p, c->stream));
  unsigned long long one = 1;
  CUDA_TRY(c, cudaMemcpyAsync(d_count, &one, sizeof one, cudaMemcpyHostToDevice, c->stream));  // m or n = 0
  if (d_mask) {  // borders (R24): row 0 = L, column 0 = U, origin 0
    CUDA_TRY(c, cudaMemsetAsync(d_mask, 4, (size_t)stride, c->stream));
    CUDA_TRY(c, cudaMemsetAsync(d_mask, 0, 1, c->stream));
    if (m > 0) CUDA_TRY(c, cudaMemset2DAsync(d_mask + stride, (size_t)stride, 2, 1, (size_t)m, c->stream));
  }
  if (m > 0 && n > 0) {
    KernelTimer kt(c, 0);
    nwk::CooptArgs A;
    A.a = ca; A.b = cb; A.prof = c->d_prof; A.K = sc->K; A.m = (int)m; A.n = (int)n; A.S = S;
    A.ticket = c->d_ints; A.progress = d_prog; A.rowH = rowH; A.rowN = rowN;
    A.mask = reinterpret_cast<uint32_t*>(d_mask); A.stride = stride; A.count = d_count;
    const int grid = std::min(S, c->sm_count * 8);
    k_coopt_fill<<<grid, 32, 0, c->stream>>>(A);
    LAUNCHED(c);
  }
  if (cap > 0) {
    KernelTimer kt(c, 1);
    const size_t sm_need = 2 * (size_t)(m + n + 1);
    const int use_smem = sm_need <= 200 * 1024;
    if (use_smem) cudaFuncSetAttribute(k_coopt_enum, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_need);
    k_coopt_enum<<<1, 32, use_smem ? sm_need : 0, c->stream>>>(
        d_mask, (int)m, (int)n, stride, sc->tie[0], sc->tie[1], sc->tie[2], cap, d_ops, ops_cap,
        d_oo, d_nf, d_rev, d_trial, use_smem);
    LAUNCHED(c);
  }
  unsigned long long hc = 0;
  int hnf = 0;
  auto bail = [&](nw_status x) { cudaFreeAsync(mem, c->stream); return x; };
  if (cudaMemcpyAsync(&hc, d_count, sizeof hc, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess)
    return bail(fail(c, NW_E_CUDA, "copy"));
  if (cap > 0 && cudaMemcpyAsync(&hnf, d_nf, sizeof hnf, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess)
    return bail(fail(c, NW_E_CUDA, "copy"));
  st = check_deferred(c);
  if (st) return bail(st);
  *count = hc;
  *saturated = hc == ~0ull ? 1 : 0;
  if (cap > 0) {
    *nfound = hnf;
    CUDA_TRY(c, cudaMemcpy(ops_off, d_oo, sizeof(long long) * ((size_t)hnf + 1), cudaMemcpyDeviceToHost));
    if (ops_off[hnf] > 0) CUDA_TRY(c, cudaMemcpy(ops, d_ops, (size_t)ops_off[hnf], cudaMemcpyDeviceToHost));
  }
  return bail(NW_OK);
}

}  // extern "C"
