/*
 * nw.h -- C ABI of the B200-native Needleman-Wunsch hot path
 *         (arXiv 2412.21103; PAPER.md = the paper text, "P:n" = its line n).
 *
 * What the library computes (DESIGN.md §1 states the readings R1-R22):
 *   Grid      (m+1) x (n+1), sequence a on the rows i, b on the columns j.   P:24, P:33-34 (Sec. 2.1)
 *   Borders   H(0,0)=0, H(i,0)=i*g, H(0,j)=j*g.                              P:43-45 (Sec. 2.2)
 *   Fill      H(i,j) = max(H(i-1,j-1)+s(a_i,b_j), H(i-1,j)+g, H(i,j-1)+g)    P:47-54 (Sec. 2.3, Eq. 1, additive reading R1)
 *   Codes     1 = diagonal, 2 = vertical (gap in b), 3 = horizontal (gap in a),
 *             the first maximal candidate in the caller's tie order.           P:90 (Sec. 3.1)
 *   Traceback from (m,n) to (0,0) along the codes, emitted in forward order.  P:65-72 (Sec. 2.4)
 *   Batch     many independent pairs, e.g. all p<q of a set: n(n-1)/2.        P:131-135 (Sec. 3.2, Eq. 2)
 *
 * Conventions shared by every entry point:
 *   - Residues are bytes; each must occur in scoring->alphabet (case-sensitive,
 *     callers upper-case first, R10). Otherwise NW_E_ALPHABET and
 *     nw_last_bad_pos() gives the first bad position (positions in b follow
 *     those of a; in a batch, the offset into `seqs`).
 *   - Host-pointer entry points are synchronous: they copy inputs to the device,
 *     run on the context's stream, copy results back and synchronise.
 *   - "_dev" entry points take device pointers, enqueue on the context's
 *     stream and return without synchronising; results are valid once the
 *     stream reaches that point. Validation that needs only sizes and the
 *     scoring happens before anything is enqueued.
 *   - Nothing aborts or throws. Every call returns an nw_status; on error the
 *     outputs are unspecified (except *len on NW_E_TRUNC) and
 *     nw_last_error(ctx) describes it.
 *   - Scores fit int32 for every accepted input: the library rejects inputs
 *     whose proven score bound |H| <= (m+n)*max(|g|, |s|) exceeds 2^30
 *     (NW_E_OVERFLOW) (R11).
 *   - One context per host thread; contexts are independent.
 */
#ifndef NW_B200_H
#define NW_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  NW_OK = 0,
  NW_E_INVAL = 1,     /* bad argument: gap >= 0, match <= mismatch, tie not a permutation of {1,2,3},
                         K out of range, NULL pointer, negative length, cap < m+n in _dev traceback */
  NW_E_ALPHABET = 2,  /* a residue is not in the alphabet (see nw_last_bad_pos) */
  NW_E_OVERFLOW = 3,  /* sizes or score bound do not fit the int32 device arithmetic */
  NW_E_NOMEM = 4,     /* device or host allocation failed */
  NW_E_CUDA = 5,      /* a CUDA runtime error (message in nw_last_error) */
  NW_E_TRUNC = 6,     /* ops buffer too small: *len holds the required length */
  NW_E_STATE = 7,     /* traceback handle belongs to another context or holds no directions */
  NW_E_DEADLOCK = 8,  /* an inter-warp dependency wait exceeded its watchdog */
  NW_E_COMM = 9       /* NCCL could not be loaded, or a collective / communicator failed
                         (dist contexts, nw_ctx_set_dist) */
} nw_status;

enum { NW_DIAG = 1, NW_UP = 2, NW_LEFT = 3 }; /* 1 diagonal, 2 vertical, 3 horizontal */

/* Scoring inputs (north_star: "sequences, alphabet, match/mismatch/gap scores and a
 * fixed traceback tie-break order"). All pointers are HOST pointers, read during the call.
 *   match, mismatch  s(x,y) when subst == NULL (+1 / -1). Requires match > mismatch.
 *   gap              linear gap score g (-1). Requires g < 0.
 *   subst            optional K*K int32 row-major matrix over `alphabet` (e.g. BLOSUM62);
 *                    when given, match/mismatch are ignored. All scores in [-31, 31]
 *                    (int8 device profile of s - 2g), 1 <= -g <= 48.
 *   alphabet, K      the K symbols, 1 <= K <= 64 (DNA "ACGT", protein 20 letters).
 *   tie              permutation of {NW_DIAG, NW_UP, NW_LEFT}, highest priority first;
 *                    {1,2,3} = diagonal > vertical > horizontal (default, P:90 code order). */
typedef struct {
  int32_t match;
  int32_t mismatch;
  int32_t gap;
  const int32_t *subst;
  const char *alphabet;
  int32_t K;
  uint8_t tie[3];
} nw_scoring;

typedef struct nw_ctx nw_ctx; /* device, stream, workspace, last error */
typedef struct nw_tb nw_tb;   /* 2-bit packed directions of one filled pair, resident on the device */

/* Create a context on CUDA device `device`, enqueuing on `cuda_stream`
 * (a cudaStream_t; NULL = the legacy default stream). *out owned by the caller,
 * released with nw_ctx_destroy. */
nw_status nw_ctx_create(int device, void *cuda_stream, nw_ctx **out);
void nw_ctx_destroy(nw_ctx *ctx);
const char *nw_strerror(nw_status st);
const char *nw_last_error(const nw_ctx *ctx);
int64_t nw_last_bad_pos(const nw_ctx *ctx);

/* ---- nw_score_only: H(m,n) in linear device memory (no directions). ----
 * Fill of Sec. 2.2-2.3; only strip-boundary rows are kept (O(n) memory).
 * a: m residues, b: n residues (m, n >= 0). *score receives H(m,n). */
nw_status nw_score_only(nw_ctx *ctx, const uint8_t *a, int64_t m, const uint8_t *b, int64_t n,
                        const nw_scoring *sc, int64_t *score);
/* Device variant: d_a, d_b device residues; d_score device int64. Alphabet errors are
 * detected on the device and reported by the next synchronising call on ctx
 * (nw_ctx_sync) as NW_E_ALPHABET. */
nw_status nw_score_only_dev(nw_ctx *ctx, const uint8_t *d_a, int64_t m, const uint8_t *d_b,
                            int64_t n, const nw_scoring *sc, int64_t *d_score);

/* ---- nw_align_pair: fill + 2-bit directions kept on the device. ----
 * Fill of Sec. 2.2-2.3 plus the P:90 code of every interior cell, packed at 2 bits
 * per cell in HBM. *score receives H(m,n). *tb receives a handle owned by the caller
 * (nw_tb_free), valid only with this ctx, consumed by nw_traceback. tb may be NULL
 * (score only, directions discarded). */
nw_status nw_align_pair(nw_ctx *ctx, const uint8_t *a, int64_t m, const uint8_t *b, int64_t n,
                        const nw_scoring *sc, int64_t *score, nw_tb **tb);
nw_status nw_align_pair_dev(nw_ctx *ctx, const uint8_t *d_a, int64_t m, const uint8_t *d_b,
                            int64_t n, const nw_scoring *sc, int64_t *d_score, nw_tb **tb);

/* ---- nw_traceback: the backtracking of Sec. 2.4. ----
 * Walks the directions of `tb` from (m,n) to (0,0) and writes the path's codes
 * (1/2/3) in forward order (first alignment column first) to ops[0..len).
 * max(m,n) <= len <= m+n. Host variant: if cap < len returns NW_E_TRUNC with *len
 * set (cap = 0 queries the length). */
nw_status nw_traceback(nw_ctx *ctx, const nw_tb *tb, uint8_t *ops, int64_t cap, int64_t *len);
/* Device variant: d_ops device buffer with cap >= m+n (else NW_E_INVAL), d_len device int64. */
nw_status nw_traceback_dev(nw_ctx *ctx, const nw_tb *tb, uint8_t *d_ops, int64_t cap,
                           int64_t *d_len);
void nw_tb_free(nw_tb *tb);

/* ---- nw_align_batch: many independent pairs. ----
 * seqs: concatenated residues; offs[0..nseq]: sequence k is seqs[offs[k]..offs[k+1]).
 * pairs: 2*npairs int32 indices (p, q) = (rows, columns) of each alignment, or NULL for
 *        all p<q in lexicographic order (npairs must then equal nseq*(nseq-1)/2).
 * flags: NW_SCORE_ONLY, or NW_TRACEBACK to also emit every pair's path.
 * scores: npairs int32 (H(m,n) per pair, in pair order).
 * With NW_TRACEBACK: ops_off: npairs+1 int64 filled by the library with the offsets
 *        (ops_off[k] = sum over k' < k of (m_k' + n_k'), the worst-case path lengths),
 *        ops: ops_off[npairs] bytes; pair k's path (forward codes) is at
 *        ops[ops_off[k] .. ops_off[k] + ops_len[k]). Unused otherwise (may be NULL).
 * Workspace (owned by ctx, kept between calls): with NW_TRACEBACK and s - 2g >= 0 for
 * every symbol pair, every pair's decision bits (about m*n/4 bytes each; C4: 7.6 GB)
 * stay in device memory until a second kernel walks them; pairs are processed in
 * waves that fit half the free device memory, NW_E_NOMEM if one pair does not. The
 * score and paths do not depend on the order pairs are processed in. */
#define NW_SCORE_ONLY 0u
#define NW_TRACEBACK 1u
nw_status nw_align_batch(nw_ctx *ctx, const uint8_t *seqs, const int64_t *offs, int32_t nseq,
                         const int32_t *pairs, int64_t npairs, const nw_scoring *sc,
                         uint32_t flags, int32_t *scores, int64_t *ops_off, uint8_t *ops,
                         int32_t *ops_len);
/* Device variant: every array is a device pointer (offs/pairs read by the host too:
 * pass host copies in h_offs / h_pairs, used for sizing and length binning;
 * h_pairs may be NULL when pairs is NULL). ops_off is then a device array the
 * caller fills (e.g. from the host prefix sum nw_batch_ops_offsets). */
nw_status nw_align_batch_dev(nw_ctx *ctx, const uint8_t *d_seqs, const int64_t *d_offs,
                             const int64_t *h_offs, int32_t nseq, const int32_t *d_pairs,
                             const int32_t *h_pairs, int64_t npairs, const nw_scoring *sc,
                             uint32_t flags, int32_t *d_scores, const int64_t *d_ops_off,
                             uint8_t *d_ops, int32_t *d_ops_len);
/* Host helper: ops_off[0..npairs] worst-case offsets for NW_TRACEBACK (see above). */
nw_status nw_batch_ops_offsets(const int64_t *h_offs, int32_t nseq, const int32_t *h_pairs,
                               int64_t npairs, int64_t *ops_off);

/* ---- distributed context: one process per GPU ----
 * "the total number of alignments is divided by the number of ranks ... the
 * data is then sent to each rank ... gathered back in the main process".
 * nw_dist_unique_id: rank 0 creates the 128-byte NCCL id; the caller hands it to every
 *   rank (any channel: torch.distributed, a file, MPI). NW_E_COMM if NCCL (libnccl.so.2,
 *   loaded at run time) is unavailable. Needs no GPU.
 * nw_ctx_set_dist: collective over the `world` ranks (each calls it with its rank on
 *   its own device's ctx); replaces an earlier communicator. world = 1 is legal (the
 *   collectives then move nothing). NW_E_COMM on NCCL failure.
 * On a dist ctx, nw_align_batch / nw_align_batch_dev take the SAME inputs on every rank
 *   and return the FULL outputs on every rank: each rank aligns the contiguous,
 *   cost-balanced range nw_batch_partition gives it (explicit pairs: pair-index ranges;
 *   pairs = NULL score-only: ranges of the length-descending rank space), then one group
 *   of in-place NCCL broadcasts gathers every range (scores, and with NW_TRACEBACK the
 *   path lengths and ops bytes). Results are identical to a single-GPU call (reading
 *   R18: the partition never changes a result). Asynchronous NCCL failures surface as
 *   NW_E_COMM at the next synchronising call. */
nw_status nw_dist_unique_id(uint8_t id[128]);
nw_status nw_ctx_set_dist(nw_ctx *ctx, int32_t rank, int32_t world, const uint8_t id[128]);
/* This ctx's rank and world (0 / 1 without nw_ctx_set_dist). */
nw_status nw_ctx_dist_info(const nw_ctx *ctx, int32_t *rank, int32_t *world);
/* Host helper (no GPU): bounds[0..world] of the dist batch partition, bounds[r] = the first
 * task of rank r. Tasks are the pairs in pair order, or (pairs == NULL) k_batch's rank
 * space: all p' < q' over the sequences sorted by length descending (stable), row-major.
 * bounds[r] is the first task whose cost prefix (sum of m*n over earlier tasks) reaches
 * r/world of the total, so every range is within one task's cost of total/world. */
nw_status nw_batch_partition(const int64_t *offs, int32_t nseq, const int32_t *pairs,
                             int64_t npairs, int32_t world, int64_t *bounds);

/* ---- column-block wavefront (giant pair across ranks) ----
 * Score-only H(m,n) computed as the multi-GPU pipeline computes it: rows in strips,
 * columns cut into blocks of block_cols (0 = automatic), block b owned by rank b % ranks,
 * strips handed down within a rank and each strip's right boundary column handed to the
 * next rank as tagged 64-bit entries. DNA-size alphabets (K <= 4).
 * With s - 2g >= 0 for every symbol pair the packed difference form runs (U crosses
 * the block edge, V the strip edge; nw_fill_d16.cuh), else int32 H'. Every call tags
 * its entries afresh (a per-context counter), so receive buffers are zeroed once, when
 * allocated, and never between calls; every rank must make the same sequence of
 * column-block calls on its context.
 * nw_score_only_cblock: all `ranks` are virtual ranks on this context's device (one
 *   launch, all warps resident); the result equals nw_score_only's. Host pointers,
 *   synchronous.
 * On a dist context (nw_ctx_set_dist) with world > 1, nw_score_only / nw_score_only_dev
 *   of a pair of >= 2^34 cells run this pipeline across the ranks' GPUs (receive buffers
 *   exchanged once through CUDA IPC, entries stored over NVLink with .sys scope), and one
 *   all-reduce gives every rank H(m,n) (NW_OPT_DIST_PIPELINE overrides the rule). */
nw_status nw_score_only_cblock(nw_ctx *ctx, const uint8_t *a, int64_t m, const uint8_t *b,
                               int64_t n, const nw_scoring *sc, int32_t ranks,
                               int32_t block_cols, int64_t *score);

/* One real rank of the same pipeline (one process per GPU), for callers that manage the
 * peer memory themselves. recv_self: this rank's receive buffer of nw_cblock_recv_bytes(m)
 * bytes, device memory the previous rank can write (a CUDA-IPC / symmetric-memory
 * mapping), zeroed on every rank before the first call; recv_next: the next rank's
 * receive buffer as mapped here. recv_self = NULL uses the buffers of
 * nw_cblock_ipc_export / nw_cblock_ipc_import (NW_E_STATE if there are none).
 * d_a, d_b, d_score device pointers; async on ctx's stream. *d_score receives H(m,n) on
 * the rank owning the last column block and 0 elsewhere (sum across ranks = the score). */
int64_t nw_cblock_recv_bytes(int64_t m);
nw_status nw_score_only_cblock_rank_dev(nw_ctx *ctx, const uint8_t *d_a, int64_t m,
                                        const uint8_t *d_b, int64_t n, const nw_scoring *sc,
                                        int32_t rank, int32_t ranks, int32_t block_cols,
                                        void *recv_self, void *recv_next, int64_t *d_score);
/* CUDA IPC plumbing for the rank entry point: export allocates (once, zeroed) this
 * context's receive buffer for m rows and returns its 64-byte cudaIpcMemHandle; import
 * opens the next rank's handle (kept until replaced or the context is destroyed). */
nw_status nw_cblock_ipc_export(nw_ctx *ctx, int64_t m, uint8_t handle[64]);
nw_status nw_cblock_ipc_import(nw_ctx *ctx, const uint8_t handle[64]);

/* ---- center-star multiple alignment ----
 * The paper's use of the batch path: scores of all n(n-1)/2 pairs (Eq. 2), the
 * center = argmax_p sum_{q != p} score(p, q) (lowest index on ties), every other
 * sequence k aligned to it (center on the rows, canonical traceback of sc->tie),
 * and the "once a gap, always a gap" merge: before center residue r the MSA has
 * G(r) = max_k g_k(r) gap columns (g_k(r) = gaps alignment k opens there), each
 * row's inserted residues left-aligned in them (R20-R23, §3.10).
 * seqs/offs as nw_align_batch (nseq >= 2, else NW_E_INVAL). Synchronous; on
 * success *out owns device rows [nseq][width] (input order, '-' = gap). Errors as
 * nw_align_batch; *out is NULL on error. */
typedef struct nw_msa nw_msa;
nw_status nw_msa_center_star(nw_ctx *ctx, const uint8_t *seqs, const int64_t *offs, int32_t nseq,
                             const nw_scoring *sc, nw_msa **out);
/* Device inputs (d_seqs, d_offs on ctx's device; h_offs the host copy of d_offs). */
nw_status nw_msa_center_star_dev(nw_ctx *ctx, const uint8_t *d_seqs, const int64_t *d_offs,
                                 const int64_t *h_offs, int32_t nseq, const nw_scoring *sc,
                                 nw_msa **out);
/* Center index and number of columns. */
nw_status nw_msa_info(const nw_msa *msa, int32_t *center, int64_t *width);
/* Copy the rows to host memory: row p at rows + p*row_stride (row_stride >= width,
 * else NW_E_TRUNC). Synchronous. */
nw_status nw_msa_rows(nw_ctx *ctx, const nw_msa *msa, uint8_t *rows, int64_t row_stride);
/* Device pointer to the rows ([nseq][width], owned by msa). */
const uint8_t *nw_msa_rows_dev(const nw_msa *msa);
void nw_msa_free(nw_msa *msa);

/* ---- checkpointed traceback for pairs whose directions do not fit ----
 * Score + canonical traceback of one pair keeping at most ~dirs_budget bytes of
 * 2-bit directions on the device (<= 0: half of the free memory): a score-only
 * pass stores the H' row every seg_rows rows (seg_rows from the budget), then
 * segments are refilled with directions bottom-up from their checkpoint row and
 * walked to their top row. Same score and ops as nw_align_pair
 * + nw_traceback for every input (the refill repeats the same decisions).
 * Host pointers, synchronous; ops/cap/len as nw_traceback (NW_E_TRUNC with *len
 * set if cap < len); extra device memory ~ 8 (n + 66) bytes per checkpoint. */
nw_status nw_align_pair_linear(nw_ctx *ctx, const uint8_t *a, int64_t m, const uint8_t *b,
                               int64_t n, const nw_scoring *sc, int64_t dirs_budget,
                               int64_t *score, uint8_t *ops, int64_t cap, int64_t *len);

/* ---- co-optimal alignments ----
 * *count = number of optimal global alignments (paths from (m,n) to (0,0) along
 * branches whose candidate equals H, borders forced), saturating at 2^64-1
 * (*saturated = 1 then). With cap > 0 also the first cap of them in depth-first
 * order, each cell's optimal branches tried in the tie order (the first is the
 * canonical traceback; R24-R25, §3.13): path k is ops[ops_off[k] ..
 * ops_off[k+1]) (forward codes 1/2/3), *nfound <= cap paths; enumeration stops
 * early if ops_cap bytes are used up. Needs (m+1)(n+1) bytes of device memory
 * for the branch masks when cap > 0. Host pointers, synchronous. */
nw_status nw_cooptimal(nw_ctx *ctx, const uint8_t *a, int64_t m, const uint8_t *b, int64_t n,
                       const nw_scoring *sc, int32_t cap, uint64_t *count, int32_t *saturated,
                       uint8_t *ops, int64_t ops_cap, int64_t *ops_off, int32_t *nfound);

/* ---- the paper's per-cell kernel, corrected ----
 * Ablation baseline, not the product path: one thread per cell spinning on its
 * up/left neighbours' direction codes (acquire/release), full H (int32) and
 * direction grids ((m+1)(n+1) x 5 bytes of device memory, NW_E_NOMEM if they do
 * not fit), serial backtrack. Same results as nw_align_pair +
 * nw_traceback. Host variant: synchronous, ops/cap/len as nw_traceback
 * (NW_E_TRUNC with *len set if cap < len). Device variant: d_ops holds m+n
 * bytes, *d_len the path length; async on ctx's stream. */
nw_status nw_align_pair_percell(nw_ctx *ctx, const uint8_t *a, int64_t m, const uint8_t *b,
                                int64_t n, const nw_scoring *sc, int64_t *score, uint8_t *ops,
                                int64_t cap, int64_t *len);
nw_status nw_align_pair_percell_dev(nw_ctx *ctx, const uint8_t *d_a, int64_t m, const uint8_t *d_b,
                                    int64_t n, const nw_scoring *sc, int64_t *d_score,
                                    uint8_t *d_ops, int64_t *d_len);

/* Wait for the context's stream and report any deferred device-side error
 * (alphabet violations, watchdog) raised by earlier _dev calls. The error flags
 * are sticky: an error raised by any _dev call since the last synchronising call
 * on ctx (this one, or any host-pointer entry point) is reported then, even if
 * later calls succeeded; the first bad position among them is kept. Reporting
 * clears the flags. */
nw_status nw_ctx_sync(nw_ctx *ctx);

/* ---- tuning and test options (explicit context state; nothing reads the environment) ----
 * Every option defaults to 0 = the measured default. They select
 * among kernels that all compute the same results (the parity tests run each
 * setting against the oracle), or shape test-only behaviour. Values < 0 or an
 * unknown option -> NW_E_INVAL. */
enum {
  NW_OPT_ROWS_PER_LANE = 0,    /* single-pair int32 fill: rows per lane 2,4,5,6,8 (10,12 with directions) */
  NW_OPT_D16_FORCE = 1,        /* score-only pair: packed difference form at this many rows per lane */
  NW_OPT_D16_KR = 2,           /* rows per lane of the tall-pair difference form (even, 12..32) */
  NW_OPT_NO_D16 = 3,           /* 1: never use the packed difference forms */
  NW_OPT_TALL_KR8 = 4,         /* 1: tall direction fills always at 8 rows per lane */
  NW_OPT_POLL_NS = 5,          /* back-off (ns) between re-polls of a late boundary entry */
  NW_OPT_TB_STEP = 6,          /* sampled-exit spacing in columns (power of two) */
  NW_OPT_TB_BAND = 7,          /* sampled exits per strip (multiple of 32) */
  NW_OPT_BATCH_KR16 = 8,       /* packed batch traceback strips: 8 or 16 rows per lane */
  NW_OPT_BATCH_NO_TRANSPOSE = 9,  /* 1: batch pairs always filled in their own orientation */
  NW_OPT_BATCH_TB_BUDGET = 10, /* bytes of kept decision words per batch wave (forces waves) */
  NW_OPT_HOST_PLAN = 11,       /* 1: plan large traceback batches on the host, not the device */
  NW_OPT_LINEAR_INT32 = 12,    /* 1: checkpoint pass of nw_align_pair_linear in int32 strips */
  NW_OPT_CBLOCK_WARPS_PER_SM = 13, /* warps per SM of the column-block launch (default 8) */
  NW_OPT_HOST_PROFILE = 14,    /* 1: print host-side phase times of batch calls to stderr */
  NW_OPT_WATCHDOG_POLLS = 15,  /* re-polls of a late boundary entry before NW_E_DEADLOCK (0: 2^28) */
  NW_OPT_TEST_WITHHOLD = 16,   /* test only: 1 + the strip whose bottom row is never published
                                  (single-pair fills), so its consumer's watchdog must fire */
  NW_OPT_DIST_VIRTUAL_WORLD = 17, /* test only, ctx without nw_ctx_set_dist: batch calls align only
                                     rank DIST_VIRTUAL_RANK's range of a world of this size and
                                     gather nothing (G sequential calls replay G ranks on one GPU) */
  NW_OPT_DIST_VIRTUAL_RANK = 18,
  NW_OPT_DIST_PIPELINE = 19,  /* dist ctx score-only pairs: 0 = column-block pipeline across the
                                 ranks when world > 1 and m*n >= 2^34; 1 = always; 2 = never */
  NW_OPT_D16_CHAINS = 20,      /* packed difference-form score-only pair fills: 2 = two independent
                                 chains per lane (rows per lane % 4 == 0; measured slower on C5),
                                 else one chain (default) */
  NW_OPT_BATCH_U16_KR = 21,    /* score-only packed H' batch sweep: rows per lane 8, 16 or 32, or 1 =
                                 32, 24 or 16 per pair, whichever sweeps less weighted area (0: by
                                 the median sequence length: 1 from 1,024, else 16 or 8) */
  NW_OPT_BATCH_BND_GLOBAL = 22, /* 1: the packed H' batch sweep keeps its boundary rows in global
                                  scratch instead of shared memory */
  NW_OPT_PAIR_FORM = 23,       /* DNA-size alphabets with s - 2g >= 0. 0 (default): tall score-only
                                  pairs, the column-block pipeline and the checkpoint pass of
                                  nw_align_pair_linear in packed H' with a moving base (nw_fill_h16),
                                  direction fills at 8+ rows per lane with long rows (n >= 128 x
                                  strips, e.g. the checkpointed refills) in its direction form;
                                  1 = the packed difference form / int32 fills throughout;
                                  2 = as 0, plus every direction fill at 4 or 8 rows per lane */
  NW_OPT_H16_REBASE = 24,      /* packed H' pair sweep: rebase period in 8-step groups (power of two,
                                  0: the largest <= 64 the value range allows); test hook */
  NW_OPT_H16_KR = 25,          /* rows per lane of the packed H' pair sweep (even, 12..32; 0: rule) */
  NW_OPT_BATCH_MIX_W = 26,     /* packed H' batch sweep, mixed strip heights: relative cost (x1000) of
                                  a 512-row strip's cell vs a 1,024-row one (0: 1100) */
  NW_OPT_BATCH_MIX_W24 = 27,   /* the same for a 768-row strip's cell (0: 1040) */
  NW_OPT_COUNT_ = 28
};
nw_status nw_ctx_set_option(nw_ctx *ctx, int32_t option, int64_t value);
/* Current value, or -1 for a NULL ctx / unknown option. */
int64_t nw_ctx_get_option(const nw_ctx *ctx, int32_t option);

/* Number of library kernels launched on this context so far (bench accounting). */
int64_t nw_ctx_launches(const nw_ctx *ctx);

/* Kernel timing (bench accounting). With enable != 0 the context brackets every
 * launch of its hot kernels with CUDA events recorded on its own stream:
 * class 0 = the DP fill (single-pair or batch kernel), class 1 = the traceback
 * (walk + reverse). nw_ctx_kernel_time synchronises, returns the summed event
 * milliseconds and launch count of one class since the last read, and resets it. */
nw_status nw_ctx_set_timing(nw_ctx *ctx, int enable);
nw_status nw_ctx_kernel_time(nw_ctx *ctx, int kernel_class, double *total_ms, int64_t *launches);

#ifdef __cplusplus
}
#endif
#endif /* NW_B200_H */
