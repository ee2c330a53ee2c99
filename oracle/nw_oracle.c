/*
 * nw_oracle.c -- plain, slow, obviously-correct CPU Needleman-Wunsch.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product path
 * (paper_2412_21103_b200/) never links, imports or executes anything in oracle/,
 * and this file shares no code, header, table or constant with it.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, "P:n" = its line n):
 *   - grid of (m+1) x (n+1) cells, sequence a on the rows (i), b on the columns
 *     (j)                                                      P:24, P:33-34 (Sec. 2.1)
 *   - borders H(0,0)=0, H(i,0)=i*g, H(0,j)=j*g ("decreases by one for each
 *     subsequent cell" with g=-1)                              P:43-45 (Sec. 2.2)
 *   - interior H(i,j) = max(H(i-1,j-1)+s(a_i,b_j), H(i-1,j)+g, H(i,j-1)+g),
 *     the additive reading of Eq. 1 (reading R1)    P:47-54 (Sec. 2.3, Eq. 1)
 *   - direction codes 1 = diagonal, 2 = vertical, 3 = horizontal, chosen as the
 *     first maximal candidate in the caller's tie order (R6)
 *                                                              P:90 (Sec. 3.1)
 *   - backtracking from (m,n) along the stored directions     P:65-72 (Sec. 2.4)
 *   - all-pairs p<q of a sequence set, n(n-1)/2 alignments    P:131-135 (Sec. 3.2, Eq. 2)
 *
 * Rules: scalar C, int64 accumulators, full uint8 direction matrix, no
 * blocking, no packing, no reordering beyond the row-major fill the
 * recurrence allows. Status codes: 0 ok, 1 invalid argument, 2 symbol not in
 * alphabet, 6 ops buffer too small (len still reported).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define OR_OK 0
#define OR_INVAL 1
#define OR_ALPHABET 2
#define OR_NOMEM 4
#define OR_TRUNC 6

enum { OR_D = 1, OR_U = 2, OR_L = 3 };

/* Map one residue byte to its index in `alphabet` (uppercase only, R10). */
static int sym_index(const char *alphabet, int K, uint8_t c) {
  for (int k = 0; k < K; ++k)
    if ((uint8_t)alphabet[k] == c) return k;
  return -1;
}

/* s(x, y): the caller's K*K row-major matrix if given, else match/mismatch. */
static int64_t subst_score(const int32_t *subst, int K, int x, int y, int32_t match,
                           int32_t mismatch) {
  if (subst) return subst[x * K + y];
  return x == y ? match : mismatch;
}

static int valid_tie(const uint8_t tie[3]) {
  int seen[4] = {0, 0, 0, 0};
  for (int t = 0; t < 3; ++t) {
    if (tie[t] < 1 || tie[t] > 3 || seen[tie[t]]) return 0;
    seen[tie[t]] = 1;
  }
  return 1;
}

/* Encode a sequence to alphabet indices; returns first bad position or -1. */
static int64_t encode(const uint8_t *s, int64_t len, const char *alphabet, int K, int *out) {
  for (int64_t p = 0; p < len; ++p) {
    int k = sym_index(alphabet, K, s[p]);
    if (k < 0) return p;
    out[p] = k;
  }
  return -1;
}

/*
 * Full fill. Follows Sec. 2.2 (borders) then Sec. 2.3 Eq. 1
 * row by row, recording the P:90 direction code of the first maximal candidate
 * in `tie`. Border codes: T(0,0)=0, T(i,0)=U, T(0,j)=L (R7).
 * H: (m+1)*(n+1) row-major int64, or NULL to keep only rows i-1 and i (then
 *    *score still receives H(m,n)).
 * T: (m+1)*(n+1) row-major uint8, or NULL.
 */
int nw_oracle_fill(const uint8_t *a, int64_t m, const uint8_t *b, int64_t n,
                   const char *alphabet, int32_t K, const int32_t *subst, int32_t match,
                   int32_t mismatch, int32_t gap, const uint8_t tie[3], int64_t *H,
                   uint8_t *T, int64_t *score, int64_t *bad_pos) {
  if (m < 0 || n < 0 || K <= 0 || !alphabet || !valid_tie(tie)) return OR_INVAL;
  const int64_t W = n + 1;
  int *ea = (int *)malloc(sizeof(int) * (size_t)(m + 1));
  int *eb = (int *)malloc(sizeof(int) * (size_t)(n + 1));
  int64_t *rows = H ? NULL : (int64_t *)malloc(sizeof(int64_t) * 2 * (size_t)W);
  if (!ea || !eb || (!H && !rows)) { free(ea); free(eb); free(rows); return OR_NOMEM; }
  int64_t bad = encode(a, m, alphabet, K, ea);
  if (bad < 0) {
    bad = encode(b, n, alphabet, K, eb);
    if (bad >= 0) bad += m; /* positions in b are reported after a's */
  }
  if (bad >= 0) {
    if (bad_pos) *bad_pos = bad;
    free(ea); free(eb); free(rows);
    return OR_ALPHABET;
  }
  /* row(i) points at H's row i, or at one of the two rolling rows */
#define ROW(i) (H ? H + (i) * W : rows + ((i) & 1) * W)
  int64_t *r0 = ROW(0);
  r0[0] = 0;
  if (T) T[0] = 0;
  for (int64_t j = 1; j <= n; ++j) { r0[j] = j * (int64_t)gap; if (T) T[j] = OR_L; }
  for (int64_t i = 1; i <= m; ++i) {
    int64_t *up = ROW(i - 1), *cur = ROW(i);
    cur[0] = i * (int64_t)gap;
    if (T) T[i * W] = OR_U;
    for (int64_t j = 1; j <= n; ++j) {
      int64_t cand[4];
      cand[OR_D] = up[j - 1] + subst_score(subst, K, ea[i - 1], eb[j - 1], match, mismatch);
      cand[OR_U] = up[j] + gap;
      cand[OR_L] = cur[j - 1] + gap;
      int64_t best = cand[OR_D];
      if (cand[OR_U] > best) best = cand[OR_U];
      if (cand[OR_L] > best) best = cand[OR_L];
      cur[j] = best;
      if (T) {
        for (int t = 0; t < 3; ++t)
          if (cand[tie[t]] == best) { T[i * W + j] = tie[t]; break; }
      }
    }
  }
  if (score) *score = ROW(m)[n];
#undef ROW
  free(ea); free(eb); free(rows);
  return OR_OK;
}

/*
 * Backtracking (Sec. 2.4): start at (m,n), follow T until (0,0):
 * D -> (i-1,j-1), U ("vertical") -> (i-1,j), L ("horizontal") -> (i,j-1).
 * Emits the codes in forward order (first column of the alignment first).
 * *len always receives the path length; OR_TRUNC if cap < len.
 */
int nw_oracle_traceback(const uint8_t *T, int64_t m, int64_t n, uint8_t *ops, int64_t cap,
                        int64_t *len) {
  if (!T || m < 0 || n < 0 || !len) return OR_INVAL;
  const int64_t W = n + 1;
  int64_t i = m, j = n, L = 0;
  while (i > 0 || j > 0) {
    uint8_t d = T[i * W + j];
    if (d == OR_D) { --i; --j; }
    else if (d == OR_U) { --i; }
    else if (d == OR_L) { --j; }
    else return OR_INVAL;
    ++L;
  }
  *len = L;
  if (cap < L) return OR_TRUNC;
  /* second walk writes from the back so the result is in forward order */
  i = m; j = n;
  int64_t k = L;
  while (i > 0 || j > 0) {
    uint8_t d = T[i * W + j];
    ops[--k] = d;
    if (d == OR_D) { --i; --j; }
    else if (d == OR_U) { --i; }
    else { --j; }
  }
  return OR_OK;
}

/*
 * Score-only with two rows: the same recurrence as
 * nw_oracle_fill, keeping only rows i-1 and i. Result identical to H(m,n).
 */
int nw_oracle_score(const uint8_t *a, int64_t m, const uint8_t *b, int64_t n,
                    const char *alphabet, int32_t K, const int32_t *subst, int32_t match,
                    int32_t mismatch, int32_t gap, int64_t *score, int64_t *bad_pos) {
  if (m < 0 || n < 0 || K <= 0 || !alphabet || !score) return OR_INVAL;
  int *ea = (int *)malloc(sizeof(int) * (size_t)(m + 1));
  int *eb = (int *)malloc(sizeof(int) * (size_t)(n + 1));
  int64_t *prev = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
  int64_t *cur = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
  if (!ea || !eb || !prev || !cur) { free(ea); free(eb); free(prev); free(cur); return OR_NOMEM; }
  int64_t bad = encode(a, m, alphabet, K, ea);
  if (bad < 0) { bad = encode(b, n, alphabet, K, eb); if (bad >= 0) bad += m; }
  if (bad >= 0) {
    if (bad_pos) *bad_pos = bad;
    free(ea); free(eb); free(prev); free(cur);
    return OR_ALPHABET;
  }
  for (int64_t j = 0; j <= n; ++j) prev[j] = j * (int64_t)gap;
  for (int64_t i = 1; i <= m; ++i) {
    cur[0] = i * (int64_t)gap;
    for (int64_t j = 1; j <= n; ++j) {
      int64_t d = prev[j - 1] + subst_score(subst, K, ea[i - 1], eb[j - 1], match, mismatch);
      int64_t u = prev[j] + gap;
      int64_t l = cur[j - 1] + gap;
      int64_t best = d;
      if (u > best) best = u;
      if (l > best) best = l;
      cur[j] = best;
    }
    int64_t *t = prev; prev = cur; cur = t;
  }
  *score = prev[n];
  free(ea); free(eb); free(prev); free(cur);
  return OR_OK;
}

/* ---- batch: P:131-135, every pair aligned independently, threads over pairs ---- */

typedef struct {
  const uint8_t *seqs; const int64_t *offs; const int32_t *pairs; int64_t npairs;
  const char *alphabet; int32_t K; const int32_t *subst; int32_t match, mismatch, gap;
  int64_t *scores; int status; int64_t next; pthread_mutex_t mu;
} batch_job;

static void *batch_worker(void *arg) {
  batch_job *jb = (batch_job *)arg;
  for (;;) {
    pthread_mutex_lock(&jb->mu);
    int64_t k = jb->next++;
    pthread_mutex_unlock(&jb->mu);
    if (k >= jb->npairs) break;
    int32_t p = jb->pairs[2 * k], q = jb->pairs[2 * k + 1];
    int64_t bad = -1;
    int st = nw_oracle_score(jb->seqs + jb->offs[p], jb->offs[p + 1] - jb->offs[p],
                             jb->seqs + jb->offs[q], jb->offs[q + 1] - jb->offs[q], jb->alphabet,
                             jb->K, jb->subst, jb->match, jb->mismatch, jb->gap, &jb->scores[k],
                             &bad);
    if (st != OR_OK) {
      pthread_mutex_lock(&jb->mu);
      jb->status = st;
      pthread_mutex_unlock(&jb->mu);
    }
  }
  return NULL;
}

/*
 * Score every listed pair (pairs[2k], pairs[2k+1]) of the concatenated set
 * `seqs` with offsets offs[0..nseq]. Pair order is the caller's; results are
 * order-independent, so `nthreads` workers pull pairs from a shared counter.
 */
int nw_oracle_batch_score(const uint8_t *seqs, const int64_t *offs, int32_t nseq,
                          const int32_t *pairs, int64_t npairs, const char *alphabet,
                          int32_t K, const int32_t *subst, int32_t match, int32_t mismatch,
                          int32_t gap, int64_t *scores, int32_t nthreads) {
  if (!seqs || !offs || nseq < 0 || (npairs > 0 && !pairs) || !scores || nthreads < 1)
    return OR_INVAL;
  for (int64_t k = 0; k < npairs; ++k)
    if (pairs[2 * k] < 0 || pairs[2 * k] >= nseq || pairs[2 * k + 1] < 0 || pairs[2 * k + 1] >= nseq)
      return OR_INVAL;
  batch_job jb;
  memset(&jb, 0, sizeof jb);
  jb.seqs = seqs; jb.offs = offs; jb.pairs = pairs; jb.npairs = npairs;
  jb.alphabet = alphabet; jb.K = K; jb.subst = subst;
  jb.match = match; jb.mismatch = mismatch; jb.gap = gap;
  jb.scores = scores; jb.status = OR_OK; jb.next = 0;
  pthread_mutex_init(&jb.mu, NULL);
  pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
  if (!th) return OR_NOMEM;
  for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, batch_worker, &jb);
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  free(th);
  pthread_mutex_destroy(&jb.mu);
  return jb.status;
}
