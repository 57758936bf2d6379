/* The paper's own beam-search selection on the CPU, in C: a timed baseline ("the paper's
 * algorithm on CPU") and a third selection oracle, pinned against the fp64 plain
 * definition in tests/test_paper_heap_c.py.
 *
 * TEST / BASELINE INFRASTRUCTURE ONLY (see oracle/__init__.py): never linked into the product.
 *
 * Per request and decode step, following PAPER.md in order:
 *   1. L361 (section 6.1): each live beam's logits are restricted to its legal children (the trie
 *      of the sorted item list), and the softmax is taken over them: m = max, Z = sum exp(x - m),
 *      lse = m + ln Z, in fp32 (the paper fixes no precision; fp32 as an NPU/GPU kernel would).
 *   2. L376 (section 6.2): log_prob accumulation, c = S_b + (x - lse).
 *   3. L156 (section 2.2.2): each beam's Top-K candidates (K = BW unless given), in descending
 *      order (L376: "the log_prob results for each beam are inherently in descending order");
 *      ties by ascending token (R4).
 *   4. L385 (section 6.2): a global min-heap of size BW; beams are visited in slot order, each
 *      beam's candidates in descending order; a candidate enters iff the heap is not full or its
 *      log_prob exceeds the heap top (strictly), otherwise that beam's traversal terminates.
 *      Extension from the sorted beam scores: once the heap is full and
 *      S_b <= heap top, no candidate of this or a later beam can enter, so the step ends.
 *   5. the heap content sorted (c desc, flat asc) is the next step's beams (L392: fixed-size
 *      state, reused).
 * Requests run on a pthread pool (one request at a time per thread).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int V, nd, w;
  int64_t n_items;
  int maxc;               /* the largest child count of any node */
  int64_t n_nodes[9];     /* nodes per level 0..nd (level 0: the root) */
  uint32_t* first[9];     /* level d: [n_nodes[d] + 1] children of node n are level-(d+1) nodes [first[n], first[n+1]) */
  uint16_t* label[9];     /* level d >= 1: [n_nodes[d]] token leading to the node */
} ph_trie;

void ph_free(ph_trie* t) {
  if (!t) return;
  for (int d = 0; d <= t->nd; ++d) {
    free(t->first[d]);
    free(t->label[d]);
  }
  free(t);
}

/* keys: the sorted, de-duplicated item keys (w bits per token, most significant token first). */
ph_trie* ph_build(const uint64_t* keys, int64_t n, int V, int nd) {
  ph_trie* t = (ph_trie*)calloc(1, sizeof(ph_trie));
  if (!t || nd < 1 || nd > 8 || n < 1) {
    free(t);
    return NULL;
  }
  int w = 1;
  while ((1 << w) < V) ++w;
  t->V = V;
  t->nd = nd;
  t->w = w;
  t->n_items = n;
  /* count the distinct prefixes of every length */
  t->n_nodes[0] = 1;
  for (int d = 1; d <= nd; ++d) {
    const int s = w * (nd - d);
    int64_t c = 0;
    for (int64_t i = 0; i < n; ++i)
      if (i == 0 || (keys[i] >> s) != (keys[i - 1] >> s)) ++c;
    t->n_nodes[d] = c;
  }
  for (int d = 0; d <= nd; ++d) {
    t->first[d] = (uint32_t*)malloc((size_t)(t->n_nodes[d] + 1) * sizeof(uint32_t));
    t->label[d] = (uint16_t*)malloc((size_t)(t->n_nodes[d] > 0 ? t->n_nodes[d] : 1) * sizeof(uint16_t));
    if (!t->first[d] || !t->label[d]) {
      ph_free(t);
      return NULL;
    }
  }
  /* level d + 1 nodes in key order; node j of level d+1 belongs to the parent that is current at
   * level d when it is created, so first[d][parent] is the first child created under it */
  int64_t cur[9];
  for (int d = 0; d <= nd; ++d) cur[d] = -1;
  cur[0] = 0;
  t->first[0][0] = 0;
  for (int64_t i = 0; i < n; ++i) {
    for (int d = 1; d <= nd; ++d) {
      const int s = w * (nd - d);
      if (i == 0 || (keys[i] >> s) != (keys[i - 1] >> s)) {
        const int64_t j = ++cur[d];
        t->label[d][j] = (uint16_t)((keys[i] >> s) & (((uint64_t)1 << w) - 1));
        if (d < nd) t->first[d][j] = (uint32_t)(cur[d + 1] + 1);
      }
    }
  }
  for (int d = 0; d < nd; ++d) t->first[d][t->n_nodes[d]] = (uint32_t)t->n_nodes[d + 1];
  t->maxc = 0;
  for (int d = 0; d < nd; ++d)
    for (int64_t j = 0; j < t->n_nodes[d]; ++j) {
      const int c = (int)(t->first[d][j + 1] - t->first[d][j]);
      if (c > t->maxc) t->maxc = c;
    }
  return t;
}

/* ---- ordering: "better" = larger c, or equal c and smaller flat (R4) -------------- */
typedef struct {
  float c;
  uint32_t flat;
} cand;

static inline int better(cand a, cand b) { return a.c > b.c || (a.c == b.c && a.flat < b.flat); }

/* min-heap under `better`: the root is the worst element */
static void heap_down(cand* h, int n, int i) {
  for (;;) {
    int l = 2 * i + 1, r = l + 1, m = i;
    if (l < n && better(h[m], h[l])) m = l;
    if (r < n && better(h[m], h[r])) m = r;
    if (m == i) return;
    cand x = h[i];
    h[i] = h[m];
    h[m] = x;
    i = m;
  }
}
static void heap_up(cand* h, int i) {
  while (i > 0) {
    int p = (i - 1) / 2;
    if (!better(h[p], h[i])) return;
    cand x = h[i];
    h[i] = h[p];
    h[p] = x;
    i = p;
  }
}
static int cmp_desc(const void* a, const void* b) {
  const cand* x = (const cand*)a;
  const cand* y = (const cand*)b;
  return better(*x, *y) ? -1 : (better(*y, *x) ? 1 : 0);
}

typedef struct {
  const ph_trie* t;
  const float* const* logits;   /* [n_req * nd]: request r, step s: [rows_s][V], rows_0 = 1 */
  int n_req, bw, topk;
  int32_t *parent, *token, *nlive;
  float* score;
  int64_t visits, cands;        /* per worker, summed by the caller */
  int next;                     /* shared request counter (lock-free claim) */
  int* counter;
} job;

static void run_request(job* J, int r, int64_t* visits, int64_t* ncand) {
  const ph_trie* t = J->t;
  const int V = t->V, nd = t->nd, BW = J->bw;
  const int K = (J->topk > 0 && J->topk < BW) ? J->topk : BW;
  uint32_t* node = (uint32_t*)malloc(sizeof(uint32_t) * BW);
  float* S = (float*)malloc(sizeof(float) * BW);
  uint32_t* node2 = (uint32_t*)malloc(sizeof(uint32_t) * BW);
  cand* heap = (cand*)malloc(sizeof(cand) * BW);
  cand* beam = (cand*)malloc(sizeof(cand) * (K + 1));
  float* x = (float*)malloc(sizeof(float) * (t->maxc + 1));
  int n_live = 1;
  node[0] = 0;
  S[0] = 0.0f;
  for (int s = 0; s < nd; ++s) {
    const float* lg = J->logits[(size_t)r * nd + s];
    int hn = 0;
    for (int b = 0; b < n_live; ++b) {
      if (hn == BW && !(S[b] > heap[0].c)) break;   /* sorted beam scores: nothing later can enter */
      const uint32_t fc = t->first[s][node[b]], fe = t->first[s][node[b] + 1];
      const uint16_t* lab = t->label[s + 1];
      const int nc = (int)(fe - fc);
      const float* row = lg + (size_t)b * V;
      float m = -INFINITY;
      for (int q = 0; q < nc; ++q) {
        x[q] = row[lab[fc + q]];
        if (x[q] > m) m = x[q];
      }
      float Z = 0.0f;
      for (int q = 0; q < nc; ++q) Z += expf(x[q] - m);
      const float lse = m + (Z > 1.0f ? logf(Z) : 0.0f);
      /* the beam's Top-K by a size-K min-heap, then sorted descending */
      int bn = 0;
      for (int q = 0; q < nc; ++q) {
        cand cd = {S[b] + (x[q] - lse), (uint32_t)b * (uint32_t)V + lab[fc + q]};
        if (bn < K) {
          beam[bn] = cd;
          heap_up(beam, bn++);
        } else if (better(cd, beam[0])) {
          beam[0] = cd;
          heap_down(beam, bn, 0);
        }
      }
      *ncand += nc;
      qsort(beam, bn, sizeof(cand), cmp_desc);
      for (int i = 0; i < bn; ++i) {
        ++*visits;
        if (hn < BW) {
          heap[hn] = beam[i];
          heap_up(heap, hn++);
        } else if (beam[i].c > heap[0].c) {
          heap[0] = beam[i];
          heap_down(heap, hn, 0);
        } else {
          break;
        }
      }
    }
    qsort(heap, hn, sizeof(cand), cmp_desc);
    int32_t* par = J->parent + ((size_t)r * nd + s) * BW;
    int32_t* tok = J->token + ((size_t)r * nd + s) * BW;
    float* sco = J->score + ((size_t)r * nd + s) * BW;
    for (int j = 0; j < BW; ++j) {
      if (j < hn) {
        const uint32_t b = heap[j].flat / (uint32_t)V, v = heap[j].flat % (uint32_t)V;
        par[j] = (int32_t)b;
        tok[j] = (int32_t)v;
        sco[j] = heap[j].c;
        /* child id: position of v among the parent's sorted child labels */
        const uint16_t* lab = t->label[s + 1];
        uint32_t lo = t->first[s][node[b]], hi = t->first[s][node[b] + 1];
        while (lo < hi) {
          uint32_t mid = (lo + hi) / 2;
          if (lab[mid] < v) lo = mid + 1; else hi = mid;
        }
        node2[j] = lo;
      } else {
        par[j] = tok[j] = -1;
        sco[j] = -INFINITY;
      }
    }
    for (int j = 0; j < hn; ++j) {
      node[j] = node2[j];
      S[j] = heap[j].c;
    }
    n_live = hn;
    J->nlive[(size_t)r * nd + s] = hn;
  }
  free(node);
  free(S);
  free(node2);
  free(heap);
  free(beam);
  free(x);
}

typedef struct {
  job* J;
  int64_t visits, cands;
} worker;

static void* work(void* p) {
  worker* W = (worker*)p;
  for (;;) {
    int r = __atomic_fetch_add(W->J->counter, 1, __ATOMIC_RELAXED);
    if (r >= W->J->n_req) break;
    run_request(W->J, r, &W->visits, &W->cands);
  }
  return NULL;
}

/* Full ND-step beam search of n_req requests. logits[r * nd + s]: fp32 [rows_s][V] (rows_0 = 1,
 * else >= bw), row-major. Outputs per request and step: parent/token/score [n_req][nd][bw] and
 * n_live [n_req][nd]. stats[0] = heap visits, stats[1] = legal candidates. Returns 0. */
int ph_run(const ph_trie* t, int n_req, const float* const* logits, int bw, int topk, int threads,
           int32_t* parent, int32_t* token, float* score, int32_t* nlive, int64_t* stats) {
  int counter = 0;
  job J = {t, logits, n_req, bw, topk, parent, token, nlive, score, 0, 0, 0, &counter};
  if (threads < 1) threads = 1;
  worker* W = (worker*)calloc(threads, sizeof(worker));
  pthread_t* th = (pthread_t*)calloc(threads, sizeof(pthread_t));
  for (int i = 0; i < threads; ++i) {
    W[i].J = &J;
    pthread_create(&th[i], NULL, work, &W[i]);
  }
  stats[0] = stats[1] = 0;
  for (int i = 0; i < threads; ++i) {
    pthread_join(th[i], NULL);
    stats[0] += W[i].visits;
    stats[1] += W[i].cands;
  }
  free(W);
  free(th);
  return 0;
}
