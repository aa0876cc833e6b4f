/*
 * oracle/seq_oracle.c — TEST INFRASTRUCTURE ONLY.  Never linked into the
 * product library; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg load it, and only as the checker.
 *
 * Plain-C restatement of the reference's independent sequential oracles
 * (/root/reference/proj/core/src/reference.cpp) and of the DOBFS direction
 * rule (primitives.cpp:131-154), operating on raw CSR arrays
 * (row_offsets u32[nv+1], col_indices u32[ne], edge_values u32[ne] or NULL).
 *
 * Pinning: tests/test_oracle.py checks every function here against
 *   (1) the golden vectors of the reference's own unit tests
 *       (tests/golden/reference_pins.json, from test_primitives.cpp /
 *       test_engine.cpp), and
 *   (2) the reference itself compiled from /root/reference into oracle/_ref
 *       (oracle/Makefile) on RMAT/grid graphs — bit-exact, including the
 *       floating-point BC / PageRank values, because the restatement keeps
 *       the reference's evaluation order.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define INF_LABEL 0xFFFFFFFFu
#define INF_DIST 0xFFFFFFFFFFFFFFFFull

/* reference.cpp:26-42 bfs_levels: FIFO queue BFS */
void mgo_bfs_levels(uint32_t nv, const uint32_t* off, const uint32_t* col, uint32_t src,
                    uint32_t* depth) {
  uint32_t* q = (uint32_t*)malloc(sizeof(uint32_t) * (nv ? nv : 1));
  size_t head = 0, tail = 0;
  for (uint32_t v = 0; v < nv; ++v) depth[v] = INF_LABEL;
  depth[src] = 0;
  q[tail++] = src;
  while (head < tail) {
    uint32_t u = q[head++];
    for (uint32_t e = off[u]; e < off[u + 1]; ++e) {
      uint32_t v = col[e];
      if (depth[v] == INF_LABEL) {
        depth[v] = depth[u] + 1;
        q[tail++] = v;
      }
    }
  }
  free(q);
}

/* ---- binary min-heap of (dist, vertex), lexicographic like std::greater<pair> */
typedef struct {
  uint64_t d;
  uint32_t v;
} item_t;

static int item_less(item_t a, item_t b) { return a.d < b.d || (a.d == b.d && a.v < b.v); }

typedef struct {
  item_t* a;
  size_t n, cap;
} heap_t;

static void heap_push(heap_t* h, item_t x) {
  if (h->n == h->cap) {
    h->cap = h->cap ? 2 * h->cap : 1024;
    h->a = (item_t*)realloc(h->a, h->cap * sizeof(item_t));
  }
  size_t i = h->n++;
  while (i > 0) {
    size_t p = (i - 1) / 2;
    if (!item_less(x, h->a[p])) break;
    h->a[i] = h->a[p];
    i = p;
  }
  h->a[i] = x;
}

static item_t heap_pop(heap_t* h) {
  item_t top = h->a[0], x = h->a[--h->n];
  size_t i = 0;
  for (;;) {
    size_t l = 2 * i + 1, r = l + 1, m = i;
    item_t best = x;
    if (l < h->n && item_less(h->a[l], best)) { m = l; best = h->a[l]; }
    if (r < h->n && item_less(h->a[r], best)) { m = r; best = h->a[r]; }
    if (m == i) break;
    h->a[i] = h->a[m];
    i = m;
  }
  if (h->n) h->a[i] = x;
  return top;
}

/* reference.cpp:44-66 dijkstra with lazy deletion; unit weight if w == NULL */
void mgo_dijkstra(uint32_t nv, const uint32_t* off, const uint32_t* col, const uint32_t* w,
                  uint32_t src, uint64_t* dist) {
  heap_t h = {0, 0, 0};
  for (uint32_t v = 0; v < nv; ++v) dist[v] = INF_DIST;
  dist[src] = 0;
  item_t s = {0, src};
  heap_push(&h, s);
  while (h.n) {
    item_t it = heap_pop(&h);
    if (it.d != dist[it.v]) continue;
    for (uint32_t e = off[it.v]; e < off[it.v + 1]; ++e) {
      uint32_t v = col[e];
      uint64_t nd = it.d + (w ? w[e] : 1u);
      if (nd < dist[v]) {
        dist[v] = nd;
        item_t x = {nd, v};
        heap_push(&h, x);
      }
    }
  }
  free(h.a);
}

/* reference.cpp:70-106 union-find with path halving; the smaller root wins,
 * so find() yields the minimum member of each component */
static uint32_t uf_find(uint32_t* parent, uint32_t x) {
  while (parent[x] != x) {
    parent[x] = parent[parent[x]];
    x = parent[x];
  }
  return x;
}

void mgo_connected_components(uint32_t nv, const uint32_t* off, const uint32_t* col,
                              uint32_t* comp) {
  for (uint32_t v = 0; v < nv; ++v) comp[v] = v;
  for (uint32_t u = 0; u < nv; ++u) {
    for (uint32_t e = off[u]; e < off[u + 1]; ++e) {
      uint32_t a = uf_find(comp, u), b = uf_find(comp, col[e]);
      if (a == b) continue;
      if (a < b) comp[b] = a;
      else comp[a] = b;
    }
  }
  for (uint32_t v = 0; v < nv; ++v) comp[v] = uf_find(comp, v);
}

/* reference.cpp:108-143 Brandes single-source dependency accumulation.
 * preds[w] are stored as a CSR-like list in discovery order (same order the
 * reference pushes them), the stack is the BFS visitation order. */
void mgo_brandes_bc(uint32_t nv, const uint32_t* off, const uint32_t* col, uint32_t src,
                    double* bc, double* sigma_out, uint32_t* dist_out) {
  double* sigma = (double*)calloc(nv ? nv : 1, sizeof(double));
  double* delta = (double*)calloc(nv ? nv : 1, sizeof(double));
  uint32_t* dist = (uint32_t*)malloc(sizeof(uint32_t) * (nv ? nv : 1));
  uint32_t* order = (uint32_t*)malloc(sizeof(uint32_t) * (nv ? nv : 1));
  /* predecessor lists: each arc (u,v) contributes at most once -> ne slots */
  uint64_t ne = nv ? off[nv] : 0;
  uint32_t* pred_head = (uint32_t*)malloc(sizeof(uint32_t) * (nv ? nv : 1));
  uint32_t* pred_next = (uint32_t*)malloc(sizeof(uint32_t) * (ne ? ne : 1));
  uint32_t* pred_val = (uint32_t*)malloc(sizeof(uint32_t) * (ne ? ne : 1));
  uint32_t* pred_tail = (uint32_t*)malloc(sizeof(uint32_t) * (nv ? nv : 1));
  uint64_t npred = 0;
  size_t head = 0, tail = 0, norder = 0;
  for (uint32_t v = 0; v < nv; ++v) {
    dist[v] = INF_LABEL;
    bc[v] = 0.0;
    pred_head[v] = pred_tail[v] = INF_LABEL;
  }
  uint32_t* q = (uint32_t*)malloc(sizeof(uint32_t) * (nv ? nv : 1));
  sigma[src] = 1.0;
  dist[src] = 0;
  q[tail++] = src;
  while (head < tail) {
    uint32_t u = q[head++];
    order[norder++] = u;
    for (uint32_t e = off[u]; e < off[u + 1]; ++e) {
      uint32_t v = col[e];
      if (dist[v] == INF_LABEL) {
        dist[v] = dist[u] + 1;
        q[tail++] = v;
      }
      if (dist[v] == dist[u] + 1) {
        sigma[v] += sigma[u];
        /* append u to preds[v], preserving push order */
        pred_val[npred] = u;
        pred_next[npred] = INF_LABEL;
        if (pred_tail[v] == INF_LABEL) pred_head[v] = (uint32_t)npred;
        else pred_next[pred_tail[v]] = (uint32_t)npred;
        pred_tail[v] = (uint32_t)npred;
        ++npred;
      }
    }
  }
  while (norder) {
    uint32_t w = order[--norder];
    for (uint32_t i = pred_head[w]; i != INF_LABEL; i = pred_next[i]) {
      uint32_t v = pred_val[i];
      delta[v] += sigma[v] / sigma[w] * (1.0 + delta[w]);
    }
    if (w != src) bc[w] += delta[w];
  }
  if (sigma_out) memcpy(sigma_out, sigma, sizeof(double) * nv);
  if (dist_out) memcpy(dist_out, dist, sizeof(uint32_t) * nv);
  free(sigma); free(delta); free(dist); free(order); free(q);
  free(pred_head); free(pred_next); free(pred_val); free(pred_tail);
}

/* reference.cpp:145-172 power iteration with uniform dangling redistribution */
uint64_t mgo_pagerank(uint32_t nv, const uint32_t* off, const uint32_t* col, double damping,
                      double epsilon, uint64_t max_iter, double* rank, double* sums,
                      uint64_t sums_cap) {
  if (nv == 0) return 0;
  double* accum = (double*)malloc(sizeof(double) * nv);
  uint64_t iters = 0;
  for (uint32_t v = 0; v < nv; ++v) rank[v] = 1.0 / nv;
  for (uint64_t it = 1; it <= max_iter; ++it) {
    double dangling = 0.0, delta_max = 0.0, sum = 0.0;
    for (uint32_t v = 0; v < nv; ++v) accum[v] = 0.0;
    for (uint32_t u = 0; u < nv; ++u) {
      uint32_t deg = off[u + 1] - off[u];
      if (deg == 0) {
        dangling += rank[u];
        continue;
      }
      double contrib = rank[u] / (double)deg;
      for (uint32_t e = off[u]; e < off[u + 1]; ++e) accum[col[e]] += contrib;
    }
    for (uint32_t v = 0; v < nv; ++v) {
      double nr = (1.0 - damping) / nv + damping * (accum[v] + dangling / nv);
      double rel = fabs(nr - rank[v]) / (nr > 1e-300 ? nr : 1e-300);
      if (rel > delta_max) delta_max = rel;
      rank[v] = nr;
      sum += nr;
    }
    iters = it;
    if (sums && it - 1 < sums_cap) sums[it - 1] = sum;
    if (delta_max < epsilon) break;
  }
  free(accum);
  return iters;
}

/* primitives.cpp:131-145 make_direction_state: FV = |Q||E|/|V|, BV = |U||V|/|P| */
void mgo_direction_estimates(uint64_t q, uint64_t u, uint64_t p, uint64_t edges,
                             uint64_t vertices, double* fv, double* bv) {
  *fv = vertices > 0 ? (double)q * (double)edges / (double)vertices : 0.0;
  *bv = p > 0 ? (double)u * (double)vertices / (double)p : 0.0;
}

/* primitives.cpp:147-154 direction_decide: 0 = forward, 1 = backward */
int mgo_direction_decide(int current, double fv, double bv, double do_a, double do_b,
                         int switched_once) {
  if (current == 0) return (!switched_once && fv > bv * do_a) ? 1 : 0;
  return fv < bv * do_b ? 0 : 1;
}
