/*
 * ORACLE TEST INFRASTRUCTURE — CPU restatement of the reference hot path.
 * See mtc_oracle.h. Every function cites the reference file:line it follows
 * (paths under /root/reference/proj). Not product code: the product never
 * links or calls this file.
 */
#include "mtc_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define MAXR 64

typedef struct {
  int order;
  uint32_t legs[MAXR];
  uint32_t dims[MAXR];
  uint64_t size;
  double* data; /* interleaved complex128 */
  int owned;
} otensor;

static int fail(char* err, size_t errlen, int code, const char* fmt, ...) {
  if (err && errlen) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(err, errlen, fmt, ap);
    va_end(ap);
  }
  return code;
}

static uint64_t shape_size(int r, const uint32_t* dims) {
  uint64_t n = 1;
  for (int i = 0; i < r; ++i) n *= dims[i];
  return n;
}

/* stride_of_leg (tensor.cpp:42-49): row-major stride of `id`, 0 if absent. */
static uint64_t stride_of(int r, const uint32_t* legs, const uint32_t* dims,
                          uint32_t id) {
  uint64_t acc = 1;
  for (int i = r; i-- > 0;) {
    if (legs[i] == id) return acc;
    acc *= dims[i];
  }
  return 0;
}

static int find_leg(int r, const uint32_t* legs, uint32_t id) {
  for (int i = 0; i < r; ++i)
    if (legs[i] == id) return i;
  return -1;
}

static int cmp_u32(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return x < y ? -1 : x > y;
}

/* contraction_result_legs + contract_pair (tensor.cpp:100-130, :150-253).
 * Reduction order: closed legs ascending by id, row-major (last fastest);
 * the first product seeds the accumulator, every later one is added once as
 * acc += (xr*yr - xi*yi), acc_i += (xr*yi + xi*yr). */
int orc_contract_pair(int ra, const uint32_t* a_legs, const uint32_t* a_dims,
                      const double* a, int rb, const uint32_t* b_legs,
                      const uint32_t* b_dims, const double* b, int nclosed,
                      const uint32_t* closed, uint32_t* out_legs,
                      uint32_t* out_dims, double* out, uint64_t* counters) {
  uint32_t cl[MAXR];
  int nc = 0;
  for (int i = 0; i < nclosed; ++i) cl[nc++] = closed[i];
  qsort(cl, nc, sizeof(uint32_t), cmp_u32);
  {
    int u = 0;
    for (int i = 0; i < nc; ++i)
      if (u == 0 || cl[u - 1] != cl[i]) cl[u++] = cl[i];
    nc = u;
  }
  for (int i = 0; i < nc; ++i)
    if (find_leg(ra, a_legs, cl[i]) < 0 || find_leg(rb, b_legs, cl[i]) < 0)
      return -1;
  for (int i = 0; i < ra; ++i) {
    int j = find_leg(rb, b_legs, a_legs[i]);
    if (j >= 0 && b_dims[j] != a_dims[i]) return -1;
  }
  /* result legs: (a ∪ b) \ closed, ascending */
  int nr = 0;
  for (int i = 0; i < ra; ++i)
    if (!bsearch(&a_legs[i], cl, nc, sizeof(uint32_t), cmp_u32)) {
      out_legs[nr] = a_legs[i];
      out_dims[nr++] = a_dims[i];
    }
  for (int i = 0; i < rb; ++i)
    if (!bsearch(&b_legs[i], cl, nc, sizeof(uint32_t), cmp_u32) &&
        find_leg(ra, a_legs, b_legs[i]) < 0) {
      out_legs[nr] = b_legs[i];
      out_dims[nr++] = b_dims[i];
    }
  for (int i = 1; i < nr; ++i) /* insertion sort by id */
    for (int j = i; j > 0 && out_legs[j - 1] > out_legs[j]; --j) {
      uint32_t t = out_legs[j]; out_legs[j] = out_legs[j - 1]; out_legs[j - 1] = t;
      t = out_dims[j]; out_dims[j] = out_dims[j - 1]; out_dims[j - 1] = t;
    }
  if (!out) return nr;

  uint64_t rdim[MAXR], rsa[MAXR], rsb[MAXR], cdim[MAXR], csa[MAXR], csb[MAXR];
  for (int i = 0; i < nr; ++i) {
    rdim[i] = out_dims[i];
    rsa[i] = stride_of(ra, a_legs, a_dims, out_legs[i]);
    rsb[i] = stride_of(rb, b_legs, b_dims, out_legs[i]);
  }
  uint64_t d_closed = 1;
  for (int i = 0; i < nc; ++i) {
    cdim[i] = a_dims[find_leg(ra, a_legs, cl[i])];
    csa[i] = stride_of(ra, a_legs, a_dims, cl[i]);
    csb[i] = stride_of(rb, b_legs, b_dims, cl[i]);
    d_closed *= cdim[i];
  }
  uint64_t d_open = shape_size(nr, out_dims);
  uint32_t ridx[MAXR] = {0}, cidx[MAXR];
  uint64_t offa = 0, offb = 0;
  for (uint64_t i = 0; i < d_open; ++i) {
    double accr = 0.0, acci = 0.0;
    uint64_t ca = offa, cb = offb;
    memset(cidx, 0, sizeof cidx);
    for (uint64_t c = 0; c < d_closed; ++c) {
      if (c > 0) { /* row-major odometer over ascending closed ids */
        for (int j = nc; j-- > 0;) {
          if (++cidx[j] < cdim[j]) {
            ca += csa[j];
            cb += csb[j];
            break;
          }
          cidx[j] = 0;
          ca -= csa[j] * (cdim[j] - 1);
          cb -= csb[j] * (cdim[j] - 1);
        }
      }
      double xr = a[2 * ca], xi = a[2 * ca + 1];
      double yr = b[2 * cb], yi = b[2 * cb + 1];
      double pr = xr * yr - xi * yi;
      double pi = xr * yi + xi * yr;
      if (c == 0) {
        accr = pr;
        acci = pi;
      } else {
        accr += pr;
        acci += pi;
      }
    }
    out[2 * i] = accr;
    out[2 * i + 1] = acci;
    for (int j = nr; j-- > 0;) {
      if (++ridx[j] < rdim[j]) {
        offa += rsa[j];
        offb += rsb[j];
        break;
      }
      ridx[j] = 0;
      offa -= rsa[j] * (rdim[j] - 1);
      offb -= rsb[j] * (rdim[j] - 1);
    }
  }
  if (counters) { /* tensor.cpp:247-251 */
    counters[0] += d_closed * d_open;
    counters[1] += (d_closed - 1) * d_open;
    counters[2] += shape_size(ra, a_dims) + shape_size(rb, b_dims) + d_open;
  }
  return nr;
}

/* project_leg (tensor.cpp:255-282): fix `leg` at `value`, drop it. */
static void project_leg(const otensor* t, uint32_t leg, uint32_t value,
                        otensor* out) {
  int pos = find_leg(t->order, t->legs, leg);
  uint64_t inner = 1;
  for (int i = pos + 1; i < t->order; ++i) inner *= t->dims[i];
  uint64_t dim = t->dims[pos];
  uint64_t outer = t->size / (inner * dim);
  out->order = 0;
  for (int i = 0; i < t->order; ++i)
    if (i != pos) {
      out->legs[out->order] = t->legs[i];
      out->dims[out->order++] = t->dims[i];
    }
  out->size = outer * inner;
  out->data = (double*)malloc(sizeof(double) * 2 * (out->size ? out->size : 1));
  out->owned = 1;
  for (uint64_t o = 0; o < outer; ++o)
    memcpy(out->data + 2 * o * inner, t->data + 2 * (o * dim + value) * inner,
           sizeof(double) * 2 * inner);
}

static void tensor_free(otensor* t) {
  if (t && t->owned) free(t->data);
  if (t) t->owned = 0;
}

/* ---- plan indexing and validation (plan.cpp:201-259) -------------------- */

typedef struct {
  const mtcg_problem* p;
  int* parent;
  int* postorder;
  int n_post;
  int* inorder_slots;
  int n_inorder;
} plan_index;

static int index_plan(const mtcg_problem* p, plan_index* ix, char* err,
                      size_t errlen) {
  const int n = p->n_nodes;
  memset(ix, 0, sizeof *ix);
  ix->p = p;
  if (p->root < 0 || p->root >= n)
    return fail(err, errlen, MTCG_ERR_DATA, "plan has no root");
  ix->parent = (int*)malloc(sizeof(int) * n);
  ix->postorder = (int*)malloc(sizeof(int) * n);
  ix->inorder_slots = (int*)malloc(sizeof(int) * (n + 1));
  for (int i = 0; i < n; ++i) ix->parent[i] = -2;
  int* stack = (int*)malloc(sizeof(int) * 2 * (n + 1));
  int sp = 0;
  stack[sp++] = p->root;
  stack[sp++] = 0;
  ix->parent[p->root] = -1;
  int rc = MTCG_OK;
  while (sp > 0) {
    int node = stack[sp - 2];
    int* phase = &stack[sp - 1];
    if (p->node_slot[node] >= 0) {
      if (p->node_slot[node] >= p->n_slots) {
        rc = fail(err, errlen, MTCG_ERR_DATA, "leaf slot %d out of range",
                  p->node_slot[node]);
        break;
      }
      ix->inorder_slots[ix->n_inorder++] = p->node_slot[node];
      ix->postorder[ix->n_post++] = node;
      sp -= 2;
      continue;
    }
    int l = p->node_left[node], r = p->node_right[node];
    if (l < 0 || r < 0 || l >= n || r >= n) {
      rc = fail(err, errlen, MTCG_ERR_DATA, "malformed plan node");
      break;
    }
    if (*phase == 0 || *phase == 1) {
      int child = *phase == 0 ? l : r;
      *phase += 1;
      if (ix->parent[child] != -2) {
        rc = fail(err, errlen, MTCG_ERR_DATA, "plan is not a tree");
        break;
      }
      ix->parent[child] = node;
      stack[sp++] = child;
      stack[sp++] = 0;
    } else {
      ix->postorder[ix->n_post++] = node;
      sp -= 2;
    }
  }
  free(stack);
  if (rc) return rc;
  char* seen = (char*)calloc(p->n_slots + 1, 1);
  for (int i = 0; i < ix->n_inorder && !rc; ++i) {
    int s = ix->inorder_slots[i];
    if (seen[s])
      rc = fail(err, errlen, MTCG_ERR_DATA, "slot %d appears twice in plan", s);
    seen[s] = 1;
  }
  free(seen);
  if (!rc && ix->n_inorder != p->n_slots)
    rc = fail(err, errlen, MTCG_ERR_DATA, "plan covers %d slots, diagram has %d",
              ix->n_inorder, p->n_slots);
  return rc;
}

static void index_free(plan_index* ix) {
  free(ix->parent);
  free(ix->postorder);
  free(ix->inorder_slots);
}

/* ---- tuple index (plan.cpp:292-333) -------------------------------------- */

typedef struct {
  uint64_t rows;
  uint32_t* row_tuples; /* rows x n_slots */
  uint64_t* row_of_request;
  uint32_t** rank;      /* [node][row] */
  uint32_t* distinct;   /* [node] */
} tuple_index;

static int g_slots; /* qsort context (the oracle is single-threaded) */

static int lex_cmp(const uint32_t* x, const uint32_t* y, int m) {
  for (int j = 0; j < m; ++j)
    if (x[j] != y[j]) return x[j] < y[j] ? -1 : 1;
  return 0;
}

static int cmp_tuple_lex(const void* a, const void* b) {
  return lex_cmp((const uint32_t*)a, (const uint32_t*)b, g_slots);
}

typedef struct {
  uint64_t key;
  uint32_t row;
} keyed;

static int cmp_keyed(const void* a, const void* b) {
  const keyed* x = (const keyed*)a;
  const keyed* y = (const keyed*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return x->row < y->row ? -1 : x->row > y->row;
}

static void build_tuple_index(const mtcg_problem* p, const plan_index* ix,
                              tuple_index* ti) {
  const int m = p->n_slots;
  const uint64_t k = p->n_requests;
  uint32_t* sorted = (uint32_t*)malloc(sizeof(uint32_t) * (k * m + 1));
  memcpy(sorted, p->tuples, sizeof(uint32_t) * k * m);
  g_slots = m;
  qsort(sorted, k, sizeof(uint32_t) * m, cmp_tuple_lex);
  uint64_t rows = 0;
  for (uint64_t i = 0; i < k; ++i)
    if (rows == 0 || lex_cmp(sorted + (rows - 1) * m, sorted + i * m, m) != 0) {
      if (rows != i) memmove(sorted + rows * m, sorted + i * m, sizeof(uint32_t) * m);
      ++rows;
    }
  ti->rows = rows;
  ti->row_tuples = sorted;
  ti->row_of_request = (uint64_t*)malloc(sizeof(uint64_t) * (k + 1));
  for (uint64_t i = 0; i < k; ++i) {
    uint64_t lo = 0, hi = rows; /* lower_bound */
    while (lo < hi) {
      uint64_t mid = (lo + hi) / 2;
      if (lex_cmp(sorted + mid * m, p->tuples + i * m, m) < 0)
        lo = mid + 1;
      else
        hi = mid;
    }
    ti->row_of_request[i] = lo;
  }
  ti->rank = (uint32_t**)calloc(p->n_nodes, sizeof(uint32_t*));
  ti->distinct = (uint32_t*)calloc(p->n_nodes, sizeof(uint32_t));
  keyed* kk = (keyed*)malloc(sizeof(keyed) * (rows + 1));
  for (int q = 0; q < ix->n_post; ++q) {
    int node = ix->postorder[q];
    uint32_t* rk = (uint32_t*)malloc(sizeof(uint32_t) * (rows + 1));
    ti->rank[node] = rk;
    for (uint64_t r = 0; r < rows; ++r) {
      if (p->node_slot[node] >= 0)
        kk[r].key = sorted[r * m + p->node_slot[node]];
      else
        kk[r].key = ((uint64_t)ti->rank[p->node_left[node]][r] << 32) |
                    ti->rank[p->node_right[node]][r];
      kk[r].row = (uint32_t)r;
    }
    qsort(kk, rows, sizeof(keyed), cmp_keyed);
    uint32_t next = 0;
    for (uint64_t r = 0; r < rows; ++r) {
      if (r > 0 && kk[r].key != kk[r - 1].key) ++next;
      rk[kk[r].row] = next;
    }
    ti->distinct[node] = rows == 0 ? 0 : next + 1;
  }
  free(kk);
}

static void tuple_index_free(const mtcg_problem* p, tuple_index* ti) {
  for (int n = 0; n < p->n_nodes; ++n) free(ti->rank[n]);
  free(ti->rank);
  free(ti->distinct);
  free(ti->row_tuples);
  free(ti->row_of_request);
}

/* ---- the multi-evaluation (multieval.cpp:384-516) ------------------------ */

typedef struct {
  const mtcg_problem* p;
  const tuple_index* ti;
  otensor** leaves;   /* [slot][value] (per-slice projected) */
  otensor** cache;    /* [node][rank] memo, NULL until computed */
  uint64_t* node_contractions;
  uint64_t* counters;
  int error;
} engine;

/* eval_naive's recursion (multieval.cpp:395-407): one cache entry per
 * (node, rank); each is a pure function of its subtree's leaf values, so the
 * result equals eval_all's bit for bit (multieval_test.cpp:118-141). */
static otensor* eval_rec(engine* e, int node, uint64_t row) {
  const mtcg_problem* p = e->p;
  if (p->node_slot[node] >= 0) {
    int slot = p->node_slot[node];
    return &e->leaves[slot][e->ti->row_tuples[row * p->n_slots + slot]];
  }
  uint32_t rk = e->ti->rank[node][row];
  if (e->cache[node][rk].data) return &e->cache[node][rk];
  otensor* ul = eval_rec(e, p->node_left[node], row);
  otensor* ur = eval_rec(e, p->node_right[node], row);
  if (!ul || !ur) return NULL;
  /* shared_legs (multieval.cpp:57-64): every shared leg is closed (:97). */
  uint32_t closed[MAXR];
  int nc = 0;
  for (int i = 0; i < ul->order; ++i)
    if (find_leg(ur->order, ur->legs, ul->legs[i]) >= 0) closed[nc++] = ul->legs[i];
  otensor* out = &e->cache[node][rk];
  int nr = orc_contract_pair(ul->order, ul->legs, ul->dims, ul->data, ur->order,
                             ur->legs, ur->dims, ur->data, nc, closed, out->legs,
                             out->dims, NULL, NULL);
  if (nr < 0) {
    e->error = 1;
    return NULL;
  }
  out->order = nr;
  out->size = shape_size(nr, out->dims);
  out->data = (double*)malloc(sizeof(double) * 2 * out->size);
  out->owned = 1;
  orc_contract_pair(ul->order, ul->legs, ul->dims, ul->data, ur->order, ur->legs,
                    ur->dims, ur->data, nc, closed, out->legs, out->dims,
                    out->data, e->counters);
  e->node_contractions[node] += 1;
  return out;
}

int orc_eval(const mtcg_problem* p, int mode, double* out_values,
             uint64_t values_capacity, uint64_t* node_contractions,
             uint64_t* counters, int32_t* out_legs, int32_t* n_out_legs,
             char* err, size_t errlen) {
  return orc_eval_slices(p, mode, 0, UINT64_MAX, out_values, values_capacity,
                         node_contractions, counters, out_legs, n_out_legs, err,
                         errlen);
}

/* The slice fold restricted to slices [s_begin, min(s_end, S)): the partial
 * sum one rank of a slice-sharded run owns. */
int orc_eval_slices(const mtcg_problem* p, int mode, uint64_t s_begin,
                    uint64_t s_end, double* out_values,
                    uint64_t values_capacity, uint64_t* node_contractions,
                    uint64_t* counters, int32_t* out_legs, int32_t* n_out_legs,
                    char* err, size_t errlen) {
  plan_index ix;
  int rc = index_plan(p, &ix, err, errlen); /* check_inputs :284-297 */
  if (rc) {
    index_free(&ix);
    return rc;
  }
  for (uint64_t i = 0; i < p->n_requests && !rc; ++i)
    for (int j = 0; j < p->n_slots; ++j)
      if (p->tuples[i * p->n_slots + j] >= (uint32_t)p->slot_n_values[j]) {
        rc = fail(err, errlen, MTCG_ERR_DATA,
                  "request tuple indexes past slot %d's value set", j);
        break;
      }
  if (!rc && mode == MTCG_EVAL_ALL && p->n_sliced > 0)
    rc = fail(err, errlen, MTCG_ERR_DATA, "plan has sliced legs; use eval_sliced");
  if (!rc && mode == MTCG_EVAL_SLICED && p->n_sliced == 0)
    rc = fail(err, errlen, MTCG_ERR_DATA, "plan has no sliced legs; use eval_all");
  /* slice_spec (multieval.cpp:332-348) */
  uint64_t n_slices = 1;
  for (int x = 0; x < p->n_sliced && !rc; ++x) {
    uint32_t l = p->sliced[x];
    if (l >= p->n_legs) {
      rc = fail(err, errlen, MTCG_ERR_DATA, "sliced leg %u does not exist", l);
      break;
    }
    if (l >= p->n_closed) {
      rc = fail(err, errlen, MTCG_ERR_DATA, "output legs cannot be sliced");
      break;
    }
    for (int y = 0; y < x; ++y)
      if (p->sliced[y] == l) rc = fail(err, errlen, MTCG_ERR_DATA,
                                       "leg %u sliced twice", l);
    n_slices *= p->leg_dims[l];
    if (!rc && n_slices > (1ull << 24))
      rc = fail(err, errlen, MTCG_ERR_DATA,
                "slice list expands to more than 2^24 slices");
  }
  if (rc) {
    index_free(&ix);
    return rc;
  }

  tuple_index ti;
  build_tuple_index(p, &ix, &ti);
  const int m = p->n_slots;
  uint64_t local_counters[3] = {0, 0, 0};
  uint64_t* nc = (uint64_t*)calloc(p->n_nodes, sizeof(uint64_t));

  /* base leaves: views of the value tensors */
  otensor** base = (otensor**)calloc(m, sizeof(otensor*));
  const double* vp = p->values;
  for (int j = 0; j < m; ++j) {
    int r = p->slot_leg_begin[j + 1] - p->slot_leg_begin[j];
    base[j] = (otensor*)calloc(p->slot_n_values[j], sizeof(otensor));
    for (int v = 0; v < p->slot_n_values[j]; ++v) {
      otensor* t = &base[j][v];
      t->order = r;
      for (int i = 0; i < r; ++i) {
        t->legs[i] = p->slot_legs[p->slot_leg_begin[j] + i];
        t->dims[i] = p->leg_dims[t->legs[i]];
      }
      t->size = shape_size(r, t->dims);
      t->data = (double*)vp;
      vp += 2 * t->size;
    }
  }

  otensor* by_row = (otensor*)calloc(ti.rows + 1, sizeof(otensor));
  uint32_t vals[MAXR];
  if (s_end > n_slices) s_end = n_slices;
  if (s_begin >= s_end && ti.rows > 0) {
    rc = fail(err, errlen, MTCG_ERR_ARGUMENT, "empty slice range");
  }
  for (uint64_t s = s_begin; s < s_end && !rc; ++s) {
    /* values_of (multieval.cpp:322-329): mixed radix, last leg fastest */
    uint64_t idx = s;
    for (int x = p->n_sliced; x-- > 0;) {
      vals[x] = (uint32_t)(idx % p->leg_dims[p->sliced[x]]);
      idx /= p->leg_dims[p->sliced[x]];
    }
    /* slice_leaves (multieval.cpp:352-367) */
    otensor** leaves = (otensor**)calloc(m, sizeof(otensor*));
    for (int j = 0; j < m; ++j) {
      leaves[j] = (otensor*)calloc(p->slot_n_values[j], sizeof(otensor));
      for (int v = 0; v < p->slot_n_values[j]; ++v) {
        otensor cur = base[j][v];
        cur.owned = 0;
        for (int x = 0; x < p->n_sliced; ++x)
          if (find_leg(cur.order, cur.legs, p->sliced[x]) >= 0) {
            otensor nxt;
            project_leg(&cur, p->sliced[x], vals[x], &nxt);
            tensor_free(&cur);
            cur = nxt;
          }
        leaves[j][v] = cur;
      }
    }
    engine e;
    e.p = p;
    e.ti = &ti;
    e.leaves = leaves;
    e.cache = (otensor**)calloc(p->n_nodes, sizeof(otensor*));
    for (int n = 0; n < p->n_nodes; ++n)
      e.cache[n] = (otensor*)calloc(ti.distinct[n] + 1, sizeof(otensor));
    e.node_contractions = nc;
    e.counters = local_counters;
    e.error = 0;
    for (uint64_t r = 0; r < ti.rows; ++r) {
      otensor* v = eval_rec(&e, p->root, r);
      if (!v) {
        rc = fail(err, errlen, MTCG_ERR_DATA, "malformed contraction operands");
        break;
      }
      /* fold in slice-index order (multieval.cpp:498-513) */
      if (s == s_begin) {
        by_row[r] = *v;
        by_row[r].data = (double*)malloc(sizeof(double) * 2 * v->size);
        by_row[r].owned = 1;
        memcpy(by_row[r].data, v->data, sizeof(double) * 2 * v->size);
      } else {
        for (uint64_t i = 0; i < 2 * v->size; ++i) by_row[r].data[i] += v->data[i];
      }
    }
    for (int n = 0; n < p->n_nodes; ++n) {
      for (uint32_t q = 0; q < ti.distinct[n]; ++q) tensor_free(&e.cache[n][q]);
      free(e.cache[n]);
    }
    free(e.cache);
    for (int j = 0; j < m; ++j) {
      for (int v = 0; v < p->slot_n_values[j]; ++v) tensor_free(&leaves[j][v]);
      free(leaves[j]);
    }
    free(leaves);
  }

  if (!rc) {
    /* fan_out (multieval.cpp:374-380) */
    uint64_t o = 0;
    for (uint64_t i = 0; i < p->n_requests; ++i) {
      const otensor* t = &by_row[ti.row_of_request[i]];
      if (o + t->size > values_capacity) {
        rc = fail(err, errlen, MTCG_ERR_ARGUMENT, "values buffer too small");
        break;
      }
      if (out_values) memcpy(out_values + 2 * o, t->data, sizeof(double) * 2 * t->size);
      o += t->size;
    }
    if (n_out_legs) {
      *n_out_legs = 0;
      if (ti.rows > 0) {
        *n_out_legs = by_row[0].order;
        for (int i = 0; i < by_row[0].order; ++i) out_legs[i] = (int32_t)by_row[0].legs[i];
      }
    }
    if (node_contractions) memcpy(node_contractions, nc, sizeof(uint64_t) * p->n_nodes);
    if (counters) memcpy(counters, local_counters, sizeof local_counters);
  }
  for (uint64_t r = 0; r < ti.rows; ++r) tensor_free(&by_row[r]);
  free(by_row);
  for (int j = 0; j < m; ++j) free(base[j]);
  free(base);
  free(nc);
  tuple_index_free(p, &ti);
  index_free(&ix);
  return rc;
}

/* compensated_sum + linear_xeb (xeb.cpp:28-50) */
int orc_linear_xeb(int n, const double* probs, uint64_t count, double* out,
                   char* err, size_t errlen) {
  if (count == 0)
    return fail(err, errlen, MTCG_ERR_DATA, "linear_xeb needs at least one sample");
  if (n < 0 || n > 1022)
    return fail(err, errlen, MTCG_ERR_DATA, "qubit count out of range");
  for (uint64_t i = 0; i < count; ++i)
    if (probs[i] < 0.0) return fail(err, errlen, MTCG_ERR_DATA, "negative probability");
  double sum = 0.0, comp = 0.0;
  for (uint64_t i = 0; i < count; ++i) {
    double x = probs[i];
    double t = sum + x;
    if (fabs(sum) >= fabs(x))
      comp += (sum - t) + x;
    else
      comp += (x - t) + sum;
    sum = t;
  }
  *out = ldexp((sum + comp) / (double)count, n) - 1.0;
  return MTCG_OK;
}
