/*
 * af_oracle_mr.c — TEST INFRASTRUCTURE ONLY (the parity checker, never the
 * product): a plain-C restatement of the reference's multiresolution path,
 * /root/reference/proj/core/src/mr_tree.cpp and mr_solver.cpp, driven by the
 * run loop of oracle/ref_harness.cpp (mr_solver.cpp:318-400 with the seeded
 * data, the CFL rule and the level-dependent threshold of af_oracle.h).
 *
 * The tree is the reference's node map (mr_tree.hpp:195, unordered_map keyed
 * by pack_key) restated as an open-addressing hash table. Every loop whose
 * order matters visits keys in the order the reference sorts them (leaves()
 * ascending, internal_keys()/coarsen descending, registers ascending), and
 * every arithmetic expression keeps the reference's association order
 * (compile with -ffp-contract=off). Exceptions become a longjmp to the run
 * loop with the reference's message text.
 *
 * Pinned bit for bit against the compiled reference (afref_mr_run) by
 * tests/test_oracle_mr.py.
 */
#include <setjmp.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "af_oracle.h"
#include "af_oracle_core.h"

/* ---- node keys (mr_tree.hpp:15-43) --------------------------------------- */
#define KB 15
typedef uint64_t key_t_;

static inline key_t_ pack_key(int l, int i, int j, int k) {
  return ((key_t_)l << (3 * KB)) | ((key_t_)i << (2 * KB)) | ((key_t_)j << KB) | (key_t_)k;
}
typedef struct {
  int level;
  int idx[3];
} node_id;
static inline node_id unpack_key(key_t_ key) {
  const key_t_ mask = ((key_t_)1 << KB) - 1;
  node_id id;
  id.idx[2] = (int)(key & mask);
  id.idx[1] = (int)((key >> KB) & mask);
  id.idx[0] = (int)((key >> (2 * KB)) & mask);
  id.level = (int)(key >> (3 * KB));
  return id;
}
static inline key_t_ key_of(const node_id* id) {
  return pack_key(id->level, id->idx[0], id->idx[1], id->idx[2]);
}
static inline key_t_ child_key(const node_id* p, int c) {
  return pack_key(p->level + 1, 2 * p->idx[0] + (c & 1), 2 * p->idx[1] + ((c >> 1) & 1),
                  2 * p->idx[2] + ((c >> 2) & 1));
}

/* ---- open-addressing map: uint64 key -> fixed-size value ----------------- */
typedef struct {
  key_t_* keys;
  unsigned char* used;
  char* vals;
  size_t vsize, cap, count;
} omap;

static size_t hash64(key_t_ x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return (size_t)x;
}
static void omap_init(omap* m, size_t vsize, size_t cap) {
  size_t c = 64;
  while (c < 2 * cap) c <<= 1;
  m->vsize = vsize;
  m->cap = c;
  m->count = 0;
  m->keys = (key_t_*)malloc(sizeof(key_t_) * c);
  m->used = (unsigned char*)calloc(c, 1);
  m->vals = (char*)malloc(vsize * c);
}
static void omap_free(omap* m) {
  free(m->keys);
  free(m->used);
  free(m->vals);
  memset(m, 0, sizeof *m);
}
static void* omap_find(const omap* m, key_t_ k) {
  size_t i = hash64(k) & (m->cap - 1);
  while (m->used[i]) {
    if (m->keys[i] == k) return m->vals + i * m->vsize;
    i = (i + 1) & (m->cap - 1);
  }
  return NULL;
}
static void omap_grow(omap* m);
/* Inserts a zeroed value (or returns the existing one). Invalidates every
 * pointer previously returned when the table grows. */
static void* omap_insert(omap* m, key_t_ k, int* fresh) {
  if (2 * (m->count + 1) > m->cap) omap_grow(m);
  size_t i = hash64(k) & (m->cap - 1);
  while (m->used[i]) {
    if (m->keys[i] == k) {
      if (fresh) *fresh = 0;
      return m->vals + i * m->vsize;
    }
    i = (i + 1) & (m->cap - 1);
  }
  m->used[i] = 1;
  m->keys[i] = k;
  memset(m->vals + i * m->vsize, 0, m->vsize);
  ++m->count;
  if (fresh) *fresh = 1;
  return m->vals + i * m->vsize;
}
static void omap_grow(omap* m) {
  omap n;
  omap_init(&n, m->vsize, m->cap);
  for (size_t i = 0; i < m->cap; ++i)
    if (m->used[i]) memcpy(omap_insert(&n, m->keys[i], NULL), m->vals + i * m->vsize, m->vsize);
  omap_free(m);
  *m = n;
}
/* Backward-shift deletion (keeps probe chains intact). */
static void omap_erase(omap* m, key_t_ k) {
  size_t i = hash64(k) & (m->cap - 1);
  while (m->used[i] && m->keys[i] != k) i = (i + 1) & (m->cap - 1);
  if (!m->used[i]) return;
  size_t hole = i;
  size_t j = i;
  for (;;) {
    j = (j + 1) & (m->cap - 1);
    if (!m->used[j]) break;
    const size_t home = hash64(m->keys[j]) & (m->cap - 1);
    /* move j into the hole when its home is not cyclically in (hole, j] */
    const int in_range = hole <= j ? (home > hole && home <= j) : (home > hole || home <= j);
    if (in_range) continue;
    m->keys[hole] = m->keys[j];
    memcpy(m->vals + hole * m->vsize, m->vals + j * m->vsize, m->vsize);
    hole = j;
  }
  m->used[hole] = 0;
  --m->count;
}

/* ---- tree (mr_tree.hpp:46-195) ------------------------------------------- */
enum { ST_LEAF = 0, ST_INTERNAL = 1, ST_VIRTUAL = 2 }; /* NodeStatus, mr_tree.hpp:45 */

typedef struct {
  afo_state q, q_old, rhs; /* MRNode, mr_tree.hpp:47-51 */
  int status;
} mr_node;

typedef struct {
  afo_state coarse, fine; /* MRSolver::Register, mr_solver.hpp:44-47 */
  int has_coarse, has_fine;
} mr_reg;

typedef struct {
  int dim, L;
  int bc[6]; /* 0 outflow, 1 periodic, 2 reflective */
  int min_leaf;
  double norms[5];
  omap nodes;
  /* threshold: eps_level[child level] when set (the harness hook), else eps */
  double eps;
  const double* eps_level;
  /* solver (mr_solver.hpp:65-73) */
  int limiter, flux;
  double gamma;
  double max_cfl;
  long fallbacks;
  double* t_old;
  double* t_new;
  omap regs;
} mr_tree;

/* error exits (the reference's exceptions) */
static jmp_buf g_jmp;
static int g_err_kind;
static char g_err[512];

static void raise_err(int kind, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  g_err_kind = kind;
  longjmp(g_jmp, 1);
}

/* the harness hook afref_eps_level(eps, child_level): the level table when
 * one is installed, else the threshold the call passes */
static inline double thr(const mr_tree* t, double eps, int child_level) {
  return t->eps_level ? t->eps_level[child_level] : eps;
}
static inline double dx_at(int level) { return 1.0 / (double)(1 << level); } /* mr_tree.hpp:74 */
static inline int periodic(const mr_tree* t, int a) { return t->bc[2 * a] == 1; } /* grid.hpp:85 */
static inline mr_node* find(const mr_tree* t, key_t_ k) { return (mr_node*)omap_find(&t->nodes, k); }
static inline mr_node* find_id(const mr_tree* t, const node_id* id) { return find(t, key_of(id)); }

static inline void st_zero(afo_state* s) { memset(s, 0, sizeof *s); }
static inline void st_add(afo_state* a, const afo_state* b) {
  for (int m = 0; m < 5; ++m) a->v[m] = a->v[m] + b->v[m];
}
static inline void st_add_scaled(afo_state* a, const afo_state* b, double s) { /* a += b * s */
  for (int m = 0; m < 5; ++m) a->v[m] = a->v[m] + b->v[m] * s;
}
static inline void st_sub_scaled(afo_state* a, const afo_state* b, double s) { /* a -= b * s */
  for (int m = 0; m < 5; ++m) a->v[m] = a->v[m] - b->v[m] * s;
}
static inline void st_scale(afo_state* a, double s) {
  for (int m = 0; m < 5; ++m) a->v[m] = a->v[m] * s;
}

static int cmp_key_asc(const void* a, const void* b) {
  const key_t_ x = *(const key_t_*)a, y = *(const key_t_*)b;
  return x < y ? -1 : x > y;
}
static int cmp_key_desc(const void* a, const void* b) { return cmp_key_asc(b, a); }

typedef struct {
  key_t_* k;
  long n;
} keylist;

/* keys with the given status and level in [lo, hi], sorted (mr_tree.cpp:100-133) */
static keylist collect(const mr_tree* t, int status, int lo, int hi, int descending) {
  keylist out;
  out.k = (key_t_*)malloc(sizeof(key_t_) * (t->nodes.count + 1));
  out.n = 0;
  for (size_t i = 0; i < t->nodes.cap; ++i) {
    if (!t->nodes.used[i]) continue;
    const mr_node* nd = (const mr_node*)(t->nodes.vals + i * t->nodes.vsize);
    if (nd->status != status) continue;
    const int l = (int)(t->nodes.keys[i] >> (3 * KB));
    if (l < lo || l > hi) continue;
    out.k[out.n++] = t->nodes.keys[i];
  }
  qsort(out.k, (size_t)out.n, sizeof(key_t_), descending ? cmp_key_desc : cmp_key_asc);
  return out;
}
static keylist leaves(const mr_tree* t) { return collect(t, ST_LEAF, 0, 1 << 20, 0); }

/* mr_tree.cpp:89-94 */
static long leaf_count(const mr_tree* t) {
  long c = 0;
  for (size_t i = 0; i < t->nodes.cap; ++i)
    if (t->nodes.used[i] &&
        ((const mr_node*)(t->nodes.vals + i * t->nodes.vsize))->status == ST_LEAF)
      ++c;
  return c;
}

/* mr_tree.cpp:128-133 */
static int coarsest_leaf_level(const mr_tree* t) {
  int l = t->L;
  for (size_t i = 0; i < t->nodes.cap; ++i)
    if (t->nodes.used[i] &&
        ((const mr_node*)(t->nodes.vals + i * t->nodes.vsize))->status == ST_LEAF) {
      const int lv = (int)(t->nodes.keys[i] >> (3 * KB));
      if (lv < l) l = lv;
    }
  return l;
}

/* map_position (mr_tree.cpp:146-172): periodic wrap, outflow clamp,
 * reflective fold with a momentum flip per fold. */
static node_id map_position(const mr_tree* t, node_id pos, int flip[3]) {
  flip[0] = flip[1] = flip[2] = 0;
  const int n = 1 << pos.level;
  for (int a = 0; a < t->dim; ++a) {
    int c = pos.idx[a];
    if (c >= 0 && c < n) continue;
    if (periodic(t, a)) {
      pos.idx[a] = ((c % n) + n) % n;
      continue;
    }
    const int kind = c < 0 ? t->bc[2 * a] : t->bc[2 * a + 1];
    if (kind == 0) {
      c = c < 0 ? 0 : (c > n - 1 ? n - 1 : c);
    } else {
      while (c < 0 || c >= n) {
        if (c < 0) c = -1 - c;
        if (c >= n) c = 2 * n - 1 - c;
        flip[a] = !flip[a];
      }
    }
    pos.idx[a] = c;
  }
  return pos;
}

/* axis_stencil (mr_tree.cpp:199-240) */
typedef struct {
  int pos[3];
  double w_low[3], w_high[3];
} axis_st;

static axis_st axis_stencil(const mr_tree* t, int level, int coord, int axis) {
  const int n = 1 << level;
  axis_st s;
  if (periodic(t, axis) || (coord > 0 && coord < n - 1)) {
    s.pos[0] = coord - 1, s.pos[1] = coord, s.pos[2] = coord + 1;
    s.w_low[0] = 1.0 / 8.0, s.w_low[1] = 1.0, s.w_low[2] = -1.0 / 8.0;
    s.w_high[0] = -1.0 / 8.0, s.w_high[1] = 1.0, s.w_high[2] = 1.0 / 8.0;
    return s;
  }
  if (n == 1) {
    s.pos[0] = s.pos[1] = s.pos[2] = 0;
    s.w_low[0] = 1.0, s.w_low[1] = 0.0, s.w_low[2] = 0.0;
    s.w_high[0] = 1.0, s.w_high[1] = 0.0, s.w_high[2] = 0.0;
    return s;
  }
  if (n == 2) { /* linear (slope) prediction */
    s.pos[0] = 0, s.pos[1] = 1, s.pos[2] = 1;
    if (coord == 0) {
      s.w_low[0] = 5.0 / 4.0, s.w_low[1] = -1.0 / 4.0, s.w_low[2] = 0.0;
      s.w_high[0] = 3.0 / 4.0, s.w_high[1] = 1.0 / 4.0, s.w_high[2] = 0.0;
    } else {
      s.w_low[0] = 1.0 / 4.0, s.w_low[1] = 3.0 / 4.0, s.w_low[2] = 0.0;
      s.w_high[0] = -1.0 / 4.0, s.w_high[1] = 5.0 / 4.0, s.w_high[2] = 0.0;
    }
    return s;
  }
  if (coord == 0) {
    s.pos[0] = 0, s.pos[1] = 1, s.pos[2] = 2;
    s.w_low[0] = 11.0 / 8.0, s.w_low[1] = -4.0 / 8.0, s.w_low[2] = 1.0 / 8.0;
    s.w_high[0] = 5.0 / 8.0, s.w_high[1] = 4.0 / 8.0, s.w_high[2] = -1.0 / 8.0;
  } else { /* coord == n - 1 */
    s.pos[0] = n - 3, s.pos[1] = n - 2, s.pos[2] = n - 1;
    s.w_low[0] = -1.0 / 8.0, s.w_low[1] = 4.0 / 8.0, s.w_low[2] = 5.0 / 8.0;
    s.w_high[0] = 1.0 / 8.0, s.w_high[1] = -4.0 / 8.0, s.w_high[2] = 11.0 / 8.0;
  }
  return s;
}

static afo_state value_at(const mr_tree* t, node_id pos);

/* predict_children (mr_tree.cpp:242-280): tensor product of the axis
 * stencils over the 3^d neighbourhood, zero weights skipped, ck -> cj -> ci. */
static void predict_children(const mr_tree* t, const node_id* parent, afo_state out[8]) {
  axis_st st[3];
  for (int a = 0; a < t->dim; ++a) st[a] = axis_stencil(t, parent->level, parent->idx[a], a);
  const int nz = t->dim == 3 ? 3 : 1;
  afo_state nb[27];
  for (int ck = 0; ck < nz; ++ck)
    for (int cj = 0; cj < 3; ++cj)
      for (int ci = 0; ci < 3; ++ci) {
        node_id pos;
        pos.level = parent->level;
        pos.idx[0] = st[0].pos[ci];
        pos.idx[1] = st[1].pos[cj];
        pos.idx[2] = t->dim == 3 ? st[2].pos[ck] : parent->idx[2];
        nb[ci + 3 * cj + 9 * ck] = value_at(t, pos);
      }
  const int children = 1 << t->dim;
  for (int c = 0; c < children; ++c) {
    const int sx = c & 1, sy = (c >> 1) & 1, sz = (c >> 2) & 1;
    const double* wx = sx ? st[0].w_high : st[0].w_low;
    const double* wy = sy ? st[1].w_high : st[1].w_low;
    const double* wz = t->dim == 3 ? (sz ? st[2].w_high : st[2].w_low) : NULL;
    afo_state acc;
    st_zero(&acc);
    for (int ck = 0; ck < nz; ++ck) {
      const double wk = t->dim == 3 ? wz[ck] : 1.0;
      if (wk == 0.0) continue;
      for (int cj = 0; cj < 3; ++cj) {
        const double wjk = wy[cj] * wk;
        if (wjk == 0.0) continue;
        for (int ci = 0; ci < 3; ++ci) {
          const double w = wx[ci] * wjk;
          if (w == 0.0) continue;
          st_add_scaled(&acc, &nb[ci + 3 * cj + 9 * ck], w);
        }
      }
    }
    out[c] = acc;
  }
}

/* predict_single (mr_tree.cpp:282-289) */
static afo_state predict_single(const mr_tree* t, const node_id* child) {
  node_id parent;
  parent.level = child->level - 1;
  for (int a = 0; a < 3; ++a) parent.idx[a] = child->idx[a] >> 1;
  const int c = (child->idx[0] & 1) | ((child->idx[1] & 1) << 1) | ((child->idx[2] & 1) << 2);
  afo_state pred[8];
  predict_children(t, &parent, pred);
  return pred[c];
}

/* value_at (mr_tree.cpp:174-183): node q if present, else the recursive
 * prediction. Periodic axes wrap; other axes are in-domain by contract. */
static afo_state value_at(const mr_tree* t, node_id pos) {
  const int n = 1 << pos.level;
  for (int a = 0; a < t->dim; ++a)
    if (periodic(t, a)) pos.idx[a] = ((pos.idx[a] % n) + n) % n;
  const mr_node* nd = find_id(t, &pos);
  if (nd) return nd->q;
  return predict_single(t, &pos);
}

/* detail / detail_between (mr_tree.cpp:291-317) */
static double detail(const mr_tree* t, const node_id* node) {
  const int children = 1 << t->dim;
  afo_state pred[8];
  predict_children(t, node, pred);
  double mag = 0.0;
  for (int c = 0; c < children; ++c) {
    const mr_node* ch = find(t, child_key(node, c));
    afo_state d;
    for (int m = 0; m < 5; ++m) d.v[m] = ch->q.v[m] - pred[c].v[m];
    for (int m = 0; m < 5; ++m) {
      const double r = fabs(d.v[m]) / t->norms[m];
      mag = mag < r ? r : mag; /* std::max(mag, r) */
    }
  }
  return mag;
}

/* split_leaf (mr_tree.cpp:340-359) */
static void split_leaf(mr_tree* t, key_t_ key) {
  const node_id id = unpack_key(key);
  afo_state pred[8];
  predict_children(t, &id, pred);
  const int children = 1 << t->dim;
  for (int c = 0; c < children; ++c) {
    mr_node* ch = (mr_node*)omap_insert(&t->nodes, child_key(&id, c), NULL);
    ch->q = pred[c];
    ch->q_old = pred[c];
    ch->status = ST_LEAF;
  }
  find(t, key)->status = ST_INTERNAL;
}

/* enforce_gradedness (mr_tree.cpp:404-444): sequential passes over the
 * sorted pass-start leaves until a pass splits nothing. */
static void enforce_gradedness(mr_tree* t) {
  int changed = 1;
  while (changed) {
    changed = 0;
    keylist lv = leaves(t);
    for (long e = 0; e < lv.n; ++e) {
      const node_id id = unpack_key(lv.k[e]);
      if (id.level >= t->L) continue;
      int need = 0;
      for (int a = 0; a < t->dim && !need; ++a)
        for (int dir = -1; dir <= 1 && !need; dir += 2) {
          node_id np = id;
          np.idx[a] += dir;
          const int n = 1 << id.level;
          if (!periodic(t, a) && (np.idx[a] < 0 || np.idx[a] >= n)) continue;
          int flip[3];
          const node_id mp = map_position(t, np, flip);
          const mr_node* nb = find_id(t, &mp);
          if (!nb || nb->status != ST_INTERNAL) continue;
          const int face_bit = dir > 0 ? 0 : 1;
          const int tzn = t->dim == 3 ? 2 : 1;
          const int b1 = a == 0 ? 1 : 0, b2 = a == 2 ? 1 : 2;
          for (int t2 = 0; t2 < tzn && !need; ++t2)
            for (int t1 = 0; t1 < 2 && !need; ++t1) {
              int ci[3];
              ci[a] = 2 * mp.idx[a] + face_bit;
              ci[b1] = 2 * mp.idx[b1] + t1;
              ci[b2] = 2 * mp.idx[b2] + (t->dim == 3 ? t2 : 0);
              const mr_node* ch = find(t, pack_key(mp.level + 1, ci[0], ci[1], ci[2]));
              if (ch && ch->status == ST_INTERNAL) need = 1;
            }
        }
      if (need) {
        split_leaf(t, lv.k[e]);
        changed = 1;
      }
    }
    free(lv.k);
  }
}

/* refine (mr_tree.cpp:361-402): split a leaf at level [1, L-1] iff its
 * parent's detail >= eps (at the leaf's level), dilate by the per-level
 * buffer (LT), split in ascending key order, then grade. */
static void refine(mr_tree* t, const int* buffer, int nbuf) {
  keylist lv = leaves(t);
  key_t_* split = (key_t_*)malloc(sizeof(key_t_) * (size_t)(lv.n + 1));
  long ns = 0;
  omap pdet;
  omap_init(&pdet, sizeof(double), 1024);
  for (long e = 0; e < lv.n; ++e) {
    const node_id id = unpack_key(lv.k[e]);
    if (id.level >= t->L || id.level == 0) continue;
    const key_t_ pk = pack_key(id.level - 1, id.idx[0] >> 1, id.idx[1] >> 1, id.idx[2] >> 1);
    int fresh = 0;
    double* d = (double*)omap_insert(&pdet, pk, &fresh);
    if (fresh) {
      const node_id pid = unpack_key(pk);
      *d = detail(t, &pid);
    }
    if (*d >= thr(t, t->eps, id.level)) split[ns++] = lv.k[e];
  }
  omap_free(&pdet);
  free(lv.k);

  if (nbuf > 0 && ns > 0) { /* std::set<NodeKey> extended */
    omap ext;
    omap_init(&ext, 1, (size_t)ns * 4);
    for (long e = 0; e < ns; ++e) omap_insert(&ext, split[e], NULL);
    for (long e = 0; e < ns; ++e) {
      const node_id id = unpack_key(split[e]);
      const int r = id.level < nbuf ? buffer[id.level] : 0;
      if (r <= 0) continue;
      const int rz = t->dim == 3 ? r : 0;
      for (int dk = -rz; dk <= rz; ++dk)
        for (int dj = -r; dj <= r; ++dj)
          for (int di = -r; di <= r; ++di) {
            if (di == 0 && dj == 0 && dk == 0) continue;
            node_id pos = id;
            pos.idx[0] += di, pos.idx[1] += dj, pos.idx[2] += dk;
            int flip[3];
            const node_id mp = map_position(t, pos, flip);
            const mr_node* nb = find_id(t, &mp);
            if (nb && nb->status == ST_LEAF) omap_insert(&ext, key_of(&mp), NULL);
          }
    }
    free(split);
    split = (key_t_*)malloc(sizeof(key_t_) * (ext.count + 1));
    ns = 0;
    for (size_t i = 0; i < ext.cap; ++i)
      if (ext.used[i]) split[ns++] = ext.keys[i];
    omap_free(&ext);
  }
  qsort(split, (size_t)ns, sizeof(key_t_), cmp_key_asc);
  for (long e = 0; e < ns; ++e)
    if (find(t, split[e])->status == ST_LEAF) split_leaf(t, split[e]);
  free(split);
  enforce_gradedness(t);
}

/* merge_allowed (mr_tree.cpp:446-471) */
static int merge_allowed(const mr_tree* t, const node_id* parent) {
  const int fl = parent->level + 1;
  const int nf = 1 << fl;
  for (int a = 0; a < t->dim; ++a)
    for (int dir = -1; dir <= 1; dir += 2) {
      const int tzn = t->dim == 3 ? 2 : 1;
      const int b1 = a == 0 ? 1 : 0, b2 = a == 2 ? 1 : 2;
      for (int t2 = 0; t2 < tzn; ++t2)
        for (int t1 = 0; t1 < 2; ++t1) {
          node_id ring;
          ring.level = fl;
          ring.idx[a] = dir > 0 ? 2 * parent->idx[a] + 2 : 2 * parent->idx[a] - 1;
          ring.idx[b1] = 2 * parent->idx[b1] + t1;
          ring.idx[b2] = 2 * parent->idx[b2] + (t->dim == 3 ? t2 : 0);
          if (!periodic(t, a) && (ring.idx[a] < 0 || ring.idx[a] >= nf)) continue;
          int flip[3];
          const node_id mp = map_position(t, ring, flip);
          const mr_node* nb = find_id(t, &mp);
          if (nb && nb->status == ST_INTERNAL) return 0;
        }
    }
  return 1;
}

/* coarsen (mr_tree.cpp:473-511): internals finest first (descending keys),
 * merge when all children are leaves, detail < eps and the fine ring has no
 * internal node; repeat passes until one merges nothing. */
static void coarsen(mr_tree* t, double eps) {
  int merged = 1;
  const int children = 1 << t->dim;
  while (merged) {
    merged = 0;
    keylist in = collect(t, ST_INTERNAL, 0, 1 << 20, 1);
    for (long e = 0; e < in.n; ++e) {
      const node_id id = unpack_key(in.k[e]);
      if (id.level < t->min_leaf) continue;
      key_t_ ck[8];
      int all = 1;
      for (int c = 0; c < children; ++c) {
        ck[c] = child_key(&id, c);
        const mr_node* ch = find(t, ck[c]);
        if (!ch || ch->status != ST_LEAF) {
          all = 0;
          break;
        }
      }
      if (!all) continue;
      if (!(detail(t, &id) < thr(t, eps, id.level + 1))) continue;
      if (!merge_allowed(t, &id)) continue;
      afo_state sum;
      st_zero(&sum);
      for (int c = 0; c < children; ++c) st_add(&sum, &find(t, ck[c])->q);
      mr_node* p = find(t, in.k[e]);
      st_scale(&sum, 1.0 / (double)children);
      p->q = sum;
      p->q_old = sum;
      p->status = ST_LEAF;
      for (int c = 0; c < children; ++c) omap_erase(&t->nodes, ck[c]);
      merged = 1;
    }
    free(in.k);
  }
}

/* add_virtual_leaves (mr_tree.cpp:513-551) */
static void add_virtual_leaves(mr_tree* t) {
  const int children = 1 << t->dim;
  keylist lv = leaves(t);
  static const int offs[4] = {-2, -1, 1, 2};
  for (long e = 0; e < lv.n; ++e) {
    const node_id id = unpack_key(lv.k[e]);
    const int n = 1 << id.level;
    for (int a = 0; a < t->dim; ++a)
      for (int o = 0; o < 4; ++o) {
        node_id pos = id;
        pos.idx[a] += offs[o];
        if (!periodic(t, a) && (pos.idx[a] < 0 || pos.idx[a] >= n)) continue;
        int flip[3];
        const node_id mp = map_position(t, pos, flip);
        if (find_id(t, &mp)) continue;
        node_id parent;
        parent.level = mp.level - 1;
        for (int b = 0; b < 3; ++b) parent.idx[b] = mp.idx[b] >> 1;
        const mr_node* pn = find_id(t, &parent);
        if (!pn || pn->status != ST_LEAF) continue;
        afo_state pred[8];
        predict_children(t, &parent, pred);
        for (int c = 0; c < children; ++c) {
          const key_t_ k = child_key(&parent, c);
          if (find(t, k)) continue;
          mr_node* v = (mr_node*)omap_insert(&t->nodes, k, NULL);
          v->q = pred[c];
          v->q_old = pred[c];
          v->status = ST_VIRTUAL;
        }
      }
  }
  free(lv.k);
}

/* remove_virtual_leaves (mr_tree.cpp:553-560) */
static void remove_virtual_leaves(mr_tree* t) {
  keylist v = collect(t, ST_VIRTUAL, 0, 1 << 20, 0);
  for (long e = 0; e < v.n; ++e) omap_erase(&t->nodes, v.k[e]);
  free(v.k);
}

/* ---- solver (mr_solver.cpp) ---------------------------------------------- */
static inline key_t_ face_key(key_t_ cell, int axis, int side_bit) { /* mr_solver.cpp:17-20 */
  return (cell << 3) | ((key_t_)axis << 1) | (key_t_)side_bit;
}

/* resolve (mr_solver.cpp:36-57) */
static afo_state resolve(const mr_tree* t, node_id pos, double tau, int lo) {
  int flip[3];
  const node_id mp = map_position(t, pos, flip);
  const mr_node* nd = find_id(t, &mp);
  afo_state q;
  if (!nd) {
    q = predict_single(t, &mp);
  } else if (nd->status == ST_VIRTUAL && mp.level - 1 < lo) {
    const int lv = mp.level - 1;
    const double denom = t->t_new[lv] - t->t_old[lv];
    double theta = 1.0;
    if (denom > 0.0) {
      theta = (tau - t->t_old[lv]) / denom;
      theta = theta < 0.0 ? 0.0 : (1.0 < theta ? 1.0 : theta); /* std::clamp */
    }
    for (int m = 0; m < 5; ++m) q.v[m] = nd->q_old.v[m] * (1.0 - theta) + nd->q.v[m] * theta;
  } else {
    q = nd->q;
  }
  for (int a = 0; a < 3; ++a)
    if (flip[a]) q.v[1 + a] = -q.v[1 + a];
  return q;
}

/* face_flux_w over four resolved states in +axis order (qa, qb | qc, qd) */
static afo_state flux4(mr_tree* t, const afo_state* qa, const afo_state* qb, const afo_state* qc,
                       const afo_state* qd, int axis) {
  const afo_prim wa = afo_primitives_unguarded(qa, t->gamma);
  const afo_prim wb = afo_primitives_unguarded(qb, t->gamma);
  const afo_prim wc = afo_primitives_unguarded(qc, t->gamma);
  const afo_prim wd = afo_primitives_unguarded(qd, t->gamma);
  return afo_face_flux_w(qb, qc, &wa, &wb, &wc, &wd, axis, t->limiter, t->flux, t->gamma,
                         &t->fallbacks);
}

/* fine_face_average (mr_solver.cpp:59-95), including the (p-2, p-1 | p, p+2)
 * stencil for dir < 0 as the reference builds it. */
static afo_state fine_face_average(mr_tree* t, const node_id* cell, int axis, int dir, double tau,
                                   int lo) {
  const int fl = cell->level + 1;
  const int tzn = t->dim == 3 ? 2 : 1;
  const int b1 = axis == 0 ? 1 : 0, b2 = axis == 2 ? 1 : 2;
  afo_state sum;
  st_zero(&sum);
  for (int t2 = 0; t2 < tzn; ++t2)
    for (int t1 = 0; t1 < 2; ++t1) {
      node_id p;
      p.level = fl;
      p.idx[axis] = 2 * cell->idx[axis] + (dir > 0 ? 1 : 0);
      p.idx[b1] = 2 * cell->idx[b1] + t1;
      p.idx[b2] = 2 * cell->idx[b2] + (t->dim == 3 ? t2 : 0);
      node_id s0 = p, s1 = p, s2 = p, s3 = p;
      s0.idx[axis] += dir > 0 ? -1 : 2;
      s2.idx[axis] += dir;
      s3.idx[axis] += 2 * dir;
      const afo_state qa = resolve(t, dir > 0 ? s0 : s3, tau, lo);
      const afo_state qb = resolve(t, dir > 0 ? s1 : s2, tau, lo);
      const afo_state qc = resolve(t, dir > 0 ? s2 : s1, tau, lo);
      const afo_state qd = resolve(t, dir > 0 ? s3 : s0, tau, lo);
      const afo_state f = flux4(t, &qa, &qb, &qc, &qd, axis);
      st_add(&sum, &f);
    }
  st_scale(&sum, 1.0 / (double)(tzn * 2));
  return sum;
}

/* face_flux_at (mr_solver.cpp:97-161) */
static afo_state face_flux_at(mr_tree* t, const node_id* cell, int axis, int dir, double tau,
                              int lo, int hi, int register_stage, double step_dt) {
  node_id np = *cell;
  np.idx[axis] += dir;
  int flip[3];
  const node_id mp = map_position(t, np, flip);
  const mr_node* nb = find_id(t, &mp);
  const int nb_status = nb ? nb->status : -1;

  node_id s0 = *cell, s2 = *cell, s3 = *cell;
  s0.idx[axis] -= dir;
  s2.idx[axis] += dir;
  s3.idx[axis] += 2 * dir;
  if (nb_status == ST_INTERNAL) {
    if (mp.level + 1 <= hi) return fine_face_average(t, cell, axis, dir, tau, lo);
    /* provisional flux from the projected neighbour (local time stepping) */
    const afo_state qa = resolve(t, dir > 0 ? s0 : s3, tau, lo);
    const afo_state qb = resolve(t, dir > 0 ? *cell : s2, tau, lo);
    const afo_state qc = resolve(t, dir > 0 ? s2 : *cell, tau, lo);
    const afo_state qd = resolve(t, dir > 0 ? s3 : s0, tau, lo);
    const afo_state f = flux4(t, &qa, &qb, &qc, &qd, axis);
    if (register_stage) {
      mr_reg* r = (mr_reg*)omap_insert(&t->regs, face_key(key_of(cell), axis, dir > 0 ? 1 : 0), NULL);
      st_add_scaled(&r->coarse, &f, step_dt);
      r->has_coarse = 1;
    }
    return f;
  }
  const afo_state qa = resolve(t, dir > 0 ? s0 : s3, tau, lo);
  const afo_state qb = resolve(t, dir > 0 ? *cell : s2, tau, lo);
  const afo_state qc = resolve(t, dir > 0 ? s2 : *cell, tau, lo);
  const afo_state qd = resolve(t, dir > 0 ? s3 : s0, tau, lo);
  const afo_state f = flux4(t, &qa, &qb, &qc, &qd, axis);
  if (register_stage && nb_status == ST_VIRTUAL && mp.level - 1 < lo) {
    /* fine share replacing the already-advanced coarse cell's flux */
    const key_t_ pk = pack_key(mp.level - 1, mp.idx[0] >> 1, mp.idx[1] >> 1, mp.idx[2] >> 1);
    const int side_bit = dir > 0 ? 0 : 1;
    mr_reg* r = (mr_reg*)omap_insert(&t->regs, face_key(pk, axis, side_bit), NULL);
    const double share = t->dim == 3 ? 0.25 : 0.5;
    st_add_scaled(&r->fine, &f, step_dt * share);
    r->has_fine = 1;
  }
  return f;
}

static void node_str(char* buf, size_t n, const node_id* id) { /* mr_solver.cpp:11-14 */
  snprintf(buf, n, "level %d (%d,%d,%d)", id->level, id->idx[0], id->idx[1], id->idx[2]);
}

/* stage (mr_solver.cpp:163-193): pass 1 fluxes per leaf (pull form), pass 2
 * q = q_old + rhs * stage_dt. */
static void stage(mr_tree* t, int lo, int hi, const keylist* lv, double tau, double stage_dt,
                  int register_stage, double step_dt) {
  for (long e = 0; e < lv->n; ++e) {
    const node_id id = unpack_key(lv->k[e]);
    const afo_state q = find(t, lv->k[e])->q;
    const afo_prim w = afo_primitives_unguarded(&q, t->gamma);
    if (!(q.v[0] > AFO_POS_TOL) || !afo_physical(&w)) {
      char s[96];
      node_str(s, sizeof s, &id);
      raise_err(1, "%s: rho=%f p=%f", s, q.v[0], w.p); /* std::to_string(double) is %f */
    }
    const double dx = dx_at(id.level);
    const double c = afo_sound_speed(&w, t->gamma);
    for (int a = 0; a < t->dim; ++a) {
      const double r = (fabs(w.v[a]) + c) * step_dt / dx;
      t->max_cfl = t->max_cfl < r ? r : t->max_cfl;
    }
    afo_state rhs;
    st_zero(&rhs);
    const double inv_dx = 1.0 / dx;
    for (int a = 0; a < t->dim; ++a) {
      const afo_state fm = face_flux_at(t, &id, a, -1, tau, lo, hi, register_stage, step_dt);
      st_add_scaled(&rhs, &fm, inv_dx);
      const afo_state fp = face_flux_at(t, &id, a, +1, tau, lo, hi, register_stage, step_dt);
      st_sub_scaled(&rhs, &fp, inv_dx);
    }
    find(t, lv->k[e])->rhs = rhs;
  }
  for (long e = 0; e < lv->n; ++e) {
    mr_node* nd = find(t, lv->k[e]);
    for (int m = 0; m < 5; ++m) nd->q.v[m] = nd->q_old.v[m] + nd->rhs.v[m] * stage_dt;
  }
}

/* refresh_virtuals (mr_solver.cpp:195-208) */
static void refresh_virtuals(mr_tree* t, const keylist* parents) {
  const int children = 1 << t->dim;
  for (long e = 0; e < parents->n; ++e) {
    const node_id pid = unpack_key(parents->k[e]);
    afo_state pred[8];
    predict_children(t, &pid, pred);
    for (int c = 0; c < children; ++c) {
      mr_node* ch = find(t, child_key(&pid, c));
      if (ch && ch->status == ST_VIRTUAL) ch->q = pred[c];
    }
  }
}

/* apply_registers (mr_solver.cpp:210-230) */
static void apply_registers(mr_tree* t, int coarse_level) {
  key_t_* keys = (key_t_*)malloc(sizeof(key_t_) * (t->regs.count + 1));
  long n = 0;
  for (size_t i = 0; i < t->regs.cap; ++i)
    if (t->regs.used[i] && unpack_key(t->regs.keys[i] >> 3).level == coarse_level)
      keys[n++] = t->regs.keys[i];
  qsort(keys, (size_t)n, sizeof(key_t_), cmp_key_asc);
  for (long e = 0; e < n; ++e) {
    const mr_reg reg = *(const mr_reg*)omap_find(&t->regs, keys[e]);
    const node_id cid = unpack_key(keys[e] >> 3);
    char s[96];
    node_str(s, sizeof s, &cid);
    if (!reg.has_coarse || !reg.has_fine) {
      free(keys);
      raise_err(2, "interface flux register at %s is missing a side", s);
    }
    mr_node* nd = find(t, keys[e] >> 3);
    if (!nd || nd->status != ST_LEAF) {
      free(keys);
      raise_err(2, "flux register target is not a leaf: %s", s);
    }
    const double sign = (keys[e] & 1) == 1 ? 1.0 : -1.0;
    const double f = sign / dx_at(cid.level);
    for (int m = 0; m < 5; ++m) nd->q.v[m] = nd->q.v[m] + (reg.coarse.v[m] - reg.fine.v[m]) * f;
    omap_erase(&t->regs, keys[e]);
  }
  free(keys);
}

/* project_range lambda of step_levels (mr_solver.cpp:268-282) */
static void project_range(mr_tree* t, int lo, int top) {
  keylist in = collect(t, ST_INTERNAL, lo, top - 1, 1);
  const int children = 1 << t->dim;
  for (long e = 0; e < in.n; ++e) {
    const node_id id = unpack_key(in.k[e]);
    afo_state sum;
    st_zero(&sum);
    for (int c = 0; c < children; ++c) st_add(&sum, &find(t, child_key(&id, c))->q);
    st_scale(&sum, 1.0 / (double)children);
    find(t, in.k[e])->q = sum;
  }
  free(in.k);
}

/* step_levels (mr_solver.cpp:232-316) */
static void step_levels(mr_tree* t, int lo, int hi, double tm, double dt) {
  keylist lv = collect(t, ST_LEAF, lo, hi, 0);
  keylist vp;
  vp.k = (key_t_*)malloc(sizeof(key_t_) * (size_t)(lv.n + 1));
  vp.n = 0;
  const int children = 1 << t->dim;
  for (long e = 0; e < lv.n; ++e) {
    mr_node* nd = find(t, lv.k[e]);
    nd->q_old = nd->q;
    const node_id id = unpack_key(lv.k[e]);
    const mr_node* c0 = find(t, pack_key(id.level + 1, 2 * id.idx[0], 2 * id.idx[1], 2 * id.idx[2]));
    if (c0 && c0->status == ST_VIRTUAL) vp.k[vp.n++] = lv.k[e];
  }
  for (int l = lo; l <= hi && l <= t->L; ++l) {
    t->t_old[l] = tm;
    t->t_new[l] = tm + dt;
  }
  refresh_virtuals(t, &vp);
  for (long e = 0; e < vp.n; ++e) {
    const node_id pid = unpack_key(vp.k[e]);
    for (int c = 0; c < children; ++c) {
      mr_node* ch = find(t, child_key(&pid, c));
      if (ch && ch->status == ST_VIRTUAL) ch->q_old = ch->q;
    }
  }
  stage(t, lo, hi, &lv, tm, 0.5 * dt, 0, dt);
  project_range(t, lo, hi);
  refresh_virtuals(t, &vp);
  stage(t, lo, hi, &lv, tm + 0.5 * dt, dt, 1, dt);
  for (long e = 0; e < lv.n; ++e) {
    const afo_state q = find(t, lv.k[e])->q;
    const afo_prim w = afo_primitives_unguarded(&q, t->gamma);
    if (!(q.v[0] > AFO_POS_TOL) || !afo_physical(&w)) {
      char s[96];
      const node_id id = unpack_key(lv.k[e]);
      node_str(s, sizeof s, &id);
      free(lv.k);
      free(vp.k);
      raise_err(1, "post-step %s", s);
    }
  }
  project_range(t, lo, hi);
  refresh_virtuals(t, &vp);
  free(lv.k);
  free(vp.k);
  int deeper = 0;
  for (size_t i = 0; i < t->nodes.cap && !deeper; ++i)
    if (t->nodes.used[i] &&
        ((const mr_node*)(t->nodes.vals + i * t->nodes.vsize))->status == ST_LEAF &&
        (int)(t->nodes.keys[i] >> (3 * KB)) > hi)
      deeper = 1;
  if (deeper) {
    step_levels(t, hi + 1, hi + 1, tm, 0.5 * dt);
    step_levels(t, hi + 1, hi + 1, tm + 0.5 * dt, 0.5 * dt);
    apply_registers(t, hi);
    project_range(t, lo, hi + 1);
  }
}

/* from_uniform + set_norms_from (mr_tree.cpp:29-87) */
static void from_uniform(mr_tree* t, const double* init) {
  const int L = t->L, n = 1 << L, nz = t->dim == 3 ? n : 1;
  double nm[5] = {0, 0, 0, 0, 0};
  long c = 0;
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i, ++c) {
        mr_node* nd = (mr_node*)omap_insert(&t->nodes, pack_key(L, i, j, k), NULL);
        for (int m = 0; m < 5; ++m) nd->q.v[m] = init[5 * c + m];
        nd->q_old = nd->q;
        nd->status = ST_LEAF;
        for (int m = 0; m < 5; ++m) {
          const double a = fabs(init[5 * c + m]);
          nm[m] = nm[m] < a ? a : nm[m];
        }
      }
  for (int l = L - 1; l >= 0; --l) {
    const int nl = 1 << l, nzl = t->dim == 3 ? nl : 1, zc = t->dim == 3 ? 2 : 1;
    const double w = t->dim == 3 ? 0.125 : 0.25;
    for (int k = 0; k < nzl; ++k)
      for (int j = 0; j < nl; ++j)
        for (int i = 0; i < nl; ++i) {
          afo_state sum;
          st_zero(&sum);
          for (int dk = 0; dk < zc; ++dk)
            for (int dj = 0; dj < 2; ++dj)
              for (int di = 0; di < 2; ++di)
                st_add(&sum, &find(t, pack_key(l + 1, 2 * i + di, 2 * j + dj, 2 * k + dk))->q);
          st_scale(&sum, w);
          mr_node* nd = (mr_node*)omap_insert(&t->nodes, pack_key(l, i, j, k), NULL);
          nd->q = sum;
          nd->q_old = sum;
          nd->status = ST_INTERNAL;
        }
  }
  double global = 1e-300;
  for (int m = 4; m >= 0; --m) global = global < nm[m] ? nm[m] : global; /* std::max({...}) */
  for (int m = 0; m < 5; ++m) {
    if (nm[m] < 1e-12 * global) nm[m] = global;
    t->norms[m] = nm[m];
  }
}

/* mr_tree.cpp:608-621 to_uniform(L) */
static void to_uniform(const mr_tree* t, double* out) {
  const int n = 1 << t->L, nz = t->dim == 3 ? n : 1;
  long c = 0;
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i, ++c) {
        node_id pos = {t->L, {i, j, k}};
        const afo_state q = value_at(t, pos);
        for (int m = 0; m < 5; ++m) out[5 * c + m] = q.v[m];
      }
}

/* MRTree::dump (mr_tree.cpp:623-641): ostream precision 17 == %.17g */
static char* dump_tree(const mr_tree* t) {
  keylist all;
  all.k = (key_t_*)malloc(sizeof(key_t_) * (t->nodes.count + 1));
  all.n = 0;
  for (size_t i = 0; i < t->nodes.cap; ++i)
    if (t->nodes.used[i]) all.k[all.n++] = t->nodes.keys[i];
  qsort(all.k, (size_t)all.n, sizeof(key_t_), cmp_key_asc);
  size_t cap = 256 * (size_t)(all.n + 1), len = 0;
  char* s = (char*)malloc(cap);
  s[0] = 0;
  for (long e = 0; e < all.n; ++e) {
    const node_id id = unpack_key(all.k[e]);
    const mr_node* nd = find(t, all.k[e]);
    const char* st = nd->status == ST_LEAF ? "leaf" : nd->status == ST_INTERNAL ? "internal"
                                                                               : "virtual";
    len += (size_t)snprintf(s + len, cap - len, "%d %d %d %d %s %.17g %.17g %.17g %.17g %.17g\n",
                            id.level, id.idx[0], id.idx[1], id.idx[2], st, nd->q.v[0],
                            nd->q.v[1], nd->q.v[2], nd->q.v[3], nd->q.v[4]);
  }
  free(all.k);
  return s;
}

static char* g_last_dump_mr;

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* The run loop of oracle/ref_harness.cpp afref_mr_run (mr_solver.cpp:318-400
 * with from_uniform(grid, 0) -> set_min_leaf_level -> coarsen(eps), the CFL
 * rule over the leaves after refine, and the per-cycle records). */
int afo_mr_run(const af_oracle_params* p, const double* init, double* out,
               uint64_t* leaf_keys, long* n_leaves, long* per_cycle, long max_cycles,
               double* dt_hist, af_oracle_result* res) {
  memset(res, 0, sizeof(*res));
  if (p->integrator != 0) {
    res->err_kind = 9;
    snprintf(res->err, sizeof res->err, "run_mr steps with RK2 only");
    return 9;
  }
  static mr_tree T; /* static: survives the longjmp */
  memset(&T, 0, sizeof T);
  mr_tree* t = &T;
  t->dim = p->dim;
  t->L = p->level;
  for (int f = 0; f < 6; ++f) t->bc[f] = p->bc[f];
  t->eps = p->eps;
  t->eps_level = p->eps_level;
  t->limiter = p->limiter;
  t->flux = p->flux;
  t->gamma = p->gamma;
  t->t_old = (double*)calloc((size_t)p->level + 2, sizeof(double));
  t->t_new = (double*)calloc((size_t)p->level + 2, sizeof(double));
  const long fine = 1L << (p->dim * p->level);
  omap_init(&t->nodes, sizeof(mr_node), (size_t)(fine + fine / 2));
  omap_init(&t->regs, sizeof(mr_reg), 1024);
  static volatile long done, cycle;
  static volatile int in_step;
  done = 0, cycle = 0, in_step = 0;
  int* buffer = (int*)calloc((size_t)p->level + 1, sizeof(int));
  if (setjmp(g_jmp)) {
    res->err_kind = g_err_kind;
    if (g_err_kind == 1 && in_step)
      snprintf(res->err, sizeof res->err, "step %ld: %.480s", (long)done, g_err);
    else
      snprintf(res->err, sizeof res->err, "%s", g_err);
    goto cleanup; /* like the harness: only the completed cycles are reported */
  }
  {
    const int L = p->level;
    t->min_leaf = 0;
    from_uniform(t, init);
    coarsen(t, 0.0); /* from_uniform(grid, 0.0): the threshold hook applies to it too */
    int ml = p->min_leaf_level;
    if (p->local_time) {
      const int g = L - p->lt_gap > 0 ? L - p->lt_gap : 0;
      ml = ml > g ? ml : g;
    }
    t->min_leaf = ml;
    coarsen(t, p->eps);
    const double dx_L = dx_at(L);
    double wall = 0.0, tm = 0.0;
    while (done < p->n_steps) {
      const double t0 = now_s();
      long sub = 1;
      int top = L;
      if (p->local_time) { /* mr_solver.cpp:345-354 */
        const int cl = coarsest_leaf_level(t);
        top = cl > t->min_leaf ? cl : t->min_leaf;
        long span = 1L << (L - top);
        while (span > p->n_steps - done) {
          span >>= 1;
          ++top;
        }
        sub = span;
        for (int l = 0; l <= L; ++l) buffer[l] = l > top + 1 ? 1 << (l - top - 1) : 1;
        refine(t, buffer, L + 1);
      } else {
        refine(t, NULL, 0);
      }
      add_virtual_leaves(t);
      const long cells = (long)t->nodes.count;
      const long nleaves = leaf_count(t);
      double excluded = 0.0;
      if (per_cycle && cycle < max_cycles) {
        const double tx = now_s();
        long upd = 0;
        keylist lv = leaves(t);
        for (long e = 0; e < lv.n; ++e) {
          const int l = unpack_key(lv.k[e]).level;
          upd += 2 * (l > top ? (1L << (l - top)) : 1L);
        }
        free(lv.k);
        excluded += now_s() - tx;
        per_cycle[5 * cycle + 0] = nleaves;
        per_cycle[5 * cycle + 1] = cells;
        per_cycle[5 * cycle + 2] = sub;
        per_cycle[5 * cycle + 3] = top;
        per_cycle[5 * cycle + 4] = upd;
      }
      double dt = p->fixed_dt;
      if (p->cfl > 0.0) {
        double smax = 0.0;
        keylist lv = leaves(t);
        for (long e = 0; e < lv.n; ++e) {
          const double s = afo_speed_sum(&find(t, lv.k[e])->q, p->gamma, p->dim);
          smax = smax < s ? s : smax;
        }
        free(lv.k);
        dt = p->cfl * dx_L / smax;
      }
      if (dt_hist && cycle < max_cycles) dt_hist[cycle] = dt;
      const double t_cycle = p->cfl > 0.0 ? tm : (double)done * p->fixed_dt;
      in_step = 1;
      if (p->local_time)
        step_levels(t, 0, top, t_cycle, (double)sub * dt); /* advance_local */
      else
        step_levels(t, 0, L, 0.0, dt); /* evolve_global */
      in_step = 0;
      remove_virtual_leaves(t);
      coarsen(t, p->eps);
      done += sub;
      tm = t_cycle + (double)sub * dt;
      ++cycle;
      wall += now_s() - t0 - excluded;
      res->steps_done = done;
      res->n_cycles = cycle;
    }
    res->max_cfl = t->max_cfl;
    res->fallbacks = t->fallbacks;
    res->wall_seconds = wall;
    if (out) to_uniform(t, out);
    keylist lv = leaves(t);
    if (n_leaves) {
      if (leaf_keys)
        for (long e = 0; e < lv.n && e < *n_leaves; ++e) leaf_keys[e] = lv.k[e];
      *n_leaves = lv.n;
    }
    free(lv.k);
    free(g_last_dump_mr);
    g_last_dump_mr = dump_tree(t);
  }
cleanup:
  free(buffer);
  free(t->t_old);
  free(t->t_new);
  omap_free(&t->nodes);
  omap_free(&t->regs);
  return res->err_kind;
}

int afo_mr_last_dump(const char* path) {
  if (!g_last_dump_mr) return -1;
  FILE* f = fopen(path, "w");
  if (!f) return -1;
  const size_t n = strlen(g_last_dump_mr);
  const int ok = fwrite(g_last_dump_mr, 1, n, f) == n;
  return (fclose(f) == 0 && ok) ? 0 : -1;
}
