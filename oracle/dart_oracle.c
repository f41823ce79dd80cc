/*
 * dart_oracle.c -- sequential CPU restatement of prefixsim.kvcache.RadixCache.
 *
 * TEST INFRASTRUCTURE ONLY (parity checker + CPU baseline); see oracle.h.
 *
 * Every function follows the reference algorithm step for step, including
 * its costs: evict() does a full scan + heapify per call with lazy key
 * revalidation (kvcache.py:425-460) and set_protection() a full scan + sort
 * (kvcache.py:364-383).  Node ids are never reused (kvcache.py:135-138), so
 * a node's id is its index in the node array and detached nodes stay
 * inspectable (last_evicted keeps node objects alive in the reference).
 */
#include "oracle.h"

#include <stdlib.h>
#include <string.h>

typedef struct {
  int64_t parent; /* -1: root or detached */
  int64_t tok_off;
  int64_t len;
  int64_t nch;
  int64_t ref, last, hits;
  int64_t seg; /* OR_SEG_NONE for None */
  int64_t aseg, aoff, snap[3];
  int64_t guard_gen;
  int8_t kind, has_anchor, akind, prot, attached;
} ONode;

/* ------------------------------------------------------------- hash maps */
#define EMPTY_U64 UINT64_MAX
#define TOMB_U64 (UINT64_MAX - 1)

typedef struct {
  uint64_t *keys;
  int64_t *vals;
  int64_t cap, live, used;
} U64Map;

static uint64_t mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

static void map_init(U64Map *m, int64_t cap) {
  m->cap = cap;
  m->live = m->used = 0;
  m->keys = (uint64_t *)malloc(sizeof(uint64_t) * cap);
  m->vals = (int64_t *)malloc(sizeof(int64_t) * cap);
  for (int64_t i = 0; i < cap; i++) m->keys[i] = EMPTY_U64;
}
static void map_free(U64Map *m) {
  free(m->keys);
  free(m->vals);
}
static int64_t map_get(const U64Map *m, uint64_t key) {
  int64_t mask = m->cap - 1, h = (int64_t)(mix64(key) & (uint64_t)mask);
  for (;;) {
    uint64_t k = m->keys[h];
    if (k == key) return m->vals[h];
    if (k == EMPTY_U64) return -1;
    h = (h + 1) & mask;
  }
}
static void map_put(U64Map *m, uint64_t key, int64_t val);
static void map_grow(U64Map *m) {
  U64Map n;
  int64_t cap = m->cap;
  if (m->live * 4 > cap) cap *= 2;
  map_init(&n, cap);
  for (int64_t i = 0; i < m->cap; i++)
    if (m->keys[i] != EMPTY_U64 && m->keys[i] != TOMB_U64) map_put(&n, m->keys[i], m->vals[i]);
  map_free(m);
  *m = n;
}
static void map_put(U64Map *m, uint64_t key, int64_t val) {
  if ((m->used + 1) * 2 > m->cap) map_grow(m);
  int64_t mask = m->cap - 1, h = (int64_t)(mix64(key) & (uint64_t)mask), tomb = -1;
  for (;;) {
    uint64_t k = m->keys[h];
    if (k == key) {
      m->vals[h] = val;
      return;
    }
    if (k == TOMB_U64 && tomb < 0) tomb = h;
    if (k == EMPTY_U64) break;
    h = (h + 1) & mask;
  }
  if (tomb >= 0) {
    h = tomb;
  } else {
    m->used++;
  }
  m->keys[h] = key;
  m->vals[h] = val;
  m->live++;
}
static void map_del(U64Map *m, uint64_t key) {
  int64_t mask = m->cap - 1, h = (int64_t)(mix64(key) & (uint64_t)mask);
  for (;;) {
    uint64_t k = m->keys[h];
    if (k == key) {
      m->keys[h] = TOMB_U64;
      m->live--;
      return;
    }
    if (k == EMPTY_U64) return;
    h = (h + 1) & mask;
  }
}

/* segment-keyed maps (priorities, active set): keys are int64 segment ids */
static uint64_t segkey(int64_t s) { return (uint64_t)s ^ 0x8000000000000000ULL; }

/* ------------------------------------------------------------------ tree */
struct OTree {
  int64_t capacity, protect_budget;
  int policy;
  ONode *nodes;
  int64_t nnodes, ncap;
  uint32_t *toks;
  int64_t ntoks, tcap;
  U64Map children; /* (parent id << 32 | first token) -> child id */
  int64_t resident, clock;
  U64Map prio;   /* seg -> index into prio_vals */
  double *prio_vals;
  int64_t nprio;
  U64Map active; /* seg set */
  int64_t *protected_ids;
  int64_t nprot;
  int64_t guard_gen;
  int64_t *last_evicted;
  int64_t nlast, lastcap;
  int64_t *vlog; /* every victim of every evict call, in order (test observability) */
  int64_t nvlog, vlogcap;
};

static uint64_t ckey(int64_t parent, uint32_t tok) { return ((uint64_t)parent << 32) | tok; }

/* _new_node (kvcache.py:135-138) */
static int64_t new_node(OTree *t, int64_t tok_off, int64_t len, int64_t parent) {
  if (t->nnodes == t->ncap) {
    t->ncap *= 2;
    t->nodes = (ONode *)realloc(t->nodes, sizeof(ONode) * t->ncap);
  }
  int64_t id = t->nnodes++;
  ONode *n = &t->nodes[id];
  memset(n, 0, sizeof(*n));
  n->parent = parent;
  n->tok_off = tok_off;
  n->len = len;
  n->kind = OR_PRIVATE; /* RadixNode.__init__ default (kvcache.py:102) */
  n->seg = OR_SEG_NONE;
  n->aseg = OR_SEG_NONE;
  n->attached = 1;
  n->guard_gen = -1;
  return id;
}

static int64_t push_tokens(OTree *t, const uint32_t *p, int64_t n) {
  if (t->ntoks + n > t->tcap) {
    while (t->ntoks + n > t->tcap) t->tcap *= 2;
    t->toks = (uint32_t *)realloc(t->toks, sizeof(uint32_t) * t->tcap);
  }
  int64_t off = t->ntoks;
  memcpy(t->toks + off, p, sizeof(uint32_t) * n);
  t->ntoks += n;
  return off;
}

OTree *ot_create(int64_t capacity_tokens, int policy, int64_t protect_budget) {
  if (capacity_tokens <= 0 || protect_budget < 0) return NULL; /* CacheConfig (kvcache.py:72-76) */
  OTree *t = (OTree *)calloc(1, sizeof(OTree));
  t->capacity = capacity_tokens;
  t->policy = policy;
  t->protect_budget = protect_budget;
  t->ncap = 1024;
  t->nodes = (ONode *)malloc(sizeof(ONode) * t->ncap);
  t->tcap = 4096;
  t->toks = (uint32_t *)malloc(sizeof(uint32_t) * t->tcap);
  map_init(&t->children, 1024);
  map_init(&t->prio, 64);
  map_init(&t->active, 64);
  t->prio_vals = NULL;
  int64_t root = new_node(t, 0, 0, -1); /* kvcache.py:123-124 */
  t->nodes[root].kind = OR_SYSTEM;
  t->lastcap = 64;
  t->last_evicted = (int64_t *)malloc(sizeof(int64_t) * t->lastcap);
  t->vlogcap = 64;
  t->vlog = (int64_t *)malloc(sizeof(int64_t) * t->vlogcap);
  return t;
}

void ot_destroy(OTree *t) {
  if (!t) return;
  free(t->nodes);
  free(t->toks);
  map_free(&t->children);
  map_free(&t->prio);
  map_free(&t->active);
  free(t->prio_vals);
  free(t->protected_ids);
  free(t->last_evicted);
  free(t->vlog);
  free(t);
}

static int64_t tick(OTree *t) { return ++t->clock; } /* kvcache.py:140-142 */

static int64_t child_of(const OTree *t, int64_t node, uint32_t tok) {
  return map_get(&t->children, ckey(node, tok));
}

/* _lcp (kvcache.py:109-114) */
static int64_t lcp(const uint32_t *a, int64_t na, const uint32_t *b, int64_t nb) {
  int64_t n = na < nb ? na : nb, i = 0;
  while (i < n && a[i] == b[i]) i++;
  return i;
}

/* match_prefix (kvcache.py:146-171) */
int64_t ot_match(OTree *t, const uint32_t *path, int64_t n, int64_t *visited, int64_t *nvisited) {
  int64_t now = tick(t), node = 0, i = 0, nv = 0;
  while (i < n) {
    int64_t c = child_of(t, node, path[i]);
    if (c < 0) break;
    ONode *cn = &t->nodes[c];
    int64_t k = lcp(t->toks + cn->tok_off, cn->len, path + i, n - i);
    if (k == 0) break;
    cn->last = now;
    cn->hits += 1;
    if (visited) visited[nv] = c;
    nv++;
    i += k;
    if (k < cn->len) break;
    node = c;
  }
  if (nvisited) *nvisited = nv;
  return i;
}

/* _walk_resident (kvcache.py:173-186) */
static int64_t walk_resident(const OTree *t, const uint32_t *path, int64_t n) {
  int64_t node = 0, i = 0;
  while (i < n) {
    int64_t c = child_of(t, node, path[i]);
    if (c < 0) break;
    const ONode *cn = &t->nodes[c];
    int64_t k = lcp(t->toks + cn->tok_off, cn->len, path + i, n - i);
    i += k;
    if (k < cn->len) break;
    node = c;
  }
  return i;
}

/* ---------------------------------------------------------------- keys */
typedef struct {
  int64_t a;
  double p;
  int64_t b, c;
} OKey;

static double prio_of(const OTree *t, int64_t seg) {
  if (seg == OR_SEG_NONE) return 0.0; /* dict.get(None, 0.0) */
  int64_t ix = map_get(&t->prio, segkey(seg));
  return ix < 0 ? 0.0 : t->prio_vals[ix];
}

/* evict_key (kvcache.py:397-414) as a fixed-width tuple */
static OKey evict_key(const OTree *t, int64_t id) {
  const ONode *n = &t->nodes[id];
  OKey k = {0, 0.0, 0, 0};
  switch (t->policy) {
    case OR_DART:
      if (n->kind == OR_PRIVATE) {
        k.a = 0;
      } else if (n->prot) {
        k.a = 2;
      } else {
        k.a = 1;
        k.p = prio_of(t, n->seg);
      }
      k.b = n->last;
      k.c = id;
      break;
    case OR_LRU:
      k.a = n->last;
      k.b = id;
      break;
    case OR_LFU:
      k.a = n->hits;
      k.b = n->last;
      k.c = id;
      break;
    default: /* LRU_ACTIVE */
      k.a = (n->seg != OR_SEG_NONE && map_get(&t->active, segkey(n->seg)) >= 0) ? 1 : 0;
      k.b = n->last;
      k.c = id;
      break;
  }
  return k;
}

/* Python tuple ordering on the key fields (all keys end in the node id) */
static int key_cmp(OKey x, OKey y) {
  if (x.a != y.a) return x.a < y.a ? -1 : 1;
  if (x.p != y.p) return x.p < y.p ? -1 : 1;
  if (x.b != y.b) return x.b < y.b ? -1 : 1;
  if (x.c != y.c) return x.c < y.c ? -1 : 1;
  return 0;
}

void ot_evict_key(const OTree *t, int64_t id, int64_t *ints, double *pri) {
  OKey k = evict_key(t, id);
  ints[0] = k.a;
  ints[1] = k.b;
  ints[2] = k.c;
  *pri = k.p;
}

/* _is_evictable (kvcache.py:416-423) */
static int is_evictable(const OTree *t, int64_t id) {
  const ONode *n = &t->nodes[id];
  if (n->parent < 0 || n->nch > 0 || n->ref > 0) return 0;
  if (n->guard_gen == t->guard_gen) return 0;
  if (t->policy == OR_DART && n->kind == OR_SYSTEM) return 0;
  return 1;
}

/* binary min-heap of (key, node id), the heapq list of kvcache.py:438 */
typedef struct {
  OKey k;
  int64_t id;
} HEnt;

static int hless(const HEnt *x, const HEnt *y) {
  int c = key_cmp(x->k, y->k);
  if (c) return c < 0;
  return x->id < y->id;
}
static void sift_down(HEnt *h, int64_t n, int64_t i) {
  for (;;) {
    int64_t l = 2 * i + 1, r = l + 1, m = i;
    if (l < n && hless(&h[l], &h[m])) m = l;
    if (r < n && hless(&h[r], &h[m])) m = r;
    if (m == i) return;
    HEnt tmp = h[i];
    h[i] = h[m];
    h[m] = tmp;
    i = m;
  }
}
static void sift_up(HEnt *h, int64_t i) {
  while (i > 0) {
    int64_t p = (i - 1) / 2;
    if (!hless(&h[i], &h[p])) return;
    HEnt tmp = h[i];
    h[i] = h[p];
    h[p] = tmp;
    i = p;
  }
}

static void record_victim(OTree *t, int64_t id) {
  if (t->nlast == t->lastcap) {
    t->lastcap *= 2;
    t->last_evicted = (int64_t *)realloc(t->last_evicted, sizeof(int64_t) * t->lastcap);
  }
  t->last_evicted[t->nlast++] = id;
  if (t->nvlog == t->vlogcap) {
    t->vlogcap *= 2;
    t->vlog = (int64_t *)realloc(t->vlog, sizeof(int64_t) * t->vlogcap);
  }
  t->vlog[t->nvlog++] = id;
}

/* evict (kvcache.py:425-460) */
int64_t ot_evict(OTree *t, int64_t k_free) {
  if (k_free < 0) return -1;
  t->nlast = 0;
  if (k_free == 0) return 0;
  /* full scan of the tree (kvcache.py:439-441) */
  int64_t cap = 16, n = 0;
  HEnt *heap = (HEnt *)malloc(sizeof(HEnt) * cap);
  for (int64_t id = 1; id < t->nnodes; id++) {
    if (!t->nodes[id].attached) continue;
    if (is_evictable(t, id)) {
      if (n == cap) {
        cap *= 2;
        heap = (HEnt *)realloc(heap, sizeof(HEnt) * cap);
      }
      heap[n].k = evict_key(t, id);
      heap[n].id = id;
      n++;
    }
  }
  for (int64_t i = n / 2 - 1; i >= 0; i--) sift_down(heap, n, i); /* heapify */
  int64_t freed = 0;
  while (freed < k_free && n > 0) {
    HEnt top = heap[0];
    heap[0] = heap[--n];
    sift_down(heap, n, 0);
    int64_t id = top.id;
    ONode *nd = &t->nodes[id];
    if (!is_evictable(t, id) || nd->parent < 0) continue;
    OKey cur = evict_key(t, id);
    if (key_cmp(cur, top.k) != 0) { /* lazy revalidation (kvcache.py:448-451) */
      if (n == cap) {
        cap *= 2;
        heap = (HEnt *)realloc(heap, sizeof(HEnt) * cap);
      }
      heap[n].k = cur;
      heap[n].id = id;
      sift_up(heap, n++);
      continue;
    }
    int64_t parent = nd->parent;
    map_del(&t->children, ckey(parent, t->toks[nd->tok_off]));
    t->nodes[parent].nch--;
    nd->parent = -1;
    nd->attached = 0;
    t->resident -= nd->len;
    freed += nd->len;
    record_victim(t, id);
    if (is_evictable(t, parent)) {
      if (n == cap) {
        cap *= 2;
        heap = (HEnt *)realloc(heap, sizeof(HEnt) * cap);
      }
      heap[n].k = evict_key(t, parent);
      heap[n].id = parent;
      sift_up(heap, n++);
    }
  }
  free(heap);
  return freed;
}

/* _reserve (kvcache.py:243-273): returns OR_OK or OR_CAPACITY */
static int reserve(OTree *t, const uint32_t *path, int64_t n) {
  int64_t missing = n - walk_resident(t, path, n);
  int64_t shortfall = t->resident + missing - t->capacity;
  if (shortfall <= 0) return OR_OK;
  /* guard the matched prefix (kvcache.py:250-265) */
  int64_t gen = ++t->guard_gen;
  int64_t node = 0, i = 0;
  while (i < n) {
    int64_t c = child_of(t, node, path[i]);
    if (c < 0) break;
    ONode *cn = &t->nodes[c];
    int64_t k = lcp(t->toks + cn->tok_off, cn->len, path + i, n - i);
    if (k == 0) break;
    cn->guard_gen = gen;
    i += k;
    if (k < cn->len) break;
    node = c;
  }
  int64_t freed = ot_evict(t, shortfall);
  t->guard_gen++; /* _insert_guard = set() */
  return freed < shortfall ? OR_CAPACITY : OR_OK;
}

/* _split (kvcache.py:275-291): returns the new upper node id */
static int64_t split(OTree *t, int64_t id, int64_t k) {
  ONode *nd = &t->nodes[id];
  int64_t parent = nd->parent, off = nd->tok_off, len = nd->len;
  int64_t up = new_node(t, off, k, parent);
  nd = &t->nodes[id]; /* realloc safety */
  ONode *u = &t->nodes[up];
  uint32_t node_first = t->toks[off + k];
  nd->tok_off = off + k;
  nd->len = len - k;
  map_put(&t->children, ckey(parent, t->toks[off]), up);
  map_put(&t->children, ckey(up, node_first), id);
  u->nch = 1;
  nd->parent = up;
  u->ref = nd->ref;
  u->last = nd->last;
  u->hits = nd->hits;
  u->kind = nd->kind;
  u->seg = nd->seg;
  return up;
}

/* _split_at_offset (kvcache.py:293-304) */
static void split_at_offset(OTree *t, const uint32_t *path, int64_t offset) {
  int64_t node = 0, depth = 0;
  while (depth < offset) {
    int64_t c = child_of(t, node, path[depth]);
    int64_t end = depth + t->nodes[c].len;
    if (end > offset) {
      split(t, c, offset - depth);
      c = child_of(t, node, path[depth]);
      end = depth + t->nodes[c].len;
    }
    depth = end;
    node = c;
  }
}

/* insert_path (kvcache.py:190-241) */
int ot_insert(OTree *t, const uint32_t *path, int64_t n, int64_t na, const int64_t *a_off,
              const int8_t *a_kind, const int64_t *a_seg, const int64_t *a_snap, int64_t *leaf) {
  for (int64_t j = 1; j < na; j++)
    if (a_off[j] < a_off[j - 1]) return OR_INVALID; /* kvcache.py:199-201 */
  if (na > 0 && a_off[na - 1] > n) return OR_INVALID; /* kvcache.py:202-203 */
  for (int64_t j = 0; j < na; j++) /* AnchorMeta.__post_init__ (kvcache.py:51-53), checked up front */
    if (a_kind[j] == OR_REUSABLE && a_seg[j] == OR_SEG_NONE) return OR_INVALID;

  if (reserve(t, path, n) != OR_OK) return OR_CAPACITY;

  int64_t now = tick(t), node = 0, i = 0;
  while (i < n) {
    int64_t c = child_of(t, node, path[i]);
    if (c < 0) {
      int64_t off = push_tokens(t, path + i, n - i);
      c = new_node(t, off, n - i, node);
      map_put(&t->children, ckey(node, path[i]), c);
      t->nodes[node].nch++;
      t->resident += n - i;
      i = n;
      t->nodes[c].last = now;
      t->nodes[c].hits += 1;
      node = c;
      break;
    }
    ONode *cn = &t->nodes[c];
    int64_t k = lcp(t->toks + cn->tok_off, cn->len, path + i, n - i);
    if (k < cn->len) c = split(t, c, k);
    t->nodes[c].last = now;
    t->nodes[c].hits += 1;
    node = c;
    i += k;
  }
  for (int64_t j = 0; j < na; j++) /* anchor splits (kvcache.py:234-236) */
    if (0 < a_off[j] && a_off[j] < n) split_at_offset(t, path, a_off[j]);

  /* _collect_path_nodes + _label_regions (kvcache.py:306-340) */
  int64_t depth = 0, idx = 0, last_node = 0;
  node = 0;
  while (depth < n) {
    int64_t c = child_of(t, node, path[depth]);
    ONode *cn = &t->nodes[c];
    depth += cn->len;
    if (na > 0 && idx < na) {
      while (idx < na && a_off[idx] < depth) idx++;
      if (idx < na) {
        cn->kind = a_kind[idx];
        cn->seg = a_seg[idx];
        if (a_off[idx] == depth) {
          cn->has_anchor = 1;
          cn->akind = a_kind[idx];
          cn->aseg = a_seg[idx];
          cn->aoff = a_off[idx];
          cn->snap[0] = a_snap[3 * idx];
          cn->snap[1] = a_snap[3 * idx + 1];
          cn->snap[2] = a_snap[3 * idx + 2];
        }
      }
    }
    node = c;
    last_node = c;
  }
  /* _pin (kvcache.py:344-348) */
  for (int64_t x = last_node; x >= 0; x = t->nodes[x].parent) t->nodes[x].ref += 1;
  *leaf = last_node;
  return OR_OK;
}

/* release_path (kvcache.py:350-360) */
int ot_release(OTree *t, int64_t leaf) {
  if (leaf < 0 || leaf >= t->nnodes) return OR_INVALID;
  /* the reference walks node.parent; a detached node has parent None */
  for (int64_t x = leaf; x >= 0; x = t->nodes[x].parent)
    if (t->nodes[x].ref <= 0) return OR_RELEASE;
  for (int64_t x = leaf; x >= 0; x = t->nodes[x].parent) t->nodes[x].ref -= 1;
  return OR_OK;
}

/* ------------------------------------------------------------ protection */
typedef struct {
  double negp;
  int64_t seg, id;
} PEnt;
static int pent_cmp(const void *x, const void *y) {
  const PEnt *a = (const PEnt *)x, *b = (const PEnt *)y;
  if (a->negp != b->negp) return a->negp < b->negp ? -1 : 1;
  if (a->seg != b->seg) return a->seg < b->seg ? -1 : 1;
  return (a->id > b->id) - (a->id < b->id);
}

/* set_protection (kvcache.py:364-383) */
int64_t ot_set_protection(OTree *t, int64_t n, const int64_t *segs, const double *vals, int64_t *out) {
  map_free(&t->prio);
  map_init(&t->prio, 64);
  free(t->prio_vals);
  t->prio_vals = (double *)malloc(sizeof(double) * (n > 0 ? n : 1));
  t->nprio = 0;
  for (int64_t i = 0; i < n; i++) {
    int64_t ix = map_get(&t->prio, segkey(segs[i]));
    if (ix >= 0) {
      t->prio_vals[ix] = vals[i];
    } else {
      t->prio_vals[t->nprio] = vals[i];
      map_put(&t->prio, segkey(segs[i]), t->nprio++);
    }
  }
  int64_t cap = 16, m = 0;
  PEnt *v = (PEnt *)malloc(sizeof(PEnt) * cap);
  for (int64_t id = 1; id < t->nnodes; id++) {
    const ONode *nd = &t->nodes[id];
    if (!nd->attached || !nd->has_anchor || nd->akind != OR_REUSABLE) continue;
    if (m == cap) {
      cap *= 2;
      v = (PEnt *)realloc(v, sizeof(PEnt) * cap);
    }
    v[m].negp = -prio_of(t, nd->seg);
    v[m].seg = nd->seg == OR_SEG_NONE ? -1 : nd->seg;
    v[m].id = id;
    m++;
  }
  qsort(v, (size_t)m, sizeof(PEnt), pent_cmp);
  for (int64_t i = 0; i < t->nprot; i++) t->nodes[t->protected_ids[i]].prot = 0;
  int64_t f = t->protect_budget < m ? t->protect_budget : m;
  free(t->protected_ids);
  t->protected_ids = (int64_t *)malloc(sizeof(int64_t) * (f > 0 ? f : 1));
  t->nprot = f;
  for (int64_t i = 0; i < f; i++) {
    t->protected_ids[i] = v[i].id;
    t->nodes[v[i].id].prot = 1;
    if (out) out[i] = v[i].id;
  }
  free(v);
  return f;
}

/* note_active_segments (kvcache.py:385-393) */
void ot_note_active(OTree *t, int64_t n, const int64_t *segs) {
  map_free(&t->active);
  map_init(&t->active, 64);
  for (int64_t i = 0; i < n; i++) map_put(&t->active, segkey(segs[i]), 1);
  for (int64_t id = 1; id < t->nnodes; id++) {
    ONode *nd = &t->nodes[id];
    if (!nd->attached || !nd->has_anchor || nd->akind != OR_REUSABLE) continue;
    nd->snap[1] = (nd->aseg != OR_SEG_NONE && map_get(&t->active, segkey(nd->aseg)) >= 0) ? 1 : 0;
  }
}

/* ---------------------------------------------------------- inspection */
int64_t ot_resident(const OTree *t) { return t->resident; }
int64_t ot_clock(const OTree *t) { return t->clock; }
int64_t ot_num_nodes(const OTree *t) { return t->nnodes; }
int64_t ot_last_evicted(const OTree *t, int64_t *out, int64_t cap) {
  int64_t n = t->nlast < cap ? t->nlast : cap;
  if (out) memcpy(out, t->last_evicted, sizeof(int64_t) * n);
  return t->nlast;
}
int64_t ot_victim_log(const OTree *t, int64_t *out, int64_t cap) {
  int64_t n = t->nvlog < cap ? t->nvlog : cap;
  if (out) memcpy(out, t->vlog, sizeof(int64_t) * n);
  return t->nvlog;
}
void ot_node_info(const OTree *t, int64_t id, int64_t *out) {
  const ONode *n = &t->nodes[id];
  out[0] = n->parent;
  out[1] = n->len;
  out[2] = n->kind;
  out[3] = n->seg;
  out[4] = n->ref;
  out[5] = n->last;
  out[6] = n->hits;
  out[7] = n->prot;
  out[8] = n->has_anchor;
  out[9] = n->attached;
  out[10] = n->len > 0 ? (int64_t)t->toks[n->tok_off] : -1;
  out[11] = n->akind;
  out[12] = n->aseg;
  out[13] = n->aoff;
  out[14] = n->snap[0];
  out[15] = n->snap[1];
  out[16] = n->snap[2];
}
int64_t ot_edge_tokens(const OTree *t, int64_t id, uint32_t *out, int64_t cap) {
  const ONode *n = &t->nodes[id];
  int64_t m = n->len < cap ? n->len : cap;
  if (out) memcpy(out, t->toks + n->tok_off, sizeof(uint32_t) * m);
  return n->len;
}

/* Every attached node (root excluded) as 11 int64 in node-id order:
 * [id, parent, edge_len, kind, seg, ref, last, hits, prot, has_anchor, first_tok]
 * -- the fields debug_nodes() lists (kvcache.py:473-492) plus the first edge
 * token, for whole-tree parity at 1M nodes without per-node calls. */
int64_t ot_dump(const OTree *t, int64_t *out, int64_t cap) {
  int64_t k = 0;
  for (int64_t id = 1; id < t->nnodes; id++) {
    const ONode *n = &t->nodes[id];
    if (!n->attached) continue;
    if (out && k < cap) {
      int64_t *o = out + 11 * k;
      o[0] = id;
      o[1] = n->parent;
      o[2] = n->len;
      o[3] = n->kind;
      o[4] = n->seg;
      o[5] = n->ref;
      o[6] = n->last;
      o[7] = n->hits;
      o[8] = n->prot;
      o[9] = n->has_anchor;
      o[10] = n->len > 0 ? (int64_t)t->toks[n->tok_off] : -1;
    }
    k++;
  }
  return k;
}
