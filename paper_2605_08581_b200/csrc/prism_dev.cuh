// prism_dev.cuh -- device-side data layout and helpers for the B200 DART tree.
//
// Layout (all slot-indexed Structure-of-Arrays in HBM, slot 0 = root):
//   nid[S]    int64  node_id (creation order, kvcache.py:135-138); -1 = free slot
//   par[S]    int32  parent slot; -1 = root / detached
//   ftok[S]   uint32 first token of the edge (the child-table key)
//   eoff[S]   int64  edge start in the token arena; elen[S] int32 edge length
//   dend[S]   int32  token depth at the END of the edge (invariant under splits
//                    of this node's lower half; breaks eviction-order ties)
//   nch/ref/last/hits/kind/seg            the reference RadixNode fields
//   prot, hasanc/akind/aseg/aoff/snap     protection flag, AnchorMeta
//   hslot[S]  int32  index of this node's entry in the child table
//   kver[S]   uint32 key version (eviction-list entries carry it)
//   wmod/wchild/waitf/guard  epoch stamps (structural change, child added,
//                    waiting for cascade exposure, insert guard)
//   kw[S], eff[S]    eviction-list build scratch (packed key, subtree max)
// Child table: open-addressed, linear probing, 16-B entries {key, slot}
//   key = parent_slot << 32 | first_token  (kvcache.py node.children dict)
// Token arena: uint32, bump allocated; compacted on demand.
#pragma once
#include <cstdint>

namespace prism {

constexpr int32_t SEG_NONE = (int32_t)0x80000000;
constexpr uint64_t HEMPTY = ~0ull;
constexpr uint64_t HTOMB = ~0ull - 1ull;
constexpr int32_t ROOT = 0;
constexpr int32_t EFF_BLOCKED = -2;
constexpr int32_t EFF_DEAD = -1;

enum { K_SYSTEM = 0, K_REUSABLE = 1, K_PRIVATE = 2 };
enum { P_DART = 0, P_LRU = 1, P_LRU_ACTIVE = 2, P_LFU = 3 };

// commit-kernel stop codes
enum {
  ST_DONE = 0,
  ST_CAPACITY = 1,
  ST_NEED_BUILD = 10,
  ST_NEED_REBUILD = 11,
  ST_NEED_SLOTS = 12,
  ST_NEED_ARENA = 13,
  ST_NEED_HASH = 14,
  ST_FATAL = 99
};
enum { OP_MATCH = 0, OP_INSERT = 1, OP_EVICT = 2 };

// limits of the single-CTA commit kernel (documented in DESIGN.md)
constexpr int MAX_PATH = 16384;  // tokens per path staged in shared memory
constexpr int MAX_PNODES = 4096; // nodes on one root-to-leaf path
constexpr int MAX_ANCH = 2048;   // anchors per insert
constexpr int PM_MAX = 64;       // chain entries recorded by the parallel pre-match
constexpr int WP_MAXP = 66;      // pieces per path of the parallel commit: sys + 64 segments + suffix

struct HEnt {
  uint64_t key;
  uint32_t val;
  uint32_t pad;
};

struct Key3 {
  uint64_t w0, w1, w2;
};

struct VRec {  // victim record, captured at eviction time (last_evicted)
  int64_t id;
  int64_t eoff;
  uint32_t ftok;
  int32_t elen;
  int32_t seg;
  int8_t kind;
  int8_t pad[3];
};

struct Ctrl {
  int64_t resident, clock, next_id, arena_top;
  int64_t hlive, htomb;
  int64_t vlog_count, evict_calls, builds;
  int64_t fast_members, slow_members;
  int64_t chain_nodes, inserted_tokens;  // algorithmic-byte accounting
  int64_t need_hint;                     // tokens the stopped evict call still needs
  int64_t resume_freed, resume_vbeg;     // an evict call split by a list rebuild
  int32_t resume, L_partial;             // resume pending; L is a strict prefix of the order
  int64_t L_n, L_cur;
  int32_t hw, free_top;
  int32_t status, op_cursor;
  int32_t L_valid, H_n;
  uint32_t epoch, gstamp;
  uint32_t vctr;
  int32_t fatal;
  int32_t n_admitted;
  int32_t splits;  // do_split count: a root path recorded before a split may be stale (k_release_par)
};

struct OpRes {
  int64_t hit;
  int64_t leaf_id;
  int64_t freed;
  int64_t vbeg, vend;
  int32_t leaf_slot;
  int32_t status;
  int32_t evicted;
  int32_t nvis;
};

struct DT {
  // slot SoA
  int64_t *nid;
  int32_t *par;
  uint32_t *ftok;
  int64_t *eoff;
  int32_t *elen;
  int32_t *dend;
  int32_t *nch;
  int32_t *ref;
  int64_t *last;
  int32_t *hits;
  uint8_t *kind;
  int32_t *seg;
  uint8_t *prot;
  uint8_t *hasanc;
  uint8_t *akind;
  int32_t *aseg;
  int32_t *aoff;
  int32_t *snap;
  int32_t *hslot;
  uint32_t *kver;
  uint32_t *wmod;
  uint32_t *wchild;
  uint32_t *waitf;
  uint32_t *guard;
  uint64_t *wchm;  // parallel wave: (epoch << 32) | ~(first member whose pre-wave chain holds the node)
  Key3 *kw;
  int32_t *eff;
  int32_t *freelist;
  int32_t S;
  int32_t policy;
  // child table
  HEnt *ht;
  uint64_t hmask;
  // arena
  uint32_t *tok;
  int64_t acap;
  // priorities (P-hat, by segment id) and LRU_ACTIVE flags
  double *pri;
  int32_t npri;
  int32_t nact;
  uint8_t *act;
  // eviction list (sorted) and the small side heap
  Key3 *Lk;
  uint64_t *Lv;
  Key3 *Hk;
  uint64_t *Hv;
  int32_t Hcap;
  int32_t pad0;
  // victim log ring
  VRec *vlog;
  int64_t vcap;
  Ctrl *ctrl;
  int64_t capacity;
};

__host__ __device__ inline uint64_t mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

__host__ __device__ inline uint64_t ckey(int32_t parent, uint32_t tok) {
  return ((uint64_t)(uint32_t)parent << 32) | (uint64_t)tok;
}

// 192-bit shift-in: a = (a << n) | v for 1 <= n <= 64, v < 2^n
__device__ inline void shl_or(Key3 &a, int n, uint64_t v) {
  if (n >= 64) {
    a.w0 = a.w1;
    a.w1 = a.w2;
    a.w2 = v;
    return;
  }
  a.w0 = (a.w0 << n) | (a.w1 >> (64 - n));
  a.w1 = (a.w1 << n) | (a.w2 >> (64 - n));
  a.w2 = (a.w2 << n) | v;
}

// branch-free (lanes comparing different keys would otherwise diverge at every
// word and reconverge per compare)
__device__ __forceinline__ bool key_less(const Key3 &a, const Key3 &b) {
  const bool l0 = a.w0 < b.w0, e0 = a.w0 == b.w0;
  const bool l1 = a.w1 < b.w1, e1 = a.w1 == b.w1;
  const bool l2 = a.w2 < b.w2;
  return l0 | (e0 & (l1 | (e1 & l2)));
}

// order-preserving map of a double onto uint64 (-0.0 folded onto +0.0, so
// Python's 0.0 == -0.0 tie semantics are kept)
__device__ inline uint64_t ord_f64(double d) {
  if (d == 0.0) d = 0.0;
  uint64_t b = (uint64_t)__double_as_longlong(d);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__device__ inline double pri_of(const DT &T, int32_t s) {
  return (s != SEG_NONE && s >= 0 && s < T.npri) ? T.pri[s] : 0.0;
}

// evict_key (kvcache.py:397-414) packed right-aligned into 192 bits:
//   DART       (class:2, P-hat:64 ordered, last:40, id:40)
//   LRU        (last:40, id:40)
//   LFU        (hits:32, last:40, id:40)
//   LRU_ACTIVE (active:1, last:40, id:40)
// the packing from already-loaded fields (pseg: P-hat of the node's segment,
// act: its LRU_ACTIVE flag; each read only by its policy)
__device__ inline Key3 make_key_v(int32_t policy, int64_t last_, int64_t nid, int kind, bool prot, double pseg,
                                  int32_t hits, bool act) {
  Key3 k = {0, 0, 0};
  const uint64_t last = (uint64_t)last_ & ((1ull << 40) - 1);
  const uint64_t id = (uint64_t)nid & ((1ull << 40) - 1);
  switch (policy) {
    case P_DART: {
      uint32_t cls = (kind == K_PRIVATE) ? 0u : (prot ? 2u : 1u);
      double p = cls == 1u ? pseg : 0.0;
      shl_or(k, 2, cls);
      shl_or(k, 64, ord_f64(p));
      break;
    }
    case P_LFU:
      shl_or(k, 32, (uint64_t)(uint32_t)hits);
      break;
    case P_LRU_ACTIVE:
      shl_or(k, 1, act ? 1ull : 0ull);
      break;
    default:
      break;
  }
  shl_or(k, 40, last);
  shl_or(k, 40, id);
  return k;
}

__device__ inline bool act_of(const DT &T, int32_t sg) {
  return sg != SEG_NONE && sg >= 0 && sg < T.nact && T.act[sg];
}

__device__ inline Key3 make_key(const DT &T, int32_t s) {
  const int32_t p = T.policy;
  const int32_t sg = (p == P_DART || p == P_LRU_ACTIVE) ? T.seg[s] : SEG_NONE;
  const int kd = p == P_DART ? (int)T.kind[s] : 0;
  const bool pr = p == P_DART && kd != K_PRIVATE && T.prot[s];
  return make_key_v(p, T.last[s], T.nid[s], kd, pr, (p == P_DART && kd != K_PRIVATE && !pr) ? pri_of(T, sg) : 0.0,
                    p == P_LFU ? T.hits[s] : 0, p == P_LRU_ACTIVE && act_of(T, sg));
}

// bits used by the eviction sort key: policy key + 32-bit depth tiebreak
__host__ __device__ inline int evict_key_bits(int policy) {
  switch (policy) {
    case P_DART: return 2 + 64 + 40 + 40 + 32;
    case P_LFU: return 32 + 40 + 40 + 32;
    case P_LRU_ACTIVE: return 1 + 40 + 40 + 32;
    default: return 40 + 40 + 32;
  }
}

// composite eviction-order key of node s whose subtree maximum key is kmax:
// (kmax, deeper first)
__device__ inline Key3 composite(Key3 kmax, int32_t dend) {
  shl_or(kmax, 32, (uint64_t)(0xFFFFFFFFu - (uint32_t)dend));
  return kmax;
}

// Function attributes (dynamic shared-memory limits) belong to a device
// context: true the first time it is called for the current device with this
// per-call-site bitmask, so a second tree / scheduler on another GPU of the
// same process sets them again.
inline bool attr_once(uint64_t &mask) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return true;
  const uint64_t bit = 1ull << (dev & 63);
  if (mask & bit) return false;
  mask |= bit;
  return true;
}

}  // namespace prism
