// dart_kernels.cuh -- sm_100a kernels of the device DART tree.
//
//   k_prematch   one warp per wave member: read-only exact-prefix match of the
//                member's path against the pre-wave tree (kvcache.py:146-171),
//                recording the node chain so the ordered commit can skip the
//                walk when nothing on the chain changed earlier in the wave.
//   k_commit     one warp, the ordered commit of match/insert/evict operations
//                with the reference's exact sequential semantics
//                (kvcache.py:190-348, 425-460; engine.py:200-213).
//   k_build_keys / k_propagate / k_gather
//                the data-parallel eviction-order build: evict_key of every
//                node, subtree-maximum propagation, and the composite sort key
//                (see DESIGN.md "Exact eviction order").
//   protection / note-active / release / rehash / compaction kernels.
#pragma once
#include "pdl.cuh"
#include "prism_dev.cuh"

namespace prism {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// ------------------------------------------------------------ child table

// warp-collective lookup of node.children[tok] (kvcache.py:158)
__device__ __forceinline__ int32_t ht_lookup(const DT &T, int32_t parent, uint32_t tok) {
  const uint64_t key = ckey(parent, tok);
  uint64_t h = mix64(key) & T.hmask;
  const int lane = lane_id();
  for (;;) {
    const uint64_t idx = (h + (uint64_t)lane) & T.hmask;
    const HEnt e = T.ht[idx];
    const unsigned meq = __ballot_sync(FULL, e.key == key);
    if (meq) return __shfl_sync(FULL, (int32_t)e.val, __ffs(meq) - 1);
    if (__ballot_sync(FULL, e.key == HEMPTY)) return -1;
    h += 32;
  }
}

// warp-collective: first EMPTY or TOMB slot on the probe sequence of key
__device__ __forceinline__ uint64_t ht_probe_free(const DT &T, uint64_t key, bool *was_tomb) {
  uint64_t h = mix64(key) & T.hmask;
  const int lane = lane_id();
  for (;;) {
    const uint64_t idx = (h + (uint64_t)lane) & T.hmask;
    const uint64_t k = T.ht[idx].key;
    const unsigned m = __ballot_sync(FULL, k == HEMPTY || k == HTOMB);
    if (m) {
      const int src = __ffs(m) - 1;
      *was_tomb = __shfl_sync(FULL, (int)(k == HTOMB), src) != 0;
      return __shfl_sync(FULL, (unsigned long long)idx, src);
    }
    h += 32;
  }
}

// warp-collective common-prefix length of a[0..lim) and b[0..lim) (kvcache.py:109-114)
// (4 x 32 tokens per step: the loads of a step are independent, so long edges
// -- a 1024-token system prompt -- cost a quarter of the round trips)
__device__ __forceinline__ int64_t warp_lcp(const uint32_t *__restrict__ a, const uint32_t *b,
                                            int64_t lim) {
  const int lane = lane_id();
  for (int64_t j = 0; j < lim; j += 128) {
    bool ne[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const int64_t i = j + 32 * u + lane;
      ne[u] = i < lim && a[i] != b[i];
    }
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const unsigned m = __ballot_sync(FULL, ne[u]);
      if (m) return j + 32 * u + __ffs(m) - 1;
    }
  }
  return lim;
}

struct WalkOut {
  int64_t hit;
  int32_t d;
  int32_t klast;
  bool partial;
  bool overflow;
};

// warp-collective read-only walk (kvcache.py:146-186): chain[d] receives the
// visited slots (lane 0 writes), the last one possibly partially matched.
__device__ inline WalkOut warp_walk(const DT &T, const uint32_t *p, int64_t n, int32_t *chain,
                                    int32_t maxch) {
  int32_t node = ROOT, d = 0, kl = 0;
  int64_t i = 0;
  bool partial = false, of = false;
  while (i < n) {
    const int32_t c = ht_lookup(T, node, p[i]);
    if (c < 0) break;
    const int64_t eo = T.eoff[c];
    const int32_t el = T.elen[c];
    const int64_t lim = (int64_t)el < n - i ? (int64_t)el : n - i;
    const int64_t k = warp_lcp(T.tok + eo, p + i, lim);
    if (k == 0) break;
    if (d < maxch) {
      if (lane_id() == 0) chain[d] = c;
    } else {
      of = true;
    }
    d++;
    i += k;
    kl = (int32_t)k;
    if (k < el) {
      partial = true;
      break;
    }
    node = c;
  }
  __syncwarp();
  return {i, d, kl, partial, of};
}

// ------------------------------------------------------------ pre-match

__global__ void k_prematch(DT T, int64_t B, const int64_t *__restrict__ poff,
                           const uint32_t *__restrict__ tok, int32_t *__restrict__ pm_meta,
                           int32_t *__restrict__ pm_chain, const int32_t *abort = nullptr) {
  pdl_wait();
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= B || (abort && *abort)) return;
  const int64_t b = poff[w], n = poff[w + 1] - b;
  const WalkOut r = warp_walk(T, tok + b, n, pm_chain + w * PM_MAX, PM_MAX);
  if (lane_id() == 0) {
    pm_meta[4 * w + 0] = (int32_t)r.hit;
    pm_meta[4 * w + 1] = r.d;
    pm_meta[4 * w + 2] = r.klast;
    pm_meta[4 * w + 3] = (r.partial ? 1 : 0) | (r.overflow ? 2 : 0);
  }
  pdl_trace_end();
}

// ------------------------------------------------------------ commit

struct CommitArgs {
  int32_t mode;  // 0 = one explicit op, 1 = wave (op o: member o>>1, MATCH then INSERT)
  int32_t reset;
  int32_t op_type;
  int32_t nops;
  int64_t op_k;
  int64_t op_n;
  int64_t op_na;
  const int64_t *poff;
  const uint32_t *tok;
  const int64_t *aoffs;
  const int32_t *a_off;
  const int8_t *a_kind;
  const int32_t *a_seg;
  const int32_t *a_snap;
  const int32_t *pm_meta;
  const int32_t *pm_chain;
  OpRes *res;
  int64_t *hits;
  int32_t *leaf_slots;
  int64_t *leaf_ids;
  int32_t *vis_slots;
  int64_t *vis_ids;
};

constexpr size_t COMMIT_SMEM = sizeof(uint32_t) * MAX_PATH + sizeof(int32_t) * 2 * MAX_PNODES +
                               sizeof(int32_t) * 5 * MAX_ANCH + MAX_ANCH;

// heap of (Key3, value) in global memory, operated by lane 0 only
__device__ inline void heap_push(const DT &T, int32_t n, Key3 k, uint64_t v) {
  int32_t i = n;
  while (i > 0) {
    const int32_t p = (i - 1) >> 1;
    const Key3 kp = T.Hk[p];
    if (!key_less(k, kp)) break;
    T.Hk[i] = kp;
    T.Hv[i] = T.Hv[p];
    i = p;
  }
  T.Hk[i] = k;
  T.Hv[i] = v;
}

__device__ inline void heap_pop(const DT &T, int32_t n) {  // n = size before pop
  const int32_t m = n - 1;
  if (m <= 0) return;
  const Key3 k = T.Hk[m];
  const uint64_t v = T.Hv[m];
  int32_t i = 0;
  for (;;) {
    const int32_t l = 2 * i + 1, r = l + 1;
    if (l >= m) break;
    int32_t c = l;
    if (r < m && key_less(T.Hk[r], T.Hk[l])) c = r;
    if (!key_less(T.Hk[c], k)) break;
    T.Hk[i] = T.Hk[c];
    T.Hv[i] = T.Hv[c];
    i = c;
  }
  T.Hk[i] = k;
  T.Hv[i] = v;
}

// warp-uniform slot allocation; assigns the next node_id (kvcache.py:135-138)
__device__ inline int32_t alloc_slot(const DT &T, Ctrl &C) {
  int32_t s;
  if (C.free_top > 0) {
    C.free_top--;
    s = T.freelist[C.free_top];
  } else {
    s = C.hw++;
  }
  C.vctr++;
  const int64_t id = C.next_id++;
  if (lane_id() == 0) {
    T.nid[s] = id;
    T.kver[s] = C.vctr;
    T.wmod[s] = C.epoch;
    T.wchild[s] = 0;
    T.waitf[s] = 0;
    T.guard[s] = 0;
    T.prot[s] = 0;
    T.hasanc[s] = 0;
  }
  return s;
}

// _split (kvcache.py:275-291): new upper node over the first k edge tokens of X
__device__ inline int32_t do_split(const DT &T, Ctrl &C, int32_t X, int32_t k) {
  const int32_t U = alloc_slot(T, C);
  C.splits++;  // (every lane: the warp's copies of the control block stay identical)
  const int32_t p = T.par[X];
  const int64_t eo = T.eoff[X];
  const int32_t el = T.elen[X];
  const uint32_t fx = T.ftok[X];
  const int32_t hs = T.hslot[X];
  const uint32_t lowfirst = T.tok[eo + k];
  bool tomb = false;
  const uint64_t hidx = ht_probe_free(T, ckey(U, lowfirst), &tomb);
  if (lane_id() == 0) {
    T.par[U] = p;
    T.ftok[U] = fx;
    T.eoff[U] = eo;
    T.elen[U] = k;
    T.dend[U] = T.dend[X] - (el - k);
    T.nch[U] = 1;
    T.ref[U] = T.ref[X];
    T.last[U] = T.last[X];
    T.hits[U] = T.hits[X];
    T.kind[U] = T.kind[X];
    T.seg[U] = T.seg[X];
    T.ht[hs].val = (uint32_t)U;
    T.hslot[U] = hs;
    HEnt e;
    e.key = ckey(U, lowfirst);
    e.val = (uint32_t)X;
    e.pad = 0;
    T.ht[hidx] = e;
    T.hslot[X] = (int32_t)hidx;
    T.eoff[X] = eo + k;
    T.elen[X] = el - k;
    T.ftok[X] = lowfirst;
    T.par[X] = U;
    T.wmod[X] = C.epoch;
  }
  C.hlive++;
  if (tomb) C.htomb--;
  __syncwarp();
  return U;
}

// exact eviction from the sorted list L merged with the side heap H
// (semantics of evict, kvcache.py:425-460)
//
// Entries of L are consumed in batches of 32: every lane prefetches one entry
// together with its node's and its parent's state (3 dependent round trips
// per batch instead of per victim); the warp then walks the batch in order
// from registers, patching the prefetched copies whenever an eviction
// changes them (child counts, duplicates, cascade-waiting flags).
struct Cand {
  Key3 k;
  int64_t id, eoff;
  int32_t s, p, nch, pnch, el, hs, seg;
  uint32_t ftok;
  int32_t kind;
  bool ok, pw;
};

__device__ inline Cand load_cand(const DT &T, const Ctrl &C, Key3 k, uint64_t v) {
  Cand c;
  c.k = k;
  c.s = (int32_t)(v & 0xffffffffu);
  const uint32_t ver = (uint32_t)(v >> 32);
  c.id = T.nid[c.s];
  const uint32_t kv = T.kver[c.s];
  c.p = T.par[c.s];
  const int32_t rf = T.ref[c.s];
  const uint32_t gd = T.guard[c.s];
  c.kind = T.kind[c.s];
  c.nch = T.nch[c.s];
  c.el = T.elen[c.s];
  c.hs = T.hslot[c.s];
  c.seg = T.seg[c.s];
  c.ftok = T.ftok[c.s];
  c.eoff = T.eoff[c.s];
  c.ok = kv == ver && c.id >= 0 && c.p >= 0 && rf == 0 && gd != C.gstamp &&
         !(T.policy == P_DART && c.kind == K_SYSTEM);
  c.pnch = 0;
  c.pw = false;
  if (c.ok) {
    c.pnch = T.nch[c.p];
    c.pw = T.waitf[c.p] == C.epoch;
  }
  return c;
}

__device__ inline Cand shfl_cand(const Cand &c, int src) {
  Cand r;
  r.k.w0 = __shfl_sync(FULL, c.k.w0, src);
  r.k.w1 = __shfl_sync(FULL, c.k.w1, src);
  r.k.w2 = __shfl_sync(FULL, c.k.w2, src);
  r.id = __shfl_sync(FULL, c.id, src);
  r.eoff = __shfl_sync(FULL, c.eoff, src);
  r.s = __shfl_sync(FULL, c.s, src);
  r.p = __shfl_sync(FULL, c.p, src);
  r.nch = __shfl_sync(FULL, c.nch, src);
  r.pnch = __shfl_sync(FULL, c.pnch, src);
  r.el = __shfl_sync(FULL, c.el, src);
  r.hs = __shfl_sync(FULL, c.hs, src);
  r.seg = __shfl_sync(FULL, c.seg, src);
  r.ftok = __shfl_sync(FULL, c.ftok, src);
  r.kind = __shfl_sync(FULL, c.kind, src);
  r.ok = __shfl_sync(FULL, (int)c.ok, src) != 0;
  r.pw = __shfl_sync(FULL, (int)c.pw, src) != 0;
  return r;
}

__device__ inline int64_t evict_loop(const DT &T, Ctrl &C, int64_t need) {
  int64_t freed = 0;
  const int lane = lane_id();
  int nb = 0, i = 0;
  int64_t base = 0;
  Cand mine;  // this lane's prefetched batch entry
  mine.ok = false;
  mine.s = mine.p = -1;
  mine.pw = false;
  while (freed < need) {
    if (i >= nb && C.L_cur < C.L_n) {  // prefetch the next batch of the sorted list
      base = C.L_cur;
      nb = (int)((C.L_n - base) < 32 ? (C.L_n - base) : 32);
      i = 0;
      mine.ok = false;
      mine.s = mine.p = -1;
      mine.pw = false;
      if (lane < nb) mine = load_cand(T, C, T.Lk[base + lane], T.Lv[base + lane]);
      __syncwarp();
    }
    const bool hasL = i < nb;
    const bool hasH = C.H_n > 0;
    if (!hasL && !hasH) break;
    Cand c;
    bool useH = false;
    if (hasL) c = shfl_cand(mine, i);
    if (hasH) {
      const Key3 kh = T.Hk[0];
      useH = !hasL || key_less(kh, c.k);
      if (useH) {
        const uint64_t hv = T.Hv[0];
        __syncwarp();
        if (lane == 0) heap_pop(T, C.H_n);
        C.H_n--;
        __syncwarp();
        c = load_cand(T, C, kh, hv);
      }
    }
    if (!useH) {
      i++;
      C.L_cur = base + i;
    }
    if (!c.ok) continue;
    const Key3 k = c.k;
    const int32_t s = c.s, p = c.p;
    if (c.nch > 0) {  // not a leaf yet: wait for its last child (cascade)
      if (lane == 0) T.waitf[s] = C.epoch;
      if (mine.p == s) mine.pw = true;
      __syncwarp();
      continue;
    }
    // detach s (kvcache.py:452-459)
    const int32_t nchp = c.pnch - 1;
    C.vctr++;
    if (lane == 0) {
      VRec rec;
      rec.id = c.id;
      rec.eoff = c.eoff;
      rec.ftok = c.ftok;
      rec.elen = c.el;
      rec.seg = c.seg;
      rec.kind = (int8_t)c.kind;
      rec.pad[0] = rec.pad[1] = rec.pad[2] = 0;
      T.nch[p] = nchp;
      T.ht[c.hs].key = HTOMB;
      T.vlog[C.vlog_count % T.vcap] = rec;
      T.nid[s] = -1;
      T.par[s] = -1;
      T.kver[s] = C.vctr;
      T.wmod[s] = C.epoch;
      T.freelist[C.free_top] = s;
    }
    // patch the prefetched batch
    if (mine.s == s) mine.ok = false;
    if (mine.s == p) mine.nch -= 1;
    if (mine.p == p) mine.pnch -= 1;
    C.free_top++;
    C.vlog_count++;
    C.hlive--;
    C.htomb++;
    C.resident -= c.el;
    freed += c.el;
    const bool pwait = c.pw;
    __syncwarp();
    if (nchp == 0 && pwait && C.H_n >= T.Hcap) C.fatal = 4;
    if (nchp == 0 && pwait && C.H_n < T.Hcap) {
      // exposed parent (kvcache.py:458-459): it is next unless its own key is larger
      Key3 kp = composite(make_key(T, p), T.dend[p]);
      if (key_less(kp, k)) kp = k;
      const uint64_t pv = ((uint64_t)T.kver[p] << 32) | (uint32_t)p;
      __syncwarp();
      if (lane == 0) heap_push(T, C.H_n, kp, pv);
      C.H_n++;
      __syncwarp();
    }
  }
  return freed;
}

__device__ inline int32_t lower_bound_i32(const int32_t *a, int32_t n, int32_t x) {
  int32_t lo = 0, hi = n;
  while (lo < hi) {
    const int32_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(32) k_commit(DT T, CommitArgs A) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t *sp = reinterpret_cast<uint32_t *>(smem);
  int32_t *Ps = reinterpret_cast<int32_t *>(sp + MAX_PATH);
  int32_t *Pe = Ps + MAX_PNODES;
  int32_t *sa_off = Pe + MAX_PNODES;
  int32_t *sa_seg = sa_off + MAX_ANCH;
  int32_t *sa_snap = sa_seg + MAX_ANCH;
  int8_t *sa_kind = reinterpret_cast<int8_t *>(sa_snap + 3 * MAX_ANCH);
  const int lane = lane_id();

  Ctrl C = *T.ctrl;
  if (A.reset) {
    C.op_cursor = 0;
    C.epoch++;
    C.L_valid = 0;
    C.L_n = 0;
    C.L_cur = 0;
    C.H_n = 0;
    C.n_admitted = 0;
    C.resume = 0;
    C.resume_freed = 0;
  }
  C.status = ST_DONE;
  int32_t chain_member = -1;  // member whose match chain sits in Ps
  int64_t c_hit = 0;
  int32_t c_d = 0, c_kl = 0;
  bool c_partial = false;

  int32_t o = C.op_cursor;
  for (; o < A.nops; o++) {
    int32_t type, member;
    int64_t pb, n, ab, na;
    if (A.mode == 1) {
      member = o >> 1;
      type = (o & 1) ? OP_INSERT : OP_MATCH;
      pb = A.poff[member];
      n = A.poff[member + 1] - pb;
      ab = A.aoffs[member];
      na = A.aoffs[member + 1] - ab;
    } else {
      member = 0;
      type = A.op_type;
      pb = 0;
      n = A.op_n;
      ab = 0;
      na = A.op_na;
    }
    if (na > MAX_ANCH) {
      C.fatal = 1;
      C.status = ST_FATAL;
      break;
    }
    if (type == OP_INSERT) {
      const int64_t need_nodes = 2 + na;
      if ((int64_t)C.free_top + (int64_t)(T.S - C.hw) < need_nodes) {
        C.status = ST_NEED_SLOTS;
        break;
      }
      if (C.arena_top + n > T.acap) {
        C.status = ST_NEED_ARENA;
        C.need_hint = n;  // (the host compacts / grows the arena for at least this)
        break;
      }
      if ((C.hlive + C.htomb + need_nodes) * 2 > (int64_t)(T.hmask + 1)) {
        C.status = ST_NEED_HASH;
        break;
      }
      if (C.L_valid && C.H_n + 2 > T.Hcap) {
        C.status = ST_NEED_REBUILD;
        break;
      }
    }
    OpRes r;
    r.hit = 0;
    r.leaf_id = -1;
    r.freed = 0;
    r.vbeg = C.vlog_count;
    r.vend = C.vlog_count;
    r.leaf_slot = -1;
    r.status = 0;
    r.evicted = 0;
    r.nvis = 0;

    if (type == OP_EVICT) {  // evict(k) (kvcache.py:425-460)
      r.evicted = 1;
      if (A.op_k > 0) {
        const int64_t need = A.op_k - C.resume_freed;
        if (!C.L_valid) {
          C.need_hint = need;
          C.status = ST_NEED_BUILD;
          break;
        }
        C.gstamp++;
        if (C.resume) r.vbeg = C.resume_vbeg;
        const int64_t got = evict_loop(T, C, need);
        if (got < need && C.L_partial) {  // list prefix exhausted: rebuild, continue
          C.resume = 1;
          C.resume_freed += got;
          C.resume_vbeg = r.vbeg;
          C.need_hint = need - got;
          C.status = ST_NEED_REBUILD;
          break;
        }
        r.freed = got + C.resume_freed;
        C.resume = 0;
        C.resume_freed = 0;
      }
      C.evict_calls++;
      r.vend = C.vlog_count;
      if (lane == 0 && A.res) A.res[o] = r;
      continue;
    }

    // stage the path in shared memory; longer paths are read from HBM in place
    const uint32_t *pth = n <= MAX_PATH ? sp : A.tok + pb;
    if (n <= MAX_PATH)
      for (int64_t i = lane; i < n; i += 32) sp[i] = A.tok[pb + i];
    if (type == OP_INSERT) {
      for (int64_t i = lane; i < na; i += 32) {
        sa_off[i] = A.a_off[ab + i];
        sa_kind[i] = A.a_kind[ab + i];
        sa_seg[i] = A.a_seg[ab + i];
        sa_snap[3 * i] = A.a_snap[3 * (ab + i)];
        sa_snap[3 * i + 1] = A.a_snap[3 * (ab + i) + 1];
        sa_snap[3 * i + 2] = A.a_snap[3 * (ab + i) + 2];
      }
    }
    __syncwarp();

    // ---- obtain the match chain
    if (!(type == OP_INSERT && chain_member == member && A.mode == 1)) {
      bool valid = false;
      if (A.mode == 1 && A.pm_meta != nullptr) {
        const int32_t hit_pre = A.pm_meta[4 * member + 0];
        const int32_t d = A.pm_meta[4 * member + 1];
        const int32_t kl = A.pm_meta[4 * member + 2];
        const int32_t fl = A.pm_meta[4 * member + 3];
        if (!(fl & 2)) {
          bool bad = false;
          for (int32_t i = lane; i < d; i += 32) {
            const int32_t c = A.pm_chain[(int64_t)member * PM_MAX + i];
            Ps[i] = c;
            bad |= T.wmod[c] == C.epoch;
          }
          // the failed child lookup at the chain end must still fail: an earlier
          // member may have added a child with exactly this first token
          if (!(fl & 1) && hit_pre < n) {
            const int32_t tnode = d > 0 ? A.pm_chain[(int64_t)member * PM_MAX + d - 1] : ROOT;
            if (ht_lookup(T, tnode, pth[hit_pre]) >= 0) bad = true;
          }
          valid = !__any_sync(FULL, bad);
          __syncwarp();
          if (valid) {
            c_hit = hit_pre;
            c_d = d;
            c_kl = kl;
            c_partial = (fl & 1) != 0;
          }
        }
      }
      if (valid) {
        C.fast_members += (type == OP_MATCH);
      } else {
        const WalkOut w = warp_walk(T, pth, n, Ps, MAX_PNODES);
        if (w.overflow) {
          C.fatal = 2;
          C.status = ST_FATAL;
          break;
        }
        c_hit = w.hit;
        c_d = w.d;
        c_kl = w.klast;
        c_partial = w.partial;
        C.slow_members += (type == OP_MATCH && A.mode == 1);
      }
      chain_member = member;
    }

    if (type == OP_MATCH) {  // match_prefix (kvcache.py:146-171)
      C.clock++;
      const int64_t now = C.clock;
      for (int32_t i = lane; i < c_d; i += 32) {
        const int32_t c = Ps[i];
        T.last[c] = now;
        T.hits[c] += 1;
        if (A.vis_slots) {
          A.vis_slots[i] = c;
          A.vis_ids[i] = T.nid[c];
        }
      }
      __syncwarp();
      r.hit = c_hit;
      r.nvis = c_d;
      if (lane == 0) {
        if (A.res) A.res[o] = r;
        if (A.hits) A.hits[member] = c_hit;
      }
      continue;
    }

    // ---- insert_path (kvcache.py:190-241)
    const int64_t hit = c_hit;
    const int64_t shortfall = C.resident + (n - hit) - T.capacity;  // _reserve (243-273)
    if (shortfall > 0) {
      if (!C.L_valid) {
        C.need_hint = shortfall;
        C.status = ST_NEED_BUILD;
        break;
      }
      C.gstamp++;
      for (int32_t i = lane; i < c_d; i += 32) T.guard[Ps[i]] = C.gstamp;
      __syncwarp();
      r.evicted = 1;
      if (C.resume) r.vbeg = C.resume_vbeg;
      const int64_t got = evict_loop(T, C, shortfall);
      if (got < shortfall && C.L_partial) {
        // the selected prefix of the eviction order ran out: rebuild the list
        // from the current tree and continue this same evict call
        C.resume = 1;
        C.resume_freed += got;
        C.resume_vbeg = r.vbeg;
        C.need_hint = shortfall - got;
        C.status = ST_NEED_REBUILD;
        break;
      }
      r.freed = got + C.resume_freed;
      C.resume = 0;
      C.resume_freed = 0;
      C.evict_calls++;
      r.vend = C.vlog_count;
      if (got < shortfall) {
        r.status = ST_CAPACITY;
        if (lane == 0 && A.res) A.res[o] = r;
        C.status = ST_CAPACITY;
        o++;  // this op is finished (raised CapacityError)
        break;
      }
    }
    C.chain_nodes += c_d;
    C.inserted_tokens += n;
    C.clock++;
    const int64_t now = C.clock;
    int32_t np = c_d;
    const int32_t nfull = c_partial ? c_d - 1 : c_d;
    for (int32_t i = lane; i < nfull; i += 32) {
      const int32_t c = Ps[i];
      T.last[c] = now;
      T.hits[c] += 1;
      Pe[i] = T.dend[c];
    }
    __syncwarp();
    if (c_partial) {
      const int32_t X = Ps[c_d - 1];
      const int32_t U = do_split(T, C, X, c_kl);
      const int32_t hu = T.hits[U];
      C.vctr++;
      const bool pushX = C.L_valid && T.ref[X] == 0 &&
                         !(T.policy == P_DART && T.kind[X] == K_SYSTEM) && C.H_n < T.Hcap;
      Key3 kx = composite(make_key(T, X), T.dend[X]);
      __syncwarp();
      if (lane == 0) {
        T.last[U] = now;
        T.hits[U] = hu + 1;
        Ps[c_d - 1] = U;
        Pe[c_d - 1] = (int32_t)hit;
        T.kver[X] = C.vctr;  // X's key changed (match touched it): re-key
        if (pushX) heap_push(T, C.H_n, kx, ((uint64_t)C.vctr << 32) | (uint32_t)X);
      }
      if (pushX) C.H_n++;
      __syncwarp();
    }
    if (hit < n) {  // tail node with the rest of the path (kvcache.py:213-222)
      const int32_t parent = c_d > 0 ? Ps[c_d - 1] : ROOT;
      const int32_t Tn = alloc_slot(T, C);
      const int64_t len = n - hit;
      const int64_t base = C.arena_top;
      for (int64_t i = lane; i < len; i += 32) T.tok[base + i] = pth[hit + i];
      bool tomb = false;
      const uint64_t hidx = ht_probe_free(T, ckey(parent, pth[hit]), &tomb);
      const int32_t pn = T.nch[parent];
      __syncwarp();
      if (lane == 0) {
        T.par[Tn] = parent;
        T.ftok[Tn] = pth[hit];
        T.eoff[Tn] = base;
        T.elen[Tn] = (int32_t)len;
        T.dend[Tn] = (int32_t)n;
        T.nch[Tn] = 0;
        T.ref[Tn] = 0;
        T.last[Tn] = now;
        T.hits[Tn] = 1;
        T.kind[Tn] = K_PRIVATE;
        T.seg[Tn] = SEG_NONE;
        HEnt e;
        e.key = ckey(parent, pth[hit]);
        e.val = (uint32_t)Tn;
        e.pad = 0;
        T.ht[hidx] = e;
        T.hslot[Tn] = (int32_t)hidx;
        T.nch[parent] = pn + 1;
        T.wchild[parent] = C.epoch;
        Ps[np] = Tn;
        Pe[np] = (int32_t)n;
      }
      np++;
      C.hlive++;
      if (tomb) C.htomb--;
      C.arena_top += len;
      C.resident += len;
      __syncwarp();
    }
    // anchor splits, ascending offsets (kvcache.py:233-236, 293-304)
    {
      int32_t q = 0;
      for (int32_t a = 0; a < (int32_t)na; a++) {
        const int32_t off = sa_off[a];
        if (!(0 < off && off < n)) continue;
        while (q < np && Pe[q] < off) q++;
        if (q >= np || Pe[q] == off) continue;
        const int32_t st = q == 0 ? 0 : Pe[q - 1];
        const int32_t V = do_split(T, C, Ps[q], off - st);
        if (lane == 0) {
          for (int32_t j = np; j > q; j--) {
            Ps[j] = Ps[j - 1];
            Pe[j] = Pe[j - 1];
          }
          Ps[q] = V;
          Pe[q] = off;
        }
        np++;
        q++;
        __syncwarp();
        if (np >= MAX_PNODES) break;
      }
    }
    if (np >= MAX_PNODES) {
      C.fatal = 3;
      C.status = ST_FATAL;
      break;
    }
    // _label_regions (kvcache.py:317-340) and _pin (344-348)
    for (int32_t q = lane; q < np; q += 32) {
      const int32_t s = Ps[q];
      if (na > 0) {
        const int32_t end = Pe[q];
        const int32_t idx = lower_bound_i32(sa_off, (int32_t)na, end);
        if (idx < na) {
          T.kind[s] = (uint8_t)sa_kind[idx];
          T.seg[s] = sa_seg[idx];
          if (sa_off[idx] == end) {
            T.hasanc[s] = 1;
            T.akind[s] = (uint8_t)sa_kind[idx];
            T.aseg[s] = sa_seg[idx];
            T.aoff[s] = end;
            T.snap[3 * (int64_t)s] = sa_snap[3 * idx];
            T.snap[3 * (int64_t)s + 1] = sa_snap[3 * idx + 1];
            T.snap[3 * (int64_t)s + 2] = sa_snap[3 * idx + 2];
          }
        }
      }
      T.ref[s] += 1;
    }
    if (lane == 0) T.ref[ROOT] += 1;
    __syncwarp();
    const int32_t leaf = np > 0 ? Ps[np - 1] : ROOT;
    r.leaf_slot = leaf;
    r.leaf_id = T.nid[leaf];
    r.hit = hit;
    if (lane == 0) {
      if (A.res) A.res[o] = r;
      if (A.leaf_slots) {
        A.leaf_slots[member] = leaf;
        A.leaf_ids[member] = r.leaf_id;
      }
    }
    if (A.mode == 1) C.n_admitted = member + 1;
    chain_member = -1;
    __syncwarp();
  }
  C.op_cursor = o;
  __syncwarp();
  if (lane == 0) *T.ctrl = C;
}

// ------------------------------------------------------------ eviction-order build

// (hw < 0: read the high-water mark from the control block -- no host sync)
__global__ void k_build_keys(DT T, int32_t hw, const int64_t *dW = nullptr) {
  pdl_wait();
  if (dW && *dW < 0) return;  // device-side control: no eviction this wave
  if (hw < 0) hw = T.ctrl->hw;
  const int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= hw) return;
  if (s == ROOT || T.nid[s] < 0 || T.par[s] < 0) {
    T.eff[s] = EFF_DEAD;
    return;
  }
  const bool blocked = T.ref[s] > 0 || (T.policy == P_DART && T.kind[s] == K_SYSTEM);
  T.kw[s] = make_key(T, s);
  T.eff[s] = blocked ? EFF_BLOCKED : s;
}

// eff[v] = slot of the maximum key in v's subtree (EFF_BLOCKED if any node of
// the subtree can never be evicted): each node carries its own value upward
// until an ancestor already holds something at least as large.
// Most walks stop after a hop or two, but a freshly touched path is one where
// every node beats its parent (same access time, larger id), so some walks
// climb ~40 levels.  One thread per node kept a whole warp -- and its block's
// SM slot -- waiting on its longest walk, wave after wave of blocks; here a
// persistent grid of warps owns contiguous slot ranges and every lane whose
// walk ends takes the next slot of its warp's range at once, so the lanes stay
// busy and the kernel lasts about one longest walk.  (Ranges claimed from a
// counter in 128-slot chunks balanced no better and cost more.)
#ifndef PRISM_PROP_TPB
#define PRISM_PROP_TPB 256
#endif
constexpr int PROP_TPB = PRISM_PROP_TPB;
__global__ void __launch_bounds__(PROP_TPB) k_propagate(DT T, int32_t hw, const int64_t *dW = nullptr,
                                                        unsigned long long *clr = nullptr, int64_t nclr = 0) {
  pdl_wait();
  // (optionally) clear the selection state for the launches that follow (in
  // place of a memset node in the wave's graph)
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nclr; i += (int64_t)gridDim.x * blockDim.x)
    clr[i] = 0ull;
  if (dW && *dW < 0) return;
  if (hw < 0) hw = T.ctrl->hw;
  const int lane = threadIdx.x & 31;
  const int64_t nwarp = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t chunk = ((int64_t)hw + nwarp - 1) / nwarp;
  // the warp's range [beg, end) in DESCENDING slot order: nodes created together
  // take ascending slots top-down, so children come first and their raises let
  // the parents skip their own walks
  const int64_t beg = w * chunk, end = min((int64_t)hw, beg + chunk);
  int64_t next = end - 1;  // (warp-uniform) the warp's next unclaimed slot
  bool act = false, blocked = false;
  int32_t val = 0, p = 0;
  Key3 kv{};
  for (;;) {
    const unsigned idle = __ballot_sync(FULL, !act);
    if (idle && next >= beg) {  // idle lanes take the next slots of the range
      if (!act) {
        const int64_t s = next - __popc(idle & ((1u << lane) - 1u));
        if (s >= beg) {
          // k_build_keys left eff[s] = s (evictable), EFF_BLOCKED or EFF_DEAD (root / free); a
          // descendant's walk may have raised it since (the node is evictable then)
          const int32_t e0 = __ldcg(&T.eff[s]);
          // raised already by a descendant (e0 >= 0, != s): that walk carries a larger key past s,
          // so s's own walk could only raise ancestors the descendant raises again -- skip it
          if (e0 != EFF_DEAD && (e0 < 0 || e0 == (int32_t)s)) {
            blocked = e0 == EFF_BLOCKED;
            val = blocked ? EFF_BLOCKED : (int32_t)s;
            if (!blocked) kv = T.kw[s];
            p = T.par[s];
            act = p > 0;
          }
        }
      }
      next -= __popc(idle);
    }
    if (!__any_sync(FULL, act)) {
      if (next < beg) break;
      continue;
    }
    if (act) {  // one hop: raise eff[p] to val, or stop
      int32_t cur = __ldcg(&T.eff[p]);  // L2-coherent read; CAS only to raise
      const int32_t pp = T.par[p];      // (in flight with it: the next hop needs no load of its own)
      // (in flight too) a descendant raised this walk's origin: its walk carries a larger key up
      // behind this one and raises whatever this one would -- stop here
      const int32_t eo = blocked ? val : __ldcg(&T.eff[val]);
      if (eo != val) act = false;
      for (; act;) {
        if (cur == EFF_BLOCKED || (!blocked && cur >= 0 && !key_less(T.kw[cur], kv))) {
          act = false;
          break;
        }
        const int32_t old = atomicCAS(&T.eff[p], cur, val);
        if (old == cur) break;
        cur = old;
      }
      if (act) {
        p = pp;
        act = p > 0;
      }
    }
  }
  pdl_trace_end();
}

__global__ void k_gather(DT T, int32_t hw, Key3 *__restrict__ ck, uint64_t *__restrict__ cv,
                         int64_t *__restrict__ cw, int64_t *__restrict__ count) {
  pdl_wait();
  if (hw < 0) hw = T.ctrl->hw;
  const int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  bool take = false;
  int32_t e = EFF_DEAD;
  if (s < hw) {
    e = T.eff[s];
    take = e >= 0;
  }
  const unsigned m = __ballot_sync(FULL, take);
  if (!m) return;
  int64_t base = 0;
  const int lane = lane_id();
  const int leader = __ffs(m) - 1;
  if (lane == leader) base = atomicAdd((unsigned long long *)count, (unsigned long long)__popc(m));
  base = __shfl_sync(FULL, (long long)base, leader);
  if (take) {
    const int64_t pos = base + __popc(m & ((1u << lane) - 1));
    ck[pos] = composite(T.kw[e], T.dend[s]);
    cv[pos] = ((uint64_t)T.kver[s] << 32) | (uint32_t)s;
    cw[pos] = T.elen[s];
  }
}

// the sorted list is ready: n entries out of `total` candidates
__global__ void k_list_ready(DT T, int64_t n, int64_t total) {
  pdl_wait();
  Ctrl *c = T.ctrl;
  c->L_n = n;
  c->L_partial = n < total ? 1 : 0;
  c->L_cur = 0;
  c->L_valid = 1;
  c->H_n = 0;
  c->builds++;
}

// ------------------------------------------------------------ protection

// set_protection sort key (kvcache.py:375-381): (-P-hat, segment or -1, node_id)
__global__ void k_prot_gather(DT T, int32_t hw, Key3 *__restrict__ ck, uint64_t *__restrict__ cv,
                              int64_t *__restrict__ cw, int64_t *__restrict__ count) {
  pdl_wait();
  const int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  bool take = false;
  if (s < hw && s != ROOT) take = T.nid[s] >= 0 && T.par[s] >= 0 && T.hasanc[s] && T.akind[s] == K_REUSABLE;
  const unsigned m = __ballot_sync(FULL, take);
  if (!m) return;
  const int lane = lane_id();
  const int leader = __ffs(m) - 1;
  int64_t base = 0;
  if (lane == leader) base = atomicAdd((unsigned long long *)count, (unsigned long long)__popc(m));
  base = __shfl_sync(FULL, (long long)base, leader);
  if (take) {
    const int64_t pos = base + __popc(m & ((1u << lane) - 1));
    const int32_t sg = T.seg[s];
    const int32_t sv = sg == SEG_NONE ? -1 : sg;
    Key3 k = {0, 0, 0};
    shl_or(k, 64, ord_f64(-pri_of(T, sg)));
    shl_or(k, 32, (uint64_t)((uint32_t)sv ^ 0x80000000u));
    shl_or(k, 40, (uint64_t)T.nid[s] & ((1ull << 40) - 1));
    ck[pos] = k;
    cv[pos] = (uint64_t)(uint32_t)s;
    cw[pos] = 1;
  }
}

__global__ void k_prot_clear(DT T, int32_t hw) {
  pdl_wait();
  const int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < hw) T.prot[s] = 0;
}

__global__ void k_prot_set(DT T, const uint64_t *__restrict__ sorted_v, int64_t f,
                           int64_t *__restrict__ out_ids) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= f) return;
  const int32_t s = (int32_t)(sorted_v[i] & 0xffffffffu);
  T.prot[s] = 1;
  out_ids[i] = T.nid[s];
}

// note_active_segments (kvcache.py:385-393): rewrite the a-bit of every
// reusable anchor's counter snapshot
__global__ void k_note_active(DT T, int32_t hw) {
  pdl_wait();
  const int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= hw || s == ROOT || T.nid[s] < 0 || T.par[s] < 0) return;
  if (!T.hasanc[s] || T.akind[s] != K_REUSABLE) return;
  const int32_t sg = T.aseg[s];
  T.snap[3 * (int64_t)s + 1] = (sg != SEG_NONE && sg >= 0 && sg < T.nact && T.act[sg]) ? 1 : 0;
}

__global__ void k_active_flags(DT T, const int32_t *__restrict__ a, const int32_t *__restrict__ nd,
                               int32_t nseg) {
  pdl_wait();
  const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < nseg) T.act[r] = (a[r] > 0 || nd[r] > 0) ? 1 : 0;
}

// ------------------------------------------------------------ release

// release_path (kvcache.py:350-360) for n leaves in order; stops at the first
// invalid one (status written to out[0] = index of failure or -1)
__global__ void k_release_seq(DT T, int64_t n, const int32_t *__restrict__ slots,
                              const int64_t *__restrict__ ids, int64_t *out) {
  pdl_wait();
  if (threadIdx.x != 0) return;
  const int32_t hw = T.ctrl->hw;
  for (int64_t i = 0; i < n; i++) {
    const int32_t s = slots[i];
    bool ok = s >= 0 && s < hw && T.nid[s] == ids[i];
    for (int32_t x = s; ok && x >= 0; x = T.par[x])
      if (T.ref[x] <= 0) ok = false;
    if (!ok) {
      out[0] = i;
      return;
    }
    for (int32_t x = s; x >= 0; x = T.par[x]) T.ref[x] -= 1;
  }
  out[0] = -1;
}

// batched release of valid pins: one warp per leaf, atomic decrements
// the lanes of a warp climb their chains in lock step; lanes standing on the
// same node (the shared upper levels: system prompt, popular segments, the
// root) release it with one combined atomic
// release_path (kvcache.py:350-362) of n leaves: -1 on every node of each
// leaf's root chain.  A leaf whose root path the last parallel commit recorded
// (same slot, same version, no split since: the path is unchanged) is released
// from that list -- thread (member j, piece row) piece-major, so the members
// sharing the upper nodes combine their decrements per warp, with no
// dependent climb (after the L2 flush each hop of a climb is an HBM round
// trip); any other leaf climbs its parent chain, lanes in lock step.
template <int PL>
__global__ void k_release_par(DT T, int64_t n, const int32_t *__restrict__ slots, const int32_t *pinl,
                              const int32_t *pinp, const uint32_t *pinv, const int32_t *pinh) {
  pdl_wait();
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const int64_t j = t % n;
  const bool live = t < n * PL;
  const int32_t leaf = live ? slots[j] : -1;
  bool listed = false;
  int P = 0;
  if (pinh && live && leaf >= 0 && j < __ldcg(&pinh[0]) && __ldcg(&pinh[1]) == T.ctrl->splits) {
    P = __ldcg(&pinp[j]);
    listed = __ldcg(&pinv[j]) == T.kver[leaf] && (P > 0 ? __ldcg(&pinl[j * WP_MAXP + P - 1]) : ROOT) == leaf;
    if (!listed) P = 0;
  }
  for (int p = (int)(t / n); __any_sync(0xffffffffu, listed && p < P); p += PL) {
    const bool on = listed && p < P;
    const int32_t s = on ? __ldcg(&pinl[j * WP_MAXP + p]) : -1 - lane;
    const unsigned peers = __match_any_sync(0xffffffffu, s);
    if (on && lane == __ffs(peers) - 1) atomicSub(&T.ref[s], __popc(peers));
  }
  const unsigned m0 = __ballot_sync(0xffffffffu, listed && t < n);  // (each listed member's root pin, once)
  if (m0 && lane == __ffs(m0) - 1) atomicSub(&T.ref[ROOT], __popc(m0));
  // the rest climb (one thread per member: the first row)
  int32_t x = (live && t < n && !listed) ? leaf : -1;
  while (__any_sync(0xffffffffu, x >= 0)) {
    const unsigned peers = __match_any_sync(0xffffffffu, x);
    if (x >= 0 && lane == __ffs(peers) - 1) atomicSub(&T.ref[x], __popc(peers));
    if (x >= 0) x = T.par[x];
  }
  pdl_trace_end();
}

// the inverse: +1 along each leaf's root chain (an explicit lock of a cached
// prefix, e.g. the SGLang-style adapter's inc_lock_ref)
__global__ void k_pin_par(DT T, int64_t n, const int32_t *__restrict__ slots) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  int32_t x = i < n ? slots[i] : -1;
  while (__any_sync(0xffffffffu, x >= 0)) {
    const unsigned peers = __match_any_sync(0xffffffffu, x);
    if (x >= 0 && lane == __ffs(peers) - 1) atomicAdd(&T.ref[x], __popc(peers));
    if (x >= 0) x = T.par[x];
  }
}

// ------------------------------------------------------------ maintenance

__global__ void k_rehash(DT T, int32_t hw, int64_t *live) {
  pdl_wait();
  const int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= hw || s == ROOT || T.nid[s] < 0 || T.par[s] < 0) return;
  const uint64_t key = ckey(T.par[s], T.ftok[s]);
  uint64_t h = mix64(key) & T.hmask;
  for (;;) {
    const unsigned long long prev =
        atomicCAS((unsigned long long *)&T.ht[h].key, (unsigned long long)HEMPTY, (unsigned long long)key);
    if (prev == HEMPTY) {
      T.ht[h].val = (uint32_t)s;
      T.hslot[s] = (int32_t)h;
      break;
    }
    h = (h + 1) & T.hmask;
  }
  atomicAdd((unsigned long long *)live, 1ull);
}

__global__ void k_compact_len(DT T, int32_t hw, int64_t *__restrict__ len) {
  pdl_wait();
  const int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= hw) return;
  len[s] = (s != ROOT && T.nid[s] >= 0 && T.par[s] >= 0) ? T.elen[s] : 0;
}

__global__ void k_compact_copy(DT T, int32_t hw, const int64_t *__restrict__ newoff,
                               uint32_t *__restrict__ dst) {
  pdl_wait();
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= hw) return;
  const int32_t s = (int32_t)w;
  if (s == ROOT || T.nid[s] < 0 || T.par[s] < 0) return;
  const int64_t src = T.eoff[s], d = newoff[s];
  const int32_t len = T.elen[s];
  for (int32_t i = lane_id(); i < len; i += 32) dst[d + i] = T.tok[src + i];
  __syncwarp();
  if (lane_id() == 0) T.eoff[s] = d;
}

__global__ void k_key_of(DT T, int32_t s, Key3 *out) {
  pdl_wait();
  if (threadIdx.x == 0) *out = make_key(T, s);
}

}  // namespace prism
