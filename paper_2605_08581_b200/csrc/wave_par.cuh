// wave_par.cuh -- exact PARALLEL commit of one segment-structured wave.
//
// The ordered commit (k_commit) replays engine.py:200-213 member by member.
// For waves produced by the fused step -- every path is
//   [system prefix sys][segment 1 .. k, chunk tokens each][private suffix]
// with anchors at every piece boundary (engine.py:269-292) and segment
// tokens unique per segment id (workload.py:136-154) -- the same result is
// computed here with data-parallel passes:
//
//   * intra-wave sharing: the longest prefix member j shares with any earlier
//     member is sys + chunk * (longest common aligned-skeleton prefix), found
//     by a first-owner table over skeleton prefixes (atomicMin of member id);
//   * hit_j = max(pre-wave match, intra-wave share) -- LCP against a union of
//     prefix-closed path sets is the max of the LCPs;
//   * node ids: member j creates its tail + one node per anchor inside it, ids
//     by an exclusive prefix sum, tail keeps the base id, uppers get base+1..
//     top-down (kvcache.py:213-236 split order);
//   * eviction: the wave's victims are a prefix of the eviction stream L
//     (subtree-max order, built on the pre-wave tree); member j's evict call
//     consumes L until the cumulative freed tokens reach its cumulative
//     demand D_j = R0 + sum_{i<=j} missing_i - capacity;
//   * touches / pins / labels: atomics (hits += 2 per traversing member, last =
//     max insert tick, ref += 1, label = last writer = max member index).
//
// A CapacityError stop (engine.py:209-212) commits in parallel too: with the
// WHOLE order listed, the first member j* whose demand exceeds every valid
// entry cannot be satisfied, so members [0, j*) commit as above, j* matches
// (its touches) and its evict call sweeps every entry still evictable at its
// time -- valid, unpinned after the earlier members' pins, not on its own
// guarded chain (kvcache.py:243-273) -- in list order, and the wave stops.
//
// Exactness guards (else the host falls back to k_commit for the wave): no
// pre-match chain overflow, no partially matched pre-wave node, pre-wave
// chain nodes aligned 1:1 with pieces, no skeleton-hash collision, no
// consumed victim on any member's pre-wave chain, enough evictable tokens.
#pragma once
#include "dart_kernels.cuh"
#include "scan.cuh"

namespace prism {

// (member, piece)-parallel kernels: WP_PL threads per member, piece p on thread p % WP_PL
#ifndef PRISM_WP_PL
#define PRISM_WP_PL 32  // (16 -> 32: 1.5% per C3 wave, same-box A/B)
#endif
constexpr int WP_PL = PRISM_WP_PL;
// device-sized scans over DS_BLOCKS partitions (k_vscan_a / k_vscan_c, the sweep)
#ifndef PRISM_DS_BLOCKS
#define PRISM_DS_BLOCKS 296
#endif
constexpr int DS_BLOCKS = PRISM_DS_BLOCKS;
enum { WPF_OVERFLOW = 1, WPF_PARTIAL = 2, WPF_ALIGN = 4, WPF_COLLIDE = 8, WPF_VICTIM = 16, WPF_CAPACITY = 32,
       WPF_SHAPE = 64 };

struct WaveIn {
  int64_t B, sys, chunk;
  const int64_t *poff;
  const uint32_t *tok;
  const int64_t *aoffs;
  const int8_t *a_kind;
  const int32_t *a_seg;
  const int32_t *a_snap;
  const int64_t *members;
  const int64_t *sk_off;
  const int32_t *aligned;
  const int32_t *pm_meta;
  const int32_t *pm_chain;
};

struct WaveTmp {
  int32_t *hit, *pre, *npieces, *p0, *lcp_level;
  int64_t *cnew, *tail, *miss;       // per member (+1 for scans)
  int64_t *idb, *arb, *dem;          // scans
  int32_t *piece_slot;               // [B * WP_MAXP] own new pieces
  int32_t *owner;                    // [B * WP_MAXP] owner member of shared pieces
  uint64_t *lt_key;                  // level table
  int32_t *lt_min;
  uint64_t lt_mask;
  int32_t *flags;                    // [1]
  int64_t *vlen, *F;                 // eviction stream prefix
  int64_t *cut;                      // per member: victims consumed through member j
  int64_t *misc;                     // [8] device scalars
  // root paths pinned by the last parallel commit (its members [0, pinh[0])),
  // for the next release (k_release_par): node slots per piece, pieces, the
  // leaf's version; pinh = {members, Ctrl::splits when recorded}
  int32_t *pinl, *pinp;              // [B * WP_MAXP], [B]
  uint32_t *pinv;                    // [B]
  int32_t *pinh;                     // [2]
};

// device-side control of one parallel wave commit: the control-block snapshot
// the wave starts from, its totals, and the stop decision -- so the whole
// commit is one stream of launches with no host round trip in the middle
enum { WC_OK = 0, WC_FALLBACK = 1, WC_MAINT = 2, WC_FULL = 3, WC_ABORT = 4 };
struct WaveCtl {
  int64_t R0, id0, clock0, arena0, vbase;  // snapshot of the control block
  int64_t ncreate, ntail, nmiss;           // totals of the plan
  int64_t W;                               // eviction-prefix tokens to select (-1: no eviction)
  int64_t nv, freed, calls;                // victims consumed, their tokens, evict calls
  int32_t ft0, hw0;
  uint32_t vctr0, epoch;
  int32_t stop, flags;                     // WC_*; fallback reason (WPF_*)
  int64_t Bc;                              // members committed (B, or j* on a CapacityError stop)
  int64_t nsw, swfreed;                    // the stopping member's sweep: victims, tokens
  int32_t trunc, pad;                      // 1: the wave stops at member Bc (CapacityError)
};

__device__ inline int64_t wp_end(const WaveIn &W, int p, int k, int64_t n) {
  // end depth of piece p: [sys][seg 0..k-1][suffix]
  const int has_sys = W.sys > 0;
  if (has_sys && p == 0) return W.sys;
  const int q = p - has_sys;  // segment index
  if (q < k) return W.sys + (int64_t)(q + 1) * W.chunk;
  return n;
}

__device__ inline int wp_level_of_piece(const WaveIn &W, int p) {
  // number of segments covered through the end of piece p
  return p + (W.sys > 0 ? 0 : 1);
}

__device__ inline uint64_t wp_level_key(int level, uint64_t h) {
  uint64_t x = mix64(h ^ (0x9E3779B97F4A7C15ull * (uint64_t)(level + 1)));
  return x >> 1;  // never HEMPTY
}

__device__ inline uint64_t wp_hash_next(uint64_t h, int32_t seg) { return mix64(h * 31 + (uint32_t)seg + 0x1234567ull); }

__device__ inline int32_t wp_table(const WaveTmp &X, uint64_t key, int32_t j, bool insert) {
  uint64_t h = mix64(key) & X.lt_mask;
  for (;;) {
    if (insert) {
      const unsigned long long prev = atomicCAS((unsigned long long *)&X.lt_key[h], (unsigned long long)HEMPTY,
                                                (unsigned long long)key);
      if (prev == HEMPTY || prev == key) {
        atomicMin(&X.lt_min[h], j);
        return (int32_t)h;
      }
    } else {
      const uint64_t k = X.lt_key[h];
      if (k == key) return X.lt_min[h];
      if (k == HEMPTY) return -1;
    }
    h = (h + 1) & X.lt_mask;
  }
}

// W1: per-member plan checks, one warp per member (lanes walk the pre-wave
// chain in parallel): shape, pre-match flags, chain nodes aligned 1:1 with the
// first pieces, and the chain marks (victim guard; first member per node)
__device__ __forceinline__ void wp_plan_body(DT T, const WaveIn &W, const WaveTmp &X, const WaveCtl *wc, int64_t blk) {
  const int64_t j = (blk * blockDim.x + threadIdx.x) >> 5;
  const int lane = lane_id();
  if (j >= W.B || wc->stop) return;  // (warp-uniform)
  const uint32_t epoch = wc->epoch;
  const int64_t m = W.members[j];
  const int k = (int)(W.sk_off[m + 1] - W.sk_off[m]);
  const int64_t n = W.poff[j + 1] - W.poff[j];
  const int64_t sfx = n - W.sys - (int64_t)k * W.chunk;
  const int P = (W.sys > 0) + k + (sfx > 0);
  int flag = 0;
  if (sfx < 0 || P > WP_MAXP || W.aoffs[j + 1] - W.aoffs[j] != P) flag |= WPF_SHAPE;
  const int32_t hit_pre = W.pm_meta[4 * j + 0], d = W.pm_meta[4 * j + 1], fl = W.pm_meta[4 * j + 3];
  if (fl & 2) flag |= WPF_OVERFLOW;
  if (fl & 1) flag |= WPF_PARTIAL;
  // pre-wave chain nodes must coincide with the first d pieces
  if (!flag) {
    if (d > P) flag |= WPF_ALIGN;
    bool bad = false;
    for (int p = lane; p < d && !(flag & WPF_ALIGN); p += 32) {
      const int32_t c = W.pm_chain[j * PM_MAX + p];
      if ((int64_t)T.dend[c] != wp_end(W, p, k, n)) bad = true;
      T.wchild[c] = epoch;  // "on some member's pre-wave chain" (victim guard)
      atomicMax((unsigned long long *)&T.wchm[c],
                ((unsigned long long)epoch << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)j));  // first such member
    }
    if (__any_sync(0xffffffffu, bad)) flag |= WPF_ALIGN;
    if (!flag && (d > 0 ? wp_end(W, d - 1, k, n) : 0) != hit_pre) flag |= WPF_ALIGN;
  }
  if (lane) return;
  if (flag) {
    atomicOr(X.flags, flag);
    return;
  }
  X.pre[j] = hit_pre;
  X.npieces[j] = P;  // (the skeleton-prefix levels go into the table in k_wp_levels)
}

// W1b: skeleton-prefix ownership table -- level L = sys piece plus the first L
// segments; the first owner of each prefix by atomicMin.  Level-major (thread
// = level L of member j, consecutive members in a warp): every member shares
// the low levels, so each warp inserts one key per distinct prefix.
__device__ __forceinline__ void wp_levels_body(const WaveIn &W, const WaveTmp &X, const WaveCtl *wc, int64_t blk) {
  if (wc->stop) return;  // (an aborted wave: no dispatch order to read)
  const int64_t t = blk * blockDim.x + threadIdx.x;
  const int64_t j = t % W.B;
  const int lane = threadIdx.x & 31;
  const bool live = t < (int64_t)W.B * WP_PL;
  int k = 0;
  const int32_t *s = nullptr;
  if (live) {
    const int64_t m = W.members[j];
    k = (int)(W.sk_off[m + 1] - W.sk_off[m]);
    s = W.aligned + W.sk_off[m];
  }
  const int lmin = W.sys > 0 ? 0 : 1;
  for (int L = (int)(t / W.B); __any_sync(0xffffffffu, live && L <= k); L += WP_PL) {
    const bool on = live && L <= k && L >= lmin;
    uint64_t key = 0;
    if (on) {
      uint64_t h = 0x51ED270B27ull;
      for (int q = 0; q < L; q++) h = wp_hash_next(h, s[q]);
      key = wp_level_key(L, h);
    }
    const unsigned peers = __match_any_sync(0xffffffffu, on ? key : ~0ull);
    const unsigned jmin = __reduce_min_sync(peers, (unsigned)j);
    if (on && lane == __ffs(peers) - 1) {
      uint64_t h = mix64(key) & X.lt_mask;
      for (;;) {
        unsigned long long prev = __ldcg((const unsigned long long *)&X.lt_key[h]);
        if (prev == (unsigned long long)HEMPTY)
          prev = atomicCAS((unsigned long long *)&X.lt_key[h], (unsigned long long)HEMPTY, (unsigned long long)key);
        if (prev == (unsigned long long)HEMPTY || prev == key) {
          atomicMin(&X.lt_min[h], (int32_t)jmin);
          break;
        }
        h = (h + 1) & X.lt_mask;
      }
    }
  }
}

// W1 + W1b in one launch (the level table needs only the dispatch order and
// the aligned skeletons, not the plan): CTAs [0, nplan) plan, the rest insert levels
__global__ void k_wp_plan_levels(DT T, WaveIn W, WaveTmp X, const WaveCtl *wc, int nplan) {
  pdl_wait();
  if ((int)blockIdx.x < nplan) wp_plan_body(T, W, X, wc, blockIdx.x);
  else wp_levels_body(W, X, wc, (int64_t)blockIdx.x - nplan);
  pdl_trace_end();
}

// W2: intra-wave share, hit, new pieces, demand -- one warp per member: lane
// q holds skeleton levels q and q + 32; every lane runs the prefix-hash chain
// (ALU + shuffles), then each looks its own levels up in the first-owner table
// at once (the lookups were a dependent sequence per member)
__global__ void k_wp_hits(DT T, WaveIn W, WaveTmp X, const WaveCtl *wc) {
  pdl_wait();
  const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = lane_id();
  if (j >= W.B || wc->stop) return;  // (warp-uniform; an aborted wave never ran the plan)
  if (*X.flags) return;
  const int64_t m = W.members[j];
  const int k = (int)(W.sk_off[m + 1] - W.sk_off[m]);
  if (k > 63) {  // (levels 0..k are held two per lane: <= 63; longer skeletons take the ordered commit)
    if (lane == 0) atomicOr(X.flags, WPF_SHAPE);
    return;
  }
  const int32_t *s = W.aligned + W.sk_off[m];
  const int64_t n = W.poff[j + 1] - W.poff[j];
  const int P = X.npieces[j];
  const int lmin = W.sys > 0 ? 0 : 1;
  // segments q = lane, lane + 32 in registers; level L hashes segments [0, L)
  const int32_t s0 = lane < k ? s[lane] : 0, s1 = lane + 32 < k ? s[lane + 32] : 0;
  uint64_t h = 0x51ED270B27ull, hL0 = 0, hL1 = 0;
  if (lane == 0) hL0 = h;
  for (int q = 0; q < k; q++) {
    const int32_t sq = __shfl_sync(0xffffffffu, q < 32 ? s0 : s1, q & 31);
    h = wp_hash_next(h, sq);
    if (q + 1 == lane) hL0 = h;
    if (q + 1 == lane + 32) hL1 = h;
  }
  // this lane's levels: ok = owned by an earlier member
  int32_t o0 = -1, o1 = -1;
  bool ok0 = true, ok1 = true;  // (levels below lmin or above k do not stop the run)
  if (lane <= k && lane >= lmin) {
    o0 = wp_table(X, wp_level_key(lane, hL0), (int32_t)j, false);
    ok0 = o0 >= 0 && o0 < j;
  }
  if (lane + 32 <= k && lane + 32 >= lmin) {
    o1 = wp_table(X, wp_level_key(lane + 32, hL1), (int32_t)j, false);
    ok1 = o1 >= 0 && o1 < j;
  }
  // lstar: the last level of the unbroken run of owned levels from lmin (-1: none)
  const unsigned bad0 = __ballot_sync(0xffffffffu, !ok0), bad1 = __ballot_sync(0xffffffffu, !ok1);
  const int first_bad = bad0 ? __ffs(bad0) - 1 : (bad1 ? 32 + __ffs(bad1) - 1 : k + 1);
  const int lstar = (first_bad > k ? k : first_bad - 1) >= lmin ? (first_bad > k ? k : first_bad - 1) : -1;
  auto own_at = [&](int L) {  // owner of level L (L <= lstar), from its lane
    const int32_t v0 = __shfl_sync(0xffffffffu, o0, L & 31), v1 = __shfl_sync(0xffffffffu, o1, L & 31);
    return L < 32 ? v0 : v1;
  };
  int64_t lcpw = 0;
  if (lstar >= 0) {
    // verify the owner really shares the skeleton prefix (hash collisions)
    const int32_t o = own_at(lstar);
    const int64_t mo = W.members[o];
    const int ko = (int)(W.sk_off[mo + 1] - W.sk_off[mo]);
    const int32_t *so = W.aligned + W.sk_off[mo];
    bool diff = false;
    if (ko < lstar) diff = true;
    for (int q = lane; q < lstar && ko >= lstar; q += 32) diff |= so[q] != s[q];
    if (__any_sync(0xffffffffu, diff)) {
      if (lane == 0) atomicOr(X.flags, WPF_COLLIDE);
      return;
    }
    lcpw = W.sys + (int64_t)lstar * W.chunk;
  }
  const int64_t hit_pre = X.pre[j];
  const int64_t hit = hit_pre > lcpw ? hit_pre : lcpw;
  // first new piece (warp-uniform) and owners of the shared (intra-wave) pieces
  int p0 = P;
  for (int p = 0; p < P; p++)
    if (wp_end(W, p, k, n) > hit) {
      p0 = p;
      break;
    }
  for (int pb = 0; pb < p0; pb += 32) {  // (all lanes join the shuffles)
    const int p = pb + lane;
    const int L = wp_level_of_piece(W, p < p0 ? p : 0);
    const int32_t ow = own_at(L > 63 ? 63 : L);
    if (p < p0) {
      const int64_t e = wp_end(W, p, k, n);
      X.owner[j * WP_MAXP + p] = (e > hit_pre && L <= lstar) ? ow : -1;
    }
  }
  if (lane) return;
  atomicAdd((unsigned long long *)&X.misc[3], (unsigned long long)n);   // inserted path tokens
  atomicAdd((unsigned long long *)&X.misc[4], (unsigned long long)p0);  // matched nodes
  X.hit[j] = (int32_t)hit;
  X.p0[j] = p0;
  X.lcp_level[j] = lstar;
  X.cnew[j] = hit < n ? (P - p0) : 0;
  X.tail[j] = n - hit;
  X.miss[j] = n - hit;
  pdl_trace_end();
}


// apply the consumed victims [0, nv) of the stream (stream order == victim order)
__global__ void k_wp_evict(DT T, const WaveCtl *wc) {
  pdl_wait();
  if (wc->stop) return;
  const int64_t nv = wc->nv;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t s = (int32_t)(T.Lv[i] & 0xffffffffu);
    const int32_t p = T.par[s];
    atomicSub(&T.nch[p], 1);
    VRec rec;
    rec.id = T.nid[s];
    rec.eoff = T.eoff[s];
    rec.ftok = T.ftok[s];
    rec.elen = T.elen[s];
    rec.seg = T.seg[s];
    rec.kind = (int8_t)T.kind[s];
    rec.pad[0] = rec.pad[1] = rec.pad[2] = 0;
    T.ht[T.hslot[s]].key = HTOMB;
    T.vlog[(wc->vbase + i) % T.vcap] = rec;
    T.nid[s] = -1;
    T.par[s] = -1;
    T.kver[s] = wc->vctr0 + (uint32_t)i + 1;
    T.wmod[s] = wc->epoch;
    T.freelist[wc->ft0 + i] = s;
  }
}

// W6a: slot of every new piece (free list LIFO, then the high-water mark)

__global__ void k_wp_alloc(DT T, WaveIn W, WaveTmp X, const WaveCtl *wc) {
  pdl_wait();
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, j = t / WP_PL;
  const int pl = (int)(t % WP_PL);
  if (j >= W.B || wc->stop || j >= wc->Bc) return;
  // label owners reset on the member's pre-wave chain (k_wp_touch elects the
  // max member per node); its intra-wave shared pieces are new nodes, reset
  // below by their creator
  const int d = W.pm_meta[4 * j + 1];
  for (int p = pl; p < d; p += WP_PL) T.eff[W.pm_chain[j * PM_MAX + p]] = -1;
  if (X.cnew[j] == 0) return;
  const int64_t id0 = wc->id0;
  const int32_t free_top = wc->ft0 + (int32_t)wc->nv, hw = wc->hw0;
  const uint32_t vctr0 = wc->vctr0 + (uint32_t)wc->nv, epoch = wc->epoch;
  const int P = X.npieces[j], p0 = X.p0[j];
  const int64_t g0 = X.idb[j];  // global index of this member's first new piece
  for (int p = p0 + pl; p < P; p += WP_PL) {
    const int64_t g = g0 + (p - p0);
    const int32_t s = g < free_top ? T.freelist[free_top - 1 - g] : (int32_t)(hw + (g - free_top));
    X.piece_slot[j * WP_MAXP + p] = s;
    // ids: the tail keeps the base id, uppers get base+1.. top-down
    const int64_t id = (p == P - 1) ? id0 + g0 : id0 + g0 + 1 + (p - p0);
    T.nid[s] = id;
    T.nch[s] = 0;
    T.ref[s] = 0;
    T.kver[s] = vctr0 + (uint32_t)g + 1;
    T.wmod[s] = epoch;
    T.wchild[s] = 0;
    T.waitf[s] = 0;
    T.guard[s] = 0;
    T.prot[s] = 0;
    T.hasanc[s] = 0;
    T.eff[s] = -1;  // label owner (reset)
  }
}

// one warp copies n uint32 tokens: 16-byte vectors (4 in flight per lane)
// when source and destination share their alignment, else words (4 in flight)
__device__ __forceinline__ void warp_copy_u32(uint32_t *dst, const uint32_t *src, int64_t n, int lane) {
  int64_t i = 0;
  if ((((uintptr_t)src ^ (uintptr_t)dst) & 15) == 0) {
    const int64_t h = (int64_t)((16 - ((uintptr_t)dst & 15)) & 15) >> 2;  // words before dst is aligned
    const int64_t head = h < n ? h : n;
    if (lane < head) dst[lane] = src[lane];
    const int64_t nv = (n - head) >> 2;
    const uint4 *s4 = reinterpret_cast<const uint4 *>(src + head);
    uint4 *d4 = reinterpret_cast<uint4 *>(dst + head);
    for (int64_t v0 = lane; v0 < nv; v0 += 128) {
      uint4 x[4];
#pragma unroll
      for (int u = 0; u < 4; u++)
        if (v0 + 32 * u < nv) x[u] = __ldg(s4 + v0 + 32 * u);
#pragma unroll
      for (int u = 0; u < 4; u++)
        if (v0 + 32 * u < nv) d4[v0 + 32 * u] = x[u];
    }
    i = head + 4 * nv;
  }
  for (int64_t i0 = i + lane; i0 < n; i0 += 128) {
    uint32_t v[4];
#pragma unroll
    for (int u = 0; u < 4; u++) v[u] = i0 + 32 * u < n ? src[i0 + 32 * u] : 0u;
#pragma unroll
    for (int u = 0; u < 4; u++)
      if (i0 + 32 * u < n) dst[i0 + 32 * u] = v[u];
  }
}

__device__ inline int32_t wp_node(const WaveIn &W, const WaveTmp &X, int64_t j, int p) {
  const int d = W.pm_meta[4 * j + 1];
  if (p < d) return W.pm_chain[j * PM_MAX + p];
  if (p < X.p0[j]) return X.piece_slot[X.owner[j * WP_MAXP + p] * WP_MAXP + p];
  return X.piece_slot[j * WP_MAXP + p];
}

// W6b: fields, child-table entries and tokens of the new pieces (warp per member)
__global__ void k_wp_create(DT T, WaveIn W, WaveTmp X, const WaveCtl *wc) {
  pdl_wait();
  // two warps per member: the even one copies the tail's tokens, the odd one
  // creates the nodes (their dependent loads overlap instead of queueing)
  const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5, j = wg >> 1;
  const int lane = lane_id();
  if (j >= W.B || wc->stop || j >= wc->Bc || X.cnew[j] == 0) return;
  const int64_t arena0 = wc->arena0, clock0 = wc->clock0;
  const int64_t n = W.poff[j + 1] - W.poff[j];
  const int64_t hit = X.hit[j];
  const uint32_t *path = W.tok + W.poff[j];
  const int64_t ab = arena0 + X.arb[j];
  if ((wg & 1) == 0) {
    warp_copy_u32(T.tok + ab, path + hit, n - hit, lane);  // the tail's tokens into the arena
    return;
  }
  const int64_t m = W.members[j];
  const int k = (int)(W.sk_off[m + 1] - W.sk_off[m]);
  const int P = X.npieces[j], p0 = X.p0[j];
  const int64_t tick = clock0 + 2 * j + 2;
  for (int p = p0 + lane; p < P; p += 32) {
    const int32_t s = X.piece_slot[j * WP_MAXP + p];
    const int64_t b = p == 0 ? 0 : wp_end(W, p - 1, k, n);
    const int64_t e = wp_end(W, p, k, n);
    const int32_t parent = p == p0 ? (p == 0 ? ROOT : wp_node(W, X, j, p - 1)) : X.piece_slot[j * WP_MAXP + p - 1];
    T.par[s] = parent;
    T.ftok[s] = path[b];
    T.eoff[s] = ab + (b - hit);
    T.elen[s] = (int32_t)(e - b);
    T.dend[s] = (int32_t)e;
    T.last[s] = tick;
    T.hits[s] = 1;
    T.kind[s] = K_PRIVATE;
    T.seg[s] = SEG_NONE;
    atomicAdd(&T.nch[parent], 1);
    const uint64_t key = ckey(parent, path[b]);
    uint64_t h = mix64(key) & T.hmask;
    for (;;) {
      const uint64_t cur = T.ht[h].key;
      if (cur == HEMPTY || cur == HTOMB) {
        const unsigned long long prev = atomicCAS((unsigned long long *)&T.ht[h].key, cur, key);
        if (prev == cur) {
          if (cur == HTOMB) atomicAdd((unsigned long long *)&X.misc[2], 1ull);  // tombstone reused
          break;
        }
        continue;  // lost the race for this cell: re-read it
      }
      h = (h + 1) & T.hmask;
    }
    T.ht[h].val = (uint32_t)s;
    T.hslot[s] = (int32_t)h;
  }
  pdl_trace_end();
}

// W7: touches of pre-existing nodes, pins, and last-writer label election
// piece-major (thread = piece p of member j, consecutive members in a warp) so
// the members sharing an upper node (the system prompt, popular segments)
// combine their touches/pins in one atomic per warp and node.  A node shared
// inside the wave is "old" (pre-existing: match + insert touches) only for the
// members after its creator, so the touches aggregate over the old peers.
__global__ void k_wp_touch(DT T, WaveIn W, WaveTmp X, const WaveCtl *wc) {
  pdl_wait();
  if (wc->stop) return;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t j = t % W.B;
  const int lane = threadIdx.x & 31;
  const bool live = t < (int64_t)W.B * WP_PL && j < wc->Bc;  // (others only vote)
  const int P = live ? X.npieces[j] : 0;
  const int own0 = live ? (X.cnew[j] ? X.p0[j] : P) : 0;
  const unsigned long long base_tick = (unsigned long long)(wc->clock0 + 2);
  for (int p = (int)(t / W.B); __any_sync(0xffffffffu, p < P); p += WP_PL) {  // rows of WP_PL pieces
    const bool on = p < P;
    const int32_t s = on ? wp_node(W, X, j, p) : -1 - lane;
    const bool old = on && p < own0;
    const unsigned peers = __match_any_sync(0xffffffffu, s);
    const unsigned jall = __reduce_max_sync(peers, (unsigned)j);
    const unsigned jold = __reduce_max_sync(peers, old ? (unsigned)j + 1u : 0u);  // 0: no old peer
    const int nold = __popc(__ballot_sync(0xffffffffu, old) & peers);
    if (on && lane == __ffs(peers) - 1) {
      if (jold) {
        atomicAdd(&T.hits[s], 2 * nold);
        atomicMax((unsigned long long *)&T.last[s], base_tick + 2ull * (jold - 1));
      }
      atomicAdd(&T.ref[s], __popc(peers));
      atomicMax(&T.eff[s], (int32_t)jall);
    }
  }
  const unsigned m0 = __ballot_sync(0xffffffffu, live && t < (int64_t)W.B);  // (members < Bc)
  if (m0 && lane == __ffs(m0) - 1) atomicAdd(&T.ref[ROOT], __popc(m0));  // _pin reaches the root (kvcache.py:344-348)
}

// W8: the elected (max-index) member writes kind/seg/anchor (kvcache.py:317-340)
__device__ inline void wp_stop_touch(DT T, const WaveIn &W, const WaveTmp &X, const WaveCtl *wc);

__global__ void k_wp_label(DT T, WaveIn W, WaveTmp X, const WaveCtl *wc, int64_t *hits, int32_t *leaf_slots,
                           int64_t *leaf_ids) {
  pdl_wait();
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x < 32) wp_stop_touch(T, W, X, wc);  // (a CapacityError stop)
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, j = t / WP_PL;
  const int pl = (int)(t % WP_PL);
  if (j >= W.B || wc->stop || j >= wc->Bc) return;
  const int64_t m = W.members[j];
  const int k = (int)(W.sk_off[m + 1] - W.sk_off[m]);
  const int64_t n = W.poff[j + 1] - W.poff[j];
  const int P = X.npieces[j];
  for (int p = pl; p < P; p += WP_PL) {
    const int32_t s = wp_node(W, X, j, p);
    X.pinl[j * WP_MAXP + p] = s;  // (the root path this member pins, for its release)
    if (T.eff[s] != (int32_t)j) continue;
    const int64_t a = W.aoffs[j] + p;
    T.kind[s] = (uint8_t)W.a_kind[a];
    T.seg[s] = W.a_seg[a];
    T.hasanc[s] = 1;
    T.akind[s] = (uint8_t)W.a_kind[a];
    T.aseg[s] = W.a_seg[a];
    T.aoff[s] = (int32_t)wp_end(W, p, k, n);
    T.snap[3 * (int64_t)s] = W.a_snap[3 * a];
    T.snap[3 * (int64_t)s + 1] = W.a_snap[3 * a + 1];
    T.snap[3 * (int64_t)s + 2] = W.a_snap[3 * a + 2];
  }
  if (pl) return;
  const int32_t leaf = P > 0 ? wp_node(W, X, j, P - 1) : ROOT;
  X.pinp[j] = P;
  X.pinv[j] = T.kver[leaf];
  if (hits) hits[j] = X.hit[j];
  if (leaf_slots) leaf_slots[j] = leaf;
  if (leaf_ids) leaf_ids[j] = T.nid[leaf];
}


// ------------------------------------------------------------ device-side control

// epoch + control-block snapshot the wave commits from
__global__ void k_wc_begin(DT T, WaveCtl *wc, const int32_t *abort, WaveTmp X, int64_t nlt) {
  pdl_wait();
  // the wave's scratch: empty level table, flags, device scalars (misc[1]:
  // the poison index "none")
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nlt; i += (int64_t)gridDim.x * blockDim.x) {
    X.lt_key[i] = ~0ull;
    X.lt_min[i] = 0x7F7F7F7F;
  }
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  *X.flags = 0;
  for (int q = 0; q < 8; q++) X.misc[q] = 0;
  X.misc[1] = 0x7F7F7F7F7F7F7F7Fll;
  X.misc[5] = 0x7F7F7F7F7F7F7F7Fll;  // j*: the first member the whole order cannot satisfy
  Ctrl *C = T.ctrl;
  C->epoch++;
  WaveCtl w{};
  if (abort && *abort) w.stop = WC_ABORT;  // the caller's stage of the wave failed: touch nothing
  w.epoch = C->epoch;
  w.R0 = C->resident;
  w.id0 = C->next_id;
  w.clock0 = C->clock;
  w.arena0 = C->arena_top;
  w.vbase = C->vlog_count;
  w.ft0 = C->free_top;
  w.hw0 = C->hw;
  w.vctr0 = C->vctr;
  w.W = -1;
  w.Bc = 0;
  *wc = w;
}

// exclusive scans cnew -> idb, tail -> arb (B + 1 entries) and the inclusive
// scan miss -> dem (B entries), one CTA
// plan verdict: fallback flags, capacity headroom (slots, arena, child table),
// and the eviction demand -> the prefix of the order to select (-1: none)
__device__ inline void wc_plan_body(DT T, int64_t B, WaveTmp X, WaveCtl *wc, int64_t slack, int32_t force_full) {
  if (wc->stop) {  // aborted before the plan
    wc->W = -1;
    return;
  }
  const int32_t flags = *X.flags;
  if (flags) {
    wc->stop = WC_FALLBACK;
    wc->flags = flags;
    wc->W = -1;
    return;
  }
  const int64_t ncreate = X.idb[B], ntail = X.arb[B], nmiss = X.dem[B - 1];
  wc->ncreate = ncreate;
  wc->ntail = ntail;
  wc->nmiss = nmiss;
  const Ctrl *C = T.ctrl;
  if ((int64_t)wc->hw0 + ncreate + 2 > (int64_t)T.S || wc->arena0 + ntail > T.acap ||
      (C->hlive + C->htomb + ncreate + 64) * 2 > (int64_t)(T.hmask + 1)) {
    wc->stop = WC_MAINT;
    wc->W = -1;
    return;
  }
  const int64_t D = wc->R0 + nmiss - T.capacity;
  wc->W = D > 0 ? (force_full ? 0 : D + D / 4 + slack) : -1;
  wc->Bc = B;
}

__global__ void __launch_bounds__(1024) k_wp_scan3(DT T, int64_t B, WaveTmp X, WaveCtl *wc, int64_t slack,
                                                  int32_t force_full) {
  pdl_wait();
  // an aborted or flagged wave has no plan to scan: straight to the verdict (uniform)
  if (wc->stop || *X.flags) {
    if (threadIdx.x == 0) wc_plan_body(T, B, X, wc, slack, force_full);
    return;
  }
  // the three scans in one pass (one load round trip; B + 1 <= 5 * 1024 items
  // make a single tile at the bench's wave size)
  block_scan4<3, 5>(
      B + 1,
      [&](int a, int64_t i) -> int64_t {
        if (i >= B) return 0;
        return a == 0 ? X.cnew[i] : (a == 1 ? X.tail[i] : X.miss[i]);
      },
      [&](int a, int64_t i, int64_t ex, int64_t in) {
        if (a == 0) X.idb[i] = ex;
        else if (a == 1) X.arb[i] = ex;
        else if (i < B) X.dem[i] = in;
      });
  // and the plan verdict (block_scan4 ends on a barrier: the sums are visible)
  if (threadIdx.x == 0) wc_plan_body(T, B, X, wc, slack, force_full);
}


__device__ inline bool wp_conflict(const DT &T, const WaveTmp &X, const int64_t *part, int64_t nv, int64_t Bc);

// the victims: nv = entries consumed through the last member, checks that the
// prefix sufficed and that no consumed entry is pinned/guarded; the number of
// evict calls (members whose cut advances) and the tokens freed
__device__ inline void wc_cut_body(DT T, int64_t B, WaveTmp X, WaveCtl *wc, const int64_t *part) {
  __shared__ int64_t s_calls[32];
  const int32_t flags = __ldcg(X.flags);
  // a CapacityError stop commits the members before it (when the whole order
  // is listed: a partial prefix proves nothing -- take the whole order)
  const bool cap = (flags & WPF_CAPACITY) != 0;
  const int64_t jstar = (int64_t)__ldcg((const unsigned long long *)&X.misc[5]);
  const int64_t Bc = cap ? (jstar < B ? jstar : B) : B;
  int64_t calls = 0;
  for (int64_t j = threadIdx.x; j < Bc; j += blockDim.x) calls += __ldcg(&X.cut[j]) > (j ? __ldcg(&X.cut[j - 1]) : 0) ? 1 : 0;
  for (int o = 16; o > 0; o >>= 1) calls += __shfl_xor_sync(0xffffffffu, calls, o);
  if ((threadIdx.x & 31) == 0) s_calls[threadIdx.x >> 5] = calls;
  // (the conflict guard over the consumed prefix, by the whole CTA; used below
  // only on the path where the victims [0, nv) are final)
  const bool conflict = wp_conflict(T, X, part, Bc > 0 ? __ldcg(&X.cut[Bc - 1]) : 0, Bc);  // (+ barrier)
  if (threadIdx.x) return;
  calls = 0;
  for (int w = 0; w < (int)(blockDim.x >> 5); w++) calls += s_calls[w];
  const int64_t poison = X.misc[1];
  if (cap && T.ctrl->L_partial) {
    wc->stop = WC_FULL;  // the selected prefix fell short: the whole order
    return;
  }
  const int64_t nv = Bc > 0 ? __ldcg(&X.cut[Bc - 1]) : 0;
  if ((flags & ~WPF_CAPACITY) || poison < nv) {
    wc->stop = WC_FALLBACK;
    wc->flags = (flags & ~WPF_CAPACITY) ? flags : WPF_VICTIM;
    return;
  }
  if (conflict) {
    wc->stop = WC_FALLBACK;
    wc->flags = WPF_VICTIM;
    return;
  }
  wc->Bc = Bc;
  wc->trunc = Bc < B ? 1 : 0;
  wc->nv = nv;
  wc->calls = calls + (Bc < B ? 1 : 0);  // the stopping member's evict call
  wc->freed = nv > 0 ? X.F[nv - 1] : 0;
}

// per member: number of list entries consumed through member j (first F >= D_j),
// one warp per member: a 32-ary search (32 probes per round, ~4 dependent
// rounds over a 400K-entry prefix instead of ~19 for a binary search); the
// last CTA to finish then takes the verdict (wc_cut_body)
__global__ void k_wp_cuts(DT T, int64_t B, WaveTmp X, WaveCtl *wc, const int64_t *part) {
  pdl_wait();
  __shared__ bool s_last;
  const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wc->stop) return;  // (uniform over the grid)
  if (j < B) {  // (warp-uniform)
    const int64_t D = wc->R0 + X.dem[j] - T.capacity;  // dem = inclusive sum of missing
    int64_t c = 0;
    if (D > 0) {
      const int64_t Tn = T.ctrl->L_n;
      int64_t lo = 0, hi = Tn;  // the first idx with F[idx] >= D lies in [lo, hi] (hi: Tn or known >= D)
      while (hi - lo > 32) {
        const int64_t step = (hi - lo + 31) >> 5, p = lo + lane * step;
        const bool ge = p < hi && __ldcg(&X.F[p]) >= D;
        const unsigned b = __ballot_sync(0xffffffffu, ge);
        const unsigned lt = __ballot_sync(0xffffffffu, p < hi && !ge);  // (a prefix of the lanes)
        if (b) {
          const int f = __ffs(b) - 1;
          hi = lo + f * step;
        }
        if (lt) lo = lo + (int64_t)(31 - __clz(lt)) * step + 1;  // past the last probe below D
      }
      const int64_t p = lo + lane;
      const unsigned b = __ballot_sync(0xffffffffu, p < hi && __ldcg(&X.F[p]) >= D);
      const int64_t a = b ? lo + __ffs(b) - 1 : hi;
      if (a >= Tn) {
        if (lane == 0) {
          atomicOr(X.flags, WPF_CAPACITY);
          atomicMin((unsigned long long *)&X.misc[5], (unsigned long long)j);
        }
        c = Tn;
      } else {
        c = a + 1;
      }
    }
    if (lane == 0) X.cut[j] = c;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0)
    s_last = atomicAdd((unsigned long long *)&X.misc[7], 1ull) == (unsigned long long)gridDim.x - 1ull;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  wc_cut_body(T, B, X, wc, part);
}

// the control block after the committed wave (what the ordered commit leaves)
__device__ inline void wc_finalize_body(DT T, int64_t B, const WaveTmp &X, const WaveCtl *wc) {
  (void)B;
  Ctrl *C = T.ctrl;
  const int64_t Bc = wc->Bc, nv = wc->nv, nsw = __ldcg(&wc->nsw);  // (nsw, swfreed: the sweep's CTAs)
  const int64_t ncreate = X.idb[Bc], ntail = X.arb[Bc], nmiss = Bc > 0 ? X.dem[Bc - 1] : 0;
  const int32_t ft1 = wc->ft0 + (int32_t)nv;
  const int64_t from_free = ncreate < ft1 ? ncreate : ft1;
  const int64_t reused = X.misc[2];
  C->free_top = ft1 - (int32_t)from_free + (int32_t)nsw;
  C->hw = wc->hw0 + (int32_t)(ncreate - from_free);
  C->resident = wc->R0 + nmiss - wc->freed - __ldcg(&wc->swfreed);
  C->clock = wc->clock0 + 2 * Bc + (wc->trunc ? 1 : 0);  // the stopping member's match tick
  C->next_id = wc->id0 + ncreate;
  C->arena_top = wc->arena0 + ntail;
  C->vlog_count += nv + nsw;
  C->hlive += ncreate - nv - nsw;
  C->htomb += nv + nsw - reused;
  C->evict_calls += wc->calls;
  C->vctr = wc->vctr0 + (uint32_t)(nv + ncreate + nsw);
  C->n_admitted = (int32_t)Bc;
  C->fast_members += Bc;
  if (wc->trunc) C->gstamp += 1;  // (the sweep's guard stamp)
  C->inserted_tokens += X.misc[3];
  C->chain_nodes += X.misc[4];
  C->status = ST_DONE;
  C->L_valid = 0;
  C->H_n = 0;
}





// the eviction stream's token lengths fused into the device-sized scan: entry
// i of the list counts elen when it is still the node it was listed as and
// evictable by the wave's members, else 0 (and marks the first such entry:
// misc[1], the victim guard).  k_vscan_a: per-block sums (+ the guard),
// k_vscan_c: each CTA reduces the sums before it, then the inclusive prefix F.
__device__ __forceinline__ int64_t wp_vlen(const DT &T, const WaveTmp &X, int64_t i, uint32_t epoch, int64_t &mark) {
  const uint64_t v = T.Lv[i];
  const int32_t s = (int32_t)(v & 0xffffffffu);
  const bool valid = T.kver[s] == (uint32_t)(v >> 32) && T.nid[s] >= 0 && T.par[s] >= 0 && T.ref[s] == 0;
  if (!valid) atomicMin((unsigned long long *)&X.misc[1], (unsigned long long)i);
  // the first member whose pre-wave chain holds it (a victim a running member matched)
  const uint64_t m = T.wchm[s];
  mark = (uint32_t)(m >> 32) == epoch ? (int64_t)(0xFFFFFFFFu - (uint32_t)m) : 0x7FFFFFFFFFFFFFFFll;
  return valid ? T.elen[s] : 0;
}

// the conflict guard, in the cut verdict: a victim consumed by the committed
// members [0, Bc) that lies on the pre-wave chain of a member that runs
// (index <= Bc: the committed ones and a stopping one) changes that member's
// match (nothing applied yet).  vlen holds the in-partition prefix minimum of
// the first-member marks, part[DS_BLOCKS + b] partition b's minimum (k_vscan_a)
__device__ inline bool wp_conflict(const DT &T, const WaveTmp &X, const int64_t *part, int64_t nv, int64_t Bc) {
  if (nv <= 0) return false;
  const int64_t n = T.ctrl->L_n, per = (n + DS_BLOCKS - 1) / DS_BLOCKS, q = (nv - 1) / per;
  bool hit = false;
  for (int64_t b = threadIdx.x; b < q; b += blockDim.x) hit |= __ldcg(&part[DS_BLOCKS + b]) <= Bc;
  if (threadIdx.x == 0) hit |= __ldcg(&X.vlen[nv - 1]) <= Bc;
  return __syncthreads_or(hit) != 0;
}

// k_vscan_a: each CTA's contiguous partition -- the entries' lengths (one
// gather pass over the list), their inclusive prefix within the partition
// into F and the partition's total; k_vscan_c: + the totals of the partitions
// before it (a streaming add; the gathers are not repeated)
__global__ void __launch_bounds__(256) k_vscan_a(DT T, WaveTmp X, int64_t *part, const WaveCtl *wc) {
  pdl_wait();
  if (wc->stop || wc->W < 0) return;
  constexpr int64_t INF = 0x7FFFFFFFFFFFFFFFll;
  __shared__ int64_t sw[8], sm[8];
  __shared__ int64_t carry, cmin;
  const int64_t n = T.ctrl->L_n, per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = blockIdx.x * per, b1 = b0 + per < n ? b0 + per : n;
  const uint32_t epoch = wc->epoch;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0, cmin = INF;
  constexpr int U = 4;  // entries per thread per round (their gathers in flight together)
  for (int64_t t0 = b0; t0 < b1; t0 += U * blockDim.x) {
    int64_t v[U], mk[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int64_t i = t0 + (int64_t)threadIdx.x * U + u;
      mk[u] = INF;
      v[u] = i < b1 ? wp_vlen(T, X, i, epoch, mk[u]) : 0;
    }
    int64_t x = 0, y = INF;
#pragma unroll
    for (int u = 0; u < U; u++) x += v[u], y = mk[u] < y ? mk[u] : y;
    const int64_t own = x;
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t a = __shfl_up_sync(0xffffffffu, x, o), b = __shfl_up_sync(0xffffffffu, y, o);
      if (lane >= o) x += a, y = b < y ? b : y;
    }
    int64_t yex = __shfl_up_sync(0xffffffffu, y, 1);  // exclusive min within the warp
    if (lane == 0) yex = INF;
    if (lane == 31) sw[wid] = x, sm[wid] = y;
    __syncthreads();
    int64_t before = carry, mbefore = cmin;
    for (int w = 0; w < wid; w++) before += sw[w], mbefore = sm[w] < mbefore ? sm[w] : mbefore;
    int64_t run = before + x - own, rmin = yex < mbefore ? yex : mbefore;
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int64_t i = t0 + (int64_t)threadIdx.x * U + u;
      run += v[u];
      rmin = mk[u] < rmin ? mk[u] : rmin;
      if (i < b1) X.F[i] = run, X.vlen[i] = rmin;  // (vlen: in-partition prefix minimum of the marks)
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = before + x, cmin = y < mbefore ? y : mbefore;
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = carry, part[DS_BLOCKS + blockIdx.x] = cmin;
}

__global__ void __launch_bounds__(256) k_vscan_c(DT T, WaveTmp X, const int64_t *part, const WaveCtl *wc) {
  pdl_wait();
  if (wc->stop || wc->W < 0) return;
  __shared__ int64_t sw[8];
  __shared__ int64_t carry;
  const int64_t n = T.ctrl->L_n, per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = blockIdx.x * per, b1 = b0 + per < n ? b0 + per : n;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  {  // this CTA's carry: the totals of the partitions before it (k_vscan_a), reduced here
    int64_t x = 0;
    for (int q = threadIdx.x; q < (int)blockIdx.x; q += blockDim.x) x += part[q];
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) sw[wid] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t c = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); w++) c += sw[w];
      carry = c;
    }
    __syncthreads();
  }
  const int64_t c = carry;
  if (c)
    for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) X.F[i] += c;
}

// ------------------------------------------------------------ CapacityError stop (member Bc = j*)

// j*'s match (kvcache.py:146-171: hits + 1, last = its match tick on every
// node of its matched prefix) and the guard of its reserve (its pre-wave
// chain, kvcache.py:252-266), one warp of k_wp_label (after the earlier
// members' pins, before the sweep)
__device__ inline void wp_stop_touch(DT T, const WaveIn &W, const WaveTmp &X, const WaveCtl *wc) {
  if (wc->stop || !wc->trunc) return;
  const int64_t j = wc->Bc;
  const int lane = lane_id();
  const int d = W.pm_meta[4 * j + 1];
  const uint32_t stamp = T.ctrl->gstamp + 1;
  for (int p = lane; p < d; p += 32) T.guard[W.pm_chain[j * PM_MAX + p]] = stamp;
  const int64_t tick = wc->clock0 + 2 * j + 1;
  for (int p = lane; p < X.p0[j]; p += 32) {
    const int32_t s = wp_node(W, X, j, p);
    atomicAdd(&T.hits[s], 1);
    atomicMax((unsigned long long *)&T.last[s], (unsigned long long)tick);
  }
}

// the sweep: list entries [nv, L_n) still evictable at j*'s time, in list order
__device__ __forceinline__ bool wp_sweepable(const DT &T, int64_t i, uint32_t stamp) {
  const uint64_t v = T.Lv[i];
  const int32_t s = (int32_t)(v & 0xffffffffu);
  return T.kver[s] == (uint32_t)(v >> 32) && T.nid[s] >= 0 && T.par[s] >= 0 && T.ref[s] == 0 && T.guard[s] != stamp;
}

__global__ void __launch_bounds__(256) k_wp_sweep_a(DT T, int64_t *part, const WaveCtl *wc) {
  pdl_wait();
  if (wc->stop || !wc->trunc) return;
  const int64_t nv = wc->nv, n = T.ctrl->L_n - nv, per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = nv + blockIdx.x * per, b1 = b0 + per < nv + n ? b0 + per : nv + n;
  const uint32_t stamp = T.ctrl->gstamp + 1;
  int64_t c = 0;
  for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) c += wp_sweepable(T, i, stamp) ? 1 : 0;
  __shared__ int64_t sw[8];
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += sw[w];
    part[blockIdx.x] = t;
  }
}

// each CTA: its carry from the counts before it, then its sweepable entries
// detached in order (victim log, free list, child table, parents' child counts)
__device__ __forceinline__ void wp_sweep_c_body(DT T, const WaveTmp &X, const int64_t *part, WaveCtl *wc) {
  __shared__ int64_t sw[8];
  __shared__ int64_t carry;
  const int64_t nv = wc->nv, n = T.ctrl->L_n - nv, per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = nv + blockIdx.x * per, b1 = b0 + per < nv + n ? b0 + per : nv + n;
  const uint32_t stamp = T.ctrl->gstamp + 1;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  {
    int64_t x = 0;
    for (int q = threadIdx.x; q < (int)blockIdx.x; q += blockDim.x) x += part[q];
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) sw[wid] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t c = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); w++) c += sw[w];
      carry = c;
    }
    __syncthreads();
  }
  const int64_t Bc = wc->Bc, ncreate = X.idb[Bc];
  const int32_t ft1 = wc->ft0 + (int32_t)nv;
  const int64_t fbase = ft1 - (ncreate < ft1 ? ncreate : ft1);  // the free list after this wave's allocations
  int64_t tok = 0;
  for (int64_t t0 = b0; t0 < b1; t0 += blockDim.x) {
    const int64_t i = t0 + threadIdx.x;
    const bool on = i < b1 && wp_sweepable(T, i, stamp);
    const unsigned bal = __ballot_sync(0xffffffffu, on);
    if (lane == 0) sw[wid] = __popc(bal);
    __syncthreads();
    int64_t before = carry;
    for (int w = 0; w < wid; w++) before += sw[w];
    before += __popc(bal & ((1u << lane) - 1u));
    if (on) {
      const int32_t s = (int32_t)(T.Lv[i] & 0xffffffffu);
      const int32_t p = T.par[s];
      atomicSub(&T.nch[p], 1);
      VRec rec;
      rec.id = T.nid[s];
      rec.eoff = T.eoff[s];
      rec.ftok = T.ftok[s];
      rec.elen = T.elen[s];
      rec.seg = T.seg[s];
      rec.kind = (int8_t)T.kind[s];
      rec.pad[0] = rec.pad[1] = rec.pad[2] = 0;
      tok += rec.elen;
      T.ht[T.hslot[s]].key = HTOMB;
      T.vlog[(wc->vbase + nv + before) % T.vcap] = rec;
      T.nid[s] = -1;
      T.par[s] = -1;
      T.kver[s] = wc->vctr0 + (uint32_t)(nv + ncreate + before) + 1;
      T.wmod[s] = wc->epoch;
      T.freelist[fbase + before] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t c = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); w++) c += sw[w];
      carry += c;
    }
    __syncthreads();
  }
  for (int o = 16; o > 0; o >>= 1) tok += __shfl_xor_sync(0xffffffffu, tok, o);
  if (lane == 0 && tok) atomicAdd((unsigned long long *)&wc->swfreed, (unsigned long long)tok);
  if (threadIdx.x == 0 && blockIdx.x == gridDim.x - 1) wc->nsw = carry;  // (the last CTA's carry: all of them)
}

// copy of a device struct to its mapped pinned host copy, 8-byte words over the CTA
template <class S>
__device__ __forceinline__ void wc_to_host(S *dst, const S *src) {
  static_assert(sizeof(S) % 8 == 0, "word copy");
  const unsigned long long *a = (const unsigned long long *)src;
  unsigned long long *b = (unsigned long long *)dst;
  for (int w = threadIdx.x; w < (int)(sizeof(S) / 8); w += blockDim.x) b[w] = __ldcg(a + w);
}

// the sweep (a CapacityError stop; else nothing), then the last CTA to finish
// writes the control block after the committed wave and the verdict + control
// block straight to the host's pinned (mapped) copies: no copy nodes
__global__ void __launch_bounds__(256) k_wp_sweep_c(DT T, int64_t B, WaveTmp X, const int64_t *part, WaveCtl *wc,
                                                   WaveCtl *h_wc, Ctrl *h_ctrl) {
  pdl_wait();
  if (!wc->stop && wc->trunc) wp_sweep_c_body(T, X, part, wc);  // (uniform)
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0)
    s_last = atomicAdd((unsigned long long *)&X.misc[6], 1ull) == (unsigned long long)gridDim.x - 1ull;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x == 0 && !__ldcg(&wc->stop)) {
    wc_finalize_body(T, B, X, wc);
    X.pinh[0] = (int32_t)wc->Bc;  // the committed members' recorded root paths
    X.pinh[1] = T.ctrl->splits;
  }
  __threadfence();
  __syncthreads();
  wc_to_host(h_wc, wc);
  wc_to_host(h_ctrl, T.ctrl);
}

}  // namespace prism
