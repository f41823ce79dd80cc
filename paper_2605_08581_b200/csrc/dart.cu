// dart.cu -- host runtime + C ABI of the device DART tree (see include/prism.h).
//
// The host side owns the device memory (slot SoA, child table, token arena,
// eviction list, victim log), launches the kernels of dart_kernels.cuh on
// one stream per tree, and services the commit kernel's resumable stops:
// NEED_BUILD (eviction order), NEED_SLOTS / NEED_ARENA / NEED_HASH (grow,
// compact, rehash).  All tree state lives in HBM; nothing is mirrored on the
// host, and there is no CPU execution path.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <cub/cub.cuh>
#include <string>
#include <vector>

#include "../../include/prism.h"
#include "pdl.cuh"
#include "dart_kernels.cuh"
#include "select.cuh"
#include "wave_par.cuh"
#include "coop.cuh"
#include "kv.cuh"

using namespace prism;

namespace {
thread_local std::string g_err;

struct Key3Decomp {
  __host__ __device__ ::cuda::std::tuple<uint64_t &, uint64_t &, uint64_t &> operator()(Key3 &k) const {
    return {k.w0, k.w1, k.w2};
  }
};

int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}

#define CK(x)                                                                                \
  do {                                                                                       \
    cudaError_t e_ = (x);                                                                    \
    if (e_ != cudaSuccess)                                                                   \
      return fail(PRISM_CUDA, std::string("CUDA error ") + cudaGetErrorString(e_) + " in " #x); \
  } while (0)

template <class T>
cudaError_t dalloc(T **p, int64_t n) {
  return cudaMalloc((void **)p, sizeof(T) * (size_t)std::max<int64_t>(n, 1));
}

int64_t next_pow2(int64_t x) {
  int64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

constexpr int TPB = 256;
inline unsigned blocks_for(int64_t n, int tpb = TPB) { return (unsigned)((n + tpb - 1) / tpb); }
}  // namespace

struct prism_tree {
  int dev = 0;
  cudaStream_t st = nullptr;
  // protection of the fused wave runs on st_aux, overlapped with the
  // serialization / pre-match / commit plan on st; st joins it (join_aux)
  // before anything reads the protected flags
  cudaStream_t st_aux = nullptr;
  cudaEvent_t ev_aux = nullptr, ev_main = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;  // caller stream <-> tree stream (graph-capturable)
  int aux_pending = 0;
  int keys_fresh = 0;  // the protection pass left the eviction keys (k_build_keys not needed)
  int prebuilt = 0;    // ... and the subtree maxima + the sample of the order (prebuild_order)
  DT d{};
  Ctrl *hctrl = nullptr;  // pinned
  int64_t protect_budget = 0;
  // candidate buffers (gather output / selection rounds / selected set), sized S
  Key3 *ck = nullptr, *ck2 = nullptr, *ks = nullptr;
  uint64_t *cv = nullptr, *cv2 = nullptr, *vs = nullptr;
  int64_t *cw = nullptr, *cw2 = nullptr;
  SelState *sel = nullptr;
  Key3 *bmin = nullptr, *bmax = nullptr;
  Key3 *kt = nullptr;  // cooperative sort scratch
  uint64_t *vt = nullptr;
  CoopState *cst = nullptr;
  int coop_grid = 0;
  int64_t *d_count = nullptr;
  int64_t *h_small = nullptr;  // pinned scratch
  void *cub_tmp = nullptr;
  size_t cub_bytes = 0;
  // per-call staging
  uint32_t *d_path = nullptr;
  int64_t path_cap = 0;
  int32_t *d_aoff = nullptr, *d_aseg = nullptr, *d_asnap = nullptr;
  int8_t *d_akind = nullptr;
  int64_t anc_cap = 0;
  OpRes *d_res = nullptr, *h_res = nullptr;
  int32_t *d_vis_slots = nullptr;
  int64_t *d_vis_ids = nullptr;
  int64_t vis_cap = 0;
  // wave staging for the host-buffer entry point
  int64_t *d_poff = nullptr, *d_aoffs = nullptr;
  int64_t woff_cap = 0;
  uint32_t *d_wtok = nullptr;
  int64_t wtok_cap = 0;
  int32_t *d_waoff = nullptr, *d_waseg = nullptr, *d_wasnap = nullptr;
  int8_t *d_wakind = nullptr;
  int64_t wanc_cap = 0;
  int64_t *d_hits = nullptr, *d_lids = nullptr;
  int32_t *d_lslots = nullptr;
  int64_t wout_cap = 0;
  // pre-match
  int32_t *d_pm_meta = nullptr, *d_pm_chain = nullptr;
  int64_t pm_cap = 0;
  // protection scratch
  int64_t *d_prot_ids = nullptr;
  int64_t prot_cap = 0;
  int64_t compactions = 0;
  uint32_t *tok_spare = nullptr;  // spare token arena (compaction target)
  int64_t spare_cap = 0;
  int64_t *cmp_len = nullptr, *cmp_off = nullptr;
  int64_t cmp_cap = 0;
  // live device-time profile per phase (CUDA events on the tree stream)
  int prof_on = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  double prof_ms[8] = {};
  int64_t prof_calls[8] = {};
  int64_t launches[8] = {};  // own kernel launches per phase (always counted)
  int64_t lib_calls = 0;     // CUB primitive invocations
  // parallel wave commit scratch and device-side control
  WaveTmp wx{};
  WaveCtl *wc = nullptr, *h_wc = nullptr;
  int64_t *ds_part = nullptr;
  int sms = 0;
  int64_t wx_cap = 0, wx_lt = 0, wx_T = 0;
  int64_t par_waves = 0, seq_waves = 0, trunc_waves = 0;
  int32_t last_fallback = 0;
  // tunables (prism_tune): eviction-list prefix sizing
  int64_t list_min_tokens = 1 << 18;   // ordered commit: select >= this many tokens
  int64_t list_slack_tokens = 4096;    // parallel commit: demand + 25% + this
  int64_t sel_min_candidates = 4096;   // below this many candidates, sort them all
  int64_t use_coop = 1;                // cooperative single-kernel build / protection
  int64_t use_sample = 1;              // sample select before the materialising selection
  int64_t prebuild = 1;                // fused wave: subtree maxima + sample on the auxiliary stream
  // paged KV payload (kv.cuh), null when disabled
  struct Kv {
    KvDev k{};
    int32_t *kvx_spare = nullptr;
    int64_t kvx_cap = 0;
    int64_t *voff = nullptr, *total = nullptr, *part = nullptr;  // part: k_kv_vsum's chunk sums (1024)
    int64_t voff_cap = 0;
  } *kv = nullptr;
};

enum { PH_COMMIT = 0, PH_BUILD = 1, PH_PROTECT = 2, PH_PREMATCH = 3, PH_RELEASE = 4, PH_NOTE = 5, PH_MAINT = 6 };

namespace {
inline void prof_begin(prism_tree *t) {
  if (t->prof_on) cudaEventRecord(t->ev0, t->st);
}
inline void prof_end(prism_tree *t, int ph) {
  t->prof_calls[ph]++;
  if (!t->prof_on) return;
  cudaEventRecord(t->ev1, t->st);
  cudaEventSynchronize(t->ev1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, t->ev0, t->ev1);
  t->prof_ms[ph] += ms;
}
}  // namespace

namespace {
inline void join_aux(prism_tree *t) {
  if (t->aux_pending) {
    cudaStreamWaitEvent(t->st, t->ev_aux, 0);
    t->aux_pending = 0;
  }
}
// public entry points: join the auxiliary stream; keys left by a protection
// pass are only trusted by the build of the same fused wave
inline void api_enter(prism_tree *t) {
  join_aux(t);
  t->keys_fresh = 0;
  t->prebuilt = 0;
}

// ----------------------------------------------------------------- slot arrays
struct SlotField {
  void **ptr;
  size_t elem;
};

std::vector<SlotField> slot_fields(prism_tree *t) {
  DT &d = t->d;
  return {
      {(void **)&d.nid, 8},    {(void **)&d.par, 4},    {(void **)&d.ftok, 4},   {(void **)&d.eoff, 8},
      {(void **)&d.elen, 4},   {(void **)&d.dend, 4},   {(void **)&d.nch, 4},    {(void **)&d.ref, 4},
      {(void **)&d.last, 8},   {(void **)&d.hits, 4},   {(void **)&d.kind, 1},   {(void **)&d.seg, 4},
      {(void **)&d.prot, 1},   {(void **)&d.hasanc, 1}, {(void **)&d.akind, 1},  {(void **)&d.aseg, 4},
      {(void **)&d.aoff, 4},   {(void **)&d.snap, 12},  {(void **)&d.hslot, 4},  {(void **)&d.kver, 4},
      {(void **)&d.wmod, 4},   {(void **)&d.wchild, 4}, {(void **)&d.waitf, 4},  {(void **)&d.guard, 4},
      {(void **)&d.wchm, 8},
      {(void **)&d.kw, sizeof(Key3)}, {(void **)&d.eff, 4}, {(void **)&d.freelist, 4},
      {(void **)&d.Lk, sizeof(Key3)}, {(void **)&d.Lv, 8},
  };
}

// candidate / selection scratch, sized with the slot capacity
int alloc_scratch(prism_tree *t, int64_t S) {
  void **bufs[] = {(void **)&t->ck, (void **)&t->cv, (void **)&t->cw, (void **)&t->ck2, (void **)&t->cv2,
                   (void **)&t->cw2, (void **)&t->ks, (void **)&t->vs, (void **)&t->kt, (void **)&t->vt};
  for (void **b : bufs)
    if (*b) CK(cudaFree(*b));
  CK(dalloc(&t->kt, S));
  CK(dalloc(&t->vt, S));
  if (!t->cst) {
    CK(dalloc(&t->cst, 1));
    CK(cudaMemset(t->cst, 0, sizeof(CoopState)));
  }
  CK(dalloc(&t->ck, S));
  CK(dalloc(&t->cv, S));
  CK(dalloc(&t->cw, S));
  CK(dalloc(&t->ck2, S));
  CK(dalloc(&t->cv2, S));
  CK(dalloc(&t->cw2, S));
  CK(dalloc(&t->ks, S));
  CK(dalloc(&t->vs, S));
  if (!t->sel) {
    CK(dalloc(&t->sel, 1));
    CK(dalloc(&t->bmin, 2048));
    CK(dalloc(&t->bmax, 2048));
  }
  return PRISM_OK;
}

int alloc_slots(prism_tree *t, int32_t S) {
  for (auto &f : slot_fields(t)) {
    CK(cudaMalloc(f.ptr, f.elem * (size_t)S));
    CK(cudaMemsetAsync(*f.ptr, 0, f.elem * (size_t)S, t->st));
  }
  int rc = alloc_scratch(t, S);
  if (rc) return rc;
  t->d.S = S;
  return PRISM_OK;
}

int grow_slots(prism_tree *t, int64_t need_total) {
  join_aux(t);  // the auxiliary stream must not touch arrays being replaced
  int64_t S2 = (int64_t)t->d.S * 2;
  while (S2 < need_total) S2 *= 2;
  if (S2 > 0x7fffff00) return fail(PRISM_FATAL, "slot capacity overflow");
  const int32_t S = t->d.S;
  for (auto &f : slot_fields(t)) {
    void *np = nullptr;
    CK(cudaMalloc(&np, f.elem * (size_t)S2));
    CK(cudaMemsetAsync(np, 0, f.elem * (size_t)S2, t->st));
    CK(cudaMemcpyAsync(np, *f.ptr, f.elem * (size_t)S, cudaMemcpyDeviceToDevice, t->st));
    CK(cudaStreamSynchronize(t->st));
    CK(cudaFree(*f.ptr));
    *f.ptr = np;
  }
  int rc = alloc_scratch(t, S2);
  if (rc) return rc;
  t->d.S = (int32_t)S2;
  return PRISM_OK;
}

int pull_ctrl(prism_tree *t) {
  CK(cudaMemcpyAsync(t->hctrl, t->d.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, t->st));
  CK(cudaStreamSynchronize(t->st));
  return PRISM_OK;
}

int push_ctrl(prism_tree *t) {
  CK(cudaMemcpyAsync(t->d.ctrl, t->hctrl, sizeof(Ctrl), cudaMemcpyHostToDevice, t->st));
  return PRISM_OK;
}

int ensure_cub(prism_tree *t, size_t bytes) {
  if (bytes <= t->cub_bytes) return PRISM_OK;
  if (t->cub_tmp) CK(cudaFree(t->cub_tmp));
  t->cub_bytes = bytes + bytes / 4 + 4096;
  CK(cudaMalloc(&t->cub_tmp, t->cub_bytes));
  return PRISM_OK;
}

// sort n Key3/uint64 pairs (kin, vin) into (kout, vout) on the low `bits` bits
int sort_pairs(prism_tree *t, int64_t n, const Key3 *kin, const uint64_t *vin, Key3 *kout, uint64_t *vout,
               int bits) {
  if (n <= 0) return PRISM_OK;
  size_t bytes = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, vin, vout, (int)n, Key3Decomp{}, 0, bits, t->st));
  int rc = ensure_cub(t, bytes);
  if (rc) return rc;
  bytes = t->cub_bytes;
  CK(cub::DeviceRadixSort::SortPairs(t->cub_tmp, bytes, kin, kout, vin, vout, (int)n, Key3Decomp{}, 0, bits,
                                     t->st));
  t->lib_calls++;
  return PRISM_OK;
}

// Sort n (Key3, value) pairs into (kout, vout): when the bits that vary across
// the set fit 64, sort the order-preserving 64-bit compression of the keys
// and gather; else sort the 192-bit keys directly.  (kin/vin != kout/vout.)
int sort_compact(prism_tree *t, int64_t n, const Key3 *kin, const uint64_t *vin, Key3 *kout, uint64_t *vout,
                 int bits) {
  if (n <= 1) {
    if (n == 1) {
      CK(cudaMemcpyAsync(kout, kin, sizeof(Key3), cudaMemcpyDeviceToDevice, t->st));
      CK(cudaMemcpyAsync(vout, vin, sizeof(uint64_t), cudaMemcpyDeviceToDevice, t->st));
    }
    return PRISM_OK;
  }
  if (n <= BSORT_MAX) {  // one CTA: bitonic sort in shared memory
    static uint64_t attr = 0;
    if (prism::attr_once(attr)) {
      CK(cudaFuncSetAttribute(k_block_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BSORT_SMEM));
    }
    k_block_sort<<<1, 1024, BSORT_SMEM, t->st>>>(kin, vin, (int)n, kout, vout);
    CK(cudaGetLastError());
    t->launches[PH_BUILD] += 1;
    return PRISM_OK;
  }
  unsigned long long *dmask = (unsigned long long *)t->d_count + 4;  // d_count has 8 slots
  CK(cudaMemsetAsync(dmask, 0, 3 * sizeof(unsigned long long), t->st));
  const unsigned nb = std::min<unsigned>(blocks_for(n, SEL_TPB), 592u);
  k_key_mask<<<nb, SEL_TPB, 0, t->st>>>(kin, n, dmask);
  Key3 mask;
  CK(cudaMemcpyAsync(&mask, dmask, sizeof(Key3), cudaMemcpyDeviceToHost, t->st));
  CK(cudaStreamSynchronize(t->st));
  const int vb = __builtin_popcountll(mask.w0) + __builtin_popcountll(mask.w1) + __builtin_popcountll(mask.w2);
  t->launches[PH_BUILD] += 1;
  if (vb > 64) return sort_pairs(t, n, kin, vin, kout, vout, bits);
  uint64_t *ck64 = t->cv2, *idx = (uint64_t *)t->cw2;
  uint64_t *sk64 = (uint64_t *)t->ck2, *sidx = (uint64_t *)t->ck2 + t->d.S;  // ck2 holds 3*S words
  k_key_compress<<<blocks_for(n), TPB, 0, t->st>>>(kin, n, mask, ck64, idx);
  size_t bytes = 0;
  const int eb = std::max(vb, 1);
  CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, ck64, sk64, idx, sidx, (int)n, 0, eb, t->st));
  int rc = ensure_cub(t, bytes);
  if (rc) return rc;
  bytes = t->cub_bytes;
  CK(cub::DeviceRadixSort::SortPairs(t->cub_tmp, bytes, ck64, sk64, idx, sidx, (int)n, 0, eb, t->st));
  k_key_gather<<<blocks_for(n), TPB, 0, t->st>>>(kin, vin, sidx, n, kout, vout);
  CK(cudaGetLastError());
  t->lib_calls++;
  t->launches[PH_BUILD] += 2;
  return PRISM_OK;
}

// select_prefix (select.cuh): from the n candidates in (ck, cv, cw), the
// smallest keys whose weights sum to >= W, into (ks, vs); returns the count
int select_prefix(prism_tree *t, int64_t n, int64_t W, int64_t *nsel) {
  const SelBufs b{t->ck, t->ck2, t->ks, t->cv, t->cv2, t->vs, t->cw, t->cw2, t->sel, t->bmin, t->bmax};
  CK(sel_run(b, n, W, t->st, nsel, &t->launches[PH_BUILD], std::min<int64_t>(SEL_SMALL, t->sel_min_candidates)));
  return PRISM_OK;
}

// ------------------------------------------------------------ cooperative kernels
int coop_grid(prism_tree *t) {
  if (t->coop_grid > 0) return t->coop_grid;
  CK(cudaFuncSetAttribute(k_build_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)COOP_SMEM));
  CK(cudaFuncSetAttribute(k_protect_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)COOP_SMEM));
  int per_sm = 0, sms = 0, dev = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_build_coop, COOP_TPB, COOP_SMEM));
  int per_sm2 = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2, k_protect_coop, COOP_TPB, COOP_SMEM));
  per_sm = std::min(per_sm, per_sm2);
  if (per_sm < 1) return fail(PRISM_FATAL, "cooperative kernels do not fit one CTA per SM");
  t->coop_grid = std::min(sms * per_sm, 2048);
  return t->coop_grid;
}

// the sample-select launches (coop.cuh) ahead of the cooperative finaliser
template <class Cand>
int sample_select(prism_tree *t, Cand cand, const CoopBufs &B, int64_t W, const int64_t *dW, int64_t min_cand,
                  bool sampled_already = false, bool big_in_finaliser = false) {
  static uint64_t attr = 0;
  if (prism::attr_once(attr)) {
    CK(cudaFuncSetAttribute(k_ss_select<EvictCand>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SS_SEL_SMEM));
    CK(cudaFuncSetAttribute(k_ss_select<ProtCand>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SS_SEL_SMEM));
    CK(cudaFuncSetAttribute(k_ss_filter<EvictCand>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SS_FILTER_SMEM));
    CK(cudaFuncSetAttribute(k_ss_filter<ProtCand>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SS_FILTER_SMEM));
    CK(cudaFuncSetAttribute(k_ss_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SS_SORT_SMEM));
    CK(cudaFuncSetAttribute(k_ss_sort_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SS_BIG_SMEM));
  }
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, t->dev));
  cudaStream_t st = t->st;
  if (!sampled_already) k_ss_sample<Cand><<<SS_SAMP / SS_TPB, SS_TPB, 0, st>>>(cand, B, W, dW, min_cand);
  k_ss_select<Cand><<<SS_CL, SS_SEL_TPB, SS_SEL_SMEM, st>>>(cand, B, W, dW);
  k_ss_filter<Cand><<<3 * sms, SS_TPB, SS_FILTER_SMEM, st>>>(cand, B);  // (3 x 72 KB per SM: one wave)
  k_ss_scatter<<<2 * sms, SS_TPB, 0, st>>>(B, W, dW);
  k_ss_sort<<<SS_SORT_PER_SM * sms, SS_SORT_TPB, SS_SORT_SMEM, st>>>(B, t->d.Lk, t->d.Lv);
  if (!big_in_finaliser) k_ss_sort_big<<<sms, 512, SS_BIG_SMEM, st>>>(B, t->d.Lk, t->d.Lv);
  CK(cudaGetLastError());
  return PRISM_OK;
}

// k_propagate's persistent grid: every warp slot of the device (8 CTAs of 256 per SM)
// launch shapes (per SM) of a few full-tree / per-victim passes (build-time knobs)
#ifndef PRISM_PROP_CTAS
#define PRISM_PROP_CTAS (2048 / PROP_TPB)
#endif
#ifndef PRISM_EVICT_CTAS
#define PRISM_EVICT_CTAS 2
#endif
#ifndef PRISM_TFSCAN_CTAS
#define PRISM_TFSCAN_CTAS 4
#endif
unsigned prop_blocks(prism_tree *t) {
  if (!t->sms) cudaDeviceGetAttribute(&t->sms, cudaDevAttrMultiProcessorCount, t->dev);
  return (unsigned)(t->sms * PRISM_PROP_CTAS);
}

CoopBufs coop_bufs(prism_tree *t) {
  return CoopBufs{t->ck, t->ck2, t->ks, t->kt, t->cv, t->cv2, t->vs, t->vt, t->cw, t->cw2, t->bmin, t->bmax,
                  t->cst, t->d_prot_ids};
}

// ------------------------------------------------------------ eviction order
// Build the eviction order of the current tree, but only the prefix whose
// tokens reach W (W <= 0: the whole order).  dW (cooperative path only): W is
// read on the device instead (< 0: no list is built at all).
int build_list(prism_tree *t, int64_t W, const int64_t *dW = nullptr) {
  join_aux(t);  // the keys read the protected flags
  if (t->use_coop) {  // one cooperative kernel, no host round trip
    int grid = coop_grid(t);
    if (grid < 0) return PRISM_FATAL;
    prof_begin(t);
    // the fused wave's build may find the subtree maxima and the sample
    // already taken on the auxiliary stream (prebuild_order)
    const bool pre = t->prebuilt && dW != nullptr;
    t->prebuilt = 0;
    const int64_t S = t->d.S;
    if (!pre) {
      CK(cudaMemsetAsync(t->cst, 0, offsetof(CoopState, ts), t->st));
      // keys / subtree maxima / gather at full occupancy over the slot range
      // (each reads hw from the control block; the count lands in cst->cand)
      if (!t->keys_fresh) k_build_keys<<<blocks_for(S), TPB, 0, t->st>>>(t->d, -1, dW);
      k_propagate<<<prop_blocks(t), PROP_TPB, 0, t->st>>>(t->d, -1, dW);
    }
    t->keys_fresh = 0;  // consumed (the commit mutates the tree next)
    CoopBufs B = coop_bufs(t);
    int64_t minc = t->sel_min_candidates, small = std::min<int64_t>(SEL_SMALL, t->sel_min_candidates);
    int32_t sampled = (t->use_sample && (dW || W > 0)) ? 1 : 0;
    if (sampled) {
      int rc = sample_select(t, EvictCand{t->d}, B, W, dW, minc, pre, true);
      if (rc) return rc;
      sampled = 2;  // k_build_coop sorts the big buckets itself
    }
    void *args[] = {(void *)&t->d, (void *)&B, (void *)&W, (void *)&dW, (void *)&minc, (void *)&small,
                    (void *)&sampled};
    CK(cudaLaunchCooperativeKernel((void *)k_build_coop, grid, COOP_TPB, args, COOP_SMEM, t->st));
    t->launches[PH_BUILD] += 3 + (sampled ? 6 : 0);
    prof_end(t, PH_BUILD);
    return PRISM_OK;
  }
  t->keys_fresh = 0;
  const int32_t hw = t->hctrl->hw;
  prof_begin(t);
  CK(cudaMemsetAsync(t->d_count, 0, 2 * sizeof(int64_t), t->st));
  k_build_keys<<<blocks_for(hw), TPB, 0, t->st>>>(t->d, hw);
  k_propagate<<<prop_blocks(t), PROP_TPB, 0, t->st>>>(t->d, hw);
  k_gather<<<blocks_for(hw), TPB, 0, t->st>>>(t->d, hw, t->ck, t->cv, t->cw, t->d_count);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(t->h_small, t->d_count, sizeof(int64_t), cudaMemcpyDeviceToHost, t->st));
  CK(cudaStreamSynchronize(t->st));
  const int64_t m = t->h_small[0];
  int64_t nsel = m;
  int rc;
  if (W > 0 && m > t->sel_min_candidates) {
    if ((rc = select_prefix(t, m, W, &nsel))) return rc;
    rc = sort_compact(t, nsel, t->ks, t->vs, t->d.Lk, t->d.Lv, evict_key_bits(t->d.policy));
  } else {
    rc = sort_compact(t, m, t->ck, t->cv, t->d.Lk, t->d.Lv, evict_key_bits(t->d.policy));
  }
  if (rc) return rc;
  k_list_ready<<<1, 1, 0, t->st>>>(t->d, nsel, m);
  CK(cudaGetLastError());
  t->launches[PH_BUILD] += 4;
  prof_end(t, PH_BUILD);
  return PRISM_OK;
}

int rehash(prism_tree *t, int64_t extra) {
  join_aux(t);  // the auxiliary stream must not touch arrays being replaced
  int64_t live = t->hctrl->hlive + extra;
  const int64_t cap = (int64_t)(t->d.hmask + 1);
  const int64_t want = std::max<int64_t>(cap, next_pow2(4 * (live + 64)));  // never shrinks
  HEnt *nt = nullptr;
  CK(dalloc(&nt, want));
  CK(cudaMemsetAsync(nt, 0xFF, sizeof(HEnt) * (size_t)want, t->st));
  CK(cudaStreamSynchronize(t->st));
  CK(cudaFree(t->d.ht));
  t->d.ht = nt;
  t->d.hmask = (uint64_t)(want - 1);
  CK(cudaMemsetAsync(t->d_count, 0, sizeof(int64_t), t->st));
  const int32_t hw = t->hctrl->hw;
  k_rehash<<<blocks_for(hw), TPB, 0, t->st>>>(t->d, hw, t->d_count);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(t->h_small, t->d_count, sizeof(int64_t), cudaMemcpyDeviceToHost, t->st));
  CK(cudaStreamSynchronize(t->st));
  t->hctrl->hlive = t->h_small[0];
  t->hctrl->htomb = 0;
  return push_ctrl(t);
}

// compaction of the token arena: live edges packed into the spare arena (kept
// allocated at the same capacity, so a steady-state compaction is two kernels
// and a scan, no allocation), then the two swap
int kv_sync(prism_tree *t, const void *src, void *dst, int64_t *out);

int compact_arena(prism_tree *t, int64_t need) {
  join_aux(t);  // the auxiliary stream must not touch arrays being replaced
  if (t->kv) {  // settle the payload first: the victims' rows and the new spans move with the arena
    int64_t o2[2];
    int rc = kv_sync(t, nullptr, nullptr, o2);
    if (rc) return rc;
  }
  const int32_t hw = t->hctrl->hw;
  if (hw + 1 > t->cmp_cap) {
    if (t->cmp_len) CK(cudaFree(t->cmp_len));
    if (t->cmp_off) CK(cudaFree(t->cmp_off));
    t->cmp_cap = next_pow2(hw + 1);
    CK(dalloc(&t->cmp_len, t->cmp_cap));
    CK(dalloc(&t->cmp_off, t->cmp_cap));
  }
  int64_t *len = t->cmp_len, *off = t->cmp_off;
  k_compact_len<<<blocks_for(hw), TPB, 0, t->st>>>(t->d, hw, len);
  size_t bytes = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, len, off, (int)hw, t->st));
  int rc = ensure_cub(t, bytes);
  if (rc) return rc;
  bytes = t->cub_bytes;
  CK(cub::DeviceScan::ExclusiveSum(t->cub_tmp, bytes, len, off, (int)hw, t->st));
  int64_t h2[2];
  CK(cudaMemcpyAsync(&h2[0], off + hw - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, t->st));
  CK(cudaMemcpyAsync(&h2[1], len + hw - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, t->st));
  CK(cudaStreamSynchronize(t->st));
  const int64_t live = h2[0] + h2[1];
  int64_t cap = t->d.acap;
  while (live + need > cap / 2) cap *= 2;
  if (cap != t->d.acap || !t->tok_spare || t->spare_cap != cap) {  // (re)size the spare
    if (t->tok_spare) CK(cudaFree(t->tok_spare));
    CK(dalloc(&t->tok_spare, cap));
    t->spare_cap = cap;
  }
  uint32_t *na = t->tok_spare;
  if (t->kv) {  // the shadow rows follow the spans (before k_compact_copy moves eoff)
    auto *K = t->kv;
    if (K->kvx_cap != cap || !K->kvx_spare) {
      if (K->kvx_spare) CK(cudaFree(K->kvx_spare));
      CK(dalloc(&K->kvx_spare, cap));
    }
    k_kv_compact<<<blocks_for((int64_t)hw * 32), TPB, 0, t->st>>>(t->d, hw, off, K->k.kvx, K->kvx_spare);
    if (K->kvx_cap == cap) {
      std::swap(K->k.kvx, K->kvx_spare);
    } else {
      CK(cudaFree(K->k.kvx));
      K->k.kvx = K->kvx_spare;
      K->kvx_spare = nullptr;
      K->kvx_cap = cap;
    }
    const int64_t mark = live;  // (every span synced above: the new arena starts settled)
    CK(cudaMemcpyAsync(K->k.ctl, &mark, sizeof(int64_t), cudaMemcpyHostToDevice, t->st));
    CK(cudaStreamSynchronize(t->st));
  }
  k_compact_copy<<<blocks_for((int64_t)hw * 32), TPB, 0, t->st>>>(t->d, hw, off, na);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(t->st));
  if (cap == t->d.acap) {  // keep the old arena as the next spare
    t->tok_spare = t->d.tok;
  } else {
    CK(cudaFree(t->d.tok));
    t->tok_spare = nullptr;
    t->spare_cap = 0;
  }
  t->d.tok = na;
  t->d.acap = cap;
  t->hctrl->arena_top = live;
  t->compactions++;
  return push_ctrl(t);
}

// run the commit kernel until DONE/CAPACITY, servicing resumable stops
int run_commit(prism_tree *t, CommitArgs a) {
  static uint64_t attr_set = 0;
  if (prism::attr_once(attr_set)) {
    CK(cudaFuncSetAttribute(k_commit, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)COMMIT_SMEM));
  }
  // a rebuild that made no progress (the prefix held only entries the stopped
  // call may not evict, e.g. its own guarded path) is retried with a doubled
  // prefix, then the whole order: any prefix gives the same victims
  int64_t last_hint = -1, last_freed = -1, lastW = 0;
  int stalls = 0;
  static const bool dbg = getenv("PRISM_DEBUG_COMMIT") != nullptr;
  int nb = 0, ns = 0, na_ = 0, nh = 0;
  auto t0 = std::chrono::steady_clock::now();
  struct Rep {
    bool on;
    int *nb, *ns, *na, *nh;
    std::chrono::steady_clock::time_point t0;
    int *iters;
    ~Rep() {
      if (!on) return;
      const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      if (ms > 2.0) fprintf(stderr, "[commit] %.2f ms iters %d builds %d slots %d arena %d hash %d\n", ms, *iters, *nb, *ns, *na, *nh);
    }
  };
  int iters = 0;
  Rep rep{dbg, &nb, &ns, &na_, &nh, t0, &iters};
  for (int iter = 0; iter < 1000000; iter++) {
    iters = iter + 1;
    prof_begin(t);
    k_commit<<<1, 32, COMMIT_SMEM, t->st>>>(t->d, a);
    CK(cudaGetLastError());
    t->launches[PH_COMMIT]++;
    prof_end(t, PH_COMMIT);
    int rc = pull_ctrl(t);
    if (rc) return rc;
    a.reset = 0;
    Ctrl &c = *t->hctrl;
    if (c.fatal) return fail(PRISM_FATAL, "device commit fatal error code " + std::to_string(c.fatal));
    switch (c.status) {
      case ST_DONE:
      case ST_CAPACITY:
        return PRISM_OK;
      case ST_NEED_BUILD:
      case ST_NEED_REBUILD: {
        // a prefix of the eviction order with 4x the tokens the stopped call
        // still needs; a call that exhausts it resumes after a rebuild
        int64_t W = std::max<int64_t>(4 * c.need_hint, t->list_min_tokens);
        const bool stalled = c.status == ST_NEED_REBUILD && c.need_hint == last_hint && c.resume_freed == last_freed;
        stalls = stalled ? stalls + 1 : 0;
        if (stalls) W = stalls > 8 || lastW <= 0 ? 0 : std::max(W, 2 * lastW);
        last_hint = c.need_hint;
        last_freed = c.resume_freed;
        lastW = W;
        nb++;
        rc = build_list(t, W);
        break;
      }
      case ST_NEED_SLOTS:
        ns++;
        rc = grow_slots(t, (int64_t)c.hw + 2 + MAX_ANCH);
        break;
      case ST_NEED_ARENA: {
        na_++;
        const int64_t n = std::max<int64_t>(a.mode == 1 ? (int64_t)MAX_PATH : a.op_n, c.need_hint);
        rc = compact_arena(t, n);
        break;
      }
      case ST_NEED_HASH:
        nh++;
        rc = rehash(t, 2 + MAX_ANCH);
        break;
      default:
        return fail(PRISM_FATAL, "unexpected commit status " + std::to_string(c.status));
    }
    if (rc) return rc;
  }
  return fail(PRISM_FATAL, "commit did not converge");
}

template <class T>
cudaError_t regrow(T **p, int64_t n) {
  if (*p) cudaFree(*p);
  return dalloc(p, n);
}

int wx_ensure(prism_tree *t, int64_t B, int64_t levels, int64_t Tn) {
  WaveTmp &X = t->wx;
  if (B > t->wx_cap || !X.hit) {
    const int64_t c = std::max<int64_t>(next_pow2(B + 1), 64);
    CK(regrow(&X.hit, c));
    CK(regrow(&X.pre, c));
    CK(regrow(&X.npieces, c));
    CK(regrow(&X.p0, c));
    CK(regrow(&X.lcp_level, c));
    CK(regrow(&X.cnew, c + 1));
    CK(regrow(&X.tail, c + 1));
    CK(regrow(&X.miss, c + 1));
    CK(regrow(&X.idb, c + 1));
    CK(regrow(&X.arb, c + 1));
    CK(regrow(&X.dem, c + 1));
    CK(regrow(&X.piece_slot, c * WP_MAXP));
    CK(regrow(&X.owner, c * WP_MAXP));
    CK(regrow(&X.cut, c));
    CK(regrow(&X.pinl, c * WP_MAXP));
    CK(regrow(&X.pinp, c));
    CK(regrow(&X.pinv, c));
    if (!X.pinh) CK(dalloc(&X.pinh, 2));
    CK(cudaMemsetAsync(X.pinh, 0, 2 * sizeof(int32_t), t->st));  // (the recorded paths are gone)
    if (!X.flags) CK(dalloc(&X.flags, 1));
    if (!X.misc) CK(dalloc(&X.misc, 8));
    t->wx_cap = c;
  }
  const int64_t lt = std::max<int64_t>(next_pow2(4 * levels + 64), 1024);
  if (lt > t->wx_lt || !X.lt_key) {
    CK(regrow(&X.lt_key, lt));
    CK(regrow(&X.lt_min, lt));
    t->wx_lt = lt;
  }
  X.lt_mask = (uint64_t)(lt - 1);
  if (Tn > t->wx_T || !X.vlen) {
    const int64_t c = std::max<int64_t>(next_pow2(Tn + 1), 1024);
    CK(regrow(&X.vlen, c));
    CK(regrow(&X.F, c));
    t->wx_T = c;
  }
  return PRISM_OK;
}

template <class In, class Out>
int cub_scan(prism_tree *t, In in, Out out, int64_t n, bool inclusive) {
  size_t bytes = 0;
  if (inclusive) CK(cub::DeviceScan::InclusiveSum(nullptr, bytes, in, out, (int)n, t->st));
  else CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, (int)n, t->st));
  int rc = ensure_cub(t, bytes);
  if (rc) return rc;
  bytes = t->cub_bytes;
  if (inclusive) CK(cub::DeviceScan::InclusiveSum(t->cub_tmp, bytes, in, out, (int)n, t->st));
  else CK(cub::DeviceScan::ExclusiveSum(t->cub_tmp, bytes, in, out, (int)n, t->st));
  t->lib_calls++;
  return PRISM_OK;
}

// Parallel commit of a segment-structured wave (wave_par.cuh), driven on the
// device: plan -> scans -> plan verdict (k_wc_plan: fallback flags, capacity
// headroom, eviction demand) -> the eviction-order prefix it needs (read on
// the device) -> victim cuts + verdict (k_wp_cuts, its last CTA) -> apply -> control block
// (k_wp_sweep_c's last CTA), one stream of launches with a single host round trip at
// the end.  Returns PRISM_OK with *applied = 1 when the wave was committed,
// *applied = 0 when an exactness guard tripped (nothing was mutated; the
// caller runs the ordered commit k_commit).  Capacity maintenance and a
// prefix that fell short are handled between attempts.
// buffers of the device-driven commit for a wave of B members
int wave_par_prepare(prism_tree *t, int64_t B, int64_t levels) {
  if (!t->wc) {
    CK(dalloc(&t->wc, 1));
    CK(cudaMallocHost(&t->h_wc, sizeof(WaveCtl)));
    CK(dalloc(&t->ds_part, 2 * DS_BLOCKS));  // partition sums, partition minima
  }
  if (!t->sms) CK(cudaDeviceGetAttribute(&t->sms, cudaDevAttrMultiProcessorCount, t->dev));
  return wx_ensure(t, B, levels, t->d.S);  // eviction-stream buffers for any prefix length
}

// one attempt of the device-driven commit, enqueued on the tree stream with
// no host wait (cooperative build path); ends by copying the verdict and the
// control block to pinned host memory.  Capturable in a CUDA graph.
int wave_par_enqueue(prism_tree *t, const WaveIn &W, int64_t *hits, int32_t *leaf_slots, int64_t *leaf_ids,
                     int32_t force_full, const int32_t *abort = nullptr) {
  const int64_t B = W.B;
  cudaStream_t st = t->st;
  const int sms = t->sms;
  WaveTmp &X = t->wx;
  WaveCtl *wc = t->wc;
  int rc;
  prof_begin(t);
  k_wc_begin<<<(int)std::min<int64_t>(std::max<int64_t>((t->wx_lt + 255) / 256, 1), 4 * sms), 256, 0, st>>>(
      t->d, wc, abort, X, t->wx_lt);
  {
    const int nplan = (int)blocks_for(B * 32);  // (warp per member) + the level table (thread per level row)
    k_wp_plan_levels<<<nplan + (int)blocks_for(B * WP_PL), TPB, 0, st>>>(t->d, W, X, wc, nplan);
  }
  k_wp_hits<<<blocks_for(B * 32), TPB, 0, st>>>(t->d, W, X, wc);  // (warp per member)
  k_wp_scan3<<<1, 1024, 0, st>>>(t->d, B, X, wc, t->list_slack_tokens, force_full);  // + the plan verdict
  CK(cudaGetLastError());
  t->launches[PH_COMMIT] += 4;
  prof_end(t, PH_COMMIT);
  const int64_t *dW = &wc->W;
  if (t->use_coop) {
    if ((rc = build_list(t, 0, dW))) return rc;
  } else {  // the multi-kernel build sizes its passes on the host: one round trip for W
    CK(cudaMemcpyAsync(t->h_wc, wc, sizeof(WaveCtl), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (!t->h_wc->stop && t->h_wc->W >= 0 && (rc = build_list(t, t->h_wc->W))) return rc;
  }
  prof_begin(t);
  k_vscan_a<<<DS_BLOCKS, 256, 0, st>>>(t->d, X, t->ds_part, wc);
  k_vscan_c<<<DS_BLOCKS, 256, 0, st>>>(t->d, X, t->ds_part, wc);
  k_wp_cuts<<<blocks_for(B * 32), TPB, 0, st>>>(t->d, B, X, wc, t->ds_part);  // + the cut and conflict verdict (last CTA)
  k_wp_evict<<<PRISM_EVICT_CTAS * sms, TPB, 0, st>>>(t->d, wc);
  k_wp_alloc<<<blocks_for(B * WP_PL), TPB, 0, st>>>(t->d, W, X, wc);  // + the label-owner reset
  k_wp_create<<<blocks_for(B * 64), TPB, 0, st>>>(t->d, W, X, wc);
  k_wp_touch<<<blocks_for(B * WP_PL), TPB, 0, st>>>(t->d, W, X, wc);
  k_wp_label<<<blocks_for(B * WP_PL), TPB, 0, st>>>(t->d, W, X, wc, hits, leaf_slots, leaf_ids);
  // a CapacityError stop: the stopping member's evict call sweeps the rest of the order
  k_wp_sweep_a<<<DS_BLOCKS, 256, 0, st>>>(t->d, t->ds_part, wc);
  // + the control block after the wave, verdict and control block to the host (last CTA)
  k_wp_sweep_c<<<DS_BLOCKS, 256, 0, st>>>(t->d, B, X, t->ds_part, wc, t->h_wc, t->hctrl);
  CK(cudaGetLastError());
  t->launches[PH_COMMIT] += 10;
  return PRISM_OK;
}

// the verdict of a completed attempt (h_wc / hctrl current): *applied = 1
// committed; *again = 1 retry (maintenance done / whole order needed,
// *force_full set); neither: an exactness guard tripped (ordered commit)
int wave_par_verdict(prism_tree *t, int *applied, int *again, int32_t *force_full) {
  *applied = *again = 0;
  const WaveCtl &H = *t->h_wc;
  int rc;
  switch (H.stop) {
    case WC_OK:
      t->last_fallback = 0;
      *applied = 1;
      return PRISM_OK;
    case WC_FALLBACK:
      t->last_fallback = H.flags;
      return PRISM_OK;
    case WC_ABORT:  // the caller's stage failed; it re-runs the wave
      return PRISM_OK;
    case WC_FULL:  // the selected prefix fell short: select the whole order
      *force_full = 1;
      *again = 1;
      return PRISM_OK;
    case WC_MAINT: {  // semantics-free capacity maintenance, then the same wave again
      Ctrl &C = *t->hctrl;
      if ((int64_t)C.hw + H.ncreate + 2 > t->d.S && (rc = grow_slots(t, (int64_t)C.hw + H.ncreate + 2))) return rc;
      if (C.arena_top + H.ntail > t->d.acap && (rc = compact_arena(t, H.ntail))) return rc;
      if ((C.hlive + C.htomb + H.ncreate + 64) * 2 > (int64_t)(t->d.hmask + 1) && (rc = rehash(t, H.ncreate + 64)))
        return rc;
      if ((rc = pull_ctrl(t))) return rc;
      *again = 1;
      return PRISM_OK;
    }
    default:
      return fail(PRISM_FATAL, "unexpected wave control stop " + std::to_string(H.stop));
  }
}

// Parallel commit of a segment-structured wave (wave_par.cuh), driven on the
// device: plan -> scans -> plan verdict (k_wc_plan: fallback flags, capacity
// headroom, eviction demand) -> the eviction-order prefix it needs (read on
// the device) -> victim cuts + verdict (k_wp_cuts, its last CTA) -> apply -> control block
// (k_wp_sweep_c's last CTA), one stream of launches with a single host round trip at
// the end.  Returns PRISM_OK with *applied = 1 when the wave was committed,
// *applied = 0 when an exactness guard tripped (nothing was mutated; the
// caller runs the ordered commit k_commit).  Capacity maintenance and a
// prefix that fell short are handled between attempts.
int admit_wave_par(prism_tree *t, const WaveIn &W, int64_t levels, int64_t *hits, int32_t *leaf_slots,
                   int64_t *leaf_ids, int *applied) {
  *applied = 0;
  int32_t force_full = 0;
  for (int attempt = 0; attempt < 8; attempt++) {
    int rc = wave_par_prepare(t, W.B, levels);
    if (rc) return rc;
    if ((rc = wave_par_enqueue(t, W, hits, leaf_slots, leaf_ids, force_full))) return rc;
    CK(cudaStreamSynchronize(t->st));  // the wave's one host round trip
    prof_end(t, PH_COMMIT);
    int again = 0;
    if ((rc = wave_par_verdict(t, applied, &again, &force_full))) return rc;
    if (!again) return PRISM_OK;
  }
  return fail(PRISM_FATAL, "parallel wave commit did not converge");
}

template <class T>
int ensure_buf(T **p, int64_t &cap, int64_t need) {
  if (need <= cap && *p) return PRISM_OK;
  if (*p) CK(cudaFree(*p));
  int64_t c = std::max<int64_t>(next_pow2(std::max<int64_t>(need, 1)), 64);
  CK(dalloc(p, c));
  cap = c;
  return PRISM_OK;
}

int stage_anchors(prism_tree *t, int64_t na, const int32_t *a_off, const int8_t *a_kind,
                  const int32_t *a_seg, const int32_t *a_snap) {
  if (na > t->anc_cap || !t->d_aoff) {
    int64_t c = std::max<int64_t>(next_pow2(na), 64);
    if (t->d_aoff) {
      CK(cudaFree(t->d_aoff));
      CK(cudaFree(t->d_akind));
      CK(cudaFree(t->d_aseg));
      CK(cudaFree(t->d_asnap));
    }
    CK(dalloc(&t->d_aoff, c));
    CK(dalloc(&t->d_akind, c));
    CK(dalloc(&t->d_aseg, c));
    CK(dalloc(&t->d_asnap, 3 * c));
    t->anc_cap = c;
  }
  if (na > 0) {
    CK(cudaMemcpyAsync(t->d_aoff, a_off, sizeof(int32_t) * na, cudaMemcpyHostToDevice, t->st));
    CK(cudaMemcpyAsync(t->d_akind, a_kind, sizeof(int8_t) * na, cudaMemcpyHostToDevice, t->st));
    CK(cudaMemcpyAsync(t->d_aseg, a_seg, sizeof(int32_t) * na, cudaMemcpyHostToDevice, t->st));
    CK(cudaMemcpyAsync(t->d_asnap, a_snap, sizeof(int32_t) * 3 * na, cudaMemcpyHostToDevice, t->st));
  }
  return PRISM_OK;
}

CommitArgs one_op(prism_tree *t, int type, int64_t n, int64_t na, int64_t k) {
  CommitArgs a{};
  a.mode = 0;
  a.reset = 1;
  a.op_type = type;
  a.nops = 1;
  a.op_k = k;
  a.op_n = n;
  a.op_na = na;
  a.tok = t->d_path;
  a.a_off = t->d_aoff;
  a.a_kind = t->d_akind;
  a.a_seg = t->d_aseg;
  a.a_snap = t->d_asnap;
  a.res = t->d_res;
  return a;
}

int validate_anchors(int64_t n, int64_t na, const int32_t *a_off, const int8_t *a_kind,
                     const int32_t *a_seg) {
  for (int64_t j = 1; j < na; j++)
    if (a_off[j] < a_off[j - 1]) return fail(PRISM_INVALID, "anchor offsets must be sorted");
  if (na > 0 && a_off[na - 1] > n) return fail(PRISM_INVALID, "anchor offset beyond path length");
  for (int64_t j = 0; j < na; j++) {
    if (a_kind[j] < 0 || a_kind[j] > 2) return fail(PRISM_INVALID, "bad anchor kind");
    if (a_kind[j] == K_REUSABLE && a_seg[j] == SEG_NONE)
      return fail(PRISM_INVALID, "reusable anchor requires segment_id");
  }
  if (na > MAX_ANCH) return fail(PRISM_INVALID, "too many anchors for one insert");
  return PRISM_OK;
}

}  // namespace

// =================================================================== C ABI
extern "C" {

const char *prism_last_error(void) { return g_err.c_str(); }
void prism_set_last_error(const char *msg) { g_err = msg ? msg : ""; }

int prism_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

prism_tree *prism_tree_create(int64_t capacity_tokens, int32_t policy, int64_t protect_budget,
                              int64_t initial_slots, int64_t initial_arena_tokens, int32_t device) {
  if (capacity_tokens <= 0 || protect_budget < 0 || policy < 0 || policy > 3) {
    fail(PRISM_INVALID, "invalid CacheConfig");
    return nullptr;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    fail(PRISM_CUDA, "no CUDA device: the PRISM device tree has no CPU fallback");
    return nullptr;
  }
  prism_tree *t = new prism_tree();
  t->dev = device;
  auto bad = [&](const char *m) {
    fail(PRISM_CUDA, std::string("prism_tree_create: ") + m + ": " + cudaGetErrorString(cudaGetLastError()));
    delete t;
    return (prism_tree *)nullptr;
  };
  if (cudaSetDevice(device) != cudaSuccess) return bad("cudaSetDevice");
  if (cudaStreamCreateWithFlags(&t->st, cudaStreamNonBlocking) != cudaSuccess) return bad("stream");
  if (cudaStreamCreateWithFlags(&t->st_aux, cudaStreamNonBlocking) != cudaSuccess) return bad("stream");
  if (cudaEventCreateWithFlags(&t->ev_aux, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&t->ev_main, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&t->ev_in, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&t->ev_out, cudaEventDisableTiming) != cudaSuccess)
    return bad("events");
  int64_t S = std::max<int64_t>(initial_slots > 0 ? initial_slots : 4096, 64);
  S = std::min<int64_t>(next_pow2(S), 1ll << 30);
  t->d.policy = policy;
  t->d.capacity = capacity_tokens;
  t->protect_budget = protect_budget;
  if (alloc_slots(t, (int32_t)S)) return bad("slots");
  const int64_t H = next_pow2(4 * S);
  if (dalloc(&t->d.ht, H) != cudaSuccess) return bad("hash");
  cudaMemsetAsync(t->d.ht, 0xFF, sizeof(HEnt) * H, t->st);
  t->d.hmask = (uint64_t)(H - 1);
  t->d.acap = std::max<int64_t>(initial_arena_tokens > 0 ? initial_arena_tokens : 1 << 16, MAX_PATH * 2);
  if (dalloc(&t->d.tok, t->d.acap) != cudaSuccess) return bad("arena");
  t->d.Hcap = 8192;
  if (dalloc(&t->d.Hk, t->d.Hcap) != cudaSuccess || dalloc(&t->d.Hv, t->d.Hcap) != cudaSuccess)
    return bad("heap");
  t->d.vcap = 1 << 20;
  if (dalloc(&t->d.vlog, t->d.vcap) != cudaSuccess) return bad("vlog");
  t->d.npri = 0;
  t->d.nact = 0;
  if (dalloc(&t->d.pri, 1) != cudaSuccess || dalloc(&t->d.act, 1) != cudaSuccess) return bad("pri");
  if (dalloc(&t->d.ctrl, 1) != cudaSuccess) return bad("ctrl");
  if (cudaMallocHost((void **)&t->hctrl, sizeof(Ctrl)) != cudaSuccess) return bad("pinned");
  if (cudaMallocHost((void **)&t->h_small, 64 * sizeof(int64_t)) != cudaSuccess) return bad("pinned");
  if (cudaMallocHost((void **)&t->h_res, sizeof(OpRes)) != cudaSuccess) return bad("pinned");
  if (dalloc(&t->d_res, 1) != cudaSuccess || dalloc(&t->d_count, 8) != cudaSuccess) return bad("res");
  // root (kvcache.py:123-124): id 0, SYSTEM, empty edge
  memset(t->hctrl, 0, sizeof(Ctrl));
  t->hctrl->hw = 1;
  t->hctrl->next_id = 1;
  int32_t negi = -1;
  uint8_t sys = K_SYSTEM;
  int32_t none = SEG_NONE;
  cudaMemcpyAsync(t->d.par, &negi, sizeof(int32_t), cudaMemcpyHostToDevice, t->st);
  cudaMemcpyAsync(t->d.kind, &sys, 1, cudaMemcpyHostToDevice, t->st);
  cudaMemcpyAsync(t->d.seg, &none, sizeof(int32_t), cudaMemcpyHostToDevice, t->st);
  cudaMemcpyAsync(t->d.hslot, &negi, sizeof(int32_t), cudaMemcpyHostToDevice, t->st);
  if (push_ctrl(t) != PRISM_OK) return bad("ctrl init");
  if (cudaStreamSynchronize(t->st) != cudaSuccess) return bad("init sync");
  return t;
}

void prism_tree_destroy(prism_tree *t) {
  if (!t) return;
  cudaSetDevice(t->dev);
  cudaStreamSynchronize(t->st);
  if (t->kv) {
    void *kb[] = {t->kv->k.pool, t->kv->k.kvx, t->kv->k.stack, t->kv->k.top, t->kv->k.moved, t->kv->kvx_spare,
                  t->kv->voff, t->kv->total, t->kv->part, t->kv->k.ctl};
    for (void *p : kb)
      if (p) cudaFree(p);
    delete t->kv;
  }
  for (auto &f : slot_fields(t)) cudaFree(*f.ptr);
  if (t->tok_spare) cudaFree(t->tok_spare);
  if (t->cmp_len) cudaFree(t->cmp_len);
  if (t->cmp_off) cudaFree(t->cmp_off);
  void *bufs[] = {t->d.ht,     t->d.tok,     t->d.Hk,      t->d.Hv,     t->d.vlog,    t->d.pri,
                  t->d.act,    t->d.ctrl,    t->ck,        t->cv,       t->d_count,   t->cub_tmp,
                  t->d_path,   t->d_aoff,    t->d_akind,   t->d_aseg,   t->d_asnap,   t->d_res,
                  t->d_vis_slots, t->d_vis_ids, t->d_poff, t->d_aoffs,  t->d_wtok,    t->d_waoff,
                  t->d_waseg,  t->d_wasnap,  t->d_wakind,  t->d_hits,   t->d_lids,    t->d_lslots,
                  t->d_pm_meta, t->d_pm_chain, t->d_prot_ids, t->ck2, t->cv2, t->cw, t->cw2, t->ks,
                  t->vs,       t->sel,       t->bmin,      t->bmax,      t->kt,       t->vt,
                  t->cst};
  for (void *p : bufs)
    if (p) cudaFree(p);
  const WaveTmp &X = t->wx;
  void *wbufs[] = {X.hit, X.pre, X.npieces, X.p0, X.lcp_level, X.cnew, X.tail, X.miss, X.idb, X.arb, X.dem,
                   X.piece_slot, X.owner, X.lt_key, X.lt_min, X.flags, X.vlen, X.F, X.cut, X.misc,
                   X.pinl, X.pinp, X.pinv, X.pinh};
  for (void *p : wbufs)
    if (p) cudaFree(p);
  if (t->ev0) cudaEventDestroy(t->ev0);
  if (t->ev1) cudaEventDestroy(t->ev1);
  cudaFreeHost(t->hctrl);
  cudaFreeHost(t->h_small);
  cudaFreeHost(t->h_res);
  cudaStreamSynchronize(t->st_aux);
  cudaStreamDestroy(t->st_aux);
  cudaEventDestroy(t->ev_aux);
  cudaEventDestroy(t->ev_main);
  cudaEventDestroy(t->ev_in);
  cudaEventDestroy(t->ev_out);
  cudaStreamDestroy(t->st);
  delete t;
}

int prism_match(prism_tree *t, const uint32_t *path, int64_t n, int64_t *hit, int32_t *visited_slots,
                int64_t *visited_ids, int64_t *n_visited) {
  api_enter(t);
  if (n < 0 || n > (int64_t)INT32_MAX) return fail(PRISM_INVALID, "path length out of range");
  cudaSetDevice(t->dev);
  int rc = ensure_buf(&t->d_path, t->path_cap, n);
  if (rc) return rc;
  if (n > t->vis_cap || !t->d_vis_slots) {
    if (t->d_vis_slots) {
      CK(cudaFree(t->d_vis_slots));
      CK(cudaFree(t->d_vis_ids));
    }
    t->vis_cap = std::max<int64_t>(next_pow2(n), 64);
    CK(dalloc(&t->d_vis_slots, t->vis_cap));
    CK(dalloc(&t->d_vis_ids, t->vis_cap));
  }
  if (n) CK(cudaMemcpyAsync(t->d_path, path, sizeof(uint32_t) * n, cudaMemcpyHostToDevice, t->st));
  CommitArgs a = one_op(t, OP_MATCH, n, 0, 0);
  a.vis_slots = t->d_vis_slots;
  a.vis_ids = t->d_vis_ids;
  rc = run_commit(t, a);
  if (rc) return rc;
  CK(cudaMemcpyAsync(t->h_res, t->d_res, sizeof(OpRes), cudaMemcpyDeviceToHost, t->st));
  CK(cudaStreamSynchronize(t->st));
  *hit = t->h_res->hit;
  const int64_t nv = t->h_res->nvis;
  if (n_visited) *n_visited = nv;
  if (nv > 0 && visited_slots)
    CK(cudaMemcpyAsync(visited_slots, t->d_vis_slots, sizeof(int32_t) * nv, cudaMemcpyDeviceToHost, t->st));
  if (nv > 0 && visited_ids)
    CK(cudaMemcpyAsync(visited_ids, t->d_vis_ids, sizeof(int64_t) * nv, cudaMemcpyDeviceToHost, t->st));
  CK(cudaStreamSynchronize(t->st));
  return PRISM_OK;
}

// last-op details for the Python binding: [evicted, vbeg, vend, freed, status]
int prism_last_op(prism_tree *t, int64_t *out) {
  api_enter(t);
  out[0] = t->h_res->evicted;
  out[1] = t->h_res->vbeg;
  out[2] = t->h_res->vend;
  out[3] = t->h_res->freed;
  out[4] = t->h_res->status;
  return PRISM_OK;
}

int prism_insert(prism_tree *t, const uint32_t *path, int64_t n, int64_t na, const int32_t *a_off,
                 const int8_t *a_kind, const int32_t *a_seg, const int32_t *a_snap, int32_t *leaf_slot,
                 int64_t *leaf_id) {
  api_enter(t);
  if (n < 0 || n > (int64_t)INT32_MAX) return fail(PRISM_INVALID, "path length out of range");
  int rc = validate_anchors(n, na, a_off, a_kind, a_seg);
  if (rc) return rc;
  cudaSetDevice(t->dev);
  rc = ensure_buf(&t->d_path, t->path_cap, n);
  if (rc) return rc;
  rc = stage_anchors(t, na, a_off, a_kind, a_seg, a_snap);
  if (rc) return rc;
  if (n) CK(cudaMemcpyAsync(t->d_path, path, sizeof(uint32_t) * n, cudaMemcpyHostToDevice, t->st));
  rc = run_commit(t, one_op(t, OP_INSERT, n, na, 0));
  if (rc) return rc;
  CK(cudaMemcpyAsync(t->h_res, t->d_res, sizeof(OpRes), cudaMemcpyDeviceToHost, t->st));
  CK(cudaStreamSynchronize(t->st));
  if (t->h_res->status == ST_CAPACITY) return fail(PRISM_CAPACITY, "path cannot fit even after maximal eviction");
  *leaf_slot = t->h_res->leaf_slot;
  *leaf_id = t->h_res->leaf_id;
  return PRISM_OK;
}

int prism_release(prism_tree *t, int64_t n, const int32_t *slots, const int64_t *ids) {
  api_enter(t);
  if (n <= 0) return PRISM_OK;
  cudaSetDevice(t->dev);
  int32_t *ds = nullptr;
  int64_t *di = nullptr, *dout = nullptr;
  CK(dalloc(&ds, n));
  CK(dalloc(&di, n));
  CK(dalloc(&dout, 1));
  CK(cudaMemcpyAsync(ds, slots, sizeof(int32_t) * n, cudaMemcpyHostToDevice, t->st));
  CK(cudaMemcpyAsync(di, ids, sizeof(int64_t) * n, cudaMemcpyHostToDevice, t->st));
  k_release_seq<<<1, 32, 0, t->st>>>(t->d, n, ds, di, dout);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(t->h_small, dout, sizeof(int64_t), cudaMemcpyDeviceToHost, t->st));
  CK(cudaStreamSynchronize(t->st));
  cudaFree(ds);
  cudaFree(di);
  cudaFree(dout);
  if (t->h_small[0] >= 0) return fail(PRISM_RELEASE, "release of a path that is not currently pinned");
  return PRISM_OK;
}

int prism_release_device(prism_tree *t, int64_t n, const int32_t *slots, const int64_t *ids, void *stream) {
  api_enter(t);
  (void)ids;
  if (n <= 0) return PRISM_OK;
  cudaSetDevice(t->dev);
  cudaStream_t s = stream ? (cudaStream_t)stream : t->st;
  // (the last parallel commit's recorded root paths, when there is one)
  const WaveTmp &X = t->wx;
  k_release_par<WP_PL><<<blocks_for(n * WP_PL), TPB, 0, s>>>(t->d, n, slots, X.pinl, X.pinp, X.pinv, X.pinh);
  CK(cudaGetLastError());
  t->launches[PH_RELEASE]++;
  return PRISM_OK;
}

int prism_pin_device(prism_tree *t, int64_t n, const int32_t *slots, void *stream) {
  api_enter(t);
  if (n <= 0) return PRISM_OK;
  cudaSetDevice(t->dev);
  cudaStream_t s = stream ? (cudaStream_t)stream : t->st;
  k_pin_par<<<blocks_for(n), TPB, 0, s>>>(t->d, n, slots);
  CK(cudaGetLastError());
  t->launches[PH_RELEASE]++;
  return PRISM_OK;
}

int prism_evict(prism_tree *t, int64_t k_free, int64_t *freed) {
  api_enter(t);
  if (k_free < 0) return fail(PRISM_INVALID, "k_free must be >= 0");
  cudaSetDevice(t->dev);
  int rc = run_commit(t, one_op(t, OP_EVICT, 0, 0, k_free));
  if (rc) return rc;
  CK(cudaMemcpyAsync(t->h_res, t->d_res, sizeof(OpRes), cudaMemcpyDeviceToHost, t->st));
  CK(cudaStreamSynchronize(t->st));
  *freed = t->h_res->freed;
  return PRISM_OK;
}

// top-f reusable anchors by (-P-hat, segment, id) with the current t->d.pri
static int protect_current(prism_tree *t, int64_t *out_ids, int64_t *n_out, int32_t keys = 0) {
  int rc;
  if (t->use_coop) {  // one cooperative kernel; no host round trip unless ids are wanted
    int grid = coop_grid(t);
    if (grid < 0) return PRISM_FATAL;
    const int64_t f = t->protect_budget;
    if ((rc = ensure_buf(&t->d_prot_ids, t->prot_cap, std::max<int64_t>(f, 1)))) return rc;
    prof_begin(t);
    CK(cudaMemsetAsync(t->cst, 0, offsetof(CoopState, ts), t->st));
    CoopBufs B = coop_bufs(t);
    int64_t minc = t->sel_min_candidates, small = std::min<int64_t>(SEL_SMALL, t->sel_min_candidates);
    int64_t ff = f;
    int32_t sampled = (t->use_sample && f > 0) ? 1 : 0;
    if (sampled && f <= TF_MAX) {  // small budget: the positive-P-hat list and its top f
      int sms = 0;
      CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, t->dev));
      k_tf_scan<<<PRISM_TFSCAN_CTAS * sms, SS_TPB, 0, t->st>>>(ProtCand{t->d, keys}, B);
      // clusters of TF_CL CTAs, at most TF_FIN / f of them (the last one's merge)
      const int ncl = (int)std::max<int64_t>(1, std::min<int64_t>(2 * sms / TF_CL, TF_FIN / std::max<int64_t>(ff, 1)));
      static uint64_t attr = 0;
      if (prism::attr_once(attr))
        CK(cudaFuncSetAttribute(k_tf_local, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TF_LOCAL_SMEM));
      k_tf_local<<<ncl * TF_CL, SS_TPB, TF_LOCAL_SMEM, t->st>>>(t->d, B, ff, keys);
      CK(cudaGetLastError());
      t->launches[PH_PROTECT] += 2;
    } else if (sampled) {
      rc = sample_select(t, ProtCand{t->d, keys}, B, ff, nullptr, minc);
      if (rc) return rc;
      t->launches[PH_PROTECT] += 5;
    }
    void *args[] = {(void *)&t->d, (void *)&B, (void *)&ff, (void *)&minc, (void *)&small, (void *)&sampled,
                    (void *)&keys};
    // the fused wave (keys): after the small top-f k_protect_coop is only the rare
    // fallback (fewer than f positive-P-hat anchors); one CTA needs no whole-GPU
    // residency, so the launch does not wait for the tree stream's kernels to drain
    const int pgrid = (keys && sampled && f <= TF_MAX) ? 1 : grid;
    CK(cudaLaunchCooperativeKernel((void *)k_protect_coop, pgrid, COOP_TPB, args, COOP_SMEM, t->st));
    t->launches[PH_PROTECT] += 1;
    prof_end(t, PH_PROTECT);
    if (out_ids || n_out) {
      int64_t nf = 0;
      CK(cudaMemcpyAsync(&nf, &t->cst->prot_n, sizeof(int64_t), cudaMemcpyDeviceToHost, t->st));
      CK(cudaStreamSynchronize(t->st));
      if (out_ids && nf > 0)
        CK(cudaMemcpyAsync(out_ids, t->d_prot_ids, sizeof(int64_t) * nf, cudaMemcpyDeviceToHost, t->st));
      CK(cudaStreamSynchronize(t->st));
      if (n_out) *n_out = nf;
    }
    return PRISM_OK;
  }
  rc = pull_ctrl(t);
  if (rc) return rc;
  const int32_t hw = t->hctrl->hw;
  prof_begin(t);
  t->launches[PH_PROTECT] += 3;
  t->lib_calls += 1;
  CK(cudaMemsetAsync(t->d_count, 0, sizeof(int64_t), t->st));
  k_prot_gather<<<blocks_for(hw), TPB, 0, t->st>>>(t->d, hw, t->ck, t->cv, t->cw, t->d_count);
  k_prot_clear<<<blocks_for(hw), TPB, 0, t->st>>>(t->d, hw);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(t->h_small, t->d_count, sizeof(int64_t), cudaMemcpyDeviceToHost, t->st));
  CK(cudaStreamSynchronize(t->st));
  const int64_t m = t->h_small[0];
  const int64_t f = std::min<int64_t>(t->protect_budget, m);
  if (f > 0) {
    // top-f: select the f smallest keys, sort only those (Lk/Lv as scratch:
    // no eviction list survives across calls)
    int64_t nsel = m;
    if (m > t->sel_min_candidates) {
      if ((rc = select_prefix(t, m, f, &nsel))) return rc;
      rc = sort_compact(t, nsel, t->ks, t->vs, t->d.Lk, t->d.Lv, 64 + 32 + 40);
    } else {
      rc = sort_compact(t, m, t->ck, t->cv, t->d.Lk, t->d.Lv, 64 + 32 + 40);
    }
    if (rc) return rc;
    rc = ensure_buf(&t->d_prot_ids, t->prot_cap, f);
    if (rc) return rc;
    k_prot_set<<<blocks_for(f), TPB, 0, t->st>>>(t->d, t->d.Lv, f, t->d_prot_ids);
    CK(cudaGetLastError());
    if (out_ids)
      CK(cudaMemcpyAsync(out_ids, t->d_prot_ids, sizeof(int64_t) * f, cudaMemcpyDeviceToHost, t->st));
  }
  prof_end(t, PH_PROTECT);
  CK(cudaStreamSynchronize(t->st));
  if (n_out) *n_out = f;
  return PRISM_OK;
}

int prism_set_protection(prism_tree *t, int64_t n, const int32_t *segs, const double *vals,
                         int64_t *out_ids, int64_t *n_out) {
  api_enter(t);
  cudaSetDevice(t->dev);
  int32_t nseg = 0;
  for (int64_t i = 0; i < n; i++) {
    if (segs[i] < 0 || segs[i] == SEG_NONE) return fail(PRISM_INVALID, "segment ids must be >= 0");
    if (vals[i] != vals[i]) return fail(PRISM_INVALID, "NaN dispatch priority");
    nseg = std::max(nseg, segs[i] + 1);
  }
  std::vector<double> dense((size_t)std::max(nseg, 1), 0.0);
  for (int64_t i = 0; i < n; i++) dense[segs[i]] = vals[i];  // dict(): last write wins
  if (nseg > t->d.npri) {
    CK(cudaFree(t->d.pri));
    CK(dalloc(&t->d.pri, nseg));
  }
  if (nseg) CK(cudaMemcpyAsync(t->d.pri, dense.data(), sizeof(double) * nseg, cudaMemcpyHostToDevice, t->st));
  t->d.npri = nseg;
  return protect_current(t, out_ids, n_out);
}

// set_protection from a dense device P-hat array (the QAS round's output)
static int prism_set_protection_device_impl(prism_tree *t, const double *d_pri, int32_t nseg,
                                           int64_t *out_ids, int64_t *n_out, int32_t keys = 0) {
  cudaSetDevice(t->dev);
  if (nseg > t->d.npri) {
    CK(cudaFree(t->d.pri));
    CK(dalloc(&t->d.pri, nseg));
  }
  if (nseg) CK(cudaMemcpyAsync(t->d.pri, d_pri, sizeof(double) * nseg, cudaMemcpyDeviceToDevice, t->st));
  t->d.npri = nseg;
  return protect_current(t, out_ids, n_out, keys);
}

int prism_set_protection_device(prism_tree *t, const double *d_pri, int32_t nseg, int64_t *out_ids,
                                int64_t *n_out) {
  api_enter(t);
  return prism_set_protection_device_impl(t, d_pri, nseg, out_ids, n_out);
}

// The first launches of the next eviction-order build, on the auxiliary
// stream right after the protection pass that left the keys: subtree maxima
// and the sample of the order.  Neither needs the wave's eviction demand W
// (k_ss_select, on the tree stream, gives the whole order when W <= 0), and
// the tree stream's commit plan in the meantime only reads the tree, so the
// two overlap.  The build of the same fused wave picks them up (t->prebuilt).
static int prebuild_order(prism_tree *t) {
  static_assert(offsetof(CoopState, ts) % 8 == 0, "CoopState clear in 8-byte words");
  k_propagate<<<prop_blocks(t), PROP_TPB, 0, t->st>>>(t->d, -1, nullptr, (unsigned long long *)t->cst,
                                                     (int64_t)(offsetof(CoopState, ts) / 8));
  CoopBufs B = coop_bufs(t);
  k_ss_sample<EvictCand><<<SS_SAMP / SS_TPB, SS_TPB, 0, t->st>>>(EvictCand{t->d}, B, 1, nullptr,
                                                                   t->sel_min_candidates);
  CK(cudaGetLastError());
  t->launches[PH_BUILD] += 2;
  t->prebuilt = 1;
  return PRISM_OK;
}

// set_protection from a dense device P-hat array, on the auxiliary stream:
// ordered after the tree stream's work so far, joined by the tree stream
// before the next eviction-order build or API call (join_aux)
int prism_set_protection_device_async(prism_tree *t, const double *d_pri, int32_t nseg) {
  cudaSetDevice(t->dev);
  api_enter(t);
  CK(cudaEventRecord(t->ev_main, t->st));
  CK(cudaStreamWaitEvent(t->st_aux, t->ev_main, 0));
  std::swap(t->st, t->st_aux);
  // the pass over every node also leaves the eviction keys (cooperative path)
  const int32_t keys = t->use_coop ? 1 : 0;
  int rc = prism_set_protection_device_impl(t, d_pri, nseg, nullptr, nullptr, keys);
  if (!rc && keys && t->use_sample && t->prebuild) rc = prebuild_order(t);
  std::swap(t->st, t->st_aux);
  if (rc) return rc;
  CK(cudaEventRecord(t->ev_aux, t->st_aux));
  t->aux_pending = 1;
  t->keys_fresh = keys;
  return PRISM_OK;
}

// LRU_ACTIVE hand-off (engine.py:195-197) from dense device counters:
// active = segments with a count > 0 over the active set or the batch
int prism_note_active_device(prism_tree *t, const int32_t *d_a, const int32_t *d_nd, int32_t nseg) {
  api_enter(t);
  cudaSetDevice(t->dev);
  if (nseg > t->d.nact) {
    CK(cudaFree(t->d.act));
    CK(dalloc(&t->d.act, nseg));
  }
  t->d.nact = nseg;
  if (nseg) k_active_flags<<<blocks_for(nseg), TPB, 0, t->st>>>(t->d, d_a, d_nd, nseg);
  int rc = pull_ctrl(t);
  if (rc) return rc;
  const int32_t hw = t->hctrl->hw;
  k_note_active<<<blocks_for(hw), TPB, 0, t->st>>>(t->d, hw);
  CK(cudaGetLastError());
  return PRISM_OK;
}

void *prism_tree_stream(prism_tree *t) { return (void *)t->st; }

int prism_tree_aux_wait(prism_tree *t, void *event) {
  cudaSetDevice(t->dev);
  CK(cudaStreamWaitEvent(t->st_aux, (cudaEvent_t)event, 0));
  return PRISM_OK;
}

// the tree's part of the fused wave can be captured in a CUDA graph: the
// cooperative (host-sync-free) build and no live profile
int32_t prism_tree_graphable(prism_tree *t) { return (t->use_coop && !t->prof_on) ? 1 : 0; }

int32_t prism_tree_policy(prism_tree *t) { return t->d.policy; }

int prism_note_active(prism_tree *t, int64_t n, const int32_t *segs) {
  api_enter(t);
  cudaSetDevice(t->dev);
  int32_t nseg = 0;
  for (int64_t i = 0; i < n; i++) {
    if (segs[i] < 0 || segs[i] == SEG_NONE) return fail(PRISM_INVALID, "segment ids must be >= 0");
    nseg = std::max(nseg, segs[i] + 1);
  }
  std::vector<uint8_t> dense((size_t)std::max(nseg, 1), 0);
  for (int64_t i = 0; i < n; i++) dense[segs[i]] = 1;
  if (nseg > t->d.nact) {
    CK(cudaFree(t->d.act));
    CK(dalloc(&t->d.act, nseg));
  }
  if (nseg) CK(cudaMemcpyAsync(t->d.act, dense.data(), (size_t)nseg, cudaMemcpyHostToDevice, t->st));
  t->d.nact = nseg;
  int rc = pull_ctrl(t);
  if (rc) return rc;
  const int32_t hw = t->hctrl->hw;
  k_note_active<<<blocks_for(hw), TPB, 0, t->st>>>(t->d, hw);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(t->st));
  return PRISM_OK;
}

int prism_admit_wave_device(prism_tree *t, int64_t B, const int64_t *path_off, const uint32_t *tokens,
                            const int64_t *anc_off, const int32_t *a_off, const int8_t *a_kind,
                            const int32_t *a_seg, const int32_t *a_snap, int64_t *hits,
                            int32_t *leaf_slots, int64_t *leaf_ids, int64_t *n_admitted_host,
                            void *stream) {
  api_enter(t);
  cudaSetDevice(t->dev);
  if (B <= 0) {
    *n_admitted_host = 0;
    return PRISM_OK;
  }
  if (stream) {  // order after the caller's producers
    cudaEvent_t ev;
    CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CK(cudaEventRecord(ev, (cudaStream_t)stream));
    CK(cudaStreamWaitEvent(t->st, ev, 0));
    CK(cudaEventDestroy(ev));
  }
  if (B > t->pm_cap || !t->d_pm_meta) {
    if (t->d_pm_meta) {
      CK(cudaFree(t->d_pm_meta));
      CK(cudaFree(t->d_pm_chain));
    }
    t->pm_cap = std::max<int64_t>(next_pow2(B), 64);
    CK(dalloc(&t->d_pm_meta, 4 * t->pm_cap));
    CK(dalloc(&t->d_pm_chain, PM_MAX * t->pm_cap));
  }
  prof_begin(t);
  k_prematch<<<blocks_for(B * 32), TPB, 0, t->st>>>(t->d, B, path_off, tokens, t->d_pm_meta, t->d_pm_chain);
  CK(cudaGetLastError());
  t->launches[PH_PREMATCH]++;
  prof_end(t, PH_PREMATCH);
  CommitArgs a{};
  a.mode = 1;
  a.reset = 1;
  a.nops = (int32_t)(2 * B);
  a.poff = path_off;
  a.tok = tokens;
  a.aoffs = anc_off;
  a.a_off = a_off;
  a.a_kind = a_kind;
  a.a_seg = a_seg;
  a.a_snap = a_snap;
  a.pm_meta = t->d_pm_meta;
  a.pm_chain = t->d_pm_chain;
  a.hits = hits;
  a.leaf_slots = leaf_slots;
  a.leaf_ids = leaf_ids;
  int rc = run_commit(t, a);
  if (rc) return rc;
  *n_admitted_host = t->hctrl->n_admitted;
  if (stream) {
    cudaEvent_t ev;
    CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CK(cudaEventRecord(ev, t->st));
    CK(cudaStreamWaitEvent((cudaStream_t)stream, ev, 0));
    CK(cudaEventDestroy(ev));
  }
  return PRISM_OK;
}

int prism_admit_wave_segmented(prism_tree *t, int64_t B, const int64_t *path_off, const uint32_t *tokens,
                               const int64_t *anc_off, const int32_t *a_off, const int8_t *a_kind,
                               const int32_t *a_seg, const int32_t *a_snap, const int64_t *members,
                               const int64_t *sk_off, const int32_t *aligned, int64_t sys_len, int64_t chunk,
                               int32_t mode, int64_t *hits, int32_t *leaf_slots, int64_t *leaf_ids,
                               int64_t *n_admitted_host, void *stream) {
  cudaSetDevice(t->dev);
  if (B <= 0) {
    *n_admitted_host = 0;
    return PRISM_OK;
  }
  if (mode != 1 && chunk > 0) {
    if (stream) {
      cudaEvent_t ev;
      CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      CK(cudaEventRecord(ev, (cudaStream_t)stream));
      CK(cudaStreamWaitEvent(t->st, ev, 0));
      CK(cudaEventDestroy(ev));
    }
    if (B > t->pm_cap || !t->d_pm_meta) {
      if (t->d_pm_meta) {
        CK(cudaFree(t->d_pm_meta));
        CK(cudaFree(t->d_pm_chain));
      }
      t->pm_cap = std::max<int64_t>(next_pow2(B), 64);
      CK(dalloc(&t->d_pm_meta, 4 * t->pm_cap));
      CK(dalloc(&t->d_pm_chain, PM_MAX * t->pm_cap));
    }
    prof_begin(t);
    k_prematch<<<blocks_for(B * 32), TPB, 0, t->st>>>(t->d, B, path_off, tokens, t->d_pm_meta, t->d_pm_chain);
    CK(cudaGetLastError());
    t->launches[PH_PREMATCH]++;
    prof_end(t, PH_PREMATCH);
    WaveIn W{B, sys_len, chunk, path_off, tokens, anc_off, a_kind, a_seg, a_snap, members, sk_off, aligned,
             t->d_pm_meta, t->d_pm_chain};
    int applied = 0;
    int rc = admit_wave_par(t, W, B * WP_MAXP, hits, leaf_slots, leaf_ids, &applied);
    if (rc) return rc;
    if (applied) {
      t->par_waves++;
      if (t->h_wc->trunc) t->trunc_waves++;
      *n_admitted_host = t->h_wc->Bc;  // (< B: the wave stopped on a CapacityError)
      if (stream) {
        cudaEvent_t ev;
        CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        CK(cudaEventRecord(ev, t->st));
        CK(cudaStreamWaitEvent((cudaStream_t)stream, ev, 0));
        CK(cudaEventDestroy(ev));
      }
      return PRISM_OK;
    }
  }
  t->seq_waves++;
  return prism_admit_wave_device(t, B, path_off, tokens, anc_off, a_off, a_kind, a_seg, a_snap, hits, leaf_slots,
                                 leaf_ids, n_admitted_host, stream);
}

// ---- the fused wave's commit split for CUDA-graph capture (prism_wave_step):
// prepare (allocations, outside any capture) -> enqueue (pre-match + one
// device-driven attempt, ordered after and joined back into `stream`, no host
// wait) -> finish (after the stream completed: the verdict; a wave that did
// not commit is re-run by the regular path, which also covers maintenance).
int prism_wave_commit_prepare(prism_tree *t, int64_t B) {
  cudaSetDevice(t->dev);
  if (B > t->pm_cap || !t->d_pm_meta) {
    if (t->d_pm_meta) {
      CK(cudaFree(t->d_pm_meta));
      CK(cudaFree(t->d_pm_chain));
    }
    t->pm_cap = std::max<int64_t>(next_pow2(B), 64);
    CK(dalloc(&t->d_pm_meta, 4 * t->pm_cap));
    CK(dalloc(&t->d_pm_chain, PM_MAX * t->pm_cap));
  }
  return wave_par_prepare(t, B, B * WP_MAXP);
}

int prism_wave_commit_enqueue(prism_tree *t, int64_t B, const int64_t *path_off, const uint32_t *tokens,
                              const int64_t *anc_off, const int8_t *a_kind, const int32_t *a_seg,
                              const int32_t *a_snap, const int64_t *members, const int64_t *sk_off,
                              const int32_t *aligned, int64_t sys_len, int64_t chunk, int64_t *hits,
                              int32_t *leaf_slots, int64_t *leaf_ids, void *stream, const int32_t *abort) {
  CK(cudaEventRecord(t->ev_in, (cudaStream_t)stream));
  CK(cudaStreamWaitEvent(t->st, t->ev_in, 0));
  k_prematch<<<blocks_for(B * 32), TPB, 0, t->st>>>(t->d, B, path_off, tokens, t->d_pm_meta, t->d_pm_chain, abort);
  t->launches[PH_PREMATCH]++;
  WaveIn W{B, sys_len, chunk, path_off, tokens, anc_off, a_kind, a_seg, a_snap, members, sk_off, aligned,
           t->d_pm_meta, t->d_pm_chain};
  int rc = wave_par_enqueue(t, W, hits, leaf_slots, leaf_ids, 0, abort);
  if (rc) return rc;
  CK(cudaEventRecord(t->ev_out, t->st));
  CK(cudaStreamWaitEvent((cudaStream_t)stream, t->ev_out, 0));
  return PRISM_OK;
}

// *applied = 1: the enqueued attempt committed the wave
int prism_wave_commit_finish(prism_tree *t, int64_t B, int32_t *applied, int64_t *n_admitted) {
  int ap = 0, again = 0;
  int32_t ff = 0;
  int rc = wave_par_verdict(t, &ap, &again, &ff);
  if (rc) return rc;
  *applied = ap;
  if (ap) t->par_waves++;
  if (ap && t->h_wc->trunc) t->trunc_waves++;
  if (n_admitted) *n_admitted = ap ? t->h_wc->Bc : 0;
  (void)B;
  return PRISM_OK;
}

// fingerprint of everything a captured commit bakes in (device layout, scratch
// pointers, tunables): a graph is reused only while it is unchanged
uint64_t prism_wave_commit_key(prism_tree *t) {
  auto mixin = [](uint64_t h, const void *p, size_t n) {
    const unsigned char *c = (const unsigned char *)p;
    for (size_t i = 0; i < n; i++) h = (h ^ c[i]) * 0x100000001B3ull;
    return h;
  };
  uint64_t h = 0xCBF29CE484222325ull;
  h = mixin(h, &t->d, sizeof(DT));
  h = mixin(h, &t->wx, sizeof(WaveTmp));
  const void *ptrs[] = {t->wc, t->ds_part, t->cst, t->d_pm_meta, t->d_pm_chain, t->ck, t->ck2, t->ks, t->kt,
                        t->cv, t->cv2, t->vs, t->vt, t->cw, t->cw2, t->bmin, t->bmax, t->d_prot_ids,
                        t->hctrl, t->h_wc, t->st, t->st_aux};
  h = mixin(h, ptrs, sizeof(ptrs));
  const int64_t knobs[] = {t->wx_lt, t->list_slack_tokens, t->sel_min_candidates, t->use_coop, t->use_sample,
                           t->protect_budget, t->sms, t->prof_on};
  h = mixin(h, knobs, sizeof(knobs));
  return h;
}

// out[3]: waves committed in parallel, waves committed in order, last fallback reason flags
int prism_wave_stats(prism_tree *t, int64_t *out) {
  api_enter(t);
  out[0] = t->par_waves;
  out[1] = t->seq_waves;
  out[2] = t->last_fallback;
  out[3] = t->trunc_waves;
  return PRISM_OK;
}

int prism_admit_wave(prism_tree *t, int64_t B, const int64_t *path_off, const uint32_t *tokens,
                     const int64_t *anc_off, const int32_t *a_off, const int8_t *a_kind, const int32_t *a_seg,
                     const int32_t *a_snap, int64_t *hits, int32_t *leaf_slots, int64_t *leaf_ids,
                     int64_t *n_admitted) {
  api_enter(t);
  cudaSetDevice(t->dev);
  if (B <= 0) {
    *n_admitted = 0;
    return PRISM_OK;
  }
  for (int64_t j = 0; j < B; j++) {
    const int64_t n = path_off[j + 1] - path_off[j];
    if (n < 0 || n > (int64_t)INT32_MAX) return fail(PRISM_INVALID, "path length out of range");
    const int64_t a0 = anc_off[j], na = anc_off[j + 1] - a0;
    int rc = validate_anchors(n, na, a_off + a0, a_kind + a0, a_seg + a0);
    if (rc) return rc;
  }
  const int64_t ntok = path_off[B], nanc = anc_off[B];
  int64_t aoffs_cap = t->woff_cap;
  int rc = ensure_buf(&t->d_poff, t->woff_cap, B + 1);
  if (rc) return rc;
  rc = ensure_buf(&t->d_aoffs, aoffs_cap, B + 1);
  if (rc) return rc;
  rc = ensure_buf(&t->d_wtok, t->wtok_cap, ntok);
  if (rc) return rc;
  if (nanc > t->wanc_cap || !t->d_waoff) {
    int64_t c = std::max<int64_t>(next_pow2(std::max<int64_t>(nanc, 1)), 64);
    if (t->d_waoff) {
      CK(cudaFree(t->d_waoff));
      CK(cudaFree(t->d_wakind));
      CK(cudaFree(t->d_waseg));
      CK(cudaFree(t->d_wasnap));
    }
    CK(dalloc(&t->d_waoff, c));
    CK(dalloc(&t->d_wakind, c));
    CK(dalloc(&t->d_waseg, c));
    CK(dalloc(&t->d_wasnap, 3 * c));
    t->wanc_cap = c;
  }
  if (B > t->wout_cap || !t->d_hits) {
    if (t->d_hits) {
      CK(cudaFree(t->d_hits));
      CK(cudaFree(t->d_lids));
      CK(cudaFree(t->d_lslots));
    }
    t->wout_cap = std::max<int64_t>(next_pow2(B), 64);
    CK(dalloc(&t->d_hits, t->wout_cap));
    CK(dalloc(&t->d_lids, t->wout_cap));
    CK(dalloc(&t->d_lslots, t->wout_cap));
  }
  CK(cudaMemcpyAsync(t->d_poff, path_off, sizeof(int64_t) * (B + 1), cudaMemcpyHostToDevice, t->st));
  CK(cudaMemcpyAsync(t->d_aoffs, anc_off, sizeof(int64_t) * (B + 1), cudaMemcpyHostToDevice, t->st));
  if (ntok) CK(cudaMemcpyAsync(t->d_wtok, tokens, sizeof(uint32_t) * ntok, cudaMemcpyHostToDevice, t->st));
  if (nanc) {
    CK(cudaMemcpyAsync(t->d_waoff, a_off, sizeof(int32_t) * nanc, cudaMemcpyHostToDevice, t->st));
    CK(cudaMemcpyAsync(t->d_wakind, a_kind, sizeof(int8_t) * nanc, cudaMemcpyHostToDevice, t->st));
    CK(cudaMemcpyAsync(t->d_waseg, a_seg, sizeof(int32_t) * nanc, cudaMemcpyHostToDevice, t->st));
    CK(cudaMemcpyAsync(t->d_wasnap, a_snap, sizeof(int32_t) * 3 * nanc, cudaMemcpyHostToDevice, t->st));
  }
  int64_t nadm = 0;
  rc = prism_admit_wave_device(t, B, t->d_poff, t->d_wtok, t->d_aoffs, t->d_waoff, t->d_wakind, t->d_waseg,
                               t->d_wasnap, t->d_hits, t->d_lslots, t->d_lids, &nadm, nullptr);
  if (rc) return rc;
  *n_admitted = nadm;
  if (nadm > 0) {
    CK(cudaMemcpyAsync(hits, t->d_hits, sizeof(int64_t) * nadm, cudaMemcpyDeviceToHost, t->st));
    CK(cudaMemcpyAsync(leaf_slots, t->d_lslots, sizeof(int32_t) * nadm, cudaMemcpyDeviceToHost, t->st));
    CK(cudaMemcpyAsync(leaf_ids, t->d_lids, sizeof(int64_t) * nadm, cudaMemcpyDeviceToHost, t->st));
  }
  CK(cudaStreamSynchronize(t->st));
  return PRISM_OK;
}

int prism_stats(prism_tree *t, int64_t *out) {
  api_enter(t);
  cudaSetDevice(t->dev);
  int rc = pull_ctrl(t);
  if (rc) return rc;
  const Ctrl &c = *t->hctrl;
  out[0] = c.resident;
  out[1] = c.clock;
  out[2] = c.next_id;
  out[3] = c.hw;
  out[4] = (int64_t)c.hw - c.free_top;
  out[5] = c.arena_top;
  out[6] = c.hlive;
  out[7] = c.htomb;
  out[8] = c.vlog_count;
  out[9] = c.evict_calls;
  out[10] = c.builds;
  out[11] = t->d.S;
  out[12] = t->d.acap;
  out[13] = (int64_t)(t->d.hmask + 1);
  out[14] = c.fast_members;
  out[15] = c.slow_members;
  return PRISM_OK;
}

int prism_victims(prism_tree *t, int64_t first, int64_t count, int64_t *ids, int8_t *kinds, int32_t *segs,
                  uint32_t *first_tok, int32_t *edge_len, int64_t *edge_off) {
  api_enter(t);
  cudaSetDevice(t->dev);
  int rc = pull_ctrl(t);
  if (rc) return rc;
  if (first < 0 || first + count > t->hctrl->vlog_count || first < t->hctrl->vlog_count - t->d.vcap)
    return fail(PRISM_INVALID, "victim log range unavailable");
  std::vector<VRec> buf((size_t)std::max<int64_t>(count, 1));
  for (int64_t i = 0; i < count;) {
    const int64_t pos = (first + i) % t->d.vcap;
    const int64_t run = std::min(count - i, t->d.vcap - pos);
    CK(cudaMemcpyAsync(buf.data() + i, t->d.vlog + pos, sizeof(VRec) * run, cudaMemcpyDeviceToHost, t->st));
    i += run;
  }
  CK(cudaStreamSynchronize(t->st));
  for (int64_t i = 0; i < count; i++) {
    if (ids) ids[i] = buf[i].id;
    if (kinds) kinds[i] = buf[i].kind;
    if (segs) segs[i] = buf[i].seg;
    if (first_tok) first_tok[i] = buf[i].ftok;
    if (edge_len) edge_len[i] = buf[i].elen;
    if (edge_off) edge_off[i] = buf[i].eoff;
  }
  return PRISM_OK;
}

int prism_snapshot(prism_tree *t, int64_t cap, int64_t *hw_out, int64_t *node_id, int32_t *parent,
                   int32_t *edge_len, int8_t *kind, int32_t *seg, int32_t *ref, int64_t *last, int32_t *hits,
                   int8_t *prot, int8_t *has_anchor, uint32_t *first_tok, int8_t *anchor_kind,
                   int32_t *anchor_seg, int32_t *anchor_off, int32_t *snap, int64_t *edge_off) {
  api_enter(t);
  cudaSetDevice(t->dev);
  int rc = pull_ctrl(t);
  if (rc) return rc;
  const int64_t hw = t->hctrl->hw;
  *hw_out = hw;
  if (cap < hw) return PRISM_OK;  // caller retries with a larger buffer
  const DT &d = t->d;
#define CP(dst, src, T)                                                                            \
  if (dst) CK(cudaMemcpyAsync(dst, src, sizeof(T) * hw, cudaMemcpyDeviceToHost, t->st))
  CP(node_id, d.nid, int64_t);
  CP(parent, d.par, int32_t);
  CP(edge_len, d.elen, int32_t);
  CP(kind, d.kind, int8_t);
  CP(seg, d.seg, int32_t);
  CP(ref, d.ref, int32_t);
  CP(last, d.last, int64_t);
  CP(hits, d.hits, int32_t);
  CP(prot, d.prot, int8_t);
  CP(has_anchor, d.hasanc, int8_t);
  CP(first_tok, d.ftok, uint32_t);
  CP(anchor_kind, d.akind, int8_t);
  CP(anchor_seg, d.aseg, int32_t);
  CP(anchor_off, d.aoff, int32_t);
  if (snap) CK(cudaMemcpyAsync(snap, d.snap, sizeof(int32_t) * 3 * hw, cudaMemcpyDeviceToHost, t->st));
  CP(edge_off, d.eoff, int64_t);
#undef CP
  CK(cudaStreamSynchronize(t->st));
  return PRISM_OK;
}

int prism_arena_read(prism_tree *t, int64_t off, int64_t n, uint32_t *out) {
  api_enter(t);
  cudaSetDevice(t->dev);
  if (off < 0 || n < 0 || off + n > t->d.acap) return fail(PRISM_INVALID, "arena range");
  if (n) CK(cudaMemcpyAsync(out, t->d.tok + off, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost, t->st));
  CK(cudaStreamSynchronize(t->st));
  return PRISM_OK;
}

int prism_evict_key(prism_tree *t, int32_t slot, uint64_t *key3) {
  api_enter(t);
  cudaSetDevice(t->dev);
  Key3 *dk = nullptr;
  CK(dalloc(&dk, 1));
  k_key_of<<<1, 32, 0, t->st>>>(t->d, slot, dk);
  CK(cudaMemcpyAsync(key3, dk, sizeof(Key3), cudaMemcpyDeviceToHost, t->st));
  CK(cudaStreamSynchronize(t->st));
  cudaFree(dk);
  return PRISM_OK;
}

int64_t prism_compactions(prism_tree *t) { return t->compactions; }

// phase timeline of the last cooperative list build: out[0..n) %globaltimer
// ns stamps (start, after each selection round, after the chunk sort, after
// each merge round, end); out[38] = 1 if the sample select produced it,
// out[39] = selected-prefix size
int prism_coop_timeline(prism_tree *t, uint64_t *out, int32_t *n) {
  api_enter(t);
  cudaSetDevice(t->dev);
  CK(cudaMemcpyAsync(out, t->cst->ts_build, 40 * sizeof(uint64_t), cudaMemcpyDeviceToHost, t->st));
  CK(cudaMemcpyAsync(n, &t->cst->nts_build, sizeof(int32_t), cudaMemcpyDeviceToHost, t->st));
  CK(cudaStreamSynchronize(t->st));
  return PRISM_OK;
}

// diagnostics: bucket offsets of the last sample select (CoopState::ss_off, up
// to cap + 1 entries); *nb = its bucket count
int prism_coop_buckets(prism_tree *t, uint32_t *off, int32_t cap, int32_t *nb) {
  api_enter(t);
  cudaSetDevice(t->dev);
  CK(cudaMemcpyAsync(nb, &t->cst->ss_nb, sizeof(int32_t), cudaMemcpyDeviceToHost, t->st));
  CK(cudaStreamSynchronize(t->st));
  const int32_t n = std::min(*nb, cap);
  if (n > 0) CK(cudaMemcpyAsync(off, t->cst->ss_off, (n + 1) * sizeof(uint32_t), cudaMemcpyDeviceToHost, t->st));
  CK(cudaStreamSynchronize(t->st));
  return PRISM_OK;
}

// diagnostics: out[4] = positive-P-hat protection candidates (tf_n), protected
// (prot_n), order candidates and the selected prefix of the last build
int prism_coop_counts(prism_tree *t, int64_t *out) {
  api_enter(t);
  cudaSetDevice(t->dev);
  CoopState *c = t->cst;
  CK(cudaMemcpyAsync(out, &c->tf_n, 8, cudaMemcpyDeviceToHost, t->st));
  CK(cudaMemcpyAsync(out + 1, &c->prot_n, 8, cudaMemcpyDeviceToHost, t->st));
  CK(cudaMemcpyAsync(out + 2, &c->ss_cand, 8, cudaMemcpyDeviceToHost, t->st));
  CK(cudaMemcpyAsync(out + 3, &c->ss_n, 8, cudaMemcpyDeviceToHost, t->st));
  CK(cudaStreamSynchronize(t->st));
  return PRISM_OK;
}

// 0: list_min_tokens, 1: list_slack_tokens, 2: sel_min_candidates (tests use
// tiny values to force partial eviction lists and their rebuild/resume path),
// 3: cooperative kernels, 4: sample select (coop.cuh) before the radix selection
int prism_tune(prism_tree *t, int32_t key, int64_t value) {
  switch (key) {
    case 0: t->list_min_tokens = std::max<int64_t>(value, 1); break;
    case 1: t->list_slack_tokens = std::max<int64_t>(value, 0); break;
    case 2: t->sel_min_candidates = std::max<int64_t>(value, 0); break;
    case 3: t->use_coop = value ? 1 : 0; break;
    case 4: t->use_sample = value ? 1 : 0; break;
    case 5: t->prebuild = value ? 1 : 0; break;
    default: return fail(PRISM_INVALID, "unknown tunable");
  }
  return PRISM_OK;
}

int prism_profile(prism_tree *t, int32_t enable) {
  cudaSetDevice(t->dev);
  if (enable && !t->ev0) {
    CK(cudaEventCreate(&t->ev0));
    CK(cudaEventCreate(&t->ev1));
  }
  t->prof_on = enable ? 1 : 0;
  return PRISM_OK;
}

// out[24]: per phase (commit, build, protect, prematch, release, note, maint, -)
// device ms [0..8), calls [8..16), own kernel launches [16..24); out[24] CUB calls;
// out[25] chain nodes, out[26] inserted tokens (SURVEY.md 8(d) byte model)
int prism_profile_read(prism_tree *t, double *out) {
  api_enter(t);
  int rc = pull_ctrl(t);
  if (rc) return rc;
  for (int i = 0; i < 8; i++) {
    out[i] = t->prof_ms[i];
    out[8 + i] = (double)t->prof_calls[i];
    out[16 + i] = (double)t->launches[i];
  }
  out[24] = (double)t->lib_calls;
  out[25] = (double)t->hctrl->chain_nodes;
  out[26] = (double)t->hctrl->inserted_tokens;
  return PRISM_OK;
}

}  // extern "C"

// ------------------------------------------------------------ paged KV payload (kv.cuh)

namespace {
__global__ void k_kv_init_stack(int32_t *stack, int64_t rows) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < rows) stack[i] = (int32_t)(rows - 1 - i);  // pops hand out rows 0, 1, 2, ...
}

// settle the payload after tree operations: rows for the arena grown since the
// last sync (new resident tokens, admission order; src: their KV, or NULL),
// the victims logged since the last sync back on the free stack (dst: their
// KV copied out in eviction order, or NULL).  out[2] = {new tokens, freed tokens}.
int kv_sync(prism_tree *t, const void *src, void *dst, int64_t *out) {
  auto *K = t->kv;
  // all on the tree's stream, sizes read on the device (no host round trip)
  const int64_t cap = t->d.vcap + 1;  // victim records of one sync at most (more: the log lost some)
  if (cap > K->voff_cap) {
    if (K->voff) CK(cudaFree(K->voff));
    K->voff_cap = next_pow2(cap);
    CK(dalloc(&K->voff, K->voff_cap));
  }
  int sms = t->sms;
  if (sms <= 0) CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, t->dev));
  if (!K->part) CK(dalloc(&K->part, 1024));
  const unsigned grid = (unsigned)(8 * sms), sgrid = (unsigned)std::min(4 * sms, 1024);
  k_kv_prep<<<1, 1, 0, t->st>>>(K->k, t->d.ctrl, t->d.vcap);
  k_kv_alloc<<<grid, TPB, 0, t->st>>>(K->k, (const uint8_t *)src);
  k_kv_vsum<<<sgrid, 1024, 0, t->st>>>(t->d.vlog, t->d.vcap, K->part, K->k);
  k_kv_vfill<<<sgrid, 1024, 0, t->st>>>(t->d.vlog, t->d.vcap, K->voff, K->part, K->k);
  k_kv_free<<<grid, TPB, 0, t->st>>>(K->k, t->d.vlog, t->d.vcap, K->voff, (uint8_t *)dst);
  k_kv_fin<<<1, 1, 0, t->st>>>(K->k, t->d.ctrl, src ? 1 : 0, dst ? 1 : 0);
  CK(cudaGetLastError());
  if (out) {  // the counts (and the error check) want the host
    int64_t c[8];
    CK(cudaMemcpyAsync(c, K->k.ctl, sizeof(c), cudaMemcpyDeviceToHost, t->st));
    CK(cudaStreamSynchronize(t->st));
    if (c[5] == 1) return fail(PRISM_CAPACITY, "KV pool exhausted (rows must cover capacity + the tokens of one sync)");
    if (c[5] == 2) return fail(PRISM_INVALID, "KV payload: more victims since the last sync than the log keeps");
    out[0] = c[6];
    out[1] = c[7];
  }
  return PRISM_OK;
}
}  // namespace

extern "C" {

int prism_kv_enable(prism_tree *t, int64_t rows, int64_t bytes_per_token) {
  api_enter(t);
  cudaSetDevice(t->dev);
  if (t->kv) return fail(PRISM_INVALID, "KV payload already enabled");
  if (rows <= 0 || rows > INT32_MAX || bytes_per_token <= 0 || bytes_per_token % 16)
    return fail(PRISM_INVALID, "KV payload: rows in (0, 2^31), bytes_per_token a positive multiple of 16");
  int rc = pull_ctrl(t);
  if (rc) return rc;
  if (t->hctrl->resident != 0) return fail(PRISM_INVALID, "KV payload: enable it on an empty tree");
  auto *K = new prism_tree::Kv();
  K->k.bpt = bytes_per_token;
  K->k.rows = rows;
  if (cudaMalloc(&K->k.pool, (size_t)rows * (size_t)bytes_per_token) != cudaSuccess) {
    delete K;
    return fail(PRISM_CUDA, "KV payload: pool allocation failed");
  }
  CK(dalloc(&K->k.kvx, t->d.acap));
  K->kvx_cap = t->d.acap;
  CK(dalloc(&K->k.stack, rows));
  CK(dalloc(&K->k.top, 1));
  CK(dalloc(&K->k.moved, 4));
  CK(dalloc(&K->total, 1));
  CK(dalloc(&K->k.ctl, 8));
  k_kv_init_stack<<<blocks_for(rows), TPB, 0, t->st>>>(K->k.stack, rows);
  CK(cudaMemcpyAsync(K->k.top, &rows, sizeof(int64_t), cudaMemcpyHostToDevice, t->st));
  CK(cudaMemsetAsync(K->k.moved, 0, 4 * sizeof(int64_t), t->st));
  const int64_t marks[8] = {t->hctrl->arena_top, t->hctrl->vlog_count, 0, 0, 0, 0, 0, 0};
  CK(cudaMemcpyAsync(K->k.ctl, marks, sizeof(marks), cudaMemcpyHostToDevice, t->st));
  CK(cudaStreamSynchronize(t->st));
  t->kv = K;
  return PRISM_OK;
}

int prism_kv_sync(prism_tree *t, const void *src, void *dst, int64_t *out) {
  api_enter(t);
  cudaSetDevice(t->dev);
  if (!t->kv) return fail(PRISM_INVALID, "KV payload not enabled");
  return kv_sync(t, src, dst, out);
}

int prism_kv_gather(prism_tree *t, int64_t n, const int32_t *leaf_slots, int64_t max_len, int32_t *table,
                    void *out, int64_t *lens) {
  api_enter(t);
  cudaSetDevice(t->dev);
  if (!t->kv) return fail(PRISM_INVALID, "KV payload not enabled");
  if (n <= 0) return PRISM_OK;
  k_kv_gather<<<(unsigned)((n * 32 + TPB - 1) / TPB), TPB, 0, t->st>>>(t->d, t->kv->k, n, leaf_slots, max_len, table,
                                                                        (uint8_t *)out, lens);
  CK(cudaGetLastError());  // (asynchronous on the tree's stream)
  return PRISM_OK;
}

// out[6]: free rows, rows, rows allocated, rows freed, bytes copied in, bytes copied out
int prism_kv_stats(prism_tree *t, int64_t *out) {
  api_enter(t);
  cudaSetDevice(t->dev);
  if (!t->kv) return fail(PRISM_INVALID, "KV payload not enabled");
  int64_t m[4];
  CK(cudaMemcpyAsync(&out[0], t->kv->k.top, sizeof(int64_t), cudaMemcpyDeviceToHost, t->st));
  CK(cudaMemcpyAsync(m, t->kv->k.moved, sizeof(m), cudaMemcpyDeviceToHost, t->st));
  CK(cudaStreamSynchronize(t->st));
  out[1] = t->kv->k.rows;
  for (int i = 0; i < 4; i++) out[2 + i] = m[i];
  return PRISM_OK;
}

}  // extern "C"

#ifdef PRISM_TRACE
// diagnostics build only (pdl.cuh): this unit's kernel start stamps
extern "C" int prism_trace_dump_dart(unsigned long long *t, char *names, int cap) {
  return prism_trace_take(t, names, cap);
}
#endif
