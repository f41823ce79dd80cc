/*
 * prism.h -- C ABI of libprism.so, the B200 (sm_100a) implementation of the
 * PRISM scheduling-memory hot path: the demand-aware radix tree (DART) and
 * the query-aware scheduler (QAS).
 *
 * Plain pointers and sizes only; no torch types cross this boundary.  Every
 * entry point replaces one reference interface (paths relative to
 * /root/reference/pkg/src/prefixsim/); the Python binding a maintainer adds
 * on the reference side is shown in INTEGRATION.md.
 *
 * Conventions
 *   - Tokens are uint32 (the reference token
 *     layout tops out near 3.0e9, workload.py:21-22).
 *   - Segment ids are int32 >= 0; PRISM_SEG_NONE stands for Python None.
 *   - Node kinds: 0 SYSTEM, 1 REUSABLE, 2 PRIVATE (kvcache.py:26-29).
 *   - Policies:   0 DART, 1 LRU, 2 LRU_ACTIVE, 3 LFU (kvcache.py:19-23).
 *   - A node handle is (slot, node_id): slot indexes the device SoA, node_id
 *     is the reference's creation-order id (kvcache.py:135-138).
 *   - Every call returns a status: PRISM_OK, PRISM_CAPACITY (the reference
 *     raises CapacityError), PRISM_RELEASE (ReleaseError), PRISM_INVALID
 *     (ValueError), PRISM_CUDA / PRISM_FATAL (device failure); the message is
 *     available from prism_last_error().
 *   - Per-call entry points take HOST buffers and are synchronous (the
 *     reference consumes each result immediately, engine.py:203-213).  The
 *     *_device variants take DEVICE buffers and a cudaStream_t (as void*).
 *   - There is no CPU fallback: without a CUDA device prism_tree_create fails.
 */
#ifndef PRISM_H
#define PRISM_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PRISM_OK 0
#define PRISM_CAPACITY 1
#define PRISM_RELEASE 2
#define PRISM_INVALID 3
#define PRISM_CUDA 4
#define PRISM_FATAL 5
#define PRISM_SIMULATION 6 /* engine.py SimulationError (no progress / path over capacity) */

#define PRISM_SEG_NONE ((int32_t)0x80000000)

typedef struct prism_tree prism_tree;

const char *prism_last_error(void);
void prism_set_last_error(const char *msg);
int prism_device_count(void);

/* RadixCache.__init__(CacheConfig) -- kvcache.py:120-131, CacheConfig kvcache.py:66-76.
 * initial_slots / initial_arena_tokens are allocation hints (0 = default);
 * all device arrays grow on demand.  device = CUDA ordinal. */
prism_tree *prism_tree_create(int64_t capacity_tokens, int32_t policy, int64_t protect_budget,
                              int64_t initial_slots, int64_t initial_arena_tokens, int32_t device);
void prism_tree_destroy(prism_tree *t);

/* RadixCache.match_prefix -- kvcache.py:146-171.
 * visited_slots / visited_ids (capacity n) may be NULL. */
int prism_match(prism_tree *t, const uint32_t *path, int64_t n, int64_t *hit,
                int32_t *visited_slots, int64_t *visited_ids, int64_t *n_visited);

/* RadixCache.insert_path -- kvcache.py:190-241 (incl. _reserve 243-273 and
 * its evict).  Anchors as parallel arrays (Anchor, kvcache.py:56-63):
 * a_off[na], a_kind[na], a_seg[na], a_snap[3*na]. */
int prism_insert(prism_tree *t, const uint32_t *path, int64_t n, int64_t na, const int32_t *a_off,
                 const int8_t *a_kind, const int32_t *a_seg, const int32_t *a_snap,
                 int32_t *leaf_slot, int64_t *leaf_id);

/* RadixCache.release_path -- kvcache.py:350-360, for n leaves in order. */
int prism_release(prism_tree *t, int64_t n, const int32_t *slots, const int64_t *ids);

/* RadixCache.evict -- kvcache.py:425-460. */
int prism_evict(prism_tree *t, int64_t k_free, int64_t *freed);

/* RadixCache.set_protection -- kvcache.py:364-383.  The dispatch priority
 * map (scheduler.py:247-251) as (segs[n], vals[n]); out_ids receives at most
 * protect_budget protected node ids, *n_out their count. */
int prism_set_protection(prism_tree *t, int64_t n, const int32_t *segs, const double *vals,
                         int64_t *out_ids, int64_t *n_out);

/* RadixCache.note_active_segments -- kvcache.py:385-393. */
int prism_note_active(prism_tree *t, int64_t n, const int32_t *segs);

/* The engine's admission loop for one wave -- engine.py:200-213: for each
 * member in order, match_prefix then insert_path; stops at the first
 * CapacityError.  Paths as CSR (path_off[B+1], tokens), anchors as CSR
 * (anc_off[B+1] into a_*).  Outputs for the admitted prefix: hits[B],
 * leaf_slots[B], leaf_ids[B]; *n_admitted.  Host buffers, synchronous. */
int prism_admit_wave(prism_tree *t, int64_t B, const int64_t *path_off, const uint32_t *tokens,
                     const int64_t *anc_off, const int32_t *a_off, const int8_t *a_kind,
                     const int32_t *a_seg, const int32_t *a_snap, int64_t *hits,
                     int32_t *leaf_slots, int64_t *leaf_ids, int64_t *n_admitted);

/* Same, with every array a DEVICE pointer; outputs written on device, the
 * admitted count to *n_admitted_host after an internal stream sync. */
int prism_admit_wave_device(prism_tree *t, int64_t B, const int64_t *path_off,
                            const uint32_t *tokens, const int64_t *anc_off, const int32_t *a_off,
                            const int8_t *a_kind, const int32_t *a_seg, const int32_t *a_snap,
                            int64_t *hits, int32_t *leaf_slots, int64_t *leaf_ids,
                            int64_t *n_admitted_host, void *stream);

/* admit_wave_device for a SEGMENT-STRUCTURED wave (every path = system prefix
 * sys_len + its aligned skeleton in chunk-token segments + a private suffix,
 * anchors at every piece boundary -- what prism_wave_step produces).  The
 * wave is committed by the exact data-parallel algorithm of wave_par.cuh;
 * if one of its exactness guards trips, by the ordered commit (mode 1 forces
 * the ordered commit).  members[B] index the pending CSR (sk_off, aligned). */
int prism_admit_wave_segmented(prism_tree *t, int64_t B, const int64_t *path_off,
                               const uint32_t *tokens, const int64_t *anc_off,
                               const int32_t *a_off, const int8_t *a_kind, const int32_t *a_seg,
                               const int32_t *a_snap, const int64_t *members,
                               const int64_t *sk_off, const int32_t *aligned, int64_t sys_len,
                               int64_t chunk, int32_t mode, int64_t *hits, int32_t *leaf_slots,
                               int64_t *leaf_ids, int64_t *n_admitted_host, void *stream);
/* out[4]: waves committed in parallel, waves committed in order, last
 * fallback reason bit-set (wave_par.cuh WPF_*), parallel waves that stopped
 * on a CapacityError (engine.py:209-212). */
int prism_wave_stats(prism_tree *t, int64_t *out);

/* Batched release of device-resident leaves (engine.py:177-181 for a whole
 * completion batch); the leaves must hold valid pins. */
int prism_release_device(prism_tree *t, int64_t n, const int32_t *slots, const int64_t *ids,
                         void *stream);
/* The inverse of prism_release_device: +1 ref along each DEVICE leaf slot's
 * root chain (an explicit lock of a cached prefix; the SGLang-style adapter's
 * inc_lock_ref).  Released with prism_release_device. */
int prism_pin_device(prism_tree *t, int64_t n, const int32_t *slots, void *stream);

/* ---------------------------------------------------------- introspection */
/* out[16]: resident_tokens, clock, next_id, slot high-water mark, live nodes,
 * arena tokens used, hash live, hash tombstones, victims logged (total),
 * evict calls, list builds, slot capacity, arena capacity, hash capacity,
 * fast-path members, slow-path members. */
int prism_stats(prism_tree *t, int64_t *out);
/* Victim records [first, first+count) of the cumulative victim log:
 * ids, kinds, segs, first_tok, edge_len, edge_off (arena offset at eviction;
 * valid until the next arena compaction). */
int prism_victims(prism_tree *t, int64_t first, int64_t count, int64_t *ids, int8_t *kinds,
                  int32_t *segs, uint32_t *first_tok, int32_t *edge_len, int64_t *edge_off);
/* Copy the slot SoA [0, hw) to host for debug_nodes (kvcache.py:473-521).
 * Arrays sized >= hw: node_id, parent slot, edge_len, kind, seg, ref, last,
 * hits, protected, has_anchor, first_tok, anchor_kind, anchor_seg, anchor_off,
 * snap (3*hw), edge_off.  *hw_out receives hw. */
int prism_snapshot(prism_tree *t, int64_t cap, int64_t *hw_out, int64_t *node_id, int32_t *parent,
                   int32_t *edge_len, int8_t *kind, int32_t *seg, int32_t *ref, int64_t *last,
                   int32_t *hits, int8_t *prot, int8_t *has_anchor, uint32_t *first_tok,
                   int8_t *anchor_kind, int32_t *anchor_seg, int32_t *anchor_off, int32_t *snap,
                   int64_t *edge_off);
/* Tokens [off, off+n) of the token arena. */
int prism_arena_read(prism_tree *t, int64_t off, int64_t n, uint32_t *out);
/* Raw evict_key (kvcache.py:397-414) of one slot as the 192-bit packed key. */
int prism_evict_key(prism_tree *t, int32_t slot, uint64_t *key3);
/* Details of the last per-call op: out[5] = evict called, victim-log begin,
 * victim-log end, tokens freed, status (what last_evicted reflects,
 * kvcache.py:435). */
int prism_last_op(prism_tree *t, int64_t *out);
/* Number of token-arena compactions so far. */
int64_t prism_compactions(prism_tree *t);
/* Sizing of the selected eviction-order prefix: key 0 = minimum tokens for
 * the ordered commit (default 2^18), 1 = slack tokens for the parallel
 * commit (4096), 2 = candidate count below which all are sorted (4096),
 * 3 = cooperative build/protection kernels (1), 4 = sample select (1),
 * 5 = fused wave: subtree maxima + sample of the order on the protection
 * stream (1).  Semantics do not depend on them (exhausted prefixes are
 * rebuilt). */
int prism_tune(prism_tree *t, int32_t key, int64_t value);
/* Phase timeline of the last cooperative eviction-list build (diagnostics):
 * out[0..*n) %globaltimer ns stamps, out[39] = selected-prefix size. */
int prism_coop_timeline(prism_tree *t, uint64_t *out, int32_t *n);
/* Live device-time profile: with enable != 0 every phase is bracketed by
 * CUDA events on the tree's stream.  prism_profile_read fills out[27]:
 * device ms per phase [0..8) (commit, list build, protection, pre-match,
 * release, note-active, maintenance), calls [8..16), own kernel launches
 * [16..24), CUB primitive calls [24], matched chain nodes [25], inserted
 * path tokens [26]. */
int prism_profile(prism_tree *t, int32_t enable);
int prism_profile_read(prism_tree *t, double *out);

/* ------------------------------------------------------------------- QAS */
typedef struct {
  int64_t dispatch_budget, cold_quota, front_width, signature_size;
  double w_g, w_a, w_n, alpha_size, beta_util;
} prism_qas_config; /* SchedulerConfig + PriorityWeights, scheduler.py:19-43 */

typedef struct prism_qas prism_qas;
prism_qas *prism_qas_create(int32_t device);
void prism_qas_destroy(prism_qas *q);

/* schedule_round -- scheduler.py:192-273 over dense segment ids [0, nseg).
 * Host buffers.  Outputs as in oracle/oracle.h oq_round. */
int prism_qas_round(prism_qas *q, int64_t P, const int64_t *ids, const double *arrival,
                    const int64_t *sk_off, const int32_t *sk, const uint8_t *reorderable,
                    int64_t A, const int64_t *act_off, const int32_t *act_sk, int32_t nseg,
                    const prism_qas_config *cfg, int64_t *hot, int64_t *nhot, int64_t *cold,
                    int64_t *ncold, int32_t *aligned, int32_t *sig, int32_t *siglen, int64_t *rank,
                    int64_t *bucket, double *bscore, int64_t *nbuckets, int32_t *g, int32_t *a,
                    int32_t *nd, double *prio, uint8_t *dom);

/* schedule_round with every input a DEVICE pointer; the outputs stay on the
 * device inside q for prism_wave_step. */
int prism_qas_round_device(prism_qas *q, int64_t P, const int64_t *ids, const double *arrival,
                           const int64_t *sk_off, const int32_t *sk, const uint8_t *reorderable,
                           int64_t A, const int64_t *act_off, const int32_t *act_sk, int32_t nseg,
                           const prism_qas_config *cfg, int64_t *nhot, int64_t *ncold,
                           int64_t *nbuckets);

/* ---------------------------------------------------- fused wave (QAS + DART) */
/* set_protection from a dense DEVICE P-hat array over [0, nseg)
 * (kvcache.py:364-383 fed by scheduler.py:247-251). out_ids may be NULL. */
int prism_set_protection_device(prism_tree *t, const double *d_pri, int32_t nseg,
                                int64_t *out_ids, int64_t *n_out);
/* The same, queued on the tree's auxiliary stream after the work queued so
 * far; the tree stream joins it before the next eviction-order build or API
 * call (used by prism_wave_step to overlap protection with serialization). */
int prism_set_protection_device_async(prism_tree *t, const double *d_pri, int32_t nseg);
/* Order the tree's auxiliary stream (the next protection pass and eviction-
 * order prebuild) after a CUDA event (cudaEvent_t as void*) -- prism_wave_step
 * gates only that stream on the previous wave's releases, which nothing on the
 * tree stream before the build reads. */
int prism_tree_aux_wait(prism_tree *t, void *event);
/* note_active_segments from dense DEVICE counters: active = a > 0 or n > 0
 * (engine.py:195-197). */
int prism_note_active_device(prism_tree *t, const int32_t *d_a, const int32_t *d_nd, int32_t nseg);
int32_t prism_tree_policy(prism_tree *t);
/* The cudaStream_t (as void*) the tree launches on (tree mutations, builds). */
void *prism_tree_stream(prism_tree *t);
/* 1 when the tree's part of the fused wave is capturable (cooperative build, no live profile). */
int32_t prism_tree_graphable(prism_tree *t);
/* The fused wave's commit split for CUDA-graph capture by prism_wave_step:
 * prepare (allocations, never inside a capture) -> enqueue (pre-match + one
 * device-driven parallel-commit attempt, ordered after and joined back into
 * `stream`, no host wait; capturable) -> finish (after `stream` completed:
 * *applied = 1 when the attempt committed the wave; otherwise the caller
 * re-runs prism_admit_wave_segmented).  key: fingerprint of everything a
 * capture bakes in (device layout, scratch pointers, tunables). */
int prism_wave_commit_prepare(prism_tree *t, int64_t B);
int prism_wave_commit_enqueue(prism_tree *t, int64_t B, const int64_t *path_off, const uint32_t *tokens,
                              const int64_t *anc_off, const int8_t *a_kind, const int32_t *a_seg,
                              const int32_t *a_snap, const int64_t *members, const int64_t *sk_off,
                              const int32_t *aligned, int64_t sys_len, int64_t chunk, int64_t *hits,
                              int32_t *leaf_slots, int64_t *leaf_ids, void *stream, const int32_t *abort);
int prism_wave_commit_finish(prism_tree *t, int64_t B, int32_t *applied, int64_t *n_admitted);
uint64_t prism_wave_commit_key(prism_tree *t);
/* The cudaStream_t (as void*) the QAS instance launches on; prism_wave_step
 * completes on it, so events recorded there bracket a whole wave. */
void *prism_qas_stream(prism_qas *q);
/* Commit used by prism_wave_step: 0 = exact parallel commit with ordered
 * fallback (default), 1 = ordered commit only (parity cross-check). */
int prism_qas_set_commit_mode(prism_qas *q, int32_t mode);
/* Rounds over <= max_p pending requests (capped at 4096) with integral weights
 * run as one launch (one CTA or a cooperative grid); 0: always the
 * multi-kernel round (parity cross-check); 1: the default cutoff. */
int prism_qas_set_small(prism_qas *q, int32_t max_p);
/* One-launch round shape: key 0 = max pending (as prism_qas_set_small),
 * 1 = CTAs of the cooperative grid (0: auto), 2 = pending requests per CTA
 * for the auto grid; key 3 writes the last round's CTA count to *out. */
int prism_qas_tune(prism_qas *q, int32_t key, int64_t value, int64_t *out);
/*   key 4: 1 (default) the fused wave's tail (protection, serialization,
 *          pre-match, commit) replayed as a CUDA graph for repeated wave
 *          shapes, 0 plain launches; key 5: out[0..1] = graph captures, replays */
/* out[4]: own kernel launches, CUB primitive calls, rounds so far, and the
 * device microseconds of those rounds when profiling is on. */
int prism_qas_counts(prism_qas *q, int64_t *out);
int prism_qas_profile(prism_qas *q, int32_t enable);
/* Phase timeline of the last profiled one-CTA round: out_ns[i] = ns from the
 * kernel's start to the end of phase i (13 phases; see qas_small.cuh). */
int prism_qas_small_timeline(prism_qas *q, int64_t *out_ns, int32_t n);
/* Copy the last round's pending demand counters g[0..nseg) (DEVICE int32) to
 * dst (DEVICE) -- the per-window counter vector the replicas all-reduce. */
int prism_qas_counters(prism_qas *q, int32_t *dst, int32_t nseg);
/* count_segments (scheduler.py:83-89) of a DEVICE pending CSR into dense G[nseg]
 * (DEVICE int32, zeroed first): a replica's per-window demand counters. */
int prism_qas_demand(prism_qas *q, int64_t P, const int64_t *sk_off, const int32_t *sk, int32_t nseg, int32_t *G);
/* Global-demand knob (multi-GPU; not in the single-instance reference): when
 * G (DEVICE int32[nseg], e.g. the all-reduce of every replica's prism_qas_demand)
 * is set, the protection hand-off of the fused wave uses
 * P-hat[r] = w_g*G[r] + w_a*a[r] + w_n*n[r] (scheduler.py:247-251 with g := G)
 * instead of the local round's.  NULL restores the reference behaviour. */
int prism_qas_set_global_demand(prism_qas *q, const int32_t *G, int32_t nseg);
/* Completions handed to the next prism_wave_step on this tree (engine.py:171-175):
 * the n pins of the DEVICE leaf slots are dropped at the start of that wave, on
 * a forked stream beside its QAS round, joined before the protection hand-off. */
int prism_qas_defer_release(prism_qas *q, int64_t n, const int32_t *slots);

/* One serving-loop wave entirely on the device (engine.py:189-213):
 * schedule_round over the DEVICE-resident pending CSR, the protection (DART)
 * or active-set (LRU_ACTIVE) hand-off, serialize_tokens of every member with
 * its aligned skeleton (token layout workload.py:136-154: system prefix
 * sys_len, chunk tokens per segment, per-request suffix length), the anchors
 * of _build_anchors (engine.py:269-292), then ordered match+insert+evict.
 * members_out[P] (dispatch order as pending indices, may be NULL), hits,
 * leaf_slots, leaf_ids are DEVICE arrays; *n_members / *n_admitted host. */
int prism_wave_step(prism_tree *t, prism_qas *q, int64_t P, const int64_t *ids,
                    const double *arrival, const int64_t *sk_off, const int32_t *sk,
                    const uint8_t *reorderable, const int32_t *suffix, int64_t A,
                    const int64_t *act_off, const int32_t *act_sk, int32_t nseg,
                    const prism_qas_config *cfg, int64_t sys_len, int64_t chunk,
                    int64_t *members_out, int64_t *hits, int32_t *leaf_slots, int64_t *leaf_ids,
                    int64_t *n_members, int64_t *n_admitted);
/* The fused wave from host memory to host memory (the e2e entry point): the
 * pending arrays may be pinned host buffers (read in place by the staging
 * kernel), release_slots (device) drops the previous wave's pins first, and
 * the dispatch order / hits are also returned in h_members / h_hits (host).
 * The active set (requests in flight, engine.py:189 active.values()) is the
 * CSR act_off[A+1] / act_sk (pinned host or device; A = 0: none). */
int prism_wave_step_host(prism_tree *t, prism_qas *q, int64_t P, const int64_t *ids, const double *arrival,
                         const int64_t *sk_off, const int32_t *sk, const uint8_t *reorderable, const int32_t *suffix,
                         int64_t A, const int64_t *act_off, const int32_t *act_sk, int32_t nseg, const prism_qas_config *cfg, int64_t sys_len, int64_t chunk,
                         int64_t release_n, const int32_t *release_slots, int64_t *members_out, int64_t *hits,
                         int32_t *leaf_slots, int64_t *leaf_ids, int64_t *h_members, int64_t *h_hits,
                         int64_t *n_members, int64_t *n_admitted);

/* ------------------------------------------------------- paged KV payload
 * north_star item (4) / SURVEY.md 8(f)3 (the reference is token-granular and
 * has no payload): every resident token owns a row of a KV
 * pool in HBM (rows x bytes_per_token, a multiple of 16), taken from a free
 * stack when the token becomes resident and returned when its node is
 * evicted.  Enable on an empty tree; rows >= capacity + the new tokens of one
 * sync.  prism_kv_sync settles the tree operations since the last sync: rows
 * for the newly resident tokens (admission order = each admitted member's
 * uncached tokens; src = their KV in that order, DEVICE, or NULL) and the
 * victims' rows back on the free stack (dst = their KV in eviction order,
 * DEVICE, or NULL), all on the tree's stream with the sizes read on the device;
 * out (may be NULL: no host wait) = {new tokens, freed tokens}, and the pool /
 * log checks.  prism_kv_gather (asynchronous on the tree's stream): per
 * leaf slot (DEVICE) the pool row of every path position into table[n, max_len]
 * (the request's req_to_token), lens[n] = path lengths, and (out != NULL) the
 * KV rows themselves into out[n, max_len, bytes_per_token] -- all DEVICE. */
int prism_kv_enable(prism_tree *t, int64_t rows, int64_t bytes_per_token);
int prism_kv_sync(prism_tree *t, const void *src, void *dst, int64_t *out);
int prism_kv_gather(prism_tree *t, int64_t n, const int32_t *leaf_slots, int64_t max_len, int32_t *table,
                    void *out, int64_t *lens);
/* out[6]: free rows, rows, rows allocated, rows freed, bytes copied in, bytes copied out */
int prism_kv_stats(prism_tree *t, int64_t *out);

/* ------------------------------------------------------- serving loop
 * engine.run_simulation (engine.py:141-266) with device-resident state: the
 * trace, the pending queue, the admission log and the per-request metrics
 * live in HBM; each wave is prism_wave_step over the gathered pending and
 * in-flight CSRs.  The trace arrays are HOST arrays in (arrival_time, id)
 * order (engine.py:158); sys_len = catalog.sys_prefix_tokens, chunk =
 * catalog.chunk_tokens (reuse_len = len(skeleton) * chunk, workload.py:296);
 * window_s / prefill_rate / decode_rate / output_tokens / decode_attenuation
 * are SchedulerConfig.window_s and SimConfig (engine.py:35-48). */
typedef struct prism_serve prism_serve;
prism_serve *prism_serve_create(prism_tree *t, prism_qas *q, int64_t n, const int64_t *ids, const double *arrival,
                                const int64_t *sk_off, const int32_t *sk, const uint8_t *reorderable,
                                const int32_t *suffix, int32_t nseg, int64_t sys_len, int64_t chunk,
                                int64_t capacity_tokens, const prism_qas_config *cfg, double window_s,
                                double prefill_rate, double decode_rate, int64_t output_tokens,
                                int32_t decode_attenuation);
void prism_serve_destroy(prism_serve *s);
/* Run up to max_waves waves (<= 0: until every request completed). */
int prism_serve_run(prism_serve *s, int64_t max_waves, int64_t *waves_run, int32_t *finished);
/* out[5]: waves, admitted, windows advanced, completed, pending */
int prism_serve_counts(prism_serve *s, int64_t *out);
/* RequestMetrics (engine.py:51-66) in trace order; any pointer may be NULL. */
int prism_serve_requests(prism_serve *s, double *admit, double *prefill_end, double *first_token,
                         double *completion, int64_t *hit, int64_t *eff);
/* WaveRecord (engine.py:69-76): members as trace indices, admission order. */
int prism_serve_waves(prism_serve *s, double *launch, double *duration, int64_t *uncached, int64_t *cached,
                      int64_t *member_off, int32_t *members);
/* Host wall time (us) of each wave (diagnostics), float[waves]. */
int prism_serve_wave_times(prism_serve *s, float *out_us);

/* ------------------------------------------------------- trace ingestion
 * workload.load_trace (workload.py:258-313) natively: a save_trace JSON-lines
 * file straight into the skeleton CSR (multi-threaded; threads <= 0: all
 * cores).  Errors: NULL + "TraceFormatError: line N: ..." as the reference. */
typedef struct prism_trace prism_trace;
prism_trace *prism_trace_load_jsonl(const char *path, int32_t threads);
/* out[6]: requests, skeleton entries, num_segments, chunk_tokens, sys_prefix_tokens, hot-set size */
int prism_trace_info(prism_trace *tr, int64_t *out);
int prism_trace_copy(prism_trace *tr, int64_t *ids, double *arrival, int64_t *sk_off, int32_t *sk,
                     uint8_t *reorderable, int32_t *suffix, int64_t *hot_set);
void prism_trace_free(prism_trace *tr);

#ifdef __cplusplus
}
#endif
#endif
