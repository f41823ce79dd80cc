/*
 * qas_oracle.c -- sequential CPU restatement of prefixsim.scheduler.schedule_round.
 *
 * TEST INFRASTRUCTURE ONLY (parity checker + CPU baseline); see oracle.h.
 *
 * Segment ids are dense in [0, nseg) (the Python wrapper remaps arbitrary
 * ids order-preservingly, so every (-pri, seg) tie-break is unchanged).
 * Float arithmetic follows the reference expression by expression with no
 * FMA contraction (built with -ffp-contract=off).  The one place the
 * reference's result depends on Python set iteration order is the utility
 * sum in bucket_score (scheduler.py:162-168); it is summed here in
 * ascending segment order, which is bit-identical whenever every partial sum
 * is exactly representable (true for the default integer-valued weights).
 */
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

/* count_segments (scheduler.py:83-89): distinct segments per request */
static void count_segments(int64_t n, const int64_t *off, const int32_t *sk, int32_t *cnt,
                           const int64_t *subset, int64_t nsub, int32_t *stamp, int32_t *gen) {
  int64_t m = subset ? nsub : n;
  for (int64_t q = 0; q < m; q++) {
    int64_t r = subset ? subset[q] : q;
    (*gen)++;
    for (int64_t j = off[r]; j < off[r + 1]; j++) {
      int32_t s = sk[j];
      if (stamp[s] != *gen) {
        stamp[s] = *gen;
        cnt[s]++;
      }
    }
  }
}

typedef struct {
  double negp;
  int32_t seg;
  int64_t idx;
} RankEnt;

static int rank_cmp(const void *x, const void *y) {
  const RankEnt *a = (const RankEnt *)x, *b = (const RankEnt *)y;
  if (a->negp != b->negp) return a->negp < b->negp ? -1 : 1;
  if (a->seg != b->seg) return a->seg < b->seg ? -1 : 1;
  return (a->idx > b->idx) - (a->idx < b->idx); /* sorted() is stable */
}

typedef struct {
  double negscore;
  int64_t order;
} BEnt;
static int bent_cmp(const void *x, const void *y) {
  const BEnt *a = (const BEnt *)x, *b = (const BEnt *)y;
  if (a->negscore != b->negscore) return a->negscore < b->negscore ? -1 : 1;
  return (a->order > b->order) - (a->order < b->order);
}

typedef struct {
  double arr;
  int64_t id, idx;
} CEnt;
static int cent_cmp(const void *x, const void *y) {
  const CEnt *a = (const CEnt *)x, *b = (const CEnt *)y;
  if (a->arr != b->arr) return a->arr < b->arr ? -1 : 1;
  return (a->id > b->id) - (a->id < b->id);
}

int oq_round(int64_t P, const int64_t *ids, const double *arrival, const int64_t *sk_off,
             const int32_t *sk, const uint8_t *reorderable, int64_t A, const int64_t *act_off,
             const int32_t *act_sk, int32_t nseg, const OQConfig *cfg, int64_t *hot, int64_t *nhot,
             int64_t *cold, int64_t *ncold, int32_t *aligned, int32_t *sig, int32_t *siglen,
             int64_t *rank, int64_t *bucket, double *bscore, int64_t *nbuckets, int32_t *g,
             int32_t *a, int32_t *nd, double *prio, uint8_t *dom) {
  if (cfg->cold_quota > cfg->dispatch_budget || cfg->signature_size < 1 ||
      cfg->front_width < cfg->signature_size)
    return OR_INVALID; /* SchedulerConfig.__post_init__ (scheduler.py:37-43) */
  const int64_t kappa = cfg->signature_size;
  int32_t *stamp = (int32_t *)calloc((size_t)nseg + 1, sizeof(int32_t));
  int32_t gen = 0;
  memset(g, 0, sizeof(int32_t) * nseg);
  memset(a, 0, sizeof(int32_t) * nseg);
  memset(nd, 0, sizeof(int32_t) * nseg);
  count_segments(P, sk_off, sk, g, NULL, 0, stamp, &gen);      /* scheduler.py:205 */
  count_segments(A, act_off, act_sk, a, NULL, 0, stamp, &gen); /* scheduler.py:206 */
  /* pri0 (scheduler.py:208-209) */
  double *pri0 = (double *)malloc(sizeof(double) * (nseg > 0 ? nseg : 1));
  for (int32_t r = 0; r < nseg; r++) {
    double x = cfg->w_g * (double)g[r];
    double y = cfg->w_a * (double)a[r];
    pri0[r] = x + y;
  }

  int64_t maxk = 0;
  for (int64_t i = 0; i < P; i++)
    if (sk_off[i + 1] - sk_off[i] > maxk) maxk = sk_off[i + 1] - sk_off[i];
  RankEnt *re = (RankEnt *)malloc(sizeof(RankEnt) * (maxk > 0 ? maxk : 1));
  uint8_t *chosen = (uint8_t *)malloc((size_t)(maxk > 0 ? maxk : 1));

  /* bucket table: signature -> bucket id, first-seen order (scheduler.py:211-223) */
  int64_t nb = 0;
  int64_t *bfirst = (int64_t *)malloc(sizeof(int64_t) * (P > 0 ? P : 1)); /* first member idx */
  int64_t *bsize = (int64_t *)calloc((size_t)(P > 0 ? P : 1), sizeof(int64_t));
  int64_t hcap = 16;
  while (hcap < 4 * (P + 1)) hcap *= 2;
  int64_t *htab = (int64_t *)malloc(sizeof(int64_t) * hcap);
  for (int64_t i = 0; i < hcap; i++) htab[i] = -1;

  for (int64_t i = 0; i < P; i++) {
    int64_t k0 = sk_off[i], k = sk_off[i + 1] - k0;
    const int32_t *s = sk + k0;
    int32_t *al = aligned + k0;
    /* front_align (scheduler.py:109-129) */
    if (!reorderable[i] || k == 0) {
      memcpy(al, s, sizeof(int32_t) * k);
    } else {
      for (int64_t j = 0; j < k; j++) {
        re[j].negp = -pri0[s[j]];
        re[j].seg = s[j];
        re[j].idx = j;
      }
      qsort(re, (size_t)k, sizeof(RankEnt), rank_cmp);
      int64_t f = cfg->front_width < k ? cfg->front_width : k;
      for (int64_t j = 0; j < k; j++) chosen[j] = 0;
      int64_t w = 0;
      for (int64_t j = 0; j < f; j++) {
        al[w++] = s[re[j].idx];
        chosen[re[j].idx] = 1;
      }
      for (int64_t j = 0; j < k; j++)
        if (!chosen[j]) al[w++] = s[j];
    }
    /* make_signature (scheduler.py:132-143) */
    int64_t sl = 0;
    if (k > 0) {
      for (int64_t j = 0; j < k; j++) {
        re[j].negp = -pri0[al[j]];
        re[j].seg = al[j];
        re[j].idx = j;
      }
      qsort(re, (size_t)k, sizeof(RankEnt), rank_cmp);
      int64_t kk = kappa < k ? kappa : k;
      for (int64_t j = 0; j < k; j++) chosen[j] = 0;
      for (int64_t j = 0; j < kk; j++) chosen[re[j].idx] = 1;
      for (int64_t j = 0; j < k; j++)
        if (chosen[j]) sig[i * kappa + sl++] = al[j];
    }
    siglen[i] = (int32_t)sl;
    /* bucket lookup by signature tuple */
    uint64_t h = 1469598103934665603ULL ^ (uint64_t)sl;
    for (int64_t j = 0; j < sl; j++) h = (h ^ (uint32_t)sig[i * kappa + j]) * 1099511628211ULL;
    int64_t slot = (int64_t)(h & (uint64_t)(hcap - 1)), b = -1;
    for (;;) {
      int64_t e = htab[slot];
      if (e < 0) break;
      int64_t f0 = bfirst[e];
      if (siglen[f0] == sl &&
          memcmp(sig + f0 * kappa, sig + i * kappa, sizeof(int32_t) * (size_t)sl) == 0) {
        b = e;
        break;
      }
      slot = (slot + 1) & (hcap - 1);
    }
    if (b < 0) {
      b = nb++;
      bfirst[b] = i;
      htab[slot] = b;
    }
    bucket[i] = b;
    rank[i] = bsize[b]++; /* rank_by_id (scheduler.py:222) */
  }

  /* bucket scores (scheduler.py:225-232, 146-171) */
  int64_t hot_cap = cfg->dispatch_budget - cfg->cold_quota;
  /* members of each bucket in pending order: counting sort by bucket */
  int64_t *bstart = (int64_t *)calloc((size_t)nb + 1, sizeof(int64_t));
  for (int64_t i = 0; i < P; i++) bstart[bucket[i] + 1]++;
  for (int64_t b = 0; b < nb; b++) bstart[b + 1] += bstart[b];
  int64_t *members = (int64_t *)malloc(sizeof(int64_t) * (P > 0 ? P : 1));
  {
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (nb > 0 ? nb : 1));
    for (int64_t b = 0; b < nb; b++) fill[b] = bstart[b];
    for (int64_t i = 0; i < P; i++) members[fill[bucket[i]]++] = i;
    free(fill);
  }
  int32_t *nb_cnt = (int32_t *)calloc((size_t)nseg + 1, sizeof(int32_t));
  uint8_t *inseg = (uint8_t *)calloc((size_t)nseg + 1, 1);
  int32_t *seglist = (int32_t *)malloc(sizeof(int32_t) * (nseg > 0 ? nseg : 1));
  for (int64_t b = 0; b < nb; b++) {
    int64_t m0 = bstart[b], msz = bstart[b + 1] - m0;
    int64_t nprov = hot_cap < msz ? (hot_cap > 0 ? hot_cap : 0) : msz;
    /* n_b = count_segments(members[:hot_cap]) */
    count_segments(0, sk_off, sk, nb_cnt, members + m0, nprov, stamp, &gen);
    int64_t ns = 0;
    for (int64_t q = 0; q < msz; q++) {
      int64_t r = members[m0 + q];
      for (int64_t j = sk_off[r]; j < sk_off[r + 1]; j++)
        if (!inseg[sk[j]]) {
          inseg[sk[j]] = 1;
          seglist[ns++] = sk[j];
        }
    }
    double util = 0.0;
    if (ns > 0) {
      /* sum in ascending segment order; see file header */
      double sum = 0.0;
      int first = 1;
      for (int64_t x = 1; x < ns; x++) { /* insertion sort: ns is small */
        int32_t v = seglist[x];
        int64_t y = x - 1;
        while (y >= 0 && seglist[y] > v) {
          seglist[y + 1] = seglist[y];
          y--;
        }
        seglist[y + 1] = v;
      }
      for (int64_t q = 0; q < ns; q++) {
        int32_t r = seglist[q];
        double t1 = cfg->w_g * (double)g[r];
        double t2 = cfg->w_a * (double)a[r];
        double t3 = cfg->w_n * (double)nb_cnt[r];
        double term = (t1 + t2) + t3;
        if (first) {
          sum = term; /* sum() starts from int 0: 0 + term == term */
          first = 0;
        } else {
          sum = sum + term;
        }
      }
      util = sum / (double)ns;
    }
    double s1 = cfg->alpha_size * (double)msz;
    double s2 = cfg->beta_util * util;
    bscore[b] = s1 + s2;
    for (int64_t q = 0; q < ns; q++) inseg[seglist[q]] = 0;
    for (int64_t q = 0; q < nprov; q++) { /* reset n_b */
      int64_t r = members[m0 + q];
      for (int64_t j = sk_off[r]; j < sk_off[r + 1]; j++) nb_cnt[sk[j]] = 0;
    }
  }

  /* hot lane (scheduler.py:234-240) */
  BEnt *be = (BEnt *)malloc(sizeof(BEnt) * (nb > 0 ? nb : 1));
  for (int64_t b = 0; b < nb; b++) {
    be[b].negscore = -bscore[b];
    be[b].order = b;
  }
  qsort(be, (size_t)nb, sizeof(BEnt), bent_cmp);
  int64_t h = 0;
  uint8_t *sel = (uint8_t *)calloc((size_t)(P > 0 ? P : 1), 1);
  for (int64_t q = 0; q < nb; q++) {
    if (h >= hot_cap) break;
    int64_t b = be[q].order, take = hot_cap - h;
    int64_t m0 = bstart[b], msz = bstart[b + 1] - m0;
    int64_t nt = take < msz ? take : msz;
    for (int64_t x = 0; x < nt; x++) {
      hot[h++] = members[m0 + x];
      sel[members[m0 + x]] = 1;
    }
  }
  *nhot = h;
  /* cold lane (scheduler.py:242-245) */
  CEnt *ce = (CEnt *)malloc(sizeof(CEnt) * (P > 0 ? P : 1));
  int64_t nl = 0;
  for (int64_t i = 0; i < P; i++)
    if (!sel[i]) {
      ce[nl].arr = arrival[i];
      ce[nl].id = ids[i];
      ce[nl].idx = i;
      nl++;
    }
  qsort(ce, (size_t)nl, sizeof(CEnt), cent_cmp);
  int64_t nc = cfg->cold_quota < nl ? cfg->cold_quota : nl;
  for (int64_t x = 0; x < nc; x++) cold[x] = ce[x].idx;
  *ncold = nc;

  /* dispatch priorities (scheduler.py:247-251) */
  count_segments(0, sk_off, sk, nd, hot, h, stamp, &gen);
  count_segments(0, sk_off, sk, nd, cold, nc, stamp, &gen);
  for (int32_t r = 0; r < nseg; r++) {
    dom[r] = (g[r] > 0 || a[r] > 0 || nd[r] > 0) ? 1 : 0;
    double x = cfg->w_n * (double)nd[r];
    prio[r] = dom[r] ? pri0[r] + x : 0.0;
  }
  *nbuckets = nb;

  free(stamp);
  free(pri0);
  free(re);
  free(chosen);
  free(bfirst);
  free(bsize);
  free(htab);
  free(bstart);
  free(members);
  free(nb_cnt);
  free(inseg);
  free(seglist);
  free(be);
  free(sel);
  free(ce);
  return OR_OK;
}
