/*
 * okt_oracle.c — plain-C restatement of the reference's Ok-Topk hot path.
 * TEST INFRASTRUCTURE ONLY (see okt_oracle.h).  Paths are relative to
 * /root/reference/proj.  Compiled with -ffp-contract=off so every double
 * operation rounds exactly as the reference's (non-FMA) build does.
 */
#include "okt_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define GAMMA 0x9e3779b97f4a7c15ULL

/* ---- rng.hpp:11-49 ------------------------------------------------------- */
uint64_t orc_splitmix64(uint64_t x) {
  x += GAMMA;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

uint64_t orc_mix64(uint64_t a, uint64_t b) {
  return orc_splitmix64(a ^ (GAMMA + b + (a << 6) + (a >> 2)));
}

static double unit_from_bits(uint64_t bits) { return (double)(bits >> 11) * 0x1.0p-53; }

/* SplitMix64::next (rng.hpp:33-39) */
static uint64_t sm_next(uint64_t* state) {
  *state += GAMMA;
  uint64_t z = *state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* tests/test_util.hpp:135-140 */
void orc_random_dense(uint64_t seed, size_t n, double* out) {
  uint64_t s = seed;
  for (size_t i = 0; i < n; ++i) out[i] = 2.0 * unit_from_bits(sm_next(&s)) - 1.0;
}

/* tests/test_util.hpp:144-153 */
void orc_random_int_dense(uint64_t seed, size_t n, int hi, double* out) {
  uint64_t s = seed;
  const uint64_t span = 2 * (uint64_t)hi + 1;
  for (size_t i = 0; i < n; ++i) out[i] = (double)((int64_t)(sm_next(&s) % span) - hi);
}

/* trainer.cpp:338-388 */
int orc_drift(int64_t t, uint64_t seed, size_t n, uint64_t rank_key, int fixed_positions, double* g) {
  if (t < 1) return -1;
  const uint64_t epoch = (uint64_t)((t - 1) / 1024);
  const double scale = pow(0.95, (double)epoch);
  if (n == 0) return 0;
  const uint64_t stream = orc_mix64(seed, orc_mix64(0x72616e6bu, rank_key));
  const uint64_t pair = (uint64_t)((t + 1) / 2);
  const double noise_sign = (t % 2 == 1) ? 1.0 : -1.0;
  const uint64_t noise_key = orc_mix64(orc_mix64(stream, 0x6e6f6973u), pair);
  for (size_t i = 0; i < n; ++i) {
    const double u = unit_from_bits(orc_mix64(noise_key, i));
    g[i] = noise_sign * 0.04 * scale * (2.0 * u - 1.0);
  }
  const uint64_t heavy_epoch = fixed_positions ? 0 : epoch;
  const uint64_t pos_key = orc_mix64(orc_mix64(seed, 0x65706f73u), heavy_epoch);
  const uint64_t mag_key = orc_mix64(orc_mix64(stream, 0x656d6167u), heavy_epoch);
  const uint64_t jit_key = orc_mix64(stream, 0x6a697474u);
  const size_t slots = n / 100 > 1 ? n / 100 : 1;
  unsigned char* taken = (unsigned char*)calloc(n, 1);
  if (!taken) return -3;
  for (size_t h = 0; h < slots; ++h) {
    size_t pos = (size_t)(orc_mix64(pos_key, h) % n);
    while (taken[pos]) pos = (pos + 1) % n;
    taken[pos] = 1;
    const uint64_t mag_bits = orc_mix64(mag_key, h);
    double mag = (1.0 + unit_from_bits(mag_bits)) * scale;
    if (!fixed_positions) {
      const double u = unit_from_bits(orc_mix64(orc_mix64(jit_key, (uint64_t)t), h));
      mag *= 1.0 + 0.08 * (2.0 * u - 1.0);
    }
    g[pos] = (mag_bits & 1u) ? mag : -mag;
  }
  free(taken);
  return 0;
}

void orc_state_init(orc_state* s) {
  memset(s, 0, sizeof(*s));
  s->tau = 64;            /* sparse.hpp:59 */
  s->tau_prime = 32;      /* sparse.hpp:60 */
  s->last_local_eval = -1;
  s->last_global_eval = -1;
  s->regions = -1;
  s->bucket_size = 4;     /* oktopk.hpp:34 */
}

/* ---- selection ----------------------------------------------------------- */
/* k-th smallest of a[0..n) (0-based kth), in place (quickselect). */
static double kth_smallest(double* a, ptrdiff_t n, ptrdiff_t kth) {
  ptrdiff_t lo = 0, hi = n - 1;
  while (lo < hi) {
    double x = a[lo], y = a[lo + (hi - lo) / 2], z = a[hi];
    double pivot = (x < y) ? ((y < z) ? y : ((x < z) ? z : x)) : ((x < z) ? x : ((y < z) ? z : y));
    ptrdiff_t i = lo, j = hi;
    while (i <= j) {
      while (a[i] < pivot) ++i;
      while (a[j] > pivot) --j;
      if (i <= j) {
        double tmp = a[i];
        a[i] = a[j];
        a[j] = tmp;
        ++i;
        --j;
      }
    }
    if (kth <= j) hi = j;
    else if (kth >= i) lo = i;
    else return a[kth];
  }
  return a[lo];
}

/* topk_from's threshold (sparse.cpp:43-71): for take = min(k, count) < count
 * the magnitude at position take-1 of the magnitude-descending order, else
 * the smallest magnitude present — in both cases the take-th largest |v|. */
double orc_kth_largest_mag(const double* v, size_t count, size_t k) {
  if (count == 0 || k == 0) return NAN;
  const size_t take = k < count ? k : count;
  double* a = (double*)malloc(count * sizeof(double));
  for (size_t i = 0; i < count; ++i) a[i] = fabs(v[i]);
  const double th = kth_smallest(a, (ptrdiff_t)count, (ptrdiff_t)(count - take));
  free(a);
  return th;
}

/* sparse.cpp:94-120 (inclusive >=) */
size_t orc_select(const double* g, size_t n, double th, uint32_t* idx, double* val) {
  size_t m = 0;
  for (size_t i = 0; i < n; ++i) {
    if (fabs(g[i]) >= th) {
      if (idx) idx[m] = (uint32_t)i;
      if (val) val[m] = g[i];
      ++m;
    }
  }
  return m;
}

static size_t select_sparse(const uint32_t* idx, const double* val, size_t nnz, double th, uint32_t* oi,
                            double* ov) {
  size_t m = 0;
  for (size_t i = 0; i < nnz; ++i)
    if (fabs(val[i]) >= th) {
      oi[m] = idx[i];
      ov[m] = val[i];
      ++m;
    }
  return m;
}

/* collectives.cpp:79-87 */
void orc_equal_slice_ends(uint64_t n, int P, uint64_t* ends) {
  const uint64_t base = n / (uint64_t)P, rem = n % (uint64_t)P;
  ends[0] = 0;
  for (int r = 0; r < P; ++r) ends[r + 1] = ends[r] + base + ((uint64_t)r < rem ? 1 : 0);
}

/* ---- sparse_sum (sparse.cpp:206-257) ---------------------------------------- */
typedef struct {
  uint32_t* idx;
  double* val;
  size_t nnz;
} part_t;

/* merge_two (sparse.cpp:206-236): union in ascending index order, a + b on ties. */
static part_t merge_two(part_t a, part_t b) {
  part_t o;
  o.idx = (uint32_t*)malloc((a.nnz + b.nnz + 1) * sizeof(uint32_t));
  o.val = (double*)malloc((a.nnz + b.nnz + 1) * sizeof(double));
  size_t i = 0, j = 0, m = 0;
  while (i < a.nnz && j < b.nnz) {
    if (a.idx[i] < b.idx[j]) {
      o.idx[m] = a.idx[i];
      o.val[m++] = a.val[i++];
    } else if (b.idx[j] < a.idx[i]) {
      o.idx[m] = b.idx[j];
      o.val[m++] = b.val[j++];
    } else {
      o.idx[m] = a.idx[i];
      o.val[m++] = a.val[i] + b.val[j];
      ++i;
      ++j;
    }
  }
  for (; i < a.nnz; ++i) {
    o.idx[m] = a.idx[i];
    o.val[m++] = a.val[i];
  }
  for (; j < b.nnz; ++j) {
    o.idx[m] = b.idx[j];
    o.val[m++] = b.val[j];
  }
  o.nnz = m;
  return o;
}

static part_t copy_part(part_t p) {
  part_t o;
  o.idx = (uint32_t*)malloc((p.nnz + 1) * sizeof(uint32_t));
  o.val = (double*)malloc((p.nnz + 1) * sizeof(double));
  memcpy(o.idx, p.idx, p.nnz * sizeof(uint32_t));
  memcpy(o.val, p.val, p.nnz * sizeof(double));
  o.nnz = p.nnz;
  return o;
}

/* stride_sum (sparse.cpp:238-245): sum(q, s) = sum(q, 2s) + sum(q+s, 2s). */
static part_t stride_sum(const part_t* parts, int P, int q, int s) {
  if (q + s >= P) return copy_part(parts[q]);
  part_t a = stride_sum(parts, P, q, 2 * s);
  part_t b = stride_sum(parts, P, q + s, 2 * s);
  part_t o = merge_two(a, b);
  free(a.idx);
  free(a.val);
  free(b.idx);
  free(b.val);
  return o;
}

size_t orc_sparse_sum(int P, const uint32_t* const* idx, const double* const* val, const size_t* nnz,
                      uint32_t* out_idx, double* out_val) {
  if (P <= 0) return 0;
  part_t parts[ORC_MAX_P];
  for (int q = 0; q < P; ++q) {
    parts[q].idx = (uint32_t*)idx[q];
    parts[q].val = (double*)val[q];
    parts[q].nnz = nnz[q];
  }
  part_t o = stride_sum(parts, P, 0, 1);
  memcpy(out_idx, o.idx, o.nnz * sizeof(uint32_t));
  memcpy(out_val, o.val, o.nnz * sizeof(double));
  const size_t m = o.nnz;
  free(o.idx);
  free(o.val);
  return m;
}

/* topk_exact (sparse.cpp:43-80): th = k-th largest magnitude; keep every
 * |g| > th and the first k - #{|g| > th} entries with |g| == th (the
 * magnitude-descending order breaks ties toward the smaller index), emitted in
 * coordinate order — the reference sorts the kept positions ascending. */
size_t orc_topk_exact(const double* g, size_t n, size_t k, uint32_t* idx, double* val) {
  if (k < 1 || k > n) return 0;
  const double th = orc_kth_largest_mag(g, n, k);
  size_t gt = 0;
  for (size_t i = 0; i < n; ++i) gt += fabs(g[i]) > th;
  size_t eq_left = k - gt, m = 0;
  for (size_t i = 0; i < n; ++i) {
    const double a = fabs(g[i]);
    int keep = a > th;
    if (!keep && a == th && eq_left) {
      keep = 1;
      --eq_left;
    }
    if (keep) {
      idx[m] = (uint32_t)i;
      val[m] = g[i];
      ++m;
    }
  }
  return m;
}

/* collectives.cpp:152-159: every rank's exact top-k, sparse_allgatherv (which
 * only moves them), sparse_sum in the stride-doubling order. */
size_t orc_topka_allreduce(int P, const double* const* g, size_t n, size_t k, uint32_t* out_idx,
                           double* out_val) {
  if (P <= 0 || P > ORC_MAX_P || k < 1 || k > n) return 0;
  uint32_t* pi[ORC_MAX_P];
  double* pv[ORC_MAX_P];
  size_t nnz[ORC_MAX_P];
  for (int q = 0; q < P; ++q) {
    pi[q] = (uint32_t*)malloc(k * sizeof(uint32_t));
    pv[q] = (double*)malloc(k * sizeof(double));
    nnz[q] = orc_topk_exact(g[q], n, k, pi[q], pv[q]);
  }
  const size_t m = orc_sparse_sum(P, (const uint32_t* const*)pi, (const double* const*)pv, nnz, out_idx, out_val);
  for (int q = 0; q < P; ++q) {
    free(pi[q]);
    free(pv[q]);
  }
  return m;
}

/* ---- ledger helpers (transport.cpp:71-93, 103-160; collectives.cpp:30-77) ---- */
static int log2i(int p) {
  int l = 0;
  while ((1 << l) < p) ++l;
  return l;
}

static void credit(orc_counters* L, int P, int r, int ph, int send, uint64_t words) {
  (void)P;
  if (!L) return;
  orc_counters* c = &L[r * ORC_PHASES + ph];
  if (send) {
    c->words_sent += words;
    c->msgs_sent += 1;
  } else {
    c->words_recv += words;
    c->msgs_recv += 1;
  }
}

/* sparse_allgatherv's recursive doubling accounting over part sizes. */
static void credit_allgatherv(orc_counters* L, int P, int ph, const uint64_t* parts) {
  const int rounds = log2i(P);
  for (int r = 0; r < P; ++r)
    for (int j = 0; j < rounds; ++j) {
      const int width = 1 << j, partner = r ^ width;
      const int mb = r & ~(width - 1), pb = partner & ~(width - 1);
      uint64_t ms = 0, ps = 0;
      for (int q = 0; q < width; ++q) {
        ms += parts[mb + q];
        ps += parts[pb + q];
      }
      credit(L, P, r, ph, 1, 2 * ms);
      credit(L, P, r, ph, 0, 2 * ps);
    }
}

/* ---- remaining Table-1 baselines (collectives.cpp:184-352) ---- */
static void free_part(part_t* p) {
  free(p->idx);
  free(p->val);
  p->idx = NULL;
  p->val = NULL;
  p->nnz = 0;
}

/* topk_exact of a sparse list (sparse.cpp:82-92): take = min(k, nnz) of its
 * values, ties toward the smaller position (= smaller index). */
static part_t topk_sparse(part_t s, size_t k) {
  part_t o;
  const size_t take = k < s.nnz ? k : s.nnz;
  o.idx = (uint32_t*)malloc((take + 1) * sizeof(uint32_t));
  o.val = (double*)malloc((take + 1) * sizeof(double));
  uint32_t* pos = (uint32_t*)malloc((take + 1) * sizeof(uint32_t));
  o.nnz = take ? orc_topk_exact(s.val, s.nnz, take, pos, o.val) : 0;
  for (size_t i = 0; i < o.nnz; ++i) o.idx[i] = s.idx[pos[i]];
  free(pos);
  return o;
}

static part_t dense_topk(const double* g, size_t n, size_t k) {
  part_t o;
  o.idx = (uint32_t*)malloc((k + 1) * sizeof(uint32_t));
  o.val = (double*)malloc((k + 1) * sizeof(double));
  o.nnz = orc_topk_exact(g, n, k, o.idx, o.val);
  return o;
}

/* gtopk_allreduce (collectives.cpp:300-325) replayed for all ranks: each level
 * merges the pair (lower rank first) and keeps the exact top-k. */
size_t orc_gtopk_allreduce(int P, const double* const* g, size_t n, size_t k, uint32_t* out_idx, double* out_val,
                           orc_counters* ledger) {
  if (P <= 0 || P > ORC_MAX_P || k < 1 || k > n) return 0;
  part_t st[ORC_MAX_P], nx[ORC_MAX_P];
  for (int r = 0; r < P; ++r) st[r] = dense_topk(g[r], n, k);
  for (int level = 1; level < P; level <<= 1) {
    for (int r = 0; r < P; ++r) {
      const int peer = r ^ level, a = r < peer ? r : peer, b = r < peer ? peer : r;
      credit(ledger, P, r, 0, 1, 2 * st[r].nnz);
      credit(ledger, P, r, 0, 0, 2 * st[peer].nnz);
      part_t m = merge_two(st[a], st[b]);
      nx[r] = topk_sparse(m, k);
      free_part(&m);
    }
    for (int r = 0; r < P; ++r) {
      free_part(&st[r]);
      st[r] = nx[r];
    }
  }
  memcpy(out_idx, st[0].idx, st[0].nnz * sizeof(uint32_t));
  memcpy(out_val, st[0].val, st[0].nnz * sizeof(double));
  const size_t m = st[0].nnz;
  for (int r = 0; r < P; ++r) free_part(&st[r]);
  return m;
}

/* dense_allreduce (collectives.cpp:89-150) replayed for all ranks in lockstep:
 * recursive-halving reduce-scatter (own slice += partner's), recursive-doubling
 * allgather; rank 0's result in out (n doubles); ledger phase 4 (dense). */
void orc_dense_allreduce(int P, const double* const* g, size_t n, double* out, orc_counters* ledger) {
  if (P <= 0 || P > ORC_MAX_P) return;
  double* buf[ORC_MAX_P];
  double* in[ORC_MAX_P];
  for (int r = 0; r < P; ++r) {
    buf[r] = (double*)malloc((n + 1) * sizeof(double));
    in[r] = (double*)malloc((n + 1) * sizeof(double));
    memcpy(buf[r], g[r], n * sizeof(double));
  }
  uint64_t ends[ORC_MAX_P + 1];
  orc_equal_slice_ends(n, P, ends);
  int lo[ORC_MAX_P], hi[ORC_MAX_P];
  for (int r = 0; r < P; ++r) {
    lo[r] = 0;
    hi[r] = P;
  }
  for (int mask = P >> 1; mask > 0; mask >>= 1) {
    int klo[ORC_MAX_P], khi[ORC_MAX_P];
    for (int r = 0; r < P; ++r) { /* messages first: the half each rank gives up */
      const int mid = lo[r] + mask, low = (r & mask) == 0;
      const int send_lo = low ? mid : lo[r], send_hi = low ? hi[r] : mid;
      klo[r] = low ? lo[r] : mid;
      khi[r] = low ? mid : hi[r];
      memcpy(in[r ^ mask], buf[r] + ends[send_lo], (ends[send_hi] - ends[send_lo]) * sizeof(double));
      credit(ledger, P, r, 4, 1, ends[send_hi] - ends[send_lo]);
    }
    for (int r = 0; r < P; ++r) {
      const uint64_t kc = ends[khi[r]] - ends[klo[r]];
      credit(ledger, P, r, 4, 0, kc);
      double* dst = buf[r] + ends[klo[r]];
      for (uint64_t i = 0; i < kc; ++i) dst[i] += in[r][i];
      lo[r] = klo[r];
      hi[r] = khi[r];
    }
  }
  for (int mask = 1; mask < P; mask <<= 1) {
    for (int r = 0; r < P; ++r) { /* every rank's reduced block, then the copies */
      const int base = r & ~(2 * mask - 1), my_lo = (r & mask) ? base + mask : base;
      memcpy(in[r] + ends[my_lo], buf[r] + ends[my_lo], (ends[my_lo + mask] - ends[my_lo]) * sizeof(double));
      credit(ledger, P, r, 4, 1, ends[my_lo + mask] - ends[my_lo]);
    }
    for (int r = 0; r < P; ++r) {
      const int partner = r ^ mask, base = partner & ~(2 * mask - 1);
      const int their_lo = (partner & mask) ? base + mask : base;
      const uint64_t tc = ends[their_lo + mask] - ends[their_lo];
      memcpy(buf[r] + ends[their_lo], in[partner] + ends[their_lo], tc * sizeof(double));
      credit(ledger, P, r, 4, 0, tc);
    }
  }
  memcpy(out, buf[0], n * sizeof(double));
  for (int r = 0; r < P; ++r) {
    free(buf[r]);
    free(in[r]);
  }
}

/* TopkDSA working set (collectives.cpp:162-182): COO or a dense window. */
typedef struct {
  int dense;
  part_t coo;
  double* win;
  uint64_t lo, hi;
} dsa_t;

static void dsa_densify(dsa_t* w, uint64_t lo, uint64_t hi) {
  if (w->dense) return;
  w->win = (double*)calloc(hi - lo + 1, sizeof(double));
  for (size_t i = 0; i < w->coo.nnz; ++i) w->win[w->coo.idx[i] - lo] = w->coo.val[i];
  w->lo = lo;
  w->hi = hi;
  w->dense = 1;
  free_part(&w->coo);
}

static part_t slice_part(part_t s, uint64_t lo, uint64_t hi) { /* sparse_slice, sparse.cpp:190-202 */
  size_t a = 0, b;
  while (a < s.nnz && s.idx[a] < lo) ++a;
  b = a;
  while (b < s.nnz && s.idx[b] < hi) ++b;
  part_t o;
  o.idx = (uint32_t*)malloc((b - a + 1) * sizeof(uint32_t));
  o.val = (double*)malloc((b - a + 1) * sizeof(double));
  memcpy(o.idx, s.idx + a, (b - a) * sizeof(uint32_t));
  memcpy(o.val, s.val + a, (b - a) * sizeof(double));
  o.nnz = b - a;
  return o;
}

/* topkdsa_allreduce (collectives.cpp:184-297) replayed for all ranks in lockstep. */
size_t orc_topkdsa_allreduce(int P, const double* const* g, size_t n, size_t k, uint32_t* out_idx, double* out_val,
                             orc_counters* ledger) {
  if (P <= 0 || P > ORC_MAX_P || k < 1 || k > n) return 0;
  dsa_t w[ORC_MAX_P];
  for (int r = 0; r < P; ++r) {
    memset(&w[r], 0, sizeof(w[r]));
    w[r].coo = dense_topk(g[r], n, k);
  }
  if (P == 1) {
    memcpy(out_idx, w[0].coo.idx, w[0].coo.nnz * sizeof(uint32_t));
    memcpy(out_val, w[0].coo.val, w[0].coo.nnz * sizeof(double));
    const size_t m = w[0].coo.nnz;
    free_part(&w[0].coo);
    return m;
  }
  uint64_t ends[ORC_MAX_P + 1];
  orc_equal_slice_ends(n, P, ends);
  int lo[ORC_MAX_P], hi[ORC_MAX_P];
  for (int r = 0; r < P; ++r) {
    lo[r] = 0;
    hi[r] = P;
  }
  for (int mask = P >> 1; mask > 0; mask >>= 1) {
    /* messages of every rank first: kind, dense half or COO slice */
    int kind[ORC_MAX_P];
    double* dmsg[ORC_MAX_P];
    part_t cmsg[ORC_MAX_P];
    uint64_t klo[ORC_MAX_P], khi[ORC_MAX_P];
    for (int r = 0; r < P; ++r) {
      const int mid = lo[r] + mask;
      int keep_lo, keep_hi, send_lo, send_hi;
      if ((r & mask) == 0) {
        keep_lo = lo[r]; keep_hi = mid; send_lo = mid; send_hi = hi[r];
      } else {
        keep_lo = mid; keep_hi = hi[r]; send_lo = lo[r]; send_hi = mid;
      }
      const uint64_t s0 = ends[send_lo], s1 = ends[send_hi];
      klo[r] = ends[keep_lo];
      khi[r] = ends[keep_hi];
      kind[r] = w[r].dense;
      dmsg[r] = NULL;
      cmsg[r].idx = NULL;
      cmsg[r].val = NULL;
      cmsg[r].nnz = 0;
      if (w[r].dense) {
        dmsg[r] = (double*)malloc((s1 - s0 + 1) * sizeof(double));
        memcpy(dmsg[r], w[r].win + (s0 - w[r].lo), (s1 - s0) * sizeof(double));
        credit(ledger, P, r, 0, 1, s1 - s0);
      } else {
        cmsg[r] = slice_part(w[r].coo, s0, s1);
        credit(ledger, P, r, 0, 1, 2 * cmsg[r].nnz);
      }
      lo[r] = keep_lo;
      hi[r] = keep_hi;
    }
    for (int r = 0; r < P; ++r) {
      const int partner = r ^ mask;
      const uint64_t k0 = klo[r], k1 = khi[r];
      credit(ledger, P, r, 0, 0, kind[partner] ? k1 - k0 : 2 * cmsg[partner].nnz);
      /* restrict to the kept half */
      if (w[r].dense) {
        double* kept = (double*)malloc((k1 - k0 + 1) * sizeof(double));
        memcpy(kept, w[r].win + (k0 - w[r].lo), (k1 - k0) * sizeof(double));
        free(w[r].win);
        w[r].win = kept;
        w[r].lo = k0;
        w[r].hi = k1;
      } else {
        part_t kept = slice_part(w[r].coo, k0, k1);
        free_part(&w[r].coo);
        w[r].coo = kept;
      }
      if (kind[partner]) {
        dsa_densify(&w[r], k0, k1);
        for (uint64_t i = 0; i < k1 - k0; ++i) w[r].win[i] += dmsg[partner][i];
      } else if (w[r].dense) {
        const part_t th = cmsg[partner];
        for (size_t i = 0; i < th.nnz; ++i) w[r].win[th.idx[i] - w[r].lo] += th.val[i];
      } else {
        part_t m = r < partner ? merge_two(w[r].coo, cmsg[partner]) : merge_two(cmsg[partner], w[r].coo);
        free_part(&w[r].coo);
        w[r].coo = m;
      }
      if (!w[r].dense && 2 * w[r].coo.nnz >= k1 - k0) dsa_densify(&w[r], k0, k1);
    }
    for (int r = 0; r < P; ++r) {
      free(dmsg[r]);
      free_part(&cmsg[r]);
    }
  }
  /* segments, concatenated in rank order; allgatherv ledger */
  size_t m = 0;
  uint64_t segn[ORC_MAX_P];
  for (int r = 0; r < P; ++r) {
    if (w[r].dense) {
      segn[r] = 0;
      for (uint64_t i = 0; i < w[r].hi - w[r].lo; ++i)
        if (w[r].win[i] != 0.0) {
          out_idx[m] = (uint32_t)(w[r].lo + i);
          out_val[m++] = w[r].win[i];
          ++segn[r];
        }
      free(w[r].win);
    } else {
      segn[r] = w[r].coo.nnz;
      memcpy(out_idx + m, w[r].coo.idx, w[r].coo.nnz * sizeof(uint32_t));
      memcpy(out_val + m, w[r].coo.val, w[r].coo.nnz * sizeof(double));
      m += w[r].coo.nnz;
      free_part(&w[r].coo);
    }
  }
  credit_allgatherv(ledger, P, 2, segn);
  return m;
}

/* gaussian_threshold (sparse.cpp:167-188): sequential fp64 mean and unbiased
 * variance, quantile at 1 - k/(2n) (raw, may be negative); with
 * scale_to_floor, gaussiank_scaled_threshold.  NAN on bad input / zero variance. */
double orc_inverse_normal_cdf(double p);
double orc_gaussian_threshold(const double* g, size_t n, size_t k, int scale_to_floor) {
  if (n < 2 || k < 1 || k > n) return NAN;
  double mean = 0.0;
  for (size_t i = 0; i < n; ++i) mean += g[i];
  mean /= (double)n;
  double ss = 0.0;
  for (size_t i = 0; i < n; ++i) {
    const double d = g[i] - mean;
    ss += d * d;
  }
  const double var = ss / (double)(n - 1);
  if (var == 0.0) return NAN;
  const double p = 1.0 - (double)k / (2.0 * (double)n);
  double th = mean + sqrt(var) * orc_inverse_normal_cdf(p);
  if (scale_to_floor) { /* gaussiank_scaled_threshold, collectives.cpp:327-340 */
    if (!(th >= 0.0)) th = 0.0;
    for (;;) {
      size_t c = 0;
      for (size_t i = 0; i < n; ++i) c += fabs(g[i]) >= th;
      if (4 * c > 3 * k) break;
      th *= 0.9;
    }
  }
  return th;
}

/* Acklam's quantile approximation + two Halley steps (sparse.cpp:122-165). */
double orc_inverse_normal_cdf(double p) {
  static const double a[] = {-3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02,
                             1.383577518672690e+02,  -3.066479806614716e+01, 2.506628277459239e+00};
  static const double b[] = {-5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02,
                             6.680131188771972e+01,  -1.328068155288572e+01};
  static const double c[] = {-7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e+00,
                             -2.549732539343734e+00, 4.374664141464968e+00,  2.938163982698783e+00};
  static const double d[] = {7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e+00,
                             3.754408661907416e+00};
  double x, q, r;
  if (p < 0.02425) {
    q = sqrt(-2.0 * log(p));
    x = (((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
        ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
  } else if (p <= 1.0 - 0.02425) {
    q = p - 0.5;
    r = q * q;
    x = (((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) * q /
        (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1.0);
  } else {
    q = sqrt(-2.0 * log(1.0 - p));
    x = -(((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
        ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
  }
  for (int it = 0; it < 2; ++it) {
    const double e = 0.5 * erfc(-x / sqrt(2.0)) - p;
    const double u = e * 2.5066282746310005 * exp(x * x / 2.0);
    x = x - u / (1.0 + x * u / 2.0);
  }
  return x;
}

/* gaussiank_allreduce (collectives.cpp:342-352): per-rank threshold selection,
 * allgatherv (ledger), sparse_sum.  out holds up to P*n entries. */
size_t orc_gaussiank_allreduce(int P, const double* const* g, size_t n, size_t k, int scale_to_floor,
                               uint32_t* out_idx, double* out_val, orc_counters* ledger) {
  if (P <= 0 || P > ORC_MAX_P) return 0;
  uint32_t* pi[ORC_MAX_P];
  double* pv[ORC_MAX_P];
  size_t nnz[ORC_MAX_P];
  uint64_t parts[ORC_MAX_P];
  for (int q = 0; q < P; ++q) {
    double th = orc_gaussian_threshold(g[q], n, k, scale_to_floor);
    if (!(th >= 0.0)) th = 0.0; /* std::max(gaussian_threshold, 0.0) */
    pi[q] = (uint32_t*)malloc((n + 1) * sizeof(uint32_t));
    pv[q] = (double*)malloc((n + 1) * sizeof(double));
    nnz[q] = orc_select(g[q], n, th, pi[q], pv[q]);
    parts[q] = nnz[q];
  }
  if (P > 1) credit_allgatherv(ledger, P, 2, parts);
  const size_t m = orc_sparse_sum(P, (const uint32_t* const*)pi, (const double* const*)pv, nnz, out_idx, out_val);
  for (int q = 0; q < P; ++q) {
    free(pi[q]);
    free(pv[q]);
  }
  return m;
}

/* ---- space_repartition (oktopk.cpp:28-61) -------------------------------------- */
void orc_space_repartition(int P, const uint32_t* const* sel, const size_t* m, uint64_t n, uint64_t* cuts,
                           orc_counters* ledger) {
  double vec[ORC_MAX_P][ORC_MAX_P + 1], nxt[ORC_MAX_P][ORC_MAX_P + 1];
  for (int r = 0; r < P; ++r) {
    vec[r][0] = 0.0;
    vec[r][P] = (double)n;
    for (int q = 1; q < P; ++q) {
      uint64_t cut;
      if (m[r] == 0) cut = (uint64_t)q * n / (uint64_t)P;
      else {
        const uint64_t pos = (uint64_t)q * m[r] / (uint64_t)P;
        cut = pos < m[r] ? sel[r][pos] : n;
      }
      vec[r][q] = (double)cut;
    }
  }
  /* small_allreduce_avg: recursive doubling, lower-rank block first. */
  const int rounds = log2i(P);
  for (int j = 0; j < rounds; ++j) {
    for (int r = 0; r < P; ++r) {
      const int partner = r ^ (1 << j);
      for (int q = 0; q <= P; ++q)
        nxt[r][q] = partner < r ? vec[partner][q] + vec[r][q] : vec[r][q] + vec[partner][q];
      credit(ledger, P, r, 3, 1, (uint64_t)(P + 1));
      credit(ledger, P, r, 3, 0, (uint64_t)(P + 1));
    }
    memcpy(vec, nxt, sizeof(vec));
  }
  cuts[0] = 0;
  cuts[P] = n;
  for (int q = 1; q < P; ++q) {
    const double avg = vec[0][q] / (double)P;
    uint64_t rounded = (uint64_t)llround(avg > 0.0 ? avg : 0.0);
    if (rounded > n) rounded = n;
    cuts[q] = rounded > cuts[q - 1] ? rounded : cuts[q - 1];
  }
}

static size_t lower_bound_u32(const uint32_t* a, size_t n, uint64_t key) {
  size_t lo = 0, hi = n;
  while (lo < hi) {
    size_t mid = (lo + hi) / 2;
    if ((uint64_t)a[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

static uint64_t bucket_count(uint64_t nnz, uint32_t bucket) {
  if (bucket == 0 || nnz <= bucket) return 1;
  return (nnz + bucket - 1) / bucket;
}

/* ---- ok_sparse_allreduce (oktopk.cpp:246-307) ------------------------------------ */
int orc_ok_sparse_allreduce(int P, orc_state* st, const double* const* g, size_t n, int64_t t, size_t k,
                            orc_counters* ledger, uint32_t* u_idx, double* u_val, size_t* U,
                            uint32_t* const* indexes, size_t* n_indexes, size_t* local_selected) {
  if (n == 0 || k < 1 || t < 1) return -1;
  if (P < 1 || P > ORC_MAX_P || (P & (P - 1))) return -5;
  for (int r = 0; r < P; ++r)
    for (size_t i = 0; i < n; ++i)
      if (!isfinite(g[r][i])) return -2;

  const int thr = (t - 1) % (int64_t)st[0].tau_prime == 0;
  const int bnd = (t - 1) % (int64_t)st[0].tau == 0;
  uint32_t* sel_idx[ORC_MAX_P];
  double* sel_val[ORC_MAX_P];
  size_t m[ORC_MAX_P];
  for (int r = 0; r < P; ++r) {
    if (thr) {
      st[r].local_th = orc_kth_largest_mag(g[r], n, k);
      st[r].last_local_eval = t;
    }
    sel_idx[r] = (uint32_t*)malloc((n + 1) * sizeof(uint32_t));
    sel_val[r] = (double*)malloc((n + 1) * sizeof(double));
    m[r] = orc_select(g[r], n, st[r].local_th, sel_idx[r], sel_val[r]);
  }
  uint64_t cuts[ORC_MAX_P + 1];
  if (bnd) {
    orc_space_repartition(P, (const uint32_t* const*)sel_idx, m, n, cuts, ledger);
    for (int r = 0; r < P; ++r) {
      memcpy(st[r].cuts, cuts, sizeof(uint64_t) * (P + 1));
      st[r].regions = P;
    }
  } else if (st[0].regions != P) {
    orc_equal_slice_ends(n, P, cuts);
    for (int r = 0; r < P; ++r) {
      memcpy(st[r].cuts, cuts, sizeof(uint64_t) * (P + 1));
      st[r].regions = P;
    }
  } else {
    memcpy(cuts, st[0].cuts, sizeof(uint64_t) * (P + 1));
  }

  /* split_and_reduce (oktopk.cpp:95-163) */
  size_t off[ORC_MAX_P][ORC_MAX_P + 1];
  for (int r = 0; r < P; ++r) {
    for (int q = 0; q < P; ++q) off[r][q] = lower_bound_u32(sel_idx[r], m[r], cuts[q]);
    off[r][P] = m[r];
  }
  for (int r = 0; r < P; ++r)
    for (int s = 1; s < P; ++s) {
      const int dst = (r + s) % P, src = (r - s + P) % P;
      const uint64_t out_n = off[r][dst + 1] - off[r][dst];
      const uint64_t in_n = off[src][r + 1] - off[src][r];
      const uint64_t ob = bucket_count(out_n, st[r].bucket_size);
      const uint64_t ib = bucket_count(in_n, st[r].bucket_size);
      if (ledger) {
        ledger[r * ORC_PHASES + 0].words_sent += 2 * out_n;
        ledger[r * ORC_PHASES + 0].msgs_sent += ob;
        ledger[r * ORC_PHASES + 0].words_recv += 2 * in_n;
        ledger[r * ORC_PHASES + 0].msgs_recv += ib;
      }
    }
  uint32_t* reg_idx[ORC_MAX_P];
  double* reg_val[ORC_MAX_P];
  size_t R[ORC_MAX_P];
  for (int o = 0; o < P; ++o) {
    const uint32_t* pi[ORC_MAX_P];
    const double* pv[ORC_MAX_P];
    size_t pn[ORC_MAX_P], tot = 0;
    for (int q = 0; q < P; ++q) {
      pi[q] = sel_idx[q] + off[q][o];
      pv[q] = sel_val[q] + off[q][o];
      pn[q] = off[q][o + 1] - off[q][o];
      tot += pn[q];
    }
    reg_idx[o] = (uint32_t*)malloc((tot + 1) * sizeof(uint32_t));
    reg_val[o] = (double*)malloc((tot + 1) * sizeof(double));
    R[o] = orc_sparse_sum(P, pi, pv, pn, reg_idx[o], reg_val[o]);
  }

  /* global threshold refresh (oktopk.cpp:277-293) */
  if (thr) {
    size_t tot = 0;
    for (int o = 0; o < P; ++o) tot += R[o];
    if (P > 1) {
      uint64_t parts[ORC_MAX_P];
      for (int o = 0; o < P; ++o) parts[o] = R[o];
      credit_allgatherv(ledger, P, 5, parts);
    }
    if (tot > 0) {
      double* all = (double*)malloc(tot * sizeof(double));
      size_t w = 0;
      for (int o = 0; o < P; ++o) {
        memcpy(all + w, reg_val[o], R[o] * sizeof(double));
        w += R[o];
      }
      const double gth = orc_kth_largest_mag(all, tot, k);
      free(all);
      for (int r = 0; r < P; ++r) st[r].global_th = gth;
    }
    for (int r = 0; r < P; ++r) st[r].last_global_eval = t;
  }

  /* balance_and_allgatherv (oktopk.cpp:165-244) */
  size_t c[ORC_MAX_P], total = 0, maxs = 0;
  uint32_t* mi[ORC_MAX_P];
  double* mv[ORC_MAX_P];
  for (int r = 0; r < P; ++r) {
    mi[r] = (uint32_t*)malloc((R[r] + 1) * sizeof(uint32_t));
    mv[r] = (double*)malloc((R[r] + 1) * sizeof(double));
    c[r] = select_sparse(reg_idx[r], reg_val[r], R[r], st[r].global_th, mi[r], mv[r]);
    total += c[r];
    if (c[r] > maxs) maxs = c[r];
  }
  if (P > 1) {
    const int rounds = log2i(P);
    for (int r = 0; r < P; ++r)
      for (int j = 0; j < rounds; ++j) {
        credit(ledger, P, r, 3, 1, (uint64_t)1 << j);
        credit(ledger, P, r, 3, 0, (uint64_t)1 << j);
      }
    uint64_t parts[ORC_MAX_P];
    for (int r = 0; r < P; ++r) parts[r] = c[r];
    if (total > 0 && (uint64_t)maxs * (uint64_t)P >= 4 * (uint64_t)total) {
      uint64_t o[ORC_MAX_P + 1], block[ORC_MAX_P + 1];
      o[0] = 0;
      for (int r = 0; r < P; ++r) o[r + 1] = o[r] + c[r];
      orc_equal_slice_ends(total, P, block);
      for (int src = 0; src < P; ++src)
        for (int dst = 0; dst < P; ++dst) {
          if (src == dst) continue;
          const uint64_t a = o[src] > block[dst] ? o[src] : block[dst];
          const uint64_t b = o[src + 1] < block[dst + 1] ? o[src + 1] : block[dst + 1];
          if (a < b) {
            credit(ledger, P, src, 1, 1, 2 * (b - a));
            credit(ledger, P, dst, 1, 0, 2 * (b - a));
          }
        }
      for (int r = 0; r < P; ++r) parts[r] = block[r + 1] - block[r];
    }
    credit_allgatherv(ledger, P, 2, parts);
  }
  size_t uw = 0;
  for (int r = 0; r < P; ++r) {
    memcpy(u_idx + uw, mi[r], c[r] * sizeof(uint32_t));
    memcpy(u_val + uw, mv[r], c[r] * sizeof(double));
    uw += c[r];
  }
  *U = uw;

  /* indexes = local selection ∩ u (oktopk.cpp:299-302) */
  for (int r = 0; r < P; ++r) {
    size_t i = 0, j = 0, w = 0;
    while (i < m[r] && j < uw) {
      if (sel_idx[r][i] < u_idx[j]) ++i;
      else if (u_idx[j] < sel_idx[r][i]) ++j;
      else {
        if (indexes && indexes[r]) indexes[r][w] = sel_idx[r][i];
        ++w;
        ++i;
        ++j;
      }
    }
    if (n_indexes) n_indexes[r] = w;
    if (local_selected) local_selected[r] = m[r];
    st[r].t = t;
  }
  for (int r = 0; r < P; ++r) {
    free(sel_idx[r]);
    free(sel_val[r]);
    free(reg_idx[r]);
    free(reg_val[r]);
    free(mi[r]);
    free(mv[r]);
  }
  return 0;
}

/* ---- oktopk_sgd_step (trainer.cpp:466-488) ---------------------------------------- */
int orc_sgd_step(int P, orc_state* st, const double* const* grad, double* const* eps, double* const* w,
                 size_t n, double alpha, int64_t t, size_t k, orc_counters* ledger, uint32_t* u_idx,
                 double* u_val, size_t* U) {
  for (int r = 0; r < P; ++r)
    for (size_t i = 0; i < n; ++i)
      if (!isfinite(grad[r][i])) return -2;
  double* acc[ORC_MAX_P];
  uint32_t* ix[ORC_MAX_P];
  size_t nix[ORC_MAX_P], sel[ORC_MAX_P];
  for (int r = 0; r < P; ++r) {
    acc[r] = (double*)malloc((n + 1) * sizeof(double));
    ix[r] = (uint32_t*)malloc((n + 1) * sizeof(uint32_t));
    for (size_t i = 0; i < n; ++i) acc[r][i] = eps[r][i] + alpha * grad[r][i];
  }
  const int rc = orc_ok_sparse_allreduce(P, st, (const double* const*)acc, n, t, k, ledger, u_idx, u_val, U, ix,
                                         nix, sel);
  if (rc == 0) {
    for (int r = 0; r < P; ++r) {
      memcpy(eps[r], acc[r], n * sizeof(double));
      for (size_t j = 0; j < nix[r]; ++j) eps[r][ix[r][j]] = 0.0;
      for (size_t j = 0; j < *U; ++j) w[r][u_idx[j]] -= u_val[j] / (double)P;
    }
  }
  for (int r = 0; r < P; ++r) {
    free(acc[r]);
    free(ix[r]);
  }
  if (rc) return rc;
  for (int r = 0; r < P; ++r)
    for (size_t i = 0; i < n; ++i)
      if (!isfinite(w[r][i])) return -2;
  return 0;
}

/* ---- COO wire codec (sparse.cpp:260-312) ---------------------------------- */
static void put_u32(uint8_t* o, uint32_t w) { /* put_u32, sparse.cpp:260-265 */
  o[0] = (uint8_t)(w & 0xff);
  o[1] = (uint8_t)((w >> 8) & 0xff);
  o[2] = (uint8_t)((w >> 16) & 0xff);
  o[3] = (uint8_t)((w >> 24) & 0xff);
}
static uint32_t get_u32(const uint8_t* b) { /* get_u32, sparse.cpp:267-272 */
  return (uint32_t)b[0] | ((uint32_t)b[1] << 8) | ((uint32_t)b[2] << 16) | ((uint32_t)b[3] << 24);
}

void orc_wire_encode(const uint32_t* idx, const double* val, size_t nnz, uint8_t* out) { /* sparse.cpp:276-285 */
  put_u32(out, (uint32_t)nnz);
  for (size_t i = 0; i < nnz; ++i) put_u32(out + 4 + 4 * i, idx[i]);
  for (size_t i = 0; i < nnz; ++i) {
    const float f = (float)val[i];
    uint32_t w;
    memcpy(&w, &f, 4);
    put_u32(out + 4 + 4 * nnz + 4 * i, w);
  }
}

int orc_wire_decode(const uint8_t* in, size_t bytes, size_t n, uint32_t* idx, double* val, size_t* nnz_out) {
  /* sparse.cpp:287-310 */
  if (bytes < 4) return 1;
  const uint32_t nnz = get_u32(in);
  if (bytes != 4 + (size_t)8 * nnz) return 1;
  for (uint32_t i = 0; i < nnz; ++i) {
    const uint32_t v = get_u32(in + 4 + 4 * (size_t)i);
    if (v >= n) return 1;
    if (i > 0 && v <= idx[i - 1]) return 1;
    idx[i] = v;
  }
  for (uint32_t i = 0; i < nnz; ++i) {
    const uint32_t w = get_u32(in + 4 + 4 * (size_t)nnz + 4 * (size_t)i);
    float f;
    memcpy(&f, &w, 4);
    val[i] = (double)f;
  }
  *nnz_out = nnz;
  return 0;
}
