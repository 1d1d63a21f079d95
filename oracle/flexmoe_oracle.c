/*
 * flexmoe_oracle.c — TEST INFRASTRUCTURE ONLY (the parity checker).
 *
 * Plain-C restatement of the reference moesim count-level algorithms on the
 * FlexMoE hot path. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this; the product library
 * (paper_2304_03946_b200/libflexmoe_b200.so) never links or calls it.
 *
 * Parity is pinned against the reference itself: tests/test_oracle_vs_ref.py
 * runs these functions and the reference sources compiled into
 * oracle/_ref/libmoesim_ref.so on the same seeded inputs, and
 * tests/golden/*.json hold vectors generated from the reference
 * (tests/golden/make_golden.py).
 *
 * Sources restated (paths relative to /root/reference/proj):
 *   orc_route                  src/router.cpp:57-169 (Alg. 3, locality-first greedy)
 *   orc_largest_remainder_round src/workload.cpp:77-114
 *   orc_static_ep_kept         src/baselines.cpp:81-122 (StaticEP capacity drops)
 *   orc_balance_ratio          src/policy.cpp:32-46 (Eq. 7)
 *   orc_generate_trace         src/workload.cpp:116-173 (+ helpers :31-52)
 * Status codes follow include/flexmoe_b200.h (0 ok, 1 invalid_argument,
 * 2 logic_error); messages land in orc_last_error().
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_INVALID 1
#define ORC_LOGIC 2

static char orc_err[256];

const char* orc_last_error(void) { return orc_err; }

static int fail(int code, const char* msg) {
  snprintf(orc_err, sizeof orc_err, "%s", msg);
  return code;
}

/* ---------------------------------------------------------------- helpers */

/* Stable ordering of `n` keys, descending by key (equal keys keep their
 * input order, i.e. ascending index) — the std::stable_sort(..., a > b)
 * used by the reference at router.cpp:125-128 and workload.cpp:89-90. */
static void stable_order_desc_i64(const int64_t* key, int* order, int n) {
  for (int i = 0; i < n; ++i) {
    int v = order[i];
    int j = i - 1;
    while (j >= 0 && key[order[j]] < key[v]) {
      order[j + 1] = order[j];
      --j;
    }
    order[j + 1] = v;
  }
}

static void stable_order_desc_f64(const double* key, int* order, int n) {
  for (int i = 0; i < n; ++i) {
    int v = order[i];
    int j = i - 1;
    while (j >= 0 && key[order[j]] < key[v]) {
      order[j + 1] = order[j];
      --j;
    }
    order[j + 1] = v;
  }
}

/* ---------------------------------------------------------------- route */

/* flows[e][src][dst] for demand D[e][g] over replica counts cnt[e][g].
 * router.cpp:57-169. */
int orc_route(const int64_t* D, const int32_t* cnt, int N, int G, int64_t* flows) {
  if (N < 0 || G < 1) return fail(ORC_INVALID, "route: bad dimensions");
  memset(flows, 0, sizeof(int64_t) * (size_t)N * G * G);
  int64_t* quota = calloc((size_t)G, sizeof(int64_t));
  int64_t* avail = calloc((size_t)G, sizeof(int64_t));
  int64_t* recv = calloc((size_t)G, sizeof(int64_t));
  int64_t* rem = calloc((size_t)G, sizeof(int64_t));
  int* host = calloc((size_t)G, sizeof(int));
  int* order = calloc((size_t)G, sizeof(int));
  int status = ORC_OK;
#define F(e, s, d) flows[((size_t)(e) * G + (s)) * G + (d)]
  for (int e = 0; e < N && status == ORC_OK; ++e) {
    const int64_t* De = D + (size_t)e * G;
    const int32_t* ce = cnt + (size_t)e * G;
    int64_t load = 0, n_e = 0;
    int nh = 0;
    for (int g = 0; g < G; ++g) {
      load += De[g];
      n_e += ce[g];
      if (ce[g] > 0) host[nh++] = g; /* ascending GPU ids, placement.cpp:109-117 */
    }
    if (load == 0) continue;
    if (n_e == 0) {
      char msg[96];
      snprintf(msg, sizeof msg, "route: expert %d has demand but no replica", e);
      status = fail(ORC_INVALID, msg);
      break;
    }
    /* Capacity share per host and the local phase. */
    for (int g = 0; g < G; ++g) recv[g] = 0;
    for (int i = 0; i < nh; ++i) {
      const int h = host[i];
      quota[h] = load * ce[h] / n_e;
      const int64_t keep = quota[h] < De[h] ? quota[h] : De[h];
      if (keep > 0) {
        F(e, h, h) = keep;
        recv[h] = keep;
      }
      avail[h] = quota[h] - recv[h];
    }
    /* Remote phase, sources in ascending id. */
    for (int src = 0; src < G; ++src) {
      int64_t left = De[src] - F(e, src, src);
      if (left == 0) continue;
      int64_t pool = 0;
      for (int i = 0; i < nh; ++i) pool += avail[host[i]];
      if (pool > 0) {
        const int64_t grant = left < pool ? left : pool;
        int64_t given = 0;
        int nr = 0;
        for (int i = 0; i < nh; ++i) {
          const int h = host[i];
          if (avail[h] == 0) continue;
          const int64_t part = grant * avail[h] / pool;
          rem[h] = grant * avail[h] % pool;
          F(e, src, h) += part;
          recv[h] += part;
          avail[h] -= part;
          given += part;
          order[nr++] = h;
        }
        stable_order_desc_i64(rem, order, nr);
        for (int i = 0; i < nr && given != grant; ++i) {
          const int h = order[i];
          if (avail[h] > 0) {
            F(e, src, h) += 1;
            recv[h] += 1;
            avail[h] -= 1;
            ++given;
          }
        }
        left -= grant;
      }
      /* Rounding leftovers: least-received host, ties to the lowest id. */
      while (left > 0) {
        int best = host[0];
        for (int i = 1; i < nh; ++i)
          if (recv[host[i]] < recv[best]) best = host[i];
        F(e, src, best) += 1;
        recv[best] += 1;
        --left;
      }
    }
    for (int src = 0; src < G; ++src) {
      int64_t routed = 0;
      for (int dst = 0; dst < G; ++dst) routed += F(e, src, dst);
      if (routed != De[src]) {
        char msg[96];
        snprintf(msg, sizeof msg, "route: conservation violated for expert %d", e);
        status = fail(ORC_LOGIC, msg);
        break;
      }
    }
  }
#undef F
  free(quota);
  free(avail);
  free(recv);
  free(rem);
  free(host);
  free(order);
  return status;
}

/* ------------------------------------------------------- rounding helpers */

/* workload.cpp:77-114. */
int orc_largest_remainder_round(const double* exact, int n, int64_t total, int64_t* out) {
  if (n <= 0) {
    if (total != 0) return fail(ORC_INVALID, "largest_remainder_round: empty input");
    return ORC_OK;
  }
  double* frac = malloc(sizeof(double) * (size_t)n);
  int* order = malloc(sizeof(int) * (size_t)n);
  int64_t assigned = 0;
  for (int i = 0; i < n; ++i) {
    const double fl = floor(exact[i]);
    out[i] = (int64_t)fl;
    frac[i] = exact[i] - fl;
    assigned += out[i];
    order[i] = i;
  }
  stable_order_desc_f64(frac, order, n);
  for (int64_t i = 0; assigned < total; ++i) {
    out[order[i % n]] += 1;
    ++assigned;
  }
  int64_t idx = n;
  while (assigned > total) {
    --idx;
    const int i = order[idx % n];
    if (out[i] > 0) {
      out[i] -= 1;
      --assigned;
    }
    if (idx == 0) idx = n;
  }
  free(frac);
  free(order);
  return ORC_OK;
}

/* StaticEP drops, baselines.cpp:89-122; tokens_per_step <= 0 means sum(D). */
int orc_static_ep_kept(const int64_t* D, int N, int G, double cf, int64_t tokens_per_step,
                       int64_t* kept, int64_t* dropped_out) {
  int64_t tokens = tokens_per_step;
  if (tokens <= 0) {
    tokens = 0;
    for (size_t i = 0; i < (size_t)N * G; ++i) tokens += D[i];
  }
  memcpy(kept, D, sizeof(int64_t) * (size_t)N * G);
  int64_t dropped = 0;
  if (!isinf(cf)) {
    const int64_t cap = (int64_t)floor(cf * (double)tokens / N);
    double* exact = malloc(sizeof(double) * (size_t)G);
    int64_t* row = malloc(sizeof(int64_t) * (size_t)G);
    for (int e = 0; e < N; ++e) {
      const int64_t* De = D + (size_t)e * G;
      int64_t load = 0;
      for (int g = 0; g < G; ++g) load += De[g];
      if (load <= cap) continue;
      for (int g = 0; g < G; ++g) exact[g] = (double)De[g] * (double)cap / (double)load;
      orc_largest_remainder_round(exact, G, cap, row);
      for (int g = 0; g < G; ++g) {
        const int64_t k = row[g] < De[g] ? row[g] : De[g];
        dropped += De[g] - k;
        kept[(size_t)e * G + g] = k;
      }
    }
    free(exact);
    free(row);
  }
  if (dropped_out) *dropped_out = dropped;
  return ORC_OK;
}

/* Eq. 7 on a routing plan, policy.cpp:32-46. */
int orc_balance_ratio(const int64_t* flows, int N, int G, double* ratio) {
  int64_t sum = 0, mx = 0;
  for (int dst = 0; dst < G; ++dst) {
    int64_t t = 0;
    for (int e = 0; e < N; ++e)
      for (int src = 0; src < G; ++src) t += flows[((size_t)e * G + src) * G + dst];
    sum += t;
    if (t > mx) mx = t;
  }
  if (sum == 0) return fail(ORC_INVALID, "balance_ratio: zero total tokens");
  const double mean = (double)sum / (double)G;
  *ratio = (double)mx / mean;
  return ORC_OK;
}

/* ---------------------------------------------------------- trace generator */

/* mt19937-64 (Matsumoto & Nishimura 2000), the engine behind the reference's
 * std::mt19937_64 (workload.cpp:135). */
typedef struct {
  uint64_t s[312];
  int i;
} orc_mt64;

static void mt64_seed(orc_mt64* m, uint64_t seed) {
  m->s[0] = seed;
  for (int i = 1; i < 312; ++i)
    m->s[i] = 6364136223846793005ULL * (m->s[i - 1] ^ (m->s[i - 1] >> 62)) + (uint64_t)i;
  m->i = 312;
}

static uint64_t mt64_next(orc_mt64* m) {
  static const uint64_t mag[2] = {0ULL, 0xB5026F5AA96619E9ULL};
  const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
  if (m->i >= 312) {
    for (int k = 0; k < 312; ++k) {
      const uint64_t y = (m->s[k] & upper) | (m->s[(k + 1) % 312] & lower);
      m->s[k] = m->s[(k + 156) % 312] ^ (y >> 1) ^ mag[y & 1ULL];
    }
    m->i = 0;
  }
  uint64_t x = m->s[m->i++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

uint64_t orc_mt64_first(uint64_t seed, int skip) {
  orc_mt64 m;
  mt64_seed(&m, seed);
  for (int i = 0; i < skip; ++i) mt64_next(&m);
  return mt64_next(&m);
}

static void normalise(double* p, int n) {
  double sum = 0.0;
  for (int i = 0; i < n; ++i) sum += p[i];
  for (int i = 0; i < n; ++i) p[i] /= sum;
}

/* workload.cpp:116-173: out[step][e][g]. */
int orc_generate_trace(int N, int G, int64_t tokens_per_step, double zipf, double drift,
                       uint64_t seed, int steps, int64_t* out) {
  if (N < 1 || G < 1 || steps < 1)
    return fail(ORC_INVALID, "generate_trace: dimensions must be positive");
  if (tokens_per_step <= 0 || tokens_per_step % G != 0)
    return fail(ORC_INVALID,
                "generate_trace: tokens_per_step must be a positive multiple of num_gpus");
  if (zipf < 0 || drift < 0 || drift > 1)
    return fail(ORC_INVALID, "generate_trace: invalid zipf_exponent or drift_rate");
  orc_mt64 rng;
  mt64_seed(&rng, seed);
  int* perm = malloc(sizeof(int) * (size_t)N);
  for (int i = 0; i < N; ++i) perm[i] = i;
  for (int i = N - 1; i > 0; --i) {
    const int j = (int)(mt64_next(&rng) % (uint64_t)(i + 1));
    const int t = perm[i];
    perm[i] = perm[j];
    perm[j] = t;
  }
  double* pop = malloc(sizeof(double) * (size_t)N);
  double* exact = malloc(sizeof(double) * (size_t)N);
  int64_t* col = malloc(sizeof(int64_t) * (size_t)N);
  for (int i = 0; i < N; ++i) pop[perm[i]] = pow((double)(i + 1), -zipf);
  normalise(pop, N);
  const int64_t per_gpu = tokens_per_step / G;
  for (int step = 0; step < steps; ++step) {
    for (int e = 0; e < N; ++e) exact[e] = pop[e] * (double)per_gpu;
    orc_largest_remainder_round(exact, N, per_gpu, col);
    int64_t* D = out + (size_t)step * N * G;
    for (int e = 0; e < N; ++e)
      for (int g = 0; g < G; ++g) D[(size_t)e * G + g] = col[e];
    if (drift > 0) {
      for (int e = 0; e < N; ++e) {
        const double u01 = (double)(mt64_next(&rng) >> 11) * 0x1.0p-53;
        pop[e] *= exp((u01 * 2.0 - 1.0) * drift);
      }
      normalise(pop, N);
    }
  }
  free(perm);
  free(pop);
  free(exact);
  free(col);
  return ORC_OK;
}

/* ---------------------------------------------------------------- layer math helper
 * bf16 storage rounding (round to nearest even) of a float32 array, in place,
 * OpenMP over the host cores — the hot elementwise op of the float32 layer
 * restatement (oracle/layer.py) that bench.py times as the CPU baseline. */
void orc_bf16_round_f32(float* a, int64_t n) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    uint32_t u;
    memcpy(&u, a + i, 4);
    u += 0x7FFFu + ((u >> 16) & 1u);
    u &= 0xFFFF0000u;
    memcpy(a + i, &u, 4);
  }
}
