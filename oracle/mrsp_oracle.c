/*
 * mrsp_oracle.c — CPU restatement of the reference's MR-SP toy path.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing in the product (paper_2507_07966_b200/)
 * links, imports or calls this file; only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs load it, as the checker.
 *
 * Every function restates the reference algorithm it cites (paths relative
 * to /root/reference/proj). Parity pinned: tests/test_oracle.py checks this
 * file against golden vectors produced by the reference itself
 * (oracle/gen_golden.cpp linked against the reference sources, fixtures in
 * tests/golden/ref_toy.json) and against the survey's known-answer values.
 *
 * Floating point: compiled with -O2 -ffp-contract=off and no -mfma, which is
 * how the reference's CMake build evaluates its loops (no -march, so GCC emits
 * no FMA even under gnu++20's default contraction). libm's tanh is used as-is,
 * exactly as policy.cpp:47 does.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- std::mt19937_64 (the standard's parameters; common.hpp:63 uses it) ---- */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (g->mt[i] & UM) | (g->mt[(i + 1) % 312] & LM);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= A;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t x = g->mt[g->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* Rng::substream — FNV-1a over the tag, splitmix64 finalizer (common.hpp:67-80). */
uint64_t oracle_substream_seed(uint64_t base, const char* tag) {
  uint64_t h = 1469598103934665603ULL;
  for (const unsigned char* c = (const unsigned char*)tag; *c; ++c) {
    h ^= *c;
    h *= 1099511628211ULL;
  }
  uint64_t z = base ^ h;
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* Rng::uniform (common.hpp:31) */
static double rng_uniform(mt64* g) { return (double)(mt64_next(g) >> 11) * 0x1.0p-53; }

/* Rng::normal — Box-Muller cosine branch (common.hpp:34-38) */
static double rng_normal(mt64* g) {
  double u1 = 1.0 - rng_uniform(g);
  double u2 = rng_uniform(g);
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925286766559 * u2);
}

/* First n raw draws of Rng::substream(base, tag) — used by the KAT tests. */
void oracle_substream_draws(uint64_t base, const char* tag, uint64_t* out, int n) {
  mt64 g;
  mt64_seed(&g, oracle_substream_seed(base, tag));
  for (int i = 0; i < n; ++i) out[i] = mt64_next(&g);
}

/* Generic seeded uniform / normal streams (Rng(seed) with a raw seed). */
void oracle_rng_uniform(uint64_t seed, double* out, long n) {
  mt64 g;
  mt64_seed(&g, seed);
  for (long i = 0; i < n; ++i) out[i] = rng_uniform(&g);
}

/* ---- plan_shards (engine.cpp:15-29) ---- */
int oracle_plan_shards(uint64_t n, int k, uint64_t* ranges /* 2k */) {
  if (k < 1) return -1;
  uint64_t base = n / (uint64_t)k, extra = n % (uint64_t)k, pos = 0;
  for (int w = 0; w < k; ++w) {
    uint64_t len = base + ((uint64_t)w < extra ? 1 : 0);
    ranges[2 * w] = pos;
    ranges[2 * w + 1] = pos + len;
    pos += len;
  }
  return 0;
}

/* ---- gen_video (mmseq.cpp:58-72): frames U[-1,1) from substream(seed,"video") ---- */
int oracle_gen_video(uint64_t seed, int frames, int feature_dim, double* out) {
  if (frames < 1 || feature_dim < 4) return -1;
  mt64 g;
  mt64_seed(&g, oracle_substream_seed(seed, "video"));
  long n = (long)frames * feature_dim;
  for (long i = 0; i < n; ++i) out[i] = 2.0 * rng_uniform(&g) - 1.0;
  return 0;
}

/* ---- EncoderParams::generate (policy.cpp:12-34) ---- */
int oracle_encoder_generate(uint64_t seed, int d, int p, double* w) {
  if (d < 1 || p < 4) return -1;
  mt64 g;
  mt64_seed(&g, oracle_substream_seed(seed, "encoder"));
  double scale = 1.0 / sqrt((double)p);
  for (int r = 0; r < d; ++r)
    for (int k = 0; k < p; ++k) w[(long)r * p + k] = scale * rng_normal(&g);
  if (d >= 4 && p % 4 == 0) {
    int group = p / 4;
    for (int gi = 0; gi < 4; ++gi)
      for (int k = 0; k < p; ++k)
        w[(long)gi * p + k] = (k >= gi * group && k < (gi + 1) * group) ? 0.3 / group : 0.0;
  }
  return 0;
}

/* ---- PolicyParams::random (policy.cpp:56-61); layout policy.hpp:39-53 ---- */
long oracle_policy_param_count(int V, int d, int h) {
  return (long)V * d + 2L * h * d + h + (long)V * h + V;
}
int oracle_policy_random(int V, int d, int h, uint64_t seed, double scale, double* theta) {
  mt64 g;
  mt64_seed(&g, oracle_substream_seed(seed, "policy-init"));
  long n = oracle_policy_param_count(V, d, h);
  for (long i = 0; i < n; ++i) theta[i] = scale * rng_normal(&g);
  return 0;
}

/* ---- encode_frame (policy.cpp:36-47) ---- */
void oracle_encode_frame(const double* w, int d, int p, const double* x, double* e) {
  for (int r = 0; r < d; ++r) {
    double z = 0.0;
    const double* row = w + (long)r * p;
    for (int k = 0; k < p; ++k) z += row[k] * x[k];
    e[r] = tanh(z);
  }
}

/* serial_encode (engine.cpp:52-57) */
void oracle_serial_encode(const double* w, int d, int p, const double* frames, long n_frames,
                          double* out) {
  for (long f = 0; f < n_frames; ++f) oracle_encode_frame(w, d, p, frames + f * p, out + f * d);
}

/* ---- step_logits + hidden_state (policy.cpp:85-119) ---- */
int oracle_step_logits(const double* theta, int V, int d, int h, const double* ctx, int prev,
                       double* logits) {
  if (prev < 0 || prev >= V) return -1;
  const double* A = theta + (long)V * d;
  const double* B = A + (long)h * d;
  const double* c = B + (long)h * d;
  const double* U = c + h;
  const double* bias = U + (long)V * h;
  const double* e_prev = theta + (long)prev * d;
  double* s = (double*)malloc(sizeof(double) * (size_t)h);
  for (int r = 0; r < h; ++r) {
    double z = c[r];
    const double* arow = A + (long)r * d;
    const double* brow = B + (long)r * d;
    for (int k = 0; k < d; ++k) z += arow[k] * ctx[k] + brow[k] * e_prev[k];
    s[r] = tanh(z);
  }
  for (int v = 0; v < V; ++v) {
    double z = bias[v];
    const double* urow = U + (long)v * h;
    for (int r = 0; r < h; ++r) z += urow[r] * s[r];
    logits[v] = z;
  }
  free(s);
  return 0;
}

/* serial_prefill (engine.cpp:59-71): rows are padded [n_rows][max_len]; out is
 * packed row-major over real positions (sum(lengths) x V). prev = EOS(1) at t=0. */
int oracle_serial_prefill(const double* theta, int V, int d, int h, const double* contexts,
                          const int32_t* rows, const uint64_t* lengths, long n_rows,
                          long max_len, double* out) {
  long o = 0;
  for (long r = 0; r < n_rows; ++r) {
    for (uint64_t t = 0; t < lengths[r]; ++t) {
      int prev = t == 0 ? 1 : rows[r * max_len + (long)t - 1];
      if (oracle_step_logits(theta, V, d, h, contexts + r * d, prev, out + o * V)) return -1;
      ++o;
    }
  }
  return 0;
}

/* ---- log_softmax (common.hpp:95-104) ---- */
void oracle_log_softmax(const double* logits, int n, double* out) {
  double m = logits[0];
  for (int i = 0; i < n; ++i) m = logits[i] > m ? logits[i] : m;
  double z = 0.0;
  for (int i = 0; i < n; ++i) z += exp(logits[i] - m);
  double lz = m + log(z);
  for (int i = 0; i < n; ++i) out[i] = logits[i] - lz;
}

/* ---- context_vector (policy.cpp:63-80) ---- */
int oracle_context_vector(const double* theta, int V, int d, const double* frame_emb, long n_frames,
                          const int32_t* text, long n_text, double* ctx) {
  long total = n_frames + n_text;
  if (total == 0) return -1;
  for (int k = 0; k < d; ++k) ctx[k] = 0.0;
  for (long f = 0; f < n_frames; ++f)
    for (int k = 0; k < d; ++k) ctx[k] += frame_emb[f * d + k];
  for (long i = 0; i < n_text; ++i) {
    if (text[i] < 0 || text[i] >= V) return -1;
    const double* row = theta + (long)text[i] * d;
    for (int k = 0; k < d; ++k) ctx[k] += row[k];
  }
  double inv = 1.0 / (double)total;
  for (int k = 0; k < d; ++k) ctx[k] *= inv;
  return 0;
}

/* ---- backward: GradAccumulator (policy.cpp:195-260) ---- */
typedef struct {
  const double* theta;
  int V, d, h;
  const double* ctx; /* context_vector(seq, theta) */
  double* grad;      /* param_count */
  double* d_ctx;     /* d */
} grad_acc;

/* add_position (policy.cpp:202-247): logits = U s + b, s = tanh(A ctx + B e_prev + c) */
static void acc_add_position(grad_acc* a, int prev, const double* g_logits) {
  const int V = a->V, d = a->d, h = a->h;
  const double* A = a->theta + (long)V * d;
  const double* B = A + (long)h * d;
  const double* c = B + (long)h * d;
  const double* U = c + h;
  const double* e_prev = a->theta + (long)prev * d;
  double* gE = a->grad;
  double* gA = gE + (long)V * d;
  double* gB = gA + (long)h * d;
  double* gc = gB + (long)h * d;
  double* gU = gc + h;
  double* gb = gU + (long)V * h;
  double* s = (double*)malloc(sizeof(double) * (size_t)h);
  double* ds = (double*)calloc((size_t)h, sizeof(double));
  for (int r = 0; r < h; ++r) { /* hidden_state (policy.cpp:85-101) */
    double z = c[r];
    for (int k = 0; k < d; ++k) z += A[(long)r * d + k] * a->ctx[k] + B[(long)r * d + k] * e_prev[k];
    s[r] = tanh(z);
  }
  for (int v = 0; v < V; ++v) {
    double g = g_logits[v];
    if (g == 0.0) continue;
    gb[v] += g;
    for (int r = 0; r < h; ++r) {
      gU[(long)v * h + r] += g * s[r];
      ds[r] += g * U[(long)v * h + r];
    }
  }
  for (int r = 0; r < h; ++r) {
    double dz = ds[r] * (1.0 - s[r] * s[r]);
    if (dz == 0.0) continue;
    gc[r] += dz;
    for (int k = 0; k < d; ++k) {
      gA[(long)r * d + k] += dz * a->ctx[k];
      gB[(long)r * d + k] += dz * e_prev[k];
      gE[(long)prev * d + k] += dz * B[(long)r * d + k];
      a->d_ctx[k] += dz * A[(long)r * d + k];
    }
  }
  free(s);
  free(ds);
}

/* take (policy.cpp:249-260): text rows receive d_context / total_len each */
static void acc_take(grad_acc* a, const int32_t* text, long n_text, long total_len) {
  double inv = 1.0 / (double)total_len;
  for (long i = 0; i < n_text; ++i)
    for (int k = 0; k < a->d; ++k) a->grad[(long)text[i] * a->d + k] += inv * a->d_ctx[k];
}

static long theta_count(int V, int d, int h) {
  return (long)V * d + 2L * h * d + h + (long)V * h + V;
}

/* grpo_gradient (grpo.cpp:122-206). Rollouts packed: tokens / old_lp are the
 * concatenation of the G rollouts (lengths[i] >= 1 each). stats = {objective,
 * mean_kl, clip_fraction, token_count}. Returns 0, or -1 on bad input. */
int oracle_grpo_gradient(const double* theta, const double* ref, int V, int d, int h,
                         const double* frame_emb, long n_frames, const int32_t* text, long n_text,
                         const int32_t* tokens, const long* lengths, long G, const double* old_lp,
                         const double* adv, double clip_eps, double kl_beta, int sampled_kl,
                         double* grad, double* stats) {
  if (G < 1) return -1;
  long n_tokens = 0;
  for (long i = 0; i < G; ++i) {
    if (lengths[i] < 1) return -1;
    n_tokens += lengths[i];
  }
  double* ctx_ref = (double*)malloc(sizeof(double) * (size_t)d);
  double* ctx_theta = (double*)malloc(sizeof(double) * (size_t)d);
  if (oracle_context_vector(ref, V, d, frame_emb, n_frames, text, n_text, ctx_ref) ||
      oracle_context_vector(theta, V, d, frame_emb, n_frames, text, n_text, ctx_theta)) {
    free(ctx_ref);
    free(ctx_theta);
    return -1;
  }
  memset(grad, 0, sizeof(double) * (size_t)theta_count(V, d, h));
  double* d_ctx = (double*)calloc((size_t)d, sizeof(double));
  grad_acc acc = {theta, V, d, h, ctx_theta, grad, d_ctx};
  double* lg = (double*)malloc(sizeof(double) * (size_t)V);
  double* lp = (double*)malloc(sizeof(double) * (size_t)V);
  double* lp_ref = (double*)malloc(sizeof(double) * (size_t)V);
  double* pi = (double*)malloc(sizeof(double) * (size_t)V);
  double* g = (double*)malloc(sizeof(double) * (size_t)V);
  double kl_sum = 0.0, policy_term = 0.0;
  long n_clipped = 0, o = 0;
  const double Gd = (double)G;
  const double kl_w = -kl_beta / (double)n_tokens;
  int bad = 0;
  for (long i = 0; i < G && !bad; ++i) {
    const double a = adv[i];
    const double tok_w = 1.0 / (Gd * (double)lengths[i]);
    double seq_term = 0.0;
    int prev = 1; /* Vocab::kEos */
    for (long t = 0; t < lengths[i]; ++t, ++o) {
      int y = tokens[o];
      if (y < 0 || y >= V) { bad = 1; break; }
      oracle_step_logits(theta, V, d, h, ctx_theta, prev, lg);
      oracle_log_softmax(lg, V, lp);
      oracle_step_logits(ref, V, d, h, ctx_ref, prev, lg);
      oracle_log_softmax(lg, V, lp_ref);
      for (int v = 0; v < V; ++v) pi[v] = exp(lp[v]);
      double ratio = exp(lp[y] - old_lp[o]);
      double lo = 1.0 - clip_eps, hi = 1.0 + clip_eps;
      double clipped = ratio < lo ? lo : (hi < ratio ? hi : ratio); /* std::clamp */
      double u1 = ratio * a, u2 = clipped * a;
      seq_term += u2 < u1 ? u2 : u1; /* std::min */
      int plateau = (a > 0 && ratio > 1.0 + clip_eps) || (a < 0 && ratio < 1.0 - clip_eps);
      if (plateau) ++n_clipped;
      for (int v = 0; v < V; ++v) g[v] = 0.0;
      if (a != 0.0 && !plateau) {
        double coeff = tok_w * a * ratio;
        for (int v = 0; v < V; ++v) g[v] -= coeff * pi[v];
        g[y] += coeff;
      }
      if (kl_beta != 0.0) {
        if (sampled_kl) {
          double lr = lp_ref[y] - lp[y];
          kl_sum += exp(lr) - 1.0 - lr;
          double coeff = kl_w * (1.0 - exp(lr));
          for (int v = 0; v < V; ++v) g[v] -= coeff * pi[v];
          g[y] += coeff;
        } else {
          double kl = 0.0;
          for (int v = 0; v < V; ++v) kl += pi[v] * (lp[v] - lp_ref[v]);
          kl_sum += kl;
          for (int v = 0; v < V; ++v) g[v] += kl_w * pi[v] * (lp[v] - lp_ref[v] - kl);
        }
      } else if (sampled_kl) {
        double lr = lp_ref[y] - lp[y];
        kl_sum += exp(lr) - 1.0 - lr;
      } else {
        double kl = 0.0;
        for (int v = 0; v < V; ++v) kl += pi[v] * (lp[v] - lp_ref[v]);
        kl_sum += kl;
      }
      acc_add_position(&acc, prev, g);
      prev = y;
    }
    policy_term += seq_term / (double)lengths[i] / Gd;
  }
  if (!bad) {
    acc_take(&acc, text, n_text, n_frames + n_text);
    stats[3] = (double)n_tokens;
    stats[1] = kl_sum / (double)n_tokens;
    stats[2] = (double)n_clipped / (double)n_tokens;
    stats[0] = policy_term - kl_beta * stats[1];
  }
  free(ctx_ref); free(ctx_theta); free(d_ctx); free(lg); free(lp); free(lp_ref); free(pi); free(g);
  return bad ? -1 : 0;
}

/* sft_loss_and_grad (grpo.cpp:208-223) */
int oracle_sft_loss_and_grad(const double* theta, int V, int d, int h, const double* frame_emb,
                             long n_frames, const int32_t* text, long n_text,
                             const int32_t* targets, long n_targets, double* loss, double* grad) {
  if (n_targets < 1) return -1;
  double* ctx = (double*)malloc(sizeof(double) * (size_t)d);
  if (oracle_context_vector(theta, V, d, frame_emb, n_frames, text, n_text, ctx)) {
    free(ctx);
    return -1;
  }
  memset(grad, 0, sizeof(double) * (size_t)theta_count(V, d, h));
  double* d_ctx = (double*)calloc((size_t)d, sizeof(double));
  grad_acc acc = {theta, V, d, h, ctx, grad, d_ctx};
  double* lg = (double*)malloc(sizeof(double) * (size_t)V);
  double* lp = (double*)malloc(sizeof(double) * (size_t)V);
  double* g = (double*)malloc(sizeof(double) * (size_t)V);
  const double inv_t = 1.0 / (double)n_targets;
  double l = 0.0;
  int prev = 1, bad = 0;
  for (long t = 0; t < n_targets; ++t) {
    int y = targets[t];
    if (y < 0 || y >= V) { bad = 1; break; }
    oracle_step_logits(theta, V, d, h, ctx, prev, lg);
    oracle_log_softmax(lg, V, lp);
    l += -lp[y];
    for (int v = 0; v < V; ++v) g[v] = inv_t * exp(lp[v]);
    g[y] -= inv_t;
    acc_add_position(&acc, prev, g);
    prev = y;
  }
  if (!bad) {
    acc_take(&acc, text, n_text, n_frames + n_text);
    *loss = l * inv_t;
  }
  free(ctx); free(d_ctx); free(lg); free(lp); free(g);
  return bad ? -1 : 0;
}
