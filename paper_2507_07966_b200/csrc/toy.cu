// toy.cu — the reference's own MR-SP model on the device, fp64, bit-exact.
//
// Kernels
//   toy_encode_kernel   encode_frame (policy.cpp:36-47) for a rank's frame range:
//                       e[f][r] = tanh(sum_k W[r][k] * x[f][k]), k ascending,
//                       each product and sum individually rounded (no FMA),
//                       tanh = glibc_tanh. One CTA per frame, one thread per r.
//   toy_prefill_kernel  step_logits (policy.cpp:85-119) for a rank's positions:
//                       s = tanh(c + sum_k (A[r][k] ctx[k] + B[r][k] E[prev][k]))
//                       logits[v] = b[v] + sum_r U[v][r] s[r].
// Both reproduce the reference's summation order exactly, so the device
// result equals the reference CPU bit for bit (tests/test_toy_gpu.py).
// Ranks are CUDA streams on the current device; each launches only its own
// ShardPlan range (engine.cpp:85-100, :117-129).
// The backward (GRPO / SFT gradients, grpo.cpp:122-223) is further down.
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "common.h"
#include "glibc_tanh.cuh"

namespace mrsp {
namespace {

__global__ void toy_encode_kernel(const double* __restrict__ w, const double* __restrict__ frames,
                                  double* __restrict__ out, int d, int p, uint64_t f_begin) {
  extern __shared__ double xs[];  // one frame
  const uint64_t f = f_begin + blockIdx.x;
  const double* x = frames + f * static_cast<uint64_t>(p);
  for (int k = threadIdx.x; k < p; k += blockDim.x) xs[k] = x[k];
  __syncthreads();
  for (int r = threadIdx.x; r < d; r += blockDim.x) {
    const double* row = w + static_cast<uint64_t>(r) * p;
    double z = 0.0;
    for (int k = 0; k < p; ++k) z = DADD(z, DMUL(row[k], xs[k]));
    out[f * static_cast<uint64_t>(d) + r] = glibc_tanh(z);
  }
}

struct Pos {
  uint32_t row;
  int32_t prev;
  uint64_t out_index;
};

__global__ void toy_prefill_kernel(const double* __restrict__ theta, const double* __restrict__ ctxs,
                                   const Pos* __restrict__ pos, double* __restrict__ out, int V,
                                   int d, int h) {
  extern __shared__ double sm[];
  double* ctx = sm;          // d
  double* e_prev = sm + d;   // d
  double* s = sm + 2 * d;    // h
  const Pos ps = pos[blockIdx.x];
  const double* E = theta;
  const double* A = theta + static_cast<uint64_t>(V) * d;
  const double* B = A + static_cast<uint64_t>(h) * d;
  const double* c = B + static_cast<uint64_t>(h) * d;
  const double* U = c + h;
  const double* bias = U + static_cast<uint64_t>(V) * h;
  for (int k = threadIdx.x; k < d; k += blockDim.x) {
    ctx[k] = ctxs[static_cast<uint64_t>(ps.row) * d + k];
    e_prev[k] = E[static_cast<uint64_t>(ps.prev) * d + k];
  }
  __syncthreads();
  for (int r = threadIdx.x; r < h; r += blockDim.x) {
    const double* arow = A + static_cast<uint64_t>(r) * d;
    const double* brow = B + static_cast<uint64_t>(r) * d;
    double z = c[r];
    for (int k = 0; k < d; ++k) z = DADD(z, DADD(DMUL(arow[k], ctx[k]), DMUL(brow[k], e_prev[k])));
    s[r] = glibc_tanh(z);
  }
  __syncthreads();
  for (int v = threadIdx.x; v < V; v += blockDim.x) {
    const double* urow = U + static_cast<uint64_t>(v) * h;
    double z = bias[v];
    for (int r = 0; r < h; ++r) z = DADD(z, DMUL(urow[r], s[r]));
    out[ps.out_index * static_cast<uint64_t>(V) + v] = z;
  }
}

// Per-process pool of rank streams (ranks = streams on the current device).
// Returns a copy of the first k handles taken under the lock: the pool only
// grows, and a concurrent caller growing it must not move a vector another
// thread is still indexing.
std::vector<cudaStream_t> rank_streams(int k) {
  static std::mutex mu;
  static std::vector<cudaStream_t> pool;
  std::lock_guard<std::mutex> lock(mu);
  while (static_cast<int>(pool.size()) < k) {
    cudaStream_t s;
    MRSP_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    pool.push_back(s);
  }
  return std::vector<cudaStream_t>(pool.begin(), pool.begin() + k);
}

template <typename T>
struct DevBuf {
  T* p = nullptr;
  explicit DevBuf(size_t n) {
    if (n) MRSP_CUDA(cudaMalloc(&p, n * sizeof(T)));
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

void check_plan(const uint64_t* ranges, int k, uint64_t total, const char* who) {
  uint64_t cursor = 0;
  for (int w = 0; w < k; ++w) {
    MRSP_REQUIRE(ranges[2 * w] <= ranges[2 * w + 1] && ranges[2 * w + 1] <= total,
                 MRSP_INVALID_ARGUMENT, std::string(who) + ": malformed plan range");
    MRSP_REQUIRE(ranges[2 * w] == cursor, MRSP_INVALID_ARGUMENT,
                 std::string(who) + ": plan ranges are not a contiguous partition");
    cursor = ranges[2 * w + 1];
  }
  MRSP_REQUIRE(cursor == total, MRSP_INVALID_ARGUMENT,
               std::string(who) + ": plan does not cover its items");
}


// ---------------------------------------------------------------------------
// Backward: the GRPO / SFT gradients of the toy policy,
// grpo.cpp:122-223 over policy.cpp:195-260 (GradAccumulator).
//
//   toy_ctx_kernel       context_vector (policy.cpp:63-80) for theta and ref.
//   toy_grad_pos_kernel  one CTA per teacher-forced position, positions sharded
//                        over the ranks' ShardPlan ranges exactly as prefill:
//                        hidden state, both models' logits, log-softmax, the
//                        ratio / clip / KL terms and the logit gradient g (V),
//                        then ds = U^T g and dz = ds (1 - s^2). Writes g, s, dz
//                        and the position's scalar terms at its packed index.
//   toy_grad_reduce_kernel  one thread per parameter (plus d for d_context):
//                        the GradAccumulator sums over positions in the
//                        reference's serial (rollout, t) order, with its
//                        zero skips — so the gradient has the same bits for
//                        every SP degree.
//   toy_grad_finish_kernel  take(): text rows += d_context / total_len, and
//                        the GroupStats / SFT loss in serial order.
// Arithmetic is explicitly rounded (no contraction) in the reference's
// operation order; tanh is glibc's (bit-exact), exp / log are CUDA's (<= 1
// ulp), so the device gradient equals the reference's within fp64 rounding.
struct GradPos {
  int32_t prev, y, row, pad_;
  uint64_t o;  // packed index: row_off[row] + t
};

struct GradCfg {
  int sft;         // 1: sft_loss_and_grad, 0: grpo_gradient
  int sampled_kl;
  double clip_eps, kl_beta, kl_w;  // kl_w = -kl_beta / n_tokens (grpo.cpp:137)
};

__global__ void toy_ctx_kernel(const double* __restrict__ theta, const double* __restrict__ ref,
                               int d, const double* __restrict__ frames, uint64_t n_frames,
                               const int32_t* __restrict__ text, uint64_t n_text,
                               double* __restrict__ ctx_t, double* __restrict__ ctx_r) {
  const double inv = DDIV(1.0, static_cast<double>(n_frames + n_text));
  for (int k = threadIdx.x; k < d; k += blockDim.x) {
    for (int m = 0; m < 2; ++m) {
      const double* E = m ? ref : theta;
      if (E == nullptr) continue;
      double z = 0.0;
      for (uint64_t f = 0; f < n_frames; ++f) z = DADD(z, frames[f * d + k]);
      for (uint64_t i = 0; i < n_text; ++i) z = DADD(z, E[static_cast<uint64_t>(text[i]) * d + k]);
      (m ? ctx_r : ctx_t)[k] = DMUL(z, inv);
    }
  }
}

__device__ __forceinline__ double dmax(double m, double v) { return m < v ? v : m; }  // std::max

// log_softmax (common.hpp:95-104), serial, in place
__device__ void log_softmax_serial(double* x, int n) {
  double m = x[0];
  for (int i = 0; i < n; ++i) m = dmax(m, x[i]);
  double z = 0.0;
  for (int i = 0; i < n; ++i) z = DADD(z, exp(DSUB(x[i], m)));
  const double lz = DADD(m, log(z));
  for (int i = 0; i < n; ++i) x[i] = DSUB(x[i], lz);
}

__global__ void toy_grad_pos_kernel(const double* __restrict__ theta,
                                    const double* __restrict__ ref, int V, int d, int h,
                                    const double* __restrict__ ctx_t,
                                    const double* __restrict__ ctx_r,
                                    const GradPos* __restrict__ pos,
                                    const double* __restrict__ old_lp,
                                    const double* __restrict__ adv,
                                    const double* __restrict__ tok_w, GradCfg cfg,
                                    double* __restrict__ g_out, double* __restrict__ s_out,
                                    double* __restrict__ dz_out, double* __restrict__ scal) {
  extern __shared__ double sm[];
  double* e_t = sm;          // d: E_theta[prev]
  double* e_r = e_t + d;     // d: E_ref[prev]
  double* s_t = e_r + d;     // h
  double* s_r = s_t + h;     // h
  double* lp = s_r + h;      // V: logits, then log-probs (theta)
  double* lq = lp + V;       // V: (ref)
  double* pi = lq + V;       // V
  double* g = pi + V;        // V
  const GradPos ps = pos[blockIdx.x];
  const bool two = !cfg.sft;
  for (int k = threadIdx.x; k < d; k += blockDim.x) {
    e_t[k] = theta[static_cast<uint64_t>(ps.prev) * d + k];
    if (two) e_r[k] = ref[static_cast<uint64_t>(ps.prev) * d + k];
  }
  __syncthreads();
  // hidden_state (policy.cpp:85-101) for both models
  for (int j = threadIdx.x; j < (two ? 2 : 1) * h; j += blockDim.x) {
    const int m = j / h, r = j % h;
    const double* P = m ? ref : theta;
    const double* ctx = m ? ctx_r : ctx_t;
    const double* e = m ? e_r : e_t;
    const double* A = P + static_cast<uint64_t>(V) * d;
    const double* B = A + static_cast<uint64_t>(h) * d;
    const double* c = B + static_cast<uint64_t>(h) * d;
    double z = c[r];
    for (int k = 0; k < d; ++k)
      z = DADD(z, DADD(DMUL(A[static_cast<uint64_t>(r) * d + k], ctx[k]),
                       DMUL(B[static_cast<uint64_t>(r) * d + k], e[k])));
    (m ? s_r : s_t)[r] = glibc_tanh(z);
  }
  __syncthreads();
  // step_logits (policy.cpp:103-119)
  for (int j = threadIdx.x; j < (two ? 2 : 1) * V; j += blockDim.x) {
    const int m = j / V, v = j % V;
    const double* P = m ? ref : theta;
    const double* U = P + static_cast<uint64_t>(V) * d + 2ull * h * d + h;
    const double* b = U + static_cast<uint64_t>(V) * h;
    const double* s = m ? s_r : s_t;
    double z = b[v];
    for (int r = 0; r < h; ++r) z = DADD(z, DMUL(U[static_cast<uint64_t>(v) * h + r], s[r]));
    (m ? lq : lp)[v] = z;
  }
  __syncthreads();
  // token terms and the logit gradient (grpo.cpp:150-196 / :214-220), serial
  if (threadIdx.x == 0) {
    const int y = ps.y;
    log_softmax_serial(lp, V);
    for (int v = 0; v < V; ++v) g[v] = 0.0;
    double* sc = scal + ps.o * 4;
    if (cfg.sft) {
      const double inv_t = tok_w[0];
      sc[0] = lp[y];
      for (int v = 0; v < V; ++v) g[v] = DMUL(inv_t, exp(lp[v]));
      g[y] = DSUB(g[y], inv_t);
    } else {
      log_softmax_serial(lq, V);
      for (int v = 0; v < V; ++v) pi[v] = exp(lp[v]);
      const double a = adv[ps.row];
      const double ratio = exp(DSUB(lp[y], old_lp[ps.o]));
      const double lo = DSUB(1.0, cfg.clip_eps), hi = DADD(1.0, cfg.clip_eps);
      const double clipped = ratio < lo ? lo : (hi < ratio ? hi : ratio);  // std::clamp
      const double u1 = DMUL(ratio, a), u2 = DMUL(clipped, a);
      sc[0] = u2 < u1 ? u2 : u1;  // std::min
      const bool plateau = (a > 0 && ratio > hi) || (a < 0 && ratio < lo);
      sc[2] = plateau ? 1.0 : 0.0;
      if (a != 0.0 && !plateau) {
        const double coeff = DMUL(DMUL(tok_w[ps.row], a), ratio);
        for (int v = 0; v < V; ++v) g[v] = DSUB(g[v], DMUL(coeff, pi[v]));
        g[y] = DADD(g[y], coeff);
      }
      double klt;
      if (cfg.sampled_kl) {
        const double lr = DSUB(lq[y], lp[y]);
        klt = DSUB(DSUB(exp(lr), 1.0), lr);
        if (cfg.kl_beta != 0.0) {
          const double coeff = DMUL(cfg.kl_w, DSUB(1.0, exp(lr)));
          for (int v = 0; v < V; ++v) g[v] = DSUB(g[v], DMUL(coeff, pi[v]));
          g[y] = DADD(g[y], coeff);
        }
      } else {
        double kl = 0.0;
        for (int v = 0; v < V; ++v) kl = DADD(kl, DMUL(pi[v], DSUB(lp[v], lq[v])));
        klt = kl;
        if (cfg.kl_beta != 0.0)
          for (int v = 0; v < V; ++v)
            g[v] = DADD(g[v], DMUL(DMUL(cfg.kl_w, pi[v]), DSUB(DSUB(lp[v], lq[v]), kl)));
      }
      sc[1] = klt;
    }
  }
  __syncthreads();
  for (int v = threadIdx.x; v < V; v += blockDim.x) g_out[ps.o * V + v] = g[v];
  // add_position (policy.cpp:202-247): ds = U^T g over nonzero g, dz = ds (1 - s^2)
  const double* U = theta + static_cast<uint64_t>(V) * d + 2ull * h * d + h;
  for (int r = threadIdx.x; r < h; r += blockDim.x) {
    double ds = 0.0;
    for (int v = 0; v < V; ++v) {
      const double gv = g[v];
      if (gv == 0.0) continue;
      ds = DADD(ds, DMUL(gv, U[static_cast<uint64_t>(v) * h + r]));
    }
    const double sr = s_t[r];
    s_out[ps.o * h + r] = sr;
    dz_out[ps.o * h + r] = DMUL(ds, DSUB(1.0, DMUL(sr, sr)));
  }
}

// One thread per theta element (then d threads for d_context): the
// accumulator's sums over positions p = 0..P-1 in serial order.
__global__ void toy_grad_reduce_kernel(const double* __restrict__ theta, int V, int d, int h,
                                       const double* __restrict__ ctx_t,
                                       const GradPos* __restrict__ pos, uint64_t P,
                                       const double* __restrict__ g, const double* __restrict__ s,
                                       const double* __restrict__ dz, double* __restrict__ grad,
                                       double* __restrict__ d_ctx) {
  const uint64_t nE = static_cast<uint64_t>(V) * d, nA = static_cast<uint64_t>(h) * d;
  const uint64_t oA = nE, oB = oA + nA, oc = oB + nA, oU = oc + h,
                 ob = oU + static_cast<uint64_t>(V) * h, n = ob + V;
  const uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n + d) return;
  const double* A = theta + oA;
  const double* B = theta + oB;
  double acc = 0.0;
  if (j < oA) {  // E_txt[t][k] += dz * B[r][k] at positions with prev == t
    const int t = static_cast<int>(j / d), k = static_cast<int>(j % d);
    for (uint64_t p = 0; p < P; ++p) {
      if (pos[p].prev != t) continue;
      for (int r = 0; r < h; ++r) {
        const double z = dz[pos[p].o * h + r];
        if (z == 0.0) continue;
        acc = DADD(acc, DMUL(z, B[static_cast<uint64_t>(r) * d + k]));
      }
    }
  } else if (j < oc) {  // A[r][k] += dz ctx[k];  B[r][k] += dz E[prev][k]
    const bool isB = j >= oB;
    const uint64_t jj = j - (isB ? oB : oA);
    const int r = static_cast<int>(jj / d), k = static_cast<int>(jj % d);
    for (uint64_t p = 0; p < P; ++p) {
      const double z = dz[pos[p].o * h + r];
      if (z == 0.0) continue;
      const double x = isB ? theta[static_cast<uint64_t>(pos[p].prev) * d + k] : ctx_t[k];
      acc = DADD(acc, DMUL(z, x));
    }
  } else if (j < oU) {  // c[r] += dz
    const int r = static_cast<int>(j - oc);
    for (uint64_t p = 0; p < P; ++p) {
      const double z = dz[pos[p].o * h + r];
      if (z != 0.0) acc = DADD(acc, z);
    }
  } else if (j < ob) {  // U[v][r] += g s[r]
    const int v = static_cast<int>((j - oU) / h), r = static_cast<int>((j - oU) % h);
    for (uint64_t p = 0; p < P; ++p) {
      const double gv = g[pos[p].o * V + v];
      if (gv != 0.0) acc = DADD(acc, DMUL(gv, s[pos[p].o * h + r]));
    }
  } else if (j < n) {  // b[v] += g
    const int v = static_cast<int>(j - ob);
    for (uint64_t p = 0; p < P; ++p) {
      const double gv = g[pos[p].o * V + v];
      if (gv != 0.0) acc = DADD(acc, gv);
    }
  } else {  // d_context[k] += dz A[r][k]
    const int k = static_cast<int>(j - n);
    for (uint64_t p = 0; p < P; ++p)
      for (int r = 0; r < h; ++r) {
        const double z = dz[pos[p].o * h + r];
        if (z == 0.0) continue;
        acc = DADD(acc, DMUL(z, A[static_cast<uint64_t>(r) * d + k]));
      }
    d_ctx[k] = acc;
    return;
  }
  grad[j] = acc;
}

// take() (policy.cpp:249-260) + GroupStats (grpo.cpp:198-205) / SFT loss
__global__ void toy_grad_finish_kernel(int V, int d, const int32_t* __restrict__ text,
                                       uint64_t n_text, double inv_total,
                                       const double* __restrict__ d_ctx,
                                       double* __restrict__ grad, const double* __restrict__ scal,
                                       const uint64_t* __restrict__ row_off, uint64_t n_rows,
                                       GradCfg cfg, double* __restrict__ stats) {
  const uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j < static_cast<uint64_t>(V) * d) {
    const int t = static_cast<int>(j / d), k = static_cast<int>(j % d);
    double x = grad[j];
    for (uint64_t i = 0; i < n_text; ++i)
      if (text[i] == t) x = DADD(x, DMUL(inv_total, d_ctx[k]));
    grad[j] = x;
  }
  if (j != 0) return;
  const uint64_t n_tok = row_off[n_rows];
  if (cfg.sft) {
    double loss = 0.0;
    for (uint64_t o = 0; o < n_tok; ++o) loss = DSUB(loss, scal[o * 4]);
    stats[0] = DMUL(loss, DDIV(1.0, static_cast<double>(n_tok)));
    return;
  }
  const double G = static_cast<double>(n_rows);
  double policy_term = 0.0, kl_sum = 0.0, n_clip = 0.0;
  for (uint64_t i = 0; i < n_rows; ++i) {
    double seq = 0.0;
    for (uint64_t o = row_off[i]; o < row_off[i + 1]; ++o) {
      seq = DADD(seq, scal[o * 4]);
      kl_sum = DADD(kl_sum, scal[o * 4 + 1]);
      n_clip += scal[o * 4 + 2];
    }
    policy_term = DADD(policy_term,
                       DDIV(DDIV(seq, static_cast<double>(row_off[i + 1] - row_off[i])), G));
  }
  const double mean_kl = DDIV(kl_sum, static_cast<double>(n_tok));
  stats[1] = mean_kl;
  stats[2] = DDIV(n_clip, static_cast<double>(n_tok));
  stats[3] = static_cast<double>(n_tok);
  stats[0] = DSUB(policy_term, DMUL(cfg.kl_beta, mean_kl));
}

// Host driver shared by grpo_gradient and sft_loss_and_grad.
void toy_backward(int sp_degree, const double* theta, const double* ref, int V, int d, int h,
                  const double* frame_emb, uint64_t n_frames, const int32_t* text,
                  uint64_t n_text, const int32_t* tokens, const uint64_t* lengths,
                  uint64_t n_rows, const double* old_lp, const double* adv, GradCfg cfg,
                  const uint64_t* ranges, double* grad, double* stats) {
  const char* who = cfg.sft ? "sft_loss_and_grad" : "grpo";
  MRSP_REQUIRE(sp_degree >= 1, MRSP_INVALID_ARGUMENT, "WorkerGroup: sp_degree must be >= 1");
  MRSP_REQUIRE(V >= 1 && d >= 1 && h >= 1, MRSP_INVALID_ARGUMENT,
               std::string(who) + ": bad policy dims");
  MRSP_REQUIRE(n_rows >= 1, MRSP_INVALID_ARGUMENT,
               cfg.sft ? "sft_loss_and_grad: empty targets" : "grpo: empty rollout group");
  MRSP_REQUIRE(n_frames + n_text > 0, MRSP_INVALID_ARGUMENT, "context_vector: empty sequence");
  for (uint64_t i = 0; i < n_text; ++i)
    MRSP_REQUIRE(text[i] >= 0 && text[i] < V, MRSP_INVALID_ARGUMENT,
                 "context_vector: token out of range");
  std::vector<uint64_t> row_off(n_rows + 1, 0);
  uint64_t max_len = 0;
  for (uint64_t i = 0; i < n_rows; ++i) {
    MRSP_REQUIRE(lengths[i] >= 1, MRSP_INVALID_ARGUMENT,
                 cfg.sft ? "sft_loss_and_grad: empty targets" : "grpo: empty rollout");
    row_off[i + 1] = row_off[i] + lengths[i];
    max_len = std::max<uint64_t>(max_len, lengths[i]);
  }
  const uint64_t P = row_off[n_rows];
  for (uint64_t o = 0; o < P; ++o)
    MRSP_REQUIRE(tokens[o] >= 0 && tokens[o] < V, MRSP_INVALID_ARGUMENT,
                 cfg.sft ? "sft_loss_and_grad: token out of range"
                         : "grpo: token out of range");
  MRSP_REQUIRE(V > 1, MRSP_INVALID_ARGUMENT,
               "step_logits: prev token out of range");  // prev = EOS (1) at t = 0
  check_plan(ranges, sp_degree, max_len, cfg.sft ? "sft_loss_and_grad" : "grpo_gradient");
  require_device();
  // positions in the serial (row, t) order, and each rank's ShardPlan slice
  std::vector<GradPos> all(P);
  for (uint64_t i = 0; i < n_rows; ++i)
    for (uint64_t t = 0; t < lengths[i]; ++t) {
      const uint64_t o = row_off[i] + t;
      all[o] = GradPos{t == 0 ? 1 : tokens[o - 1], tokens[o], static_cast<int32_t>(i), 0, o};
    }
  std::vector<GradPos> by_rank;
  std::vector<uint64_t> rank_off(sp_degree + 1, 0);
  for (int w = 0; w < sp_degree; ++w) {
    for (uint64_t i = 0; i < n_rows; ++i) {
      const uint64_t stop = std::min(ranges[2 * w + 1], lengths[i]);
      for (uint64_t t = ranges[2 * w]; t < stop; ++t) by_rank.push_back(all[row_off[i] + t]);
    }
    rank_off[w + 1] = by_rank.size();
  }
  std::vector<double> tok_w(cfg.sft ? 1 : n_rows);
  if (cfg.sft)
    tok_w[0] = 1.0 / static_cast<double>(P);  // grpo.cpp:212
  else
    for (uint64_t i = 0; i < n_rows; ++i)  // grpo.cpp:142
      tok_w[i] = 1.0 / (static_cast<double>(n_rows) * static_cast<double>(lengths[i]));
  const uint64_t n_theta = static_cast<uint64_t>(V) * d + 2ull * h * d + h +
                           static_cast<uint64_t>(V) * h + V;
  const auto streams = rank_streams(sp_degree);
  cudaStream_t s0 = streams[0];
  DevBuf<double> dth(n_theta), dref(cfg.sft ? 0 : n_theta), dfr(n_frames * d), dctx(2 * d),
      dold(cfg.sft ? 0 : P), dadv(cfg.sft ? 0 : n_rows), dtw(tok_w.size()), dg(P * V), ds(P * h),
      ddz(P * h), dscal(P * 4), dgrad(n_theta), ddctx(d), dstats(4);
  DevBuf<int32_t> dtext(n_text);
  DevBuf<GradPos> dall(P), drank(P);
  DevBuf<uint64_t> drow(n_rows + 1);
  auto h2d = [&](void* dst, const void* src, size_t bytes) {
    if (bytes) MRSP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s0));
  };
  h2d(dth.p, theta, sizeof(double) * n_theta);
  if (!cfg.sft) {
    h2d(dref.p, ref, sizeof(double) * n_theta);
    h2d(dold.p, old_lp, sizeof(double) * P);
    h2d(dadv.p, adv, sizeof(double) * n_rows);
  }
  h2d(dfr.p, frame_emb, sizeof(double) * n_frames * d);
  h2d(dtext.p, text, sizeof(int32_t) * n_text);
  h2d(dtw.p, tok_w.data(), sizeof(double) * tok_w.size());
  h2d(dall.p, all.data(), sizeof(GradPos) * P);
  h2d(drank.p, by_rank.data(), sizeof(GradPos) * P);
  h2d(drow.p, row_off.data(), sizeof(uint64_t) * (n_rows + 1));
  toy_ctx_kernel<<<1, std::min(256, ((d + 31) / 32) * 32), 0, s0>>>(
      dth.p, cfg.sft ? nullptr : dref.p, d, dfr.p, n_frames, dtext.p, n_text, dctx.p, dctx.p + d);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
  cudaEvent_t ready;
  MRSP_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  MRSP_CUDA(cudaEventRecord(ready, s0));
  const int threads = std::min(256, ((std::max(std::max(2 * V, 2 * h), d) + 31) / 32) * 32);
  const size_t smem = sizeof(double) * (2 * d + 2 * h + 4 * V);
  for (int w = 0; w < sp_degree; ++w) {
    const uint64_t n = rank_off[w + 1] - rank_off[w];
    if (n == 0) continue;
    MRSP_CUDA(cudaStreamWaitEvent(streams[w], ready, 0));
    toy_grad_pos_kernel<<<static_cast<unsigned>(n), threads, smem, streams[w]>>>(
        dth.p, cfg.sft ? dth.p : dref.p, V, d, h, dctx.p, dctx.p + d, drank.p + rank_off[w],
        dold.p, dadv.p, dtw.p, cfg, dg.p, ds.p, ddz.p, dscal.p);
    count_launch();
    MRSP_CUDA(cudaGetLastError());
  }
  // join the ranks, then reduce in the serial position order on rank 0's stream
  std::vector<cudaEvent_t> done(sp_degree);
  for (int w = 0; w < sp_degree; ++w) {
    MRSP_CUDA(cudaEventCreateWithFlags(&done[w], cudaEventDisableTiming));
    MRSP_CUDA(cudaEventRecord(done[w], streams[w]));
    MRSP_CUDA(cudaStreamWaitEvent(s0, done[w], 0));
  }
  const unsigned rb = static_cast<unsigned>((n_theta + d + 127) / 128);
  toy_grad_reduce_kernel<<<rb, 128, 0, s0>>>(dth.p, V, d, h, dctx.p, dall.p, P, dg.p, ds.p, ddz.p,
                                             dgrad.p, ddctx.p);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
  const uint64_t nE = static_cast<uint64_t>(V) * d;
  toy_grad_finish_kernel<<<static_cast<unsigned>((nE + 127) / 128), 128, 0, s0>>>(
      V, d, dtext.p, n_text, 1.0 / static_cast<double>(n_frames + n_text), ddctx.p, dgrad.p,
      dscal.p, drow.p, n_rows, cfg, dstats.p);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
  MRSP_CUDA(cudaMemcpyAsync(grad, dgrad.p, sizeof(double) * n_theta, cudaMemcpyDeviceToHost, s0));
  MRSP_CUDA(cudaMemcpyAsync(stats, dstats.p, sizeof(double) * (cfg.sft ? 1 : 4),
                            cudaMemcpyDeviceToHost, s0));
  MRSP_CUDA(cudaStreamSynchronize(s0));
  cudaEventDestroy(ready);
  for (auto e : done) cudaEventDestroy(e);
}

}  // namespace
}  // namespace mrsp

using namespace mrsp;

extern "C" mrsp_status mrsp_toy_encode(int sp_degree, const double* enc_w, int d, int p,
                                       const double* frames, uint64_t n_frames,
                                       const uint64_t* ranges, double* out,
                                       uint64_t* rank_items) {
  return guard([&] {
    MRSP_REQUIRE(sp_degree >= 1, MRSP_INVALID_ARGUMENT, "WorkerGroup: sp_degree must be >= 1");
    MRSP_REQUIRE(d >= 1 && p >= 1, MRSP_INVALID_ARGUMENT, "encode_frame: frame dimension mismatch");
    check_plan(ranges, sp_degree, n_frames, "parallel_encode");
    require_device();
    if (n_frames == 0) {
      for (int w = 0; w < sp_degree; ++w) rank_items[w] = 0;
      return;
    }
    const auto streams = rank_streams(sp_degree);
    DevBuf<double> dw(static_cast<size_t>(d) * p), dx(n_frames * p), dout(n_frames * d);
    MRSP_CUDA(cudaMemcpyAsync(dw.p, enc_w, sizeof(double) * d * p, cudaMemcpyHostToDevice, streams[0]));
    MRSP_CUDA(cudaMemcpyAsync(dx.p, frames, sizeof(double) * n_frames * p, cudaMemcpyHostToDevice,
                              streams[0]));
    cudaEvent_t ready;
    MRSP_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    MRSP_CUDA(cudaEventRecord(ready, streams[0]));
    const int threads = std::min(256, ((d + 31) / 32) * 32);
    for (int w = 0; w < sp_degree; ++w) {
      const uint64_t b = ranges[2 * w], e = ranges[2 * w + 1];
      rank_items[w] = e - b;
      if (e == b) continue;
      MRSP_CUDA(cudaStreamWaitEvent(streams[w], ready, 0));
      toy_encode_kernel<<<static_cast<unsigned>(e - b), threads, sizeof(double) * p, streams[w]>>>(
          dw.p, dx.p, dout.p, d, p, b);
      count_launch();
      MRSP_CUDA(cudaGetLastError());
      // each rank's slice lands in its own range of the gathered buffer
      MRSP_CUDA(cudaMemcpyAsync(out + b * d, dout.p + b * d, sizeof(double) * (e - b) * d,
                                cudaMemcpyDeviceToHost, streams[w]));
    }
    for (int w = 0; w < sp_degree; ++w) MRSP_CUDA(cudaStreamSynchronize(streams[w]));
    cudaEventDestroy(ready);
  });
}

extern "C" mrsp_status mrsp_toy_prefill(int sp_degree, const double* theta, int V, int d, int h,
                                        const double* contexts, const int32_t* rows,
                                        const uint64_t* lengths, uint64_t n_rows,
                                        uint64_t max_len, const uint64_t* ranges, double* out,
                                        uint64_t* pad_reads) {
  return guard([&] {
    MRSP_REQUIRE(sp_degree >= 1, MRSP_INVALID_ARGUMENT, "WorkerGroup: sp_degree must be >= 1");
    MRSP_REQUIRE(V >= 1 && d >= 1 && h >= 1, MRSP_INVALID_ARGUMENT, "prefill: bad policy dims");
    check_plan(ranges, sp_degree, max_len, "parallel_prefill");
    require_device();
    *pad_reads = 0;
    // Output offsets of each row in the packed [sum(len)][V] result.
    std::vector<uint64_t> row_off(n_rows + 1, 0);
    for (uint64_t r = 0; r < n_rows; ++r) {
      MRSP_REQUIRE(lengths[r] <= max_len, MRSP_INVALID_ARGUMENT, "prefill: row longer than max_len");
      row_off[r + 1] = row_off[r] + lengths[r];
    }
    const uint64_t total = row_off[n_rows];
    if (total == 0) return;
    // Each rank's position list: t in [b, min(e, len_r)) for every row
    // (engine.cpp:120-123); prev is read only below len_r, so no pad reads.
    std::vector<std::vector<Pos>> plist(sp_degree);
    for (int w = 0; w < sp_degree; ++w) {
      const uint64_t b = ranges[2 * w], e = ranges[2 * w + 1];
      for (uint64_t r = 0; r < n_rows; ++r) {
        const uint64_t stop = std::min(e, static_cast<uint64_t>(lengths[r]));
        for (uint64_t t = b; t < stop; ++t) {
          int32_t prev = 1;  // Vocab::kEos
          if (t > 0) {
            if (t - 1 >= lengths[r]) ++*pad_reads;
            prev = rows[r * max_len + t - 1];
          }
          MRSP_REQUIRE(prev >= 0 && prev < V, MRSP_INVALID_ARGUMENT,
                       "step_logits: prev token out of range");
          plist[w].push_back(Pos{static_cast<uint32_t>(r), prev, row_off[r] + t});
        }
      }
    }
    const uint64_t n_theta = static_cast<uint64_t>(V) * d + 2ull * h * d + h +
                             static_cast<uint64_t>(V) * h + V;
    const auto streams = rank_streams(sp_degree);
    DevBuf<double> dtheta(n_theta), dctx(n_rows * d), dout(total * V);
    DevBuf<Pos> dpos(total);
    MRSP_CUDA(cudaMemcpyAsync(dtheta.p, theta, sizeof(double) * n_theta, cudaMemcpyHostToDevice,
                              streams[0]));
    MRSP_CUDA(cudaMemcpyAsync(dctx.p, contexts, sizeof(double) * n_rows * d, cudaMemcpyHostToDevice,
                              streams[0]));
    uint64_t off = 0;
    std::vector<uint64_t> pos_off(sp_degree);
    for (int w = 0; w < sp_degree; ++w) {
      pos_off[w] = off;
      if (!plist[w].empty())
        MRSP_CUDA(cudaMemcpyAsync(dpos.p + off, plist[w].data(), sizeof(Pos) * plist[w].size(),
                                  cudaMemcpyHostToDevice, streams[0]));
      off += plist[w].size();
    }
    cudaEvent_t ready;
    MRSP_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    MRSP_CUDA(cudaEventRecord(ready, streams[0]));
    const int threads = std::min(256, ((std::max(std::max(V, h), d) + 31) / 32) * 32);
    const size_t smem = sizeof(double) * (2 * d + h);
    for (int w = 0; w < sp_degree; ++w) {
      if (plist[w].empty()) continue;
      MRSP_CUDA(cudaStreamWaitEvent(streams[w], ready, 0));
      toy_prefill_kernel<<<static_cast<unsigned>(plist[w].size()), threads, smem, streams[w]>>>(
          dtheta.p, dctx.p, dpos.p + pos_off[w], dout.p, V, d, h);
      count_launch();
      MRSP_CUDA(cudaGetLastError());
    }
    for (int w = 0; w < sp_degree; ++w) MRSP_CUDA(cudaStreamSynchronize(streams[w]));
    MRSP_CUDA(cudaMemcpy(out, dout.p, sizeof(double) * total * V, cudaMemcpyDeviceToHost));
    cudaEventDestroy(ready);
  });
}

extern "C" mrsp_status mrsp_toy_grpo_gradient(
    int sp_degree, const double* theta, const double* ref, int V, int d, int h,
    const double* frame_emb, uint64_t n_frames, const int32_t* text_tokens, uint64_t n_text,
    const int32_t* tokens, const uint64_t* lengths, uint64_t n_rollouts,
    const double* old_logprobs, const double* advantages, double clip_eps, double kl_beta,
    int sampled_kl, const uint64_t* ranges, double* grad, double* stats) {
  return guard([&] {
    uint64_t n_tok = 0;
    for (uint64_t i = 0; i < n_rollouts; ++i) n_tok += lengths[i];
    GradCfg cfg{0, sampled_kl, clip_eps, kl_beta,
                n_tok ? -kl_beta / static_cast<double>(n_tok) : 0.0};
    toy_backward(sp_degree, theta, ref, V, d, h, frame_emb, n_frames, text_tokens, n_text, tokens,
                 lengths, n_rollouts, old_logprobs, advantages, cfg, ranges, grad, stats);
  });
}

extern "C" mrsp_status mrsp_toy_sft_loss_and_grad(int sp_degree, const double* theta, int V,
                                                  int d, int h, const double* frame_emb,
                                                  uint64_t n_frames, const int32_t* text_tokens,
                                                  uint64_t n_text, const int32_t* targets,
                                                  uint64_t n_targets, const uint64_t* ranges,
                                                  double* loss, double* grad) {
  return guard([&] {
    MRSP_REQUIRE(n_targets >= 1, MRSP_INVALID_ARGUMENT, "sft_loss_and_grad: empty targets");
    GradCfg cfg{1, 0, 0.0, 0.0, 0.0};
    toy_backward(sp_degree, theta, nullptr, V, d, h, frame_emb, n_frames, text_tokens, n_text,
                 targets, &n_targets, 1, nullptr, nullptr, cfg, ranges, grad, loss);
  });
}
