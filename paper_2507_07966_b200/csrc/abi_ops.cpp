// abi_ops.cpp — C-ABI wrappers of the HBM-bound device operators (misc.h).
#include <cmath>

#include "common.h"
#include "misc.h"

using namespace mrsp;

namespace {
inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }
}  // namespace

extern "C" {

mrsp_status mrsp_op_rmsnorm(const float* x, int ldx, const float* w, void* out, int ldo, int n,
                            int d, float eps, const int32_t* rows, void* stream) {
  return guard([&] {
    require_device();
    rmsnorm(x, ldx, w, static_cast<__nv_bfloat16*>(out), ldo, n, d, eps, rows, S(stream));
  });
}

mrsp_status mrsp_op_layernorm(const float* x, int ldx, const float* w, const float* b, void* out,
                              int ldo, int n, int d, float eps, void* stream) {
  return guard([&] {
    require_device();
    layernorm(x, ldx, w, b, static_cast<__nv_bfloat16*>(out), ldo, n, d, eps, S(stream));
  });
}

mrsp_status mrsp_op_rope(void* qkv, int ld, int col0, int n_heads, const int32_t* pos, int n,
                         float theta, void* stream) {
  return guard([&] {
    require_device();
    float inv[64];
    rope_inv_freq(theta, inv);
    set_rope_inv_freq(inv, S(stream));
    rope(static_cast<__nv_bfloat16*>(qkv), ld, col0, n_heads, pos, n, S(stream));
  });
}

mrsp_status mrsp_op_patchify(const float* pixels, void* out, int F, int H, int W, int P, int kpad,
                             void* stream) {
  return guard([&] {
    require_device();
    MRSP_REQUIRE(kpad >= 3 * P * P && H % P == 0 && W % P == 0, MRSP_INVALID_ARGUMENT,
                 "patchify: bad geometry");
    patchify(pixels, static_cast<__nv_bfloat16*>(out), F, H, W, P, kpad, S(stream));
  });
}

mrsp_status mrsp_op_pack_sequence(const void* frame_emb, int n_frame_tok, const int32_t* question,
                                  int n_q, const int32_t* resp, const int32_t* lengths, int Lmax,
                                  const void* embed, int d, int64_t p0, int n, float* hidden,
                                  int32_t* pos_ids, uint8_t* pad_mask, int32_t* tokens,
                                  void* stream) {
  return guard([&] {
    require_device();
    pack_sequence(static_cast<const __nv_bfloat16*>(frame_emb), n_frame_tok, question, n_q, resp,
                  lengths, Lmax, static_cast<const __nv_bfloat16*>(embed), d, p0, n, hidden,
                  pos_ids, pad_mask, tokens, S(stream));
  });
}

}  // extern "C"
