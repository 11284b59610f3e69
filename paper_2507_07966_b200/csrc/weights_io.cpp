// weights_io.cpp — engine weights to / from safetensors (SURVEY §8f rank 4:
// the on-disk format either side of the path).
//
// Tensor names follow the Hugging Face conventions of the model families the
// engine is shaped after, so a real checkpoint maps without renaming:
//   SigLIP tower    vision_model.embeddings.{patch_embedding,position_embedding}.*,
//                   vision_model.encoder.layers.N.{layer_norm1,self_attn.{q,k,v,out}_proj,
//                   layer_norm2,mlp.fc1,mlp.fc2}.*, vision_model.post_layernorm.*
//   projector       mm_projector.{0,2}.{weight,bias}   (Linear, GELU, Linear)
//   Qwen2 LLM       model.embed_tokens.weight, model.layers.N.{input_layernorm,
//                   self_attn.{q,k,v,o}_proj, post_attention_layernorm,
//                   mlp.{gate,up,down}_proj}.*, model.norm.weight, lm_head.weight
// (the reference model of the GRPO pair is saved with the prefix "ref.").
// Logical tensors are the unpadded HF shapes; the engine's storage transforms
// (q/k/v concatenation, gate/up interleaved in 128-row blocks, vision heads at
// the engine's head stride, patch K padded to a multiple of 8) are described per
// tensor as 2-D strided segments, so save and load are exact inverses.
#include <cuda_runtime.h>

#include <algorithm>
#include <cctype>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "common.h"
#include "engine.h"

namespace mrsp {
namespace {

enum DType { BF16 = 0, F32 = 1 };

// One 2-D piece of a logical tensor: `rows` rows of `width` bytes, at
// `log_off` + r * `log_pitch` in the contiguous logical tensor and at
// `dev` + r * `dev_pitch` in engine storage.
struct Seg {
  void* dev;
  size_t dev_pitch, log_off, log_pitch, width, rows;
};
struct TensorDesc {
  std::string name;
  DType dtype;
  std::vector<long> shape;
  std::vector<Seg> segs;
  size_t bytes() const {
    size_t n = dtype == BF16 ? 2 : 4;
    for (long s : shape) n *= static_cast<size_t>(s);
    return n;
  }
};

Seg contiguous(void* dev, size_t bytes) { return Seg{dev, bytes, 0, bytes, bytes, 1}; }

// ---- minimal JSON reader for the safetensors header ------------------------
struct JsonTensor {
  std::string dtype;
  std::vector<long> shape;
  size_t begin = 0, end = 0;
};

class HeaderParser {
 public:
  explicit HeaderParser(const std::string& s) : s_(s) {}
  std::map<std::string, JsonTensor> parse() {
    std::map<std::string, JsonTensor> out;
    expect('{');
    if (peek() == '}') return out;
    for (;;) {
      const std::string key = str();
      expect(':');
      if (key == "__metadata__") {
        skip_value();
      } else {
        out[key] = tensor();
      }
      if (peek() == ',') {
        ++i_;
        continue;
      }
      expect('}');
      return out;
    }
  }

 private:
  const std::string& s_;
  size_t i_ = 0;
  void ws() {
    while (i_ < s_.size() && std::isspace(static_cast<unsigned char>(s_[i_]))) ++i_;
  }
  char peek() {
    ws();
    MRSP_REQUIRE(i_ < s_.size(), MRSP_INVALID_ARGUMENT, "safetensors: truncated header");
    return s_[i_];
  }
  void expect(char c) {
    MRSP_REQUIRE(peek() == c, MRSP_INVALID_ARGUMENT,
                 std::string("safetensors: malformed header (expected '") + c + "')");
    ++i_;
  }
  std::string str() {
    expect('"');
    std::string r;
    while (i_ < s_.size() && s_[i_] != '"') {
      if (s_[i_] == '\\' && i_ + 1 < s_.size()) ++i_;
      r += s_[i_++];
    }
    expect('"');
    return r;
  }
  long num() {
    ws();
    size_t j = i_;
    while (j < s_.size() && (std::isdigit(static_cast<unsigned char>(s_[j])) || s_[j] == '-')) ++j;
    MRSP_REQUIRE(j > i_, MRSP_INVALID_ARGUMENT, "safetensors: expected a number");
    const long v = std::stol(s_.substr(i_, j - i_));
    i_ = j;
    return v;
  }
  std::vector<long> ints() {
    std::vector<long> v;
    expect('[');
    if (peek() == ']') {
      ++i_;
      return v;
    }
    for (;;) {
      v.push_back(num());
      if (peek() == ',') {
        ++i_;
        continue;
      }
      expect(']');
      return v;
    }
  }
  JsonTensor tensor() {
    JsonTensor t;
    expect('{');
    for (;;) {
      const std::string k = str();
      expect(':');
      if (k == "dtype") {
        t.dtype = str();
      } else if (k == "shape") {
        t.shape = ints();
      } else if (k == "data_offsets") {
        const auto o = ints();
        MRSP_REQUIRE(o.size() == 2 && o[0] >= 0 && o[1] >= o[0], MRSP_INVALID_ARGUMENT,
                     "safetensors: bad data_offsets");
        t.begin = static_cast<size_t>(o[0]);
        t.end = static_cast<size_t>(o[1]);
      } else {
        skip_value();
      }
      if (peek() == ',') {
        ++i_;
        continue;
      }
      expect('}');
      return t;
    }
  }
  void skip_value() {
    const char c = peek();
    if (c == '"') {
      str();
    } else if (c == '{' || c == '[') {
      const char close = c == '{' ? '}' : ']';
      int depth = 0;
      do {
        if (s_[i_] == '"') {
          str();
          continue;
        }
        if (s_[i_] == c) ++depth;
        if (s_[i_] == close) --depth;
        ++i_;
      } while (depth > 0 && i_ < s_.size());
    } else {
      while (i_ < s_.size() && s_[i_] != ',' && s_[i_] != '}') ++i_;
    }
  }
};

uint16_t f32_to_bf16(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return static_cast<uint16_t>((u >> 16) | 0x40);  // NaN
  u += 0x7fffu + ((u >> 16) & 1u);  // round to nearest even
  return static_cast<uint16_t>(u >> 16);
}
float bf16_to_f32(uint16_t h) {
  const uint32_t u = static_cast<uint32_t>(h) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

}  // namespace

// The engine's tensors as logical (HF-shaped) tensors. part: 0 = vision tower +
// projector, 1 = policy LLM, 2 = reference LLM.
static std::vector<TensorDesc> describe(const mrsp_model_config& c, const VisionW& vis,
                                        const LlmW& llm, int part, const std::string& pre,
                                        int tokens_per_frame, int vs_) {
  std::vector<TensorDesc> t;
  const size_t P = c.patch, kreal = 3 * P * P, kpad = (kreal + 7) / 8 * 8;
  const size_t vd = c.v_dim, vh = c.v_heads, vhd = c.v_head_dim, vs = vs_;
  const size_t vq = vh * vs;
  const size_t d = c.dim, nq = c.n_q_heads, nkv = c.n_kv_heads, mlp = c.mlp, V = c.vocab;
  auto plain = [&](const std::string& name, DType dt, std::vector<long> shape, void* dev) {
    TensorDesc x{pre + name, dt, shape, {}};
    x.segs.push_back(contiguous(dev, x.bytes()));
    t.push_back(std::move(x));
  };
  if (part == 0) {
    const std::string e = "vision_model.embeddings.";
    {  // conv weight [vd][3][P][P] -> patch_w [vd][kpad] (first kreal columns)
      TensorDesc x{pre + e + "patch_embedding.weight", BF16,
                   {static_cast<long>(vd), 3, static_cast<long>(P), static_cast<long>(P)}, {}};
      x.segs.push_back(Seg{vis.patch_w, kpad * 2, 0, kreal * 2, kreal * 2, vd});
      t.push_back(std::move(x));
    }
    plain(e + "patch_embedding.bias", F32, {static_cast<long>(vd)}, vis.patch_b);
    plain(e + "position_embedding.weight", F32, {tokens_per_frame, static_cast<long>(vd)}, vis.pos);
    for (size_t l = 0; l < vis.layers.size(); ++l) {
      const auto& L = vis.layers[l];
      const std::string p = "vision_model.encoder.layers." + std::to_string(l) + ".";
      plain(p + "layer_norm1.weight", F32, {static_cast<long>(vd)}, L.ln1_w);
      plain(p + "layer_norm1.bias", F32, {static_cast<long>(vd)}, L.ln1_b);
      const char* qkv[3] = {"q_proj", "k_proj", "v_proj"};
      for (int part3 = 0; part3 < 3; ++part3) {
        // rows h*vhd .. +vhd  ->  engine rows part*vq + h*vs (head stride vs >= vhd)
        TensorDesc w{pre + p + "self_attn." + qkv[part3] + ".weight", BF16,
                     {static_cast<long>(vd), static_cast<long>(vd)}, {}};
        TensorDesc b{pre + p + "self_attn." + qkv[part3] + ".bias", F32, {static_cast<long>(vd)}, {}};
        for (size_t h = 0; h < vh; ++h) {
          w.segs.push_back(Seg{L.wqkv + (part3 * vq + h * vs) * vd, vhd * vd * 2, h * vhd * vd * 2,
                               vhd * vd * 2, vhd * vd * 2, 1});
          b.segs.push_back(Seg{L.bqkv + part3 * vq + h * vs, vhd * 4, h * vhd * 4, vhd * 4,
                               vhd * 4, 1});
        }
        t.push_back(std::move(w));
        t.push_back(std::move(b));
      }
      {  // out_proj [vd][vd]: column block h*vhd .. -> engine columns h*vs ..
        TensorDesc w{pre + p + "self_attn.out_proj.weight", BF16,
                     {static_cast<long>(vd), static_cast<long>(vd)}, {}};
        for (size_t h = 0; h < vh; ++h)
          w.segs.push_back(Seg{L.wo + h * vs, vq * 2, h * vhd * 2, vd * 2, vhd * 2, vd});
        t.push_back(std::move(w));
      }
      plain(p + "self_attn.out_proj.bias", F32, {static_cast<long>(vd)}, L.bo);
      plain(p + "layer_norm2.weight", F32, {static_cast<long>(vd)}, L.ln2_w);
      plain(p + "layer_norm2.bias", F32, {static_cast<long>(vd)}, L.ln2_b);
      plain(p + "mlp.fc1.weight", BF16, {c.v_mlp, static_cast<long>(vd)}, L.w1);
      plain(p + "mlp.fc1.bias", F32, {c.v_mlp}, L.b1);
      plain(p + "mlp.fc2.weight", BF16, {static_cast<long>(vd), c.v_mlp}, L.w2);
      plain(p + "mlp.fc2.bias", F32, {static_cast<long>(vd)}, L.b2);
    }
    plain("vision_model.post_layernorm.weight", F32, {static_cast<long>(vd)}, vis.post_w);
    plain("vision_model.post_layernorm.bias", F32, {static_cast<long>(vd)}, vis.post_b);
    plain("mm_projector.0.weight", BF16, {static_cast<long>(d), static_cast<long>(vd)}, vis.p1_w);
    plain("mm_projector.0.bias", F32, {static_cast<long>(d)}, vis.p1_b);
    plain("mm_projector.2.weight", BF16, {static_cast<long>(d), static_cast<long>(d)}, vis.p2_w);
    plain("mm_projector.2.bias", F32, {static_cast<long>(d)}, vis.p2_b);
    return t;
  }
  plain("model.embed_tokens.weight", BF16, {static_cast<long>(V), static_cast<long>(d)}, llm.embed);
  for (size_t l = 0; l < llm.layers.size(); ++l) {
    const auto& L = llm.layers[l];
    const std::string p = "model.layers." + std::to_string(l) + ".";
    plain(p + "input_layernorm.weight", F32, {static_cast<long>(d)}, L.attn_norm);
    const size_t rows[3] = {nq * 128, nkv * 128, nkv * 128};
    const size_t row0[3] = {0, nq * 128, (nq + nkv) * 128};
    const char* names[3] = {"q_proj", "k_proj", "v_proj"};
    for (int k = 0; k < 3; ++k) {
      plain(p + "self_attn." + names[k] + ".weight", BF16,
            {static_cast<long>(rows[k]), static_cast<long>(d)}, L.wqkv + row0[k] * d);
      plain(p + "self_attn." + names[k] + ".bias", F32, {static_cast<long>(rows[k])},
            L.bqkv + row0[k]);
    }
    plain(p + "self_attn.o_proj.weight", BF16, {static_cast<long>(d), static_cast<long>(nq * 128)},
          L.wo);
    plain(p + "post_attention_layernorm.weight", F32, {static_cast<long>(d)}, L.mlp_norm);
    for (int k = 0; k < 2; ++k) {  // gate / up: 128-row blocks interleaved [gate | up]
      TensorDesc w{pre + p + (k ? "mlp.up_proj.weight" : "mlp.gate_proj.weight"), BF16,
                   {static_cast<long>(mlp), static_cast<long>(d)}, {}};
      w.segs.push_back(Seg{L.wgu + k * 128 * d, 256 * d * 2, 0, 128 * d * 2, 128 * d * 2, mlp / 128});
      t.push_back(std::move(w));
    }
    plain(p + "mlp.down_proj.weight", BF16, {static_cast<long>(d), static_cast<long>(mlp)}, L.wdown);
  }
  plain("model.norm.weight", F32, {static_cast<long>(d)}, llm.final_norm);
  plain("lm_head.weight", BF16, {static_cast<long>(V), static_cast<long>(d)}, llm.lm_head);
  return t;
}

static void write_safetensors(const std::string& path, const std::vector<TensorDesc>& all,
                              const char* what) {
  std::string hdr = "{\"__metadata__\":{\"format\":\"pt\",\"producer\":\"mrsp-b200\"}";
  size_t off = 0;
  for (const auto& x : all) {
    hdr += ",\"" + x.name + "\":{\"dtype\":\"" + (x.dtype == BF16 ? "BF16" : "F32") +
           "\",\"shape\":[";
    for (size_t i = 0; i < x.shape.size(); ++i) hdr += (i ? "," : "") + std::to_string(x.shape[i]);
    hdr += "],\"data_offsets\":[" + std::to_string(off) + "," + std::to_string(off + x.bytes()) +
           "]}";
    off += x.bytes();
  }
  hdr += "}";
  while (hdr.size() % 8) hdr += ' ';
  FILE* f = std::fopen(path.c_str(), "wb");
  MRSP_REQUIRE(f != nullptr, MRSP_RUNTIME_ERROR, std::string(what) + ": cannot open " + path);
  const uint64_t hlen = hdr.size();
  bool ok = std::fwrite(&hlen, 8, 1, f) == 1 && std::fwrite(hdr.data(), 1, hdr.size(), f) == hdr.size();
  std::vector<uint8_t> host;
  for (const auto& x : all) {
    if (!ok) break;
    host.assign(x.bytes(), 0);
    for (const auto& sg : x.segs)
      MRSP_CUDA(cudaMemcpy2D(host.data() + sg.log_off, sg.log_pitch, sg.dev, sg.dev_pitch,
                             sg.width, sg.rows, cudaMemcpyDeviceToHost));
    ok = std::fwrite(host.data(), 1, host.size(), f) == host.size();
  }
  const bool closed = std::fclose(f) == 0;
  MRSP_REQUIRE(ok && closed, MRSP_RUNTIME_ERROR, std::string(what) + ": write failed: " + path);
}

void Engine::save_weights(const std::string& path) {
  std::lock_guard<std::mutex> run(run_mu_);
  std::vector<TensorDesc> all;
  for (int part = 0; part < (has_ref_ ? 3 : 2); ++part) {
    auto v = describe(cfg_, vis_, llm_[part == 2 ? 1 : 0], part, part == 2 ? "ref." : "",
                      tokens_per_frame(), vstride_);
    all.insert(all.end(), v.begin(), v.end());
  }
  write_safetensors(path, all, "save_weights");
}

// The fp32 gradients of the policy LLM (grads_, engine_bwd.cu) under the
// policy's tensor names: grads_ mirrors the weight layout element for element
// with 4-byte elements, so the bf16 weight descriptors are re-used with every
// byte extent doubled.
void Engine::save_grads(const std::string& path) {
  std::lock_guard<std::mutex> run(run_mu_);
  MRSP_REQUIRE(have_grads_, MRSP_INVALID_ARGUMENT, "save_grads: no gradients (run grpo_backward)");
  std::vector<TensorDesc> all = describe(cfg_, vis_, grads_, 1, "", tokens_per_frame(), vstride_);
  // the descriptors address sub-blocks (q / k / v rows, gate / up blocks) by
  // bf16 pointer arithmetic from a tensor's base: rebase those offsets too
  std::vector<uintptr_t> bases = {reinterpret_cast<uintptr_t>(grads_.embed),
                                  reinterpret_cast<uintptr_t>(grads_.lm_head)};
  for (const auto& L : grads_.layers)
    for (const void* q : {static_cast<const void*>(L.wqkv), static_cast<const void*>(L.wo),
                          static_cast<const void*>(L.wgu), static_cast<const void*>(L.wdown)})
      bases.push_back(reinterpret_cast<uintptr_t>(q));
  std::sort(bases.begin(), bases.end());
  for (auto& x : all) {
    if (x.dtype != BF16) continue;
    x.dtype = F32;
    for (auto& sg : x.segs) {
      const uintptr_t a = reinterpret_cast<uintptr_t>(sg.dev);
      const uintptr_t b = *(std::upper_bound(bases.begin(), bases.end(), a) - 1);
      sg.dev = reinterpret_cast<void*>(b + 2 * (a - b));
      sg.dev_pitch *= 2;
      sg.log_off *= 2;
      sg.log_pitch *= 2;
      sg.width *= 2;
    }
  }
  write_safetensors(path, all, "save_grads");
}

void Engine::load_weights(const std::string& path, int part, const std::string& prefix) {
  MRSP_REQUIRE(part >= 0 && part <= 2, MRSP_INVALID_ARGUMENT,
               "load_weights: part is 0 (vision + projector), 1 (policy) or 2 (reference)");
  MRSP_REQUIRE(part != 2 || has_ref_, MRSP_INVALID_ARGUMENT,
               "load_weights: the engine was created without a separate reference model");
  std::lock_guard<std::mutex> run(run_mu_);
  FILE* f = std::fopen(path.c_str(), "rb");
  MRSP_REQUIRE(f != nullptr, MRSP_RUNTIME_ERROR, "load_weights: cannot open " + path);
  uint64_t hlen = 0;
  std::string hdr;
  bool ok = std::fread(&hlen, 8, 1, f) == 1 && hlen > 1 && hlen < (1ull << 30);
  if (ok) {
    hdr.resize(hlen);
    ok = std::fread(&hdr[0], 1, hlen, f) == hlen;
  }
  if (!ok) {
    std::fclose(f);
    fail(MRSP_INVALID_ARGUMENT, "load_weights: not a safetensors file: " + path);
  }
  std::map<std::string, JsonTensor> table;
  try {
    table = HeaderParser(hdr).parse();
  } catch (...) {
    std::fclose(f);
    throw;
  }
  const long data0 = static_cast<long>(8 + hlen);
  const auto want =
      describe(cfg_, vis_, llm_[part == 2 ? 1 : 0], part, prefix, tokens_per_frame(), vstride_);
  std::vector<uint8_t> raw, host;
  for (const auto& x : want) {
    auto it = table.find(x.name);
    if (it == table.end()) {
      std::fclose(f);
      fail(MRSP_INVALID_ARGUMENT, "load_weights: missing tensor " + x.name);
    }
    const JsonTensor& jt = it->second;
    const bool src_bf16 = jt.dtype == "BF16", src_f32 = jt.dtype == "F32";
    size_t n = 1;
    for (long s : x.shape) n *= static_cast<size_t>(s);
    if (jt.shape != x.shape || !(src_bf16 || src_f32) ||
        jt.end - jt.begin != n * (src_bf16 ? 2 : 4)) {
      std::fclose(f);
      fail(MRSP_INVALID_ARGUMENT, "load_weights: " + x.name + " has shape/dtype " + jt.dtype +
                                      " that does not match the engine geometry");
    }
    raw.resize(jt.end - jt.begin);
    if (std::fseek(f, data0 + static_cast<long>(jt.begin), SEEK_SET) != 0 ||
        std::fread(raw.data(), 1, raw.size(), f) != raw.size()) {
      std::fclose(f);
      fail(MRSP_RUNTIME_ERROR, "load_weights: truncated file " + path);
    }
    // convert to the engine's storage dtype (checkpoints often keep norms in bf16)
    const uint8_t* src = raw.data();
    if (x.dtype == BF16 && src_f32) {
      host.resize(n * 2);
      for (size_t i = 0; i < n; ++i) {
        float v;
        std::memcpy(&v, raw.data() + 4 * i, 4);
        const uint16_t h = f32_to_bf16(v);
        std::memcpy(host.data() + 2 * i, &h, 2);
      }
      src = host.data();
    } else if (x.dtype == F32 && src_bf16) {
      host.resize(n * 4);
      for (size_t i = 0; i < n; ++i) {
        uint16_t h;
        std::memcpy(&h, raw.data() + 2 * i, 2);
        const float v = bf16_to_f32(h);
        std::memcpy(host.data() + 4 * i, &v, 4);
      }
      src = host.data();
    }
    for (const auto& sg : x.segs)
      MRSP_CUDA(cudaMemcpy2D(sg.dev, sg.dev_pitch, src + sg.log_off, sg.log_pitch, sg.width,
                             sg.rows, cudaMemcpyHostToDevice));
  }
  std::fclose(f);
  if (part == 0) {  // cached embeddings were produced by the old tower
    std::lock_guard<std::mutex> lock(cache_mu_);
    cache_.clear();
  }
}

}  // namespace mrsp
