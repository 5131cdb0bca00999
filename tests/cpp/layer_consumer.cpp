// A compiled C++ consumer of include/cad.h, written the way a cadsim
// maintainer would call it: the scheduler on BASELINE config
// 1 (the reference's golden 2-server plan, P/tests/test_scheduler.cpp:163-180)
// and then -- with `gpu` -- one CA layer of that plan executed by the per-layer
// executor (cad_layer_ctx, two ranks in this process on device 0, LOCAL
// transport, the per-layer entry points cad_layer_begin / cad_dispatch /
// cad_layer_compute / cad_return / cad_layer_finish), checked against the same batch
// computed whole by cad_ca_fwd/cad_ca_bwd. Exit status 0 = pass.
//   layer_consumer [cpu|gpu]
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "cad.h"

#define CHECK(x)                                                                  \
  do {                                                                            \
    const int rc_ = (x);                                                          \
    if (rc_ != CAD_OK) {                                                          \
      std::fprintf(stderr, "%s:%d %s -> %d: %s\n", __FILE__, __LINE__, #x, rc_,   \
                   cad_last_error());                                             \
      return 1;                                                                   \
    }                                                                             \
  } while (0)
#define CUDA(x)                                                                   \
  do {                                                                            \
    const cudaError_t e_ = (x);                                                   \
    if (e_ != cudaSuccess) {                                                      \
      std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x,              \
                   cudaGetErrorString(e_));                                       \
      return 1;                                                                   \
    }                                                                             \
  } while (0)

static const char* kGolden =
    "# plan v1\n"
    "# doc q_begin q_end kv_extent ht_mirror layout source server core bytes\n"
    "0 0 2560 2560 0 contiguous 0 0 6553600 0\n"
    "0 3584 4096 4096 0 contiguous 0 0 3932160 0\n"
    "1 0 1024 1024 0 contiguous 1 1 1048576 0\n"
    "2 0 1024 1024 0 contiguous 1 1 1048576 0\n"
    "3 0 1024 1024 0 contiguous 1 1 1048576 0\n"
    "4 0 1024 1024 0 contiguous 1 1 1048576 0\n"
    "0 2560 3584 3584 0 contiguous 0 1 6291456 46137344\n";

static uint16_t to_bf16(float f) {  // round to nearest even
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7fffu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}
static float from_bf16(uint16_t h) {
  const uint32_t u = static_cast<uint32_t>(h) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::string(argv[1]) == "gpu";
  // ---------------------------------------------------------------- scheduler
  const int64_t lengths[5] = {4096, 1024, 1024, 1024, 1024};
  cad_item items[16];
  int64_t n_items = 0;
  CHECK(cad_place_sequential(lengths, 5, 2, 4096, items, 16, &n_items));
  cad_sched_cfg cfg;
  cad_sched_cfg_default(&cfg);
  cfg.epsilon = 0.0;  // P/tests/test_scheduler.cpp:29-38
  cfg.e_threshold = 1e-9;
  cfg.tile_size = 128;
  cfg.alpha_ca = 1.0;
  cfg.size_q = 16384;
  cfg.size_kv = 8192;
  cad_plan* plan = nullptr;
  CHECK(cad_schedule(items, n_items, 2, &cfg, &plan));
  char text[4096];
  size_t need = 0;
  CHECK(cad_plan_to_text(plan, text, sizeof text, &need));
  if (std::strcmp(text, kGolden) != 0) {
    std::fprintf(stderr, "plan text differs from the golden fixture:\n%s", text);
    return 1;
  }
  std::printf("golden plan ok (%lld items)\n", static_cast<long long>(n_items));
  if (!gpu) {
    cad_plan_free(plan);
    return 0;
  }
  // ---------------------------------------------------------------- one layer
  const int hq = 8, hkv = 8, d = 128, T = 8192, W = 2;
  const size_t qn = size_t(T) * hq * d, kn = size_t(T) * hkv * d;
  std::vector<uint16_t> hq_(qn), hk_(kn), hv_(kn), hdo_(qn);
  uint64_t s = 12345;
  auto rnd = [&]() {  // uniform(-2, 2) from a 64-bit LCG
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    return static_cast<float>((s >> 11) * (1.0 / 9007199254740992.0) * 4.0 - 2.0);
  };
  for (auto* v : {&hq_, &hk_, &hv_, &hdo_})
    for (auto& x : *v) x = to_bf16(rnd());
  auto dev_copy = [](const std::vector<uint16_t>& h, void** d_) {
    if (cudaMalloc(d_, h.size() * 2) != cudaSuccess) return false;
    return cudaMemcpy(*d_, h.data(), h.size() * 2, cudaMemcpyHostToDevice) == cudaSuccess;
  };
  void *q, *k, *v, *dout;
  if (!dev_copy(hq_, &q) || !dev_copy(hk_, &k) || !dev_copy(hv_, &v) || !dev_copy(hdo_, &dout)) return 1;
  // whole batch on one "server": every document one task
  cad_ca_task whole[5];
  int64_t off = 0;
  for (int i = 0; i < 5; ++i) {
    whole[i] = {off, lengths[i], off, lengths[i]};
    off += lengths[i];
  }
  cad_ca_shape shape{hq, hkv, d, 0.0f, T, T};
  cad_ca_plan* ca = nullptr;
  CHECK(cad_ca_plan_create(whole, 5, &shape, &ca));
  cad_ca_plan_info info;
  CHECK(cad_ca_plan_info_get(ca, &info));
  void *o_ref, *dq_ref, *dk_ref, *dv_ref, *ws;
  float* lse_ref;
  CUDA(cudaMalloc(&o_ref, qn * 2));
  CUDA(cudaMalloc(&dq_ref, qn * 2));
  CUDA(cudaMalloc(&dk_ref, kn * 2));
  CUDA(cudaMalloc(&dv_ref, kn * 2));
  CUDA(cudaMalloc(&lse_ref, size_t(hq) * T * 4));
  CUDA(cudaMalloc(&ws, info.workspace_bytes));
  CHECK(cad_ca_fwd(ca, q, k, v, o_ref, lse_ref, nullptr));
  CHECK(cad_ca_bwd(ca, q, k, v, o_ref, lse_ref, dout, dq_ref, dk_ref, dv_ref, ws, info.workspace_bytes, nullptr));
  // the same layer through the per-layer executor: rank r's home rows are
  // tokens [4096 r, 4096 r + 4096) of the batch (place_sequential)
  cad_layer_ctx* ctx[W];
  void *o[W], *dq[W], *dk[W], *dv[W];
  float* lse[W];
  cad_layer_io io[W];
  std::vector<uint8_t> blobs;
  for (int r = 0; r < W; ++r) {
    cad_layer_cfg lc{};
    lc.rank = r;
    lc.world = W;
    lc.h_q = hq;
    lc.h_kv = hkv;
    lc.head_dim = d;
    lc.transport = CAD_TRANSPORT_LOCAL;
    lc.layers = 1;
    CHECK(cad_layer_ctx_create(plan, items, n_items, &lc, &ctx[r]));
    cad_layer_ctx_info li;
    CHECK(cad_layer_ctx_info_get(ctx[r], &li));
    if (li.home_rows != 4096) return 1;
    CUDA(cudaMalloc(&o[r], qn));  // half the batch each
    CUDA(cudaMalloc(&dq[r], qn));
    CUDA(cudaMalloc(&dk[r], kn));
    CUDA(cudaMalloc(&dv[r], kn));
    CUDA(cudaMalloc(&lse[r], size_t(hq) * 4096 * 4));
    CHECK(cad_layer_ctx_bind_outputs(ctx[r], o[r], lse[r], dq[r]));
    const size_t row_q = size_t(hq) * d * 2, row_k = size_t(hkv) * d * 2;
    io[r] = cad_layer_io{static_cast<char*>(q) + r * 4096 * row_q, static_cast<char*>(k) + r * 4096 * row_k,
                         static_cast<char*>(v) + r * 4096 * row_k, static_cast<char*>(dout) + r * 4096 * row_q,
                         o[r], lse[r], dq[r], dk[r], dv[r], nullptr, nullptr};
    std::vector<uint8_t> b(static_cast<size_t>(li.blob_bytes));
    size_t nb = 0;
    CHECK(cad_layer_ctx_export(ctx[r], b.data(), b.size(), &nb));
    blobs.insert(blobs.end(), b.begin(), b.begin() + static_cast<long>(nb));
  }
  for (int r = 0; r < W; ++r) CHECK(cad_layer_ctx_connect(ctx[r], blobs.data(), blobs.size() / W));
  // LOCAL contexts run phase by phase in dependency order across the ranks
  // (one process per GPU would call cad_layer_step instead); two steps, so
  // the second runs on the flags' next generation
  cudaStream_t st;
  CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  if (cad_layer_step(ctx[0], &io[0], CAD_STEP_PINGPONG, st) != CAD_ERR_CONFIG) {
    std::fprintf(stderr, "cad_layer_step on a LOCAL context must be refused\n");
    return 1;
  }
  for (int rep = 0; rep < 2; ++rep) {
    for (int r = 0; r < W; ++r) CHECK(cad_layer_begin(ctx[r], st));
    const int32_t phases[2][2] = {{CAD_DISPATCH_QKV, CAD_RETURN_O}, {CAD_DISPATCH_DO, CAD_RETURN_GRAD}};
    for (int p = 0; p < 2; ++p) {
      for (int h = 0; h < 2; ++h)
        for (int r = 0; r < W; ++r) CHECK(cad_dispatch(ctx[r], 0, h, phases[p][0], &io[r], st));
      for (int h = 0; h < 2; ++h)
        for (int r = 0; r < W; ++r) CHECK(cad_layer_compute(ctx[r], 0, h, p, st));
      for (int h = 0; h < 2; ++h)
        for (int r = 0; r < W; ++r) CHECK(cad_return(ctx[r], 0, h, phases[p][1], &io[r], st));
    }
    for (int r = 0; r < W; ++r) CHECK(cad_layer_finish(ctx[r], &io[r], st));
  }
  CUDA(cudaDeviceSynchronize());
  // compare home rows with the whole-batch rows
  double worst[4] = {0, 0, 0, 0};
  const char* names[4] = {"o", "dq", "dk", "dv"};
  void* refs[4] = {o_ref, dq_ref, dk_ref, dv_ref};
  for (int r = 0; r < W; ++r) {
    void* outs[4] = {o[r], dq[r], dk[r], dv[r]};
    for (int t = 0; t < 4; ++t) {
      const size_t n = (t < 2 ? qn : kn) / 2;
      std::vector<uint16_t> a(n), b(n);
      CUDA(cudaMemcpy(a.data(), outs[t], n * 2, cudaMemcpyDeviceToHost));
      CUDA(cudaMemcpy(b.data(), static_cast<char*>(refs[t]) + size_t(r) * n * 2, n * 2, cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < n; ++i) {
        const double rb = from_bf16(b[i]);
        const double e = std::fabs(from_bf16(a[i]) - rb) / std::fmax(1.0, std::fabs(rb));
        if (!(e <= worst[t])) worst[t] = std::isnan(e) ? INFINITY : e;
      }
    }
  }
  int bad = 0;
  for (int t = 0; t < 4; ++t) {
    std::printf("%s: worst |layer - whole| / max(1, |whole|) = %.3e\n", names[t], worst[t]);
    bad += !(worst[t] <= 2e-2);
  }
  for (int r = 0; r < W; ++r) CHECK(cad_layer_ctx_destroy(ctx[r]));
  CHECK(cad_ca_plan_destroy(ca));
  cad_plan_free(plan);
  std::printf(bad ? "FAIL\n" : "layer ok\n");
  return bad ? 1 : 0;
}
