// sgmv_cuda.cpp -- the lorasim:: SGMV operators re-implemented on the B200.
//
// Value-type validation mirrors the reference exactly (sgmv.cpp:31-101,
// 143-148: same checks, same order, same std::invalid_argument messages);
// everything after validation runs through the C-ABI (include/lsg_sgmv.h).
// Each call stages its operands in a per-thread device arena (grown, never
// shrunk), runs on a per-thread stream and synchronises before returning the
// host Matrix, as the value-semantic API requires.
#include <cublas_v2.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <limits>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "lorasim/b200.hpp"
#include "lorasim/sgmv.hpp"
#include "lsg_sgmv.h"

namespace lorasim {

// ---- value types (reference invariants, sgmv.cpp:31-64) -----------------------------
Segments::Segments(std::vector<std::size_t> boundaries) : bounds_(std::move(boundaries)) {
  if (bounds_.empty()) throw std::invalid_argument("Segments: boundary list empty");
  if (bounds_[0] != 0) throw std::invalid_argument("Segments: s_0 must be 0");
  for (std::size_t i = 1; i < bounds_.size(); ++i)
    if (!(bounds_[i] > bounds_[i - 1]))
      throw std::invalid_argument("Segments: boundaries must be strictly increasing");
}

Segments Segments::single(std::size_t rows) {
  return rows == 0 ? Segments(std::vector<std::size_t>{0}) : Segments(std::vector<std::size_t>{0, rows});
}

LoraModel::LoraModel(LoraId id_in, Matrix a_in, Matrix b_in) : id(id_in), a(std::move(a_in)), b(std::move(b_in)) {
  const std::size_t r = a.cols();
  if (r == 0) throw std::invalid_argument("LoraModel: rank must be >= 1");
  if (b.rows() != r) throw std::invalid_argument("LoraModel: A columns != B rows");
  if (r > a.rows() || r > b.cols()) throw std::invalid_argument("LoraModel: rank exceeds min(h_in, h_out)");
  auto all_finite = [](const Matrix& m) {
    for (double v : m.data())
      if (!std::isfinite(v)) return false;
    return true;
  };
  if (!all_finite(a)) throw std::invalid_argument("LoraModel: non-finite entry in A");
  if (!all_finite(b)) throw std::invalid_argument("LoraModel: non-finite entry in B");
}

Batch::Batch(Matrix x_in, Segments segs, std::vector<LoraModel> ms)
    : x(std::move(x_in)), segments(std::move(segs)), models(std::move(ms)) {
  if (x.rows() != segments.total_rows()) throw std::invalid_argument("Batch: x row count != segment total");
  if (models.size() != segments.count()) throw std::invalid_argument("Batch: model count != segment count");
}

namespace b200 {

namespace {
Precision g_precision = Precision::F16;
}

void set_precision(Precision p) { g_precision = p; }
Precision precision() { return g_precision; }

// Round-to-nearest-even onto the fp16 / bf16 grid, computed exactly in fp64.
double quantize(double v, Precision p) {
  if (!std::isfinite(v) || v == 0.0) return v;
  const int mant = p == Precision::F16 ? 11 : 8;         // significand bits incl. hidden
  const int emin = p == Precision::F16 ? -14 : -126;     // min normal exponent
  const double maxv = p == Precision::F16 ? 65504.0 : 3.3895313892515355e38;
  int e;
  std::frexp(v, &e);  // |v| = f * 2^e, f in [0.5, 1)
  int exp = e - 1;
  if (exp < emin) exp = emin;
  const double ulp = std::ldexp(1.0, exp - (mant - 1));
  const double q = std::nearbyint(v / ulp) * ulp;  // default rounding mode: ties to even
  if (std::fabs(q) > maxv) return std::copysign(std::numeric_limits<double>::infinity(), v);
  return q;
}

}  // namespace b200

namespace {

using b200::Precision;

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("lorasim b200: ") + what + ": " + cudaGetErrorString(e));
}

void lsg_check(int st, const char* what) {
  if (st != LSG_OK)
    throw std::runtime_error(std::string("lorasim b200: ") + what + ": " + lsg_status_string(st) + ": " +
                             lsg_last_error());
}

uint16_t to_bits(double v, Precision p) {
  const float f = static_cast<float>(b200::quantize(v, p));  // exact: already on the grid
  uint16_t u;
  if (p == Precision::F16) {
    const __half h = __float2half_rn(f);
    std::memcpy(&u, &h, 2);
  } else {
    const __nv_bfloat16 h = __float2bfloat16_rn(f);
    std::memcpy(&u, &h, 2);
  }
  return u;
}

double from_bits(uint16_t u, Precision p) {
  if (p == Precision::F16) {
    __half h;
    std::memcpy(&h, &u, 2);
    return static_cast<double>(__half2float(h));
  }
  __nv_bfloat16 h;
  std::memcpy(&h, &u, 2);
  return static_cast<double>(__bfloat162float(h));
}

// Per-thread device staging: one growing buffer per role + a stream + cuBLAS.
struct Arena {
  std::map<int, std::pair<void*, std::size_t>> bufs;
  cudaStream_t stream = nullptr;
  cublasHandle_t blas = nullptr;

  Arena() = default;
  ~Arena() {
    for (auto& kv : bufs) cudaFree(kv.second.first);
    if (blas) cublasDestroy(blas);
    if (stream) cudaStreamDestroy(stream);
  }
  cudaStream_t s() {
    if (!stream) cuda_check(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "cudaStreamCreate");
    return stream;
  }
  void* get(int role, std::size_t bytes) {
    auto& b = bufs[role];
    if (b.second < bytes) {
      if (b.first) cudaFree(b.first);
      b.first = nullptr;
      cuda_check(cudaMalloc(&b.first, bytes < 256 ? 256 : bytes), "cudaMalloc");
      b.second = bytes;
    }
    return b.first;
  }
};

thread_local Arena t_arena;

enum Role { kX = 0, kY, kV, kA, kB, kPtrA, kPtrB, kSeg, kSlot, kRowSlot, kW };

template <typename T>
T* upload(int role, const std::vector<T>& host) {
  void* d = t_arena.get(role, host.size() * sizeof(T));
  if (!host.empty())
    cuda_check(cudaMemcpyAsync(d, host.data(), host.size() * sizeof(T), cudaMemcpyHostToDevice, t_arena.s()),
               "cudaMemcpyAsync H2D");
  return static_cast<T*>(d);
}

std::vector<uint16_t> to_bits(const std::vector<double>& v, Precision p) {
  std::vector<uint16_t> out(v.size());
  for (std::size_t i = 0; i < v.size(); ++i) out[i] = to_bits(v[i], p);
  return out;
}

// One-layer pool holding the batch's models: slot s = segment s.
struct StagedModels {
  lsg_weight_table tbl{};
};

StagedModels stage_models(const std::vector<LoraModel>& models, std::size_t h_in, std::size_t rank,
                          std::size_t h_out, bool need_a, bool need_b, Precision p) {
  const std::size_t n = models.size();
  std::vector<uint16_t> a(need_a ? n * h_in * rank : 0), b(need_b ? n * rank * h_out : 0);
  for (std::size_t s = 0; s < n; ++s) {
    if (need_a)
      for (std::size_t i = 0; i < h_in * rank; ++i) a[s * h_in * rank + i] = to_bits(models[s].a.data()[i], p);
    if (need_b)
      for (std::size_t i = 0; i < rank * h_out; ++i) b[s * rank * h_out + i] = to_bits(models[s].b.data()[i], p);
  }
  uint16_t* da = upload(kA, a.empty() ? std::vector<uint16_t>(8) : a);
  uint16_t* db = upload(kB, b.empty() ? std::vector<uint16_t>(8) : b);
  std::vector<const void*> pa(n), pb(n);
  for (std::size_t s = 0; s < n; ++s) {
    pa[s] = need_a ? da + s * h_in * rank : da;
    pb[s] = need_b ? db + s * rank * h_out : db;
  }
  StagedModels sm;
  sm.tbl.a_ptr = upload(kPtrA, pa);
  sm.tbl.b_ptr = upload(kPtrB, pb);
  sm.tbl.a_layer_stride = static_cast<int64_t>(h_in * rank);
  sm.tbl.b_layer_stride = static_cast<int64_t>(rank * h_out);
  sm.tbl.num_slots = static_cast<int32_t>(n);
  sm.tbl.num_layers = 1;
  sm.tbl.h_in = static_cast<int32_t>(h_in);
  sm.tbl.h_out = static_cast<int32_t>(h_out);
  sm.tbl.rank = static_cast<int32_t>(rank);
  sm.tbl.dtype = p == Precision::F16 ? LSG_F16 : LSG_BF16;
  return sm;
}

int32_t to_i32(std::size_t v, const char* what) {
  if (v > static_cast<std::size_t>(std::numeric_limits<int32_t>::max()))
    throw std::invalid_argument(std::string("lorasim b200: ") + what + " exceeds int32");
  return static_cast<int32_t>(v);
}

const int32_t* upload_segments(const Segments& segs) {
  std::vector<int32_t> b(segs.boundaries().size());
  for (std::size_t i = 0; i < b.size(); ++i) b[i] = to_i32(segs.boundaries()[i], "segment boundary");
  return upload(kSeg, b);
}

const int32_t* upload_identity_slots(std::size_t n) {
  std::vector<int32_t> s(n);
  for (std::size_t i = 0; i < n; ++i) s[i] = static_cast<int32_t>(i);
  return upload(kSlot, s);
}

Matrix download(const void* d, std::size_t rows, std::size_t cols, Precision p) {
  std::vector<uint16_t> h(rows * cols);
  if (!h.empty())
    cuda_check(cudaMemcpyAsync(h.data(), d, h.size() * 2, cudaMemcpyDeviceToHost, t_arena.s()), "cudaMemcpyAsync D2H");
  cuda_check(cudaStreamSynchronize(t_arena.s()), "cudaStreamSynchronize");
  Matrix m(rows, cols);
  for (std::size_t i = 0; i < h.size(); ++i) m.data()[i] = from_bits(h[i], p);
  return m;
}

// ---- reference-equivalent validation (sgmv.cpp:66-101) ---------------------------------
struct Dims {
  std::size_t rank;
  std::size_t h_in;
};

Dims shrink_dims(const Batch& batch) {
  if (batch.models.empty()) return {0, batch.x.cols()};
  const std::size_t r = batch.models.front().rank();
  for (const auto& m : batch.models) {
    if (m.rank() != r) throw std::invalid_argument("sgmv: heterogeneous adapter ranks in one batch");
    if (m.h_in() != batch.x.cols()) throw std::invalid_argument("sgmv: adapter input dim != batch hidden dim");
  }
  return {r, batch.x.cols()};
}

std::size_t expand_dims(const Matrix& v, const Segments& segments, const std::vector<LoraModel>& models) {
  if (v.rows() != segments.total_rows()) throw std::invalid_argument("sgmv_expand: v row count != segment total");
  if (models.size() != segments.count()) throw std::invalid_argument("sgmv_expand: model count != segment count");
  if (models.empty()) return 0;
  const std::size_t h_out = models.front().h_out();
  for (const auto& m : models) {
    if (m.rank() != v.cols()) throw std::invalid_argument("sgmv_expand: adapter rank != v column count");
    if (m.h_out() != h_out) throw std::invalid_argument("sgmv_expand: adapters disagree on output dim");
  }
  return h_out;
}

std::size_t common_h_out(const Batch& batch, const char* who) {
  const std::size_t h_out = batch.models.front().h_out();
  for (const auto& m : batch.models)
    if (m.h_out() != h_out) throw std::invalid_argument(std::string(who) + ": adapters disagree on output dim");
  return h_out;
}

enum class Form { Fused, TwoLaunch, PerRow };

// y = x . A . B for the whole batch on the GPU, in one of the three formulations.
Matrix addon_on_device(const Batch& batch, std::size_t rank, std::size_t h_out, Form form, const Matrix* w) {
  const Precision p = b200::precision();
  const std::size_t rows = batch.rows(), h_in = batch.x.cols(), n = batch.models.size();
  const int32_t rows32 = to_i32(rows, "row count"), n32 = to_i32(n, "segment count");
  cudaStream_t st = t_arena.s();
  auto* dx = upload(kX, to_bits(batch.x.data(), p));
  void* dy = t_arena.get(kY, rows * h_out * 2);
  if (w != nullptr) {
    // backbone x*W (cuBLAS, fp32 accumulate, rounded to the working precision); LoRA adds into it
    auto* dw = upload(kW, to_bits(w->data(), p));
    if (!t_arena.blas) {
      if (cublasCreate(&t_arena.blas) != CUBLAS_STATUS_SUCCESS) throw std::runtime_error("lorasim b200: cublasCreate");
    }
    cublasSetStream(t_arena.blas, st);
    const float one = 1.f, zero = 0.f;
    const cudaDataType_t dt = p == Precision::F16 ? CUDA_R_16F : CUDA_R_16BF;
    // row-major y[rows,h_out] = x[rows,h_in] W[h_in,h_out]  <=>  column-major y^T = W^T x^T
    const cublasStatus_t cs = cublasGemmEx(t_arena.blas, CUBLAS_OP_N, CUBLAS_OP_N, static_cast<int>(h_out),
                                           static_cast<int>(rows), static_cast<int>(h_in), &one, dw, dt,
                                           static_cast<int>(h_out), dx, dt, static_cast<int>(h_in), &zero, dy, dt,
                                           static_cast<int>(h_out), CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
    if (cs != CUBLAS_STATUS_SUCCESS) throw std::runtime_error("lorasim b200: cublasGemmEx failed");
  } else {
    cuda_check(cudaMemsetAsync(dy, 0, rows * h_out * 2, st), "cudaMemsetAsync");
  }
  const StagedModels sm = stage_models(batch.models, h_in, rank, h_out, true, true, p);
  auto* seg = upload_segments(batch.segments);
  auto* slot = upload_identity_slots(n);
  auto lst = reinterpret_cast<lsg_stream_t>(st);
  switch (form) {
    case Form::Fused: {
      // The drop-in keeps decode-length segments on the canonical CUDA-core arithmetic (the
      // segment-tile MMA pair off), so lora_addon, lora_loop_oracle and gather_bmm_oracle agree
      // bit for bit -- verify_sgmv's tolerance (experiments.cpp:79-80) assumes that.
      const lsg_call_opts opts{-1, -1, -1, 1 << 30};
      lsg_check(lsg_sgmv_ex(dy, static_cast<int64_t>(h_out), dx, static_cast<int64_t>(h_in), &sm.tbl, seg, slot, n32,
                            rows32, 0, nullptr, 0, &opts, lst),
                "lsg_sgmv_ex");
      break;
    }
    case Form::TwoLaunch: {
      auto* dv = static_cast<float*>(t_arena.get(kV, rows * rank * 4));
      lsg_check(lsg_sgmv_shrink(dv, dx, static_cast<int64_t>(h_in), &sm.tbl, seg, slot, n32, rows32, 0, lst),
                "lsg_sgmv_shrink");
      lsg_check(lsg_sgmv_expand(dy, static_cast<int64_t>(h_out), dv, &sm.tbl, seg, slot, n32, rows32, 0, lst),
                "lsg_sgmv_expand");
      break;
    }
    case Form::PerRow: {
      std::vector<int32_t> row_slot(rows);
      for (std::size_t s = 0; s < n; ++s)
        for (std::size_t j = batch.segments.begin_of(s); j < batch.segments.end_of(s); ++j)
          row_slot[j] = static_cast<int32_t>(s);
      auto* drs = upload(kRowSlot, row_slot);
      lsg_check(lsg_bgmv(dy, static_cast<int64_t>(h_out), dx, static_cast<int64_t>(h_in), &sm.tbl, drs, rows32, 0,
                         lst),
                "lsg_bgmv");
      break;
    }
  }
  return download(dy, rows, h_out, p);
}

}  // namespace

// ---- operators ---------------------------------------------------------------------------
Matrix sgmv_shrink(const Batch& batch) {
  const Dims d = shrink_dims(batch);
  if (batch.models.empty() || batch.rows() == 0) return Matrix(batch.rows(), d.rank);
  const Precision p = b200::precision();
  const std::size_t rows = batch.rows(), n = batch.models.size();
  auto* dx = upload(kX, to_bits(batch.x.data(), p));
  const StagedModels sm = stage_models(batch.models, d.h_in, d.rank, d.rank, true, false, p);
  auto* dv = static_cast<float*>(t_arena.get(kV, rows * d.rank * 4));
  lsg_check(lsg_sgmv_shrink(dv, dx, static_cast<int64_t>(d.h_in), &sm.tbl, upload_segments(batch.segments),
                            upload_identity_slots(n), to_i32(n, "segment count"), to_i32(rows, "row count"), 0,
                            reinterpret_cast<lsg_stream_t>(t_arena.s())),
            "lsg_sgmv_shrink");
  std::vector<float> hv(rows * d.rank);
  cuda_check(cudaMemcpyAsync(hv.data(), dv, hv.size() * 4, cudaMemcpyDeviceToHost, t_arena.s()), "D2H v");
  cuda_check(cudaStreamSynchronize(t_arena.s()), "cudaStreamSynchronize");
  Matrix v(rows, d.rank);
  for (std::size_t i = 0; i < hv.size(); ++i) v.data()[i] = hv[i];
  return v;
}

Matrix sgmv_expand(const Matrix& v, const Segments& segments, const std::vector<LoraModel>& models) {
  const std::size_t h_out = expand_dims(v, segments, models);
  if (models.empty() || v.rows() == 0) return Matrix(v.rows(), h_out);
  const Precision p = b200::precision();
  const std::size_t rows = v.rows(), rank = v.cols(), n = models.size();
  std::vector<float> hv(v.data().begin(), v.data().end());
  auto* dv = upload(kV, hv);
  void* dy = t_arena.get(kY, rows * h_out * 2);
  cuda_check(cudaMemsetAsync(dy, 0, rows * h_out * 2, t_arena.s()), "cudaMemsetAsync");
  const StagedModels sm = stage_models(models, rank, rank, h_out, false, true, p);
  lsg_weight_table tbl = sm.tbl;
  tbl.h_in = static_cast<int32_t>(models.front().h_in());  // only rank <= h_in is checked for expand
  tbl.a_layer_stride = static_cast<int64_t>(tbl.h_in) * static_cast<int64_t>(rank);
  lsg_check(lsg_sgmv_expand(dy, static_cast<int64_t>(h_out), dv, &tbl, upload_segments(segments),
                            upload_identity_slots(n), to_i32(n, "segment count"), to_i32(rows, "row count"), 0,
                            reinterpret_cast<lsg_stream_t>(t_arena.s())),
            "lsg_sgmv_expand");
  return download(dy, rows, h_out, p);
}

Matrix lora_addon(const Batch& batch) {
  if (batch.models.empty()) return Matrix(0, 0);
  const Dims d = shrink_dims(batch);
  // expand-side checks of the reference composition (sgmv_expand on shrink's output)
  const std::size_t h_out = common_h_out(batch, "sgmv_expand");
  return addon_on_device(batch, d.rank, h_out, Form::Fused, nullptr);
}

Matrix dense_projection(const Batch& batch, const Matrix& w) {
  if (w.rows() != batch.x.cols()) throw std::invalid_argument("dense_projection: w rows != batch hidden dim");
  for (const auto& m : batch.models)
    if (m.h_out() != w.cols()) throw std::invalid_argument("dense_projection: adapter output dim != w columns");
  if (batch.rows() == 0) return Matrix(0, w.cols());
  const Dims d = shrink_dims(batch);
  return addon_on_device(batch, d.rank, w.cols(), Form::Fused, &w);
}

Matrix lora_loop_oracle(const Batch& batch) {
  const Dims d = shrink_dims(batch);
  if (batch.models.empty()) return Matrix(0, 0);
  const std::size_t h_out = common_h_out(batch, "lora_loop_oracle");
  return addon_on_device(batch, d.rank, h_out, Form::TwoLaunch, nullptr);
}

Matrix gather_bmm_oracle(const Batch& batch) {
  const Dims d = shrink_dims(batch);
  if (batch.models.empty()) return Matrix(0, 0);
  const std::size_t h_out = common_h_out(batch, "gather_bmm_oracle");
  return addon_on_device(batch, d.rank, h_out, Form::PerRow, nullptr);
}

// ---- serving-side pool -----------------------------------------------------------------
namespace b200 {

struct AdapterPool::Impl {
  int slots, layers, h_in, h_out, rank;
  Precision p;
  uint16_t* a = nullptr;
  uint16_t* b = nullptr;
  const void** pa = nullptr;
  const void** pb = nullptr;
  lsg_weight_table tbl{};
  std::map<LoraId, int> slot_of;
  int next = 0;
};

AdapterPool::AdapterPool(int slots, int layers, int h_in, int h_out, int rank, Precision p) : impl_(new Impl) {
  if (slots < 1 || layers < 1 || rank < 1 || rank > h_in || rank > h_out)
    throw std::invalid_argument("AdapterPool: invalid geometry");
  Impl& m = *impl_;
  m.slots = slots;
  m.layers = layers;
  m.h_in = h_in;
  m.h_out = h_out;
  m.rank = rank;
  m.p = p;
  const std::size_t sa = static_cast<std::size_t>(layers) * h_in * rank, sb = static_cast<std::size_t>(layers) * rank * h_out;
  cuda_check(cudaMalloc(&m.a, sa * slots * 2), "cudaMalloc pool A");
  cuda_check(cudaMalloc(&m.b, sb * slots * 2), "cudaMalloc pool B");
  std::vector<const void*> pa(slots), pb(slots);
  for (int s = 0; s < slots; ++s) {
    pa[s] = m.a + sa * s;
    pb[s] = m.b + sb * s;
  }
  cuda_check(cudaMalloc(&m.pa, slots * sizeof(void*)), "cudaMalloc table");
  cuda_check(cudaMalloc(&m.pb, slots * sizeof(void*)), "cudaMalloc table");
  cuda_check(cudaMemcpy(m.pa, pa.data(), slots * sizeof(void*), cudaMemcpyHostToDevice), "table H2D");
  cuda_check(cudaMemcpy(m.pb, pb.data(), slots * sizeof(void*), cudaMemcpyHostToDevice), "table H2D");
  m.tbl.a_ptr = m.pa;
  m.tbl.b_ptr = m.pb;
  m.tbl.a_layer_stride = static_cast<int64_t>(h_in) * rank;
  m.tbl.b_layer_stride = static_cast<int64_t>(rank) * h_out;
  m.tbl.num_slots = slots;
  m.tbl.num_layers = layers;
  m.tbl.h_in = h_in;
  m.tbl.h_out = h_out;
  m.tbl.rank = rank;
  m.tbl.dtype = p == Precision::F16 ? LSG_F16 : LSG_BF16;
}

AdapterPool::~AdapterPool() {
  cudaFree(impl_->a);
  cudaFree(impl_->b);
  cudaFree(impl_->pa);
  cudaFree(impl_->pb);
  delete impl_;
}

int AdapterPool::load(LoraId id, int layer, const Matrix& a, const Matrix& b) {
  Impl& m = *impl_;
  if (layer < 0 || layer >= m.layers) throw std::invalid_argument("AdapterPool::load: layer out of range");
  if (a.rows() != static_cast<std::size_t>(m.h_in) || a.cols() != static_cast<std::size_t>(m.rank) ||
      b.rows() != static_cast<std::size_t>(m.rank) || b.cols() != static_cast<std::size_t>(m.h_out))
    throw std::invalid_argument("AdapterPool::load: adapter shape does not match the pool");
  auto it = m.slot_of.find(id);
  int slot;
  if (it != m.slot_of.end()) {
    slot = it->second;
  } else {
    if (m.next >= m.slots) throw std::runtime_error("AdapterPool::load: pool full");
    slot = m.next++;
    m.slot_of[id] = slot;
  }
  const std::size_t sa = static_cast<std::size_t>(m.layers) * m.h_in * m.rank;
  const std::size_t sb = static_cast<std::size_t>(m.layers) * m.rank * m.h_out;
  const auto ha = to_bits(a.data(), m.p), hb = to_bits(b.data(), m.p);
  cuda_check(cudaMemcpy(m.a + sa * slot + static_cast<std::size_t>(layer) * m.h_in * m.rank, ha.data(), ha.size() * 2,
                        cudaMemcpyHostToDevice), "pool H2D");
  cuda_check(cudaMemcpy(m.b + sb * slot + static_cast<std::size_t>(layer) * m.rank * m.h_out, hb.data(), hb.size() * 2,
                        cudaMemcpyHostToDevice), "pool H2D");
  return slot;
}

int AdapterPool::slot_of(LoraId id) const {
  auto it = impl_->slot_of.find(id);
  return it == impl_->slot_of.end() ? -1 : it->second;
}

const lsg_weight_table& AdapterPool::table() const { return impl_->tbl; }

}  // namespace b200
}  // namespace lorasim
