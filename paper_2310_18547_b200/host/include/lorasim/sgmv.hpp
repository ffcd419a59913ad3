// lorasim/sgmv.hpp -- B200 drop-in for the reference's SGMV operator API
// (proj/core/include/lorasim/sgmv.hpp:11-83, proj/core/src/sgmv.cpp).
//
// Link this library (liblorasim_b200.so) instead of the reference's sgmv.cpp
// and every caller -- verify_sgmv, bench_sgmv, dense_projection users, the
// unit tests -- runs on the B200 through the C-ABI in include/lsg_sgmv.h:
//
//   sgmv_shrink        -> lsg_sgmv_shrink   (cluster split-K shrink, fp32 v)
//   sgmv_expand        -> lsg_sgmv_expand   (expand fused with y +=, 128-bit stores)
//   lora_addon         -> lsg_sgmv          (one fused shrink+expand launch)
//   dense_projection   -> cuBLAS x*W (the plain backbone GEMM) + lsg_sgmv (+= into it)
//   lora_loop_oracle   -> lsg_sgmv_shrink + lsg_sgmv_expand (the two-launch formulation)
//   gather_bmm_oracle  -> lsg_bgmv (the per-row gather formulation)
//
// The two reference "oracles" are, on the GPU, the two alternative kernel
// formulations of the same operator; the CPU fp64 oracles used to CHECK this
// library live in oracle/ (tests only).  Every operator validates its inputs
// exactly like the reference (same std::invalid_argument messages) before any
// device work; device failures throw std::runtime_error.  There is no CPU path:
// without a usable GPU the operators throw.
//
// Numerics: x, A, B are rounded to the working precision (fp16 by default,
// see lorasim/b200.hpp), accumulation is fp32, v stays fp32, y is rounded once
// and widened back to double.
#pragma once

#include <cstdint>
#include <vector>

#include "lorasim/matrix.hpp"

namespace lorasim {

using LoraId = std::int64_t;

// Boundaries s_0 = 0 < s_1 < ... < s_n of contiguous row segments.
class Segments {
 public:
  explicit Segments(std::vector<std::size_t> boundaries);

  static Segments single(std::size_t rows);
  static Segments empty() { return Segments(std::vector<std::size_t>{0}); }

  std::size_t count() const { return bounds_.size() - 1; }
  std::size_t total_rows() const { return bounds_.back(); }
  std::size_t begin_of(std::size_t i) const { return bounds_[i]; }
  std::size_t end_of(std::size_t i) const { return bounds_[i + 1]; }
  std::size_t size_of(std::size_t i) const { return end_of(i) - begin_of(i); }
  const std::vector<std::size_t>& boundaries() const { return bounds_; }

  bool operator==(const Segments& other) const { return bounds_ == other.bounds_; }

 private:
  std::vector<std::size_t> bounds_;
};

// A LoRA adapter: a is h_in x rank, b is rank x h_out; 1 <= rank <= min(h_in, h_out).
struct LoraModel {
  LoraModel(LoraId id, Matrix a, Matrix b);

  std::size_t rank() const { return a.cols(); }
  std::size_t h_in() const { return a.rows(); }
  std::size_t h_out() const { return b.cols(); }

  LoraId id;
  Matrix a;
  Matrix b;
};

// Token rows plus their segmentation; models[i] serves rows [s_i, s_{i+1}).
struct Batch {
  Batch(Matrix x, Segments segments, std::vector<LoraModel> models);

  std::size_t rows() const { return segments.total_rows(); }
  std::size_t h_in() const { return x.cols(); }

  Matrix x;
  Segments segments;
  std::vector<LoraModel> models;
};

Matrix sgmv_shrink(const Batch& batch);
Matrix sgmv_expand(const Matrix& v, const Segments& segments, const std::vector<LoraModel>& models);
Matrix lora_addon(const Batch& batch);
Matrix dense_projection(const Batch& batch, const Matrix& w);
Matrix lora_loop_oracle(const Batch& batch);
Matrix gather_bmm_oracle(const Batch& batch);

}  // namespace lorasim
