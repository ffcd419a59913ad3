// cost_model.cpp -- SGMV formulas (reference: cost_model.cpp:8-40, 55-61).
#include "lorasim/cost_model.hpp"

#include <algorithm>
#include <stdexcept>

namespace lorasim {

namespace {
double d(std::int64_t v) { return static_cast<double>(v); }
}  // namespace

double sgmv_flop(const SgmvShape& s) { return 2.0 * d(s.total_rows) * d(s.h_in) * d(s.h_out); }

double sgmv_io_bytes(const SgmvShape& s, int elem_bytes) {
  const double activations = d(s.total_rows) * (d(s.h_in) + d(s.h_out));
  const double weights = d(s.num_models) * d(s.h_in) * d(s.h_out);
  return (activations + weights) * static_cast<double>(elem_bytes);
}

double arithmetic_intensity(const SgmvShape& s, int elem_bytes) {
  const double io = sgmv_io_bytes(s, elem_bytes);
  if (io <= 0.0) throw std::invalid_argument("arithmetic_intensity: zero-I/O shape");
  return sgmv_flop(s) / io;
}

double sgmv_latency(const SgmvShape& s, const CostParams& p) {
  return std::max({sgmv_flop(s) / p.peak_flops, sgmv_io_bytes(s, p.elem_bytes) / p.mem_bw, p.kernel_overhead});
}

double gather_bmm_extra_elements(const SgmvShape& s) { return 2.0 * d(s.total_rows) * d(s.h_in) * d(s.h_out); }

double gather_bmm_extra_io_bytes(const SgmvShape& s, int elem_bytes) {
  return gather_bmm_extra_elements(s) * static_cast<double>(elem_bytes);
}

double adapter_pair_io_bytes(double rows, double models, double hidden, double rank, int elem_bytes) {
  return 2.0 * (rows * (hidden + rank) + models * hidden * rank) * static_cast<double>(elem_bytes);
}

double adapter_pair_flop(double rows, double hidden, double rank) { return 4.0 * rows * hidden * rank; }

}  // namespace lorasim
