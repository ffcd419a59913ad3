// lorasim/cost_model.hpp -- B200 drop-in, the SGMV formula part of the
// reference's cost model (proj/core/include/lorasim/cost_model.hpp): FLOP and
// byte counts of one segmented launch, arithmetic intensity, the roofline
// latency, the gather-BMM overhead, and the shrink+expand pair bytes that the
// benchmark uses as its algorithmic-bytes numerator.  The simulated decode
// clock (decode_step_latency, adapter_load_latency) is out of scope.
#pragma once

#include <cstdint>

namespace lorasim {

struct CostParams {
  double peak_flops = 312e12;
  double mem_bw = 2.0e12;
  double kernel_overhead = 38e-6;
  double pcie_bw = 32e9;
  int elem_bytes = 2;
  int layers = 32;
  int hidden_dim = 4096;
  int lora_rank = 16;
  int projections_per_layer = 7;
  double attn_coeff = 9e-9;
  double proj_coeff = 1.0 / (0.5 * 312e12);
};

// n adapters over s_n rows, h_in -> h_out.
struct SgmvShape {
  std::int64_t num_models = 0;
  std::int64_t total_rows = 0;
  std::int64_t h_in = 0;
  std::int64_t h_out = 0;
};

double sgmv_flop(const SgmvShape& shape);                        // 2 s_n h_in h_out
double sgmv_io_bytes(const SgmvShape& shape, int elem_bytes = 2);  // (s_n(h_in+h_out) + n h_in h_out) e
double arithmetic_intensity(const SgmvShape& shape, int elem_bytes = 2);
double sgmv_latency(const SgmvShape& shape, const CostParams& params);
double gather_bmm_extra_elements(const SgmvShape& shape);
double gather_bmm_extra_io_bytes(const SgmvShape& shape, int elem_bytes = 2);

// One LoRA projection site = shrink (h -> r) + expand (r -> h): the operator
// the paper times.  Bytes = 2 (s_n (h + r) + n h r) e.
double adapter_pair_io_bytes(double rows, double models, double hidden, double rank, int elem_bytes = 2);
double adapter_pair_flop(double rows, double hidden, double rank);

}  // namespace lorasim
