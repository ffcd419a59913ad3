// lorasim/experiments.hpp -- B200 drop-in, the SGMV harnesses of the
// reference's experiments layer (proj/core/include/lorasim/experiments.hpp):
// the randomised three-formulation equivalence check behind `verify-sgmv`, and
// the roofline sweep behind `roofline`.  The simulator arms (run_simulation,
// compare_modes) are out of scope.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "lorasim/cost_model.hpp"
#include "lorasim/workload.hpp"

namespace lorasim {

struct VerifyCase {
  int trial = 0;
  Popularity popularity = Popularity::Distinct;
  std::size_t h_in = 0;
  std::size_t h_out = 0;
  std::size_t rank = 0;
  std::size_t rows = 0;
  std::size_t models = 0;
  double deviation = 0.0;
  bool passed = true;
};

struct VerifyReport {
  int trials = 0;
  int failures = 0;
  double worst_deviation = 0.0;
  double tolerance = 1e-10;
  std::vector<VerifyCase> failed_cases;

  bool passed() const { return failures == 0; }
};

// Same trial generator as the reference (experiments.cpp:35-102).  On the B200
// the three formulations compared are the fused launch (lora_addon), the
// two-launch shrink/expand (lora_loop_oracle) and the per-row BGMV
// (gather_bmm_oracle); with the library's fixed reduction order they agree
// bit for bit, so the reference's 1e-10 tolerance still applies.
VerifyReport verify_sgmv(int trials, std::uint64_t seed, bool inject_fault = false);

struct RooflineRow {
  int batch_size = 0;
  Popularity distribution = Popularity::Distinct;
  double flop = 0.0;
  double io_bytes = 0.0;
  double intensity = 0.0;
  double est_latency = 0.0;
};

std::vector<RooflineRow> roofline_sweep(const CostParams& params, int max_batch = 64);
std::string roofline_csv(const std::vector<RooflineRow>& rows);

}  // namespace lorasim
