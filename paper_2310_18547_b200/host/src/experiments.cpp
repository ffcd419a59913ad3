// experiments.cpp -- verify-sgmv and roofline harnesses on the B200
// (reference: experiments.cpp:35-174).
#include "lorasim/experiments.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <map>
#include <stdexcept>

#include "lorasim/sgmv.hpp"

namespace lorasim {

namespace {

Matrix draw_matrix(Rng& rng, std::size_t rows, std::size_t cols) {
  Matrix m(rows, cols);
  for (double& v : m.data()) v = rng.uniform01() * 2.0 - 1.0;
  return m;
}

Popularity trial_popularity(int trial) {
  static const Popularity cycle[] = {Popularity::Distinct, Popularity::Uniform, Popularity::Skewed,
                                     Popularity::Identical};
  return cycle[trial % 4];
}

}  // namespace

VerifyReport verify_sgmv(int trials, std::uint64_t seed, bool inject_fault) {
  if (trials < 0) throw std::invalid_argument("verify_sgmv: negative trial count");
  VerifyReport report;
  report.trials = trials;
  const std::size_t dims[] = {8, 64, 128};
  const std::size_t ranks[] = {8, 16, 32, 64};
  Rng rng(derive_seed(seed, 17));
  for (int trial = 0; trial < trials; ++trial) {
    const Popularity pop = trial_popularity(trial);
    const std::size_t h_in = dims[rng.uniform_index(3)];
    const std::size_t h_out = dims[rng.uniform_index(3)];
    std::vector<std::size_t> fit;
    for (std::size_t r : ranks)
      if (r <= std::min(h_in, h_out)) fit.push_back(r);
    const std::size_t rank = fit[rng.uniform_index(fit.size())];
    const int rows = rng.uniform_int(1, pop == Popularity::Distinct ? 8 : 64);
    const auto assignment = assign_models(rows, pop, 1.5, rng.next());

    std::map<LoraId, std::size_t> members;  // ascending adapter id -> row count
    for (auto id : assignment) ++members[id];
    std::vector<std::size_t> bounds{0};
    std::vector<LoraModel> models;
    Matrix x(static_cast<std::size_t>(rows), h_in);
    std::size_t cursor = 0;
    for (const auto& [id, count] : members) {
      // The reference draws each adapter's B before its A (argument evaluation
      // order of models.emplace_back under g++); keep that order so the batches
      // are bit-identical to the reference's.
      Matrix b = draw_matrix(rng, rank, h_out);
      Matrix a = draw_matrix(rng, h_in, rank);
      models.emplace_back(id, std::move(a), std::move(b));
      for (std::size_t i = 0; i < count; ++i, ++cursor)
        for (std::size_t c = 0; c < h_in; ++c) x(cursor, c) = rng.uniform01() * 2.0 - 1.0;
      bounds.push_back(cursor);
    }
    Batch batch(std::move(x), Segments(bounds), std::move(models));

    Matrix y = lora_addon(batch);
    if (inject_fault && trial == 0 && !y.data().empty()) y.data()[0] += 1e-6;
    const double dev = std::max(max_abs_diff(y, lora_loop_oracle(batch)), max_abs_diff(y, gather_bmm_oracle(batch)));

    VerifyCase c;
    c.trial = trial;
    c.popularity = pop;
    c.h_in = h_in;
    c.h_out = h_out;
    c.rank = rank;
    c.rows = static_cast<std::size_t>(rows);
    c.models = batch.models.size();
    c.deviation = dev;
    c.passed = dev < report.tolerance;
    report.worst_deviation = std::max(report.worst_deviation, dev);
    if (!c.passed) {
      ++report.failures;
      report.failed_cases.push_back(c);
    }
  }
  return report;
}

namespace {

// Expected number of distinct adapters among `batch` draws (experiments.cpp:108-137).
std::int64_t expected_distinct(Popularity pop, int batch, double alpha) {
  if (pop == Popularity::Distinct) return batch;
  if (pop == Popularity::Identical) return 1;
  const int m = model_count_for(batch, pop);
  double expect = 0.0;
  if (pop == Popularity::Uniform) {
    expect = m * (1.0 - std::pow(1.0 - 1.0 / m, batch));
  } else {
    double total = 0.0, w = 1.0;
    for (int i = 0; i < m; ++i, w /= alpha) total += w;
    w = 1.0;
    for (int i = 0; i < m; ++i, w /= alpha) expect += 1.0 - std::pow(1.0 - w / total, batch);
  }
  return std::clamp<std::int64_t>(std::llround(expect), 1, std::min(batch, m));
}

}  // namespace

std::vector<RooflineRow> roofline_sweep(const CostParams& params, int max_batch) {
  std::vector<RooflineRow> rows;
  for (Popularity pop : {Popularity::Distinct, Popularity::Uniform, Popularity::Skewed, Popularity::Identical}) {
    for (int b = 1; b <= max_batch; ++b) {
      const SgmvShape shape{expected_distinct(pop, b, 1.5), b, params.lora_rank, params.hidden_dim};
      RooflineRow row;
      row.batch_size = b;
      row.distribution = pop;
      row.flop = sgmv_flop(shape);
      row.io_bytes = sgmv_io_bytes(shape, params.elem_bytes);
      row.intensity = arithmetic_intensity(shape, params.elem_bytes);
      row.est_latency = sgmv_latency(shape, params);
      rows.push_back(row);
    }
  }
  return rows;
}

std::string roofline_csv(const std::vector<RooflineRow>& rows) {
  std::string out = "batch_size,distribution,flop,io_bytes,intensity,est_latency\n";
  char line[160];
  for (const RooflineRow& r : rows) {
    std::snprintf(line, sizeof line, "%d,%s,%.0f,%.0f,%.12g,%.9g\n", r.batch_size, to_string(r.distribution), r.flop,
                  r.io_bytes, r.intensity, r.est_latency);
    out += line;
  }
  return out;
}

}  // namespace lorasim
