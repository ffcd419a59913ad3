// sim_b200.cpp -- SURVEY 8(f-4): the reference's system-level experiments re-run with the SGMV
// cost model recalibrated to B200 measurements.
//
// The reference's simulator (proj/core/src/simulator.cpp, experiments.cpp; built in place by
// integration/CMakeLists.txt) models every LoRA projection with adapter_pair_latency
// (cost_model.cpp:55-61), i.e. max(flop / peak, io / mem_bw, kernel_overhead), on A100-era
// constants (config.hpp:20-34: 312 TFLOP/s, 2 TB/s, a 38 us launch floor).  This driver runs the
// reference's own experiments unchanged -- the throughput comparison at saturation (compare_modes,
// acceptance_main.cpp:355-411, configs/saturation.json), the calibration anchors
// (acceptance_main.cpp:106-135, configs/default.json) and the cluster replay
// (configs/cluster_replay.json) -- once with the shipped constants and once with the constants
// fitted to this repo's B200 measurements (profiles/round1/b200_cost_params.json via
// scripts/calibrate_cost_model.py: the measured launch floor, the effective SGMV bandwidth, the
// measured bf16 peak and PCIe rate).  Nothing of the simulator is reimplemented here.
//
//   sim_b200 <reference proj dir> <b200_cost_params.json>
#include <cstdio>
#include <fstream>
#include <span>
#include <string>
#include <vector>

#include "json.hpp"
#include "lorasim/config.hpp"
#include "lorasim/cost_model.hpp"
#include "lorasim/experiments.hpp"
#include "lorasim/simulator.hpp"

using namespace lorasim;

namespace {

void apply_b200(ExperimentConfig& cfg, const nlohmann::json& j) {
  cfg.cost_model.peak_flops = j.at("peak_flops").get<double>();
  cfg.cost_model.mem_bw = j.at("mem_bw").get<double>();
  cfg.cost_model.kernel_overhead = j.at("kernel_overhead").get<double>();
  cfg.cost_model.pcie_bw = j.at("pcie_bw").get<double>();
}

void anchors(const ExperimentConfig& cfg, const char* label) {
  const CostParams p = cfg.cost_params();
  const auto step = [&](int batch, int seq) {
    std::vector<StepInput> in(static_cast<std::size_t>(batch), StepInput{seq, false, 0});
    return decode_step_latency(std::span<const StepInput>(in), p) * 1e3;
  };
  std::printf("%-6s decode step (ms): b=1 s=128 %.2f | b=32 s=128 %.2f | b=32 s=1600 %.2f | b32/b1 at s=512 %.3f\n",
              label, step(1, 128), step(32, 128), step(32, 1600), step(32, 512) / step(1, 512));
}

void compare(const ExperimentConfig& cfg, const char* label) {
  const CompareReport rep = compare_modes(cfg);
  std::printf("%-6s compare_modes (configs/saturation.json):\n", label);
  for (const CompareRow& r : rep.rows)
    std::printf("         %-10s multi %9.0f tok/s (p50 batch %2d, p50 token %.2f ms) | single %9.0f tok/s "
                "(p50 batch %2d) | ratio %6.2f\n",
                to_string(r.distribution), r.multi.throughput_tok_s, r.multi.batch_size_p50,
                r.multi.p50_token_latency_s * 1e3, r.single.throughput_tok_s, r.single.batch_size_p50,
                r.throughput_ratio);
}

void replay(const ExperimentConfig& cfg, const char* label) {
  Simulator sim(cfg);
  const Summary s = sim.run().summarize();
  std::printf("%-6s cluster replay (configs/cluster_replay.json): %d/%d finished, %.0f tok/s, makespan %.1f s, "
              "p50 token %.2f ms, p99 %.2f ms, peak GPUs busy %d, migrations %d\n",
              label, s.finished_requests, s.total_requests, s.throughput_tok_s, s.makespan_s,
              s.p50_token_latency_s * 1e3, s.p99_token_latency_s * 1e3, s.peak_gpus_busy, s.migrations);
}

}  // namespace

int main(int argc, char** argv) {
  if (argc != 3) {
    std::fprintf(stderr, "usage: sim_b200 <reference proj dir> <b200_cost_params.json>\n");
    return 2;
  }
  const std::string proj = argv[1];
  std::ifstream f(argv[2]);
  const nlohmann::json b200 = nlohmann::json::parse(f);
  for (int pass = 0; pass < 2; ++pass) {
    const char* label = pass == 0 ? "A100" : "B200";
    ExperimentConfig def = load_config_file(proj + "/configs/default.json");
    ExperimentConfig sat = load_config_file(proj + "/configs/saturation.json");
    ExperimentConfig rep = load_config_file(proj + "/configs/cluster_replay.json");
    if (pass == 1) {
      apply_b200(def, b200);
      apply_b200(sat, b200);
      apply_b200(rep, b200);
    }
    const CostParams p = def.cost_params();
    std::printf("%-6s cost model: peak %.0f TFLOP/s, mem_bw %.2f TB/s, kernel floor %.2f us, pcie %.1f GB/s\n", label,
                def.cost_model.peak_flops / 1e12, def.cost_model.mem_bw / 1e12, def.cost_model.kernel_overhead * 1e6,
                def.cost_model.pcie_bw / 1e9);
    (void)p;
    anchors(def, label);
    compare(sat, label);
    replay(rep, label);
  }
  return 0;
}
