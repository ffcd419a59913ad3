// lorasim_b200 -- the SGMV verbs of the reference CLI (tools/lorasim_cli.cpp:46-73)
// running on the B200:
//
//   lorasim_b200 [--seed N] [--out DIR] [--precision fp16|bf16] verify-sgmv [--trials N] [--inject-fault]
//   lorasim_b200 [--out DIR] roofline [--max-batch N]
//
// Exit codes as in the reference (lorasim_cli.cpp:16-18): 0 ok, 1 verification
// failure, 2 usage error.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <string>
#include <vector>

#include "lorasim/b200.hpp"
#include "lorasim/experiments.hpp"

namespace {

int usage() {
  std::fprintf(stderr,
               "usage: lorasim_b200 [--seed N] [--out DIR] [--precision fp16|bf16] <verb> [flags]\n"
               "  verify-sgmv [--trials N] [--inject-fault]\n"
               "  roofline [--max-batch N]\n");
  return 2;
}

}  // namespace

int main(int argc, char** argv) {
  std::vector<std::string> args(argv + 1, argv + argc);
  std::uint64_t seed = 42;
  std::string out = "out";
  std::string verb;
  int trials = 1000, max_batch = 64;
  bool inject = false;
  try {
    for (std::size_t i = 0; i < args.size(); ++i) {
      const std::string& a = args[i];
      auto value = [&]() -> std::string {
        if (i + 1 >= args.size()) throw std::invalid_argument("missing value for " + a);
        return args[++i];
      };
      if (a == "--seed") seed = std::stoull(value());
      else if (a == "--out") out = value();
      else if (a == "--precision") {
        const std::string p = value();
        if (p == "fp16") lorasim::b200::set_precision(lorasim::b200::Precision::F16);
        else if (p == "bf16") lorasim::b200::set_precision(lorasim::b200::Precision::BF16);
        else throw std::invalid_argument("--precision must be fp16 or bf16");
      } else if (a == "--trials") trials = std::stoi(value());
      else if (a == "--max-batch") max_batch = std::stoi(value());
      else if (a == "--inject-fault") inject = true;
      else if (verb.empty() && (a == "verify-sgmv" || a == "roofline")) verb = a;
      else throw std::invalid_argument("unknown argument " + a);
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "lorasim_b200: %s\n", e.what());
    return usage();
  }
  if (verb.empty()) return usage();

  if (verb == "verify-sgmv") {
    try {
      const lorasim::VerifyReport r = lorasim::verify_sgmv(trials, seed, inject);
      std::printf("verify-sgmv: %d trials, %d failures, worst deviation %.3e (tolerance %.0e) on B200\n", r.trials,
                  r.failures, r.worst_deviation, r.tolerance);
      for (const auto& c : r.failed_cases)
        std::printf("  trial %d %s h_in=%zu h_out=%zu r=%zu rows=%zu models=%zu deviation %.3e\n", c.trial,
                    lorasim::to_string(c.popularity), c.h_in, c.h_out, c.rank, c.rows, c.models, c.deviation);
      return r.passed() ? 0 : 1;
    } catch (const std::exception& e) {
      std::fprintf(stderr, "lorasim_b200: %s\n", e.what());
      return 1;
    }
  }
  const auto rows = lorasim::roofline_sweep(lorasim::CostParams{}, max_batch);
  std::filesystem::create_directories(out);
  std::ofstream(std::filesystem::path(out) / "roofline.csv") << lorasim::roofline_csv(rows);
  std::printf("roofline: %zu rows -> %s/roofline.csv\n", rows.size(), out.c_str());
  return 0;
}
