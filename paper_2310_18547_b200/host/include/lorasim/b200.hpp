// lorasim/b200.hpp -- B200-specific knobs and the serving-side adapter pool of
// the drop-in library (no reference counterpart).
#pragma once

#include <cstddef>
#include <cstdint>
#include <map>
#include <vector>

#include "lorasim/sgmv.hpp"

struct lsg_weight_table;

namespace lorasim::b200 {

enum class Precision { F16 = 0, BF16 = 1 };

// Working precision of the value-semantic operators in lorasim/sgmv.hpp.
void set_precision(Precision p);
Precision precision();

// Round a double to the working precision (round-to-nearest-even) and back.
double quantize(double v, Precision p);

// Device-resident adapter pool for one projection site across `layers` layers:
// slot -> [layers][h_in][rank] (A) and [layers][rank][h_out] (B) in the working
// precision, plus the device pointer table the kernels index with.  LoraId ->
// slot mapping is kept on the host (the role GpuState::adapter_ready_time plays
// in the reference simulator, scheduler.hpp:39-48).
class AdapterPool {
 public:
  AdapterPool(int slots, int layers, int h_in, int h_out, int rank, Precision p = Precision::F16);
  ~AdapterPool();
  AdapterPool(const AdapterPool&) = delete;
  AdapterPool& operator=(const AdapterPool&) = delete;

  // Upload one adapter's layer (double -> working precision); returns its slot.
  int load(LoraId id, int layer, const Matrix& a, const Matrix& b);
  int slot_of(LoraId id) const;  // -1 if not resident
  const lsg_weight_table& table() const;

 private:
  struct Impl;
  Impl* impl_;
};

}  // namespace lorasim::b200
