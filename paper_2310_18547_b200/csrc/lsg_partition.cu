// lsg_partition.cu -- request-partitioned multi-GPU plan (host only, no device code).
//
// SGMV rows are independent: row j of segment s depends only on x[j] and the
// adapter of s (reference sgmv.cpp:108-116, 125-134).  A batch therefore shards
// across GPUs with no collective on the data path, the way the reference's
// scheduler places whole requests on GPUs (scheduler.cpp:12-29).  This planner
// cuts one decode step's segments into pieces and assigns them to ranks:
//
//   * the unit of placement is a segment (all rows of one adapter on one rank,
//     so that adapter's A and B are read from HBM once);
//   * a segment whose algorithmic bytes exceed the ideal per-rank share
//     (Identical / Skewed popularity) is cut into near-equal row ranges, each of
//     which pays the adapter's h*r weights again on its own rank;
//   * pieces go to ranks by LPT greedy on algorithmic bytes
//     rows*(h_in+h_out)*e + h_in*r*e + r*h_out*e (the two SGMV halves of
//     cost_model.cpp:13-19 / :59): largest piece first (ties: lower segment, then
//     lower row), onto the least-loaded rank (ties: lower rank).
//
// Pure integer arithmetic: every rank computes the same plan from the same
// seg_starts without communicating.
#include <algorithm>
#include <cstdint>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/lsg_sgmv.h"

namespace lsg {
int fail(int status, const std::string& msg);
}

extern "C" int lsg_partition_segments(const int32_t* seg_starts, int32_t num_segments, int32_t h_in, int32_t h_out,
                                      int32_t rank, int32_t elem_bytes, int32_t world, int32_t max_pieces,
                                      lsg_piece* pieces, int32_t* num_pieces) {
  using lsg::fail;
  if (num_pieces == nullptr) return fail(LSG_EINVAL, "lsg_partition_segments: num_pieces is NULL");
  *num_pieces = 0;
  if (num_segments < 0 || world < 1 || h_in < 1 || h_out < 1 || rank < 1 || elem_bytes < 1 || max_pieces < 0)
    return fail(LSG_EINVAL, "lsg_partition_segments: bad sizes");
  if (num_segments == 0) return LSG_OK;
  if (seg_starts == nullptr) return fail(LSG_EINVAL, "lsg_partition_segments: seg_starts is NULL");
  if (seg_starts[0] != 0) return fail(LSG_EINVAL, "lsg_partition_segments: seg_starts[0] must be 0");
  for (int s = 0; s < num_segments; ++s)
    if (seg_starts[s + 1] < seg_starts[s]) return fail(LSG_EINVAL, "lsg_partition_segments: seg_starts decreasing");

  const int64_t row_bytes = static_cast<int64_t>(h_in + h_out) * elem_bytes;
  const int64_t adapter_bytes = (static_cast<int64_t>(h_in) * rank + static_cast<int64_t>(rank) * h_out) * elem_bytes;
  auto bytes_of = [&](int64_t rows) { return rows * row_bytes + adapter_bytes; };
  int64_t total = 0;
  for (int s = 0; s < num_segments; ++s)
    if (seg_starts[s + 1] > seg_starts[s]) total += bytes_of(seg_starts[s + 1] - seg_starts[s]);
  const int64_t share = (total + world - 1) / world;

  struct Cand {
    int32_t seg, row0, row1;
    int64_t bytes;
  };
  std::vector<Cand> cands;
  for (int s = 0; s < num_segments; ++s) {
    const int32_t b = seg_starts[s], e = seg_starts[s + 1];
    const int32_t len = e - b;
    if (len == 0) continue;
    int32_t parts = 1;
    if (world > 1 && bytes_of(len) > share) {
      // smallest part count whose row ranges each fit the share (at most one per rank, one row each)
      parts = static_cast<int32_t>((bytes_of(len) + share - 1) / share);
      while (parts < std::min<int64_t>(len, world) && bytes_of((len + parts - 1) / parts) > share) ++parts;
      parts = static_cast<int32_t>(std::min<int64_t>({static_cast<int64_t>(parts), len, world}));
    }
    for (int32_t k = 0; k < parts; ++k) {
      const int32_t r0 = b + static_cast<int32_t>(static_cast<int64_t>(len) * k / parts);
      const int32_t r1 = b + static_cast<int32_t>(static_cast<int64_t>(len) * (k + 1) / parts);
      cands.push_back({s, r0, r1, bytes_of(r1 - r0)});
    }
  }
  if (static_cast<int64_t>(cands.size()) > max_pieces || pieces == nullptr) {
    *num_pieces = static_cast<int32_t>(cands.size());
    return fail(LSG_EINVAL, "lsg_partition_segments: max_pieces too small (num_pieces holds the count needed)");
  }
  std::vector<int> order(cands.size());
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cands[a].bytes > cands[b].bytes; });
  std::vector<int64_t> load(world, 0);
  std::vector<int32_t> owner(cands.size(), 0);
  for (int i : order) {
    const int r = static_cast<int>(std::min_element(load.begin(), load.end()) - load.begin());
    owner[i] = r;
    load[r] += cands[i].bytes;
  }
  // Output in (rank, segment, row) order: each rank's pieces form its local batch.
  // Adjacent row ranges of one segment that landed on the same rank are merged
  // (one local segment, the adapter read once).
  int32_t n = 0;
  for (int r = 0; r < world; ++r)
    for (size_t i = 0; i < cands.size(); ++i) {
      if (owner[i] != r) continue;
      if (n > 0 && pieces[n - 1].rank == r && pieces[n - 1].seg == cands[i].seg && pieces[n - 1].row1 == cands[i].row0)
        pieces[n - 1].row1 = cands[i].row1;
      else
        pieces[n++] = lsg_piece{r, cands[i].seg, cands[i].row0, cands[i].row1};
    }
  *num_pieces = n;
  return LSG_OK;
}
