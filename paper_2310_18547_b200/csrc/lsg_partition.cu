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
//   * with a slot-sharded pool (seg_owner != NULL) a segment whose adapter lives
//     on one rank only goes to that rank, whole -- the request is routed to the
//     GPU that holds its adapter, as Scheduler::place routes requests to the GPU
//     with the adapter in its working set (scheduler.cpp:12-29);
//   * the remaining (replicated) segments may be cut into row ranges, each of
//     which pays the adapter's h*r weights again on its own rank.  A cut is kept
//     only when it lowers the largest rank load: the planner grows the part count
//     of the segment with the largest piece one step at a time (at most world-1
//     extra pieces in all), evaluates the LPT makespan after each step, and keeps
//     the best plan seen (ties: fewer pieces);
//   * pieces go to ranks by LPT greedy on algorithmic bytes
//     rows*(h_in+h_out)*e + h_in*r*e + r*h_out*e (the two SGMV halves of
//     cost_model.cpp:13-19 / :59): largest piece first (ties: lower segment, then
//     lower row), onto the least-loaded rank (ties: lower rank).
//
// So a plan has at most (non-empty segments) + world - 1 pieces.
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

namespace {

struct Piece {
  int32_t seg, row0, row1;
  int64_t bytes;
};

// Cut segment s of length len into k near-equal row ranges.
void cut(std::vector<Piece>& out, int32_t s, int32_t b, int32_t len, int32_t k, int64_t row_bytes,
         int64_t adapter_bytes) {
  for (int32_t j = 0; j < k; ++j) {
    const int32_t r0 = b + static_cast<int32_t>(static_cast<int64_t>(len) * j / k);
    const int32_t r1 = b + static_cast<int32_t>(static_cast<int64_t>(len) * (j + 1) / k);
    out.push_back({s, r0, r1, (r1 - r0) * row_bytes + adapter_bytes});
  }
}

// LPT onto ranks whose loads start at `base`; returns the makespan, fills owner.
int64_t lpt(const std::vector<Piece>& pcs, const std::vector<int64_t>& base, std::vector<int32_t>& owner) {
  std::vector<int> order(pcs.size());
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return pcs[a].bytes > pcs[b].bytes; });
  std::vector<int64_t> load = base;
  owner.assign(pcs.size(), 0);
  for (int i : order) {
    const int r = static_cast<int>(std::min_element(load.begin(), load.end()) - load.begin());
    owner[i] = r;
    load[r] += pcs[i].bytes;
  }
  return *std::max_element(load.begin(), load.end());
}

}  // namespace
}  // namespace lsg

extern "C" int lsg_partition_segments(const int32_t* seg_starts, const int32_t* seg_owner, int32_t num_segments,
                                      int32_t h_in, int32_t h_out, int32_t rank, int32_t elem_bytes, int32_t world,
                                      int32_t max_pieces, lsg_piece* pieces, int32_t* num_pieces) {
  using lsg::fail;
  if (num_pieces == nullptr) return fail(LSG_EINVAL, "lsg_partition_segments: num_pieces is NULL");
  *num_pieces = 0;
  if (num_segments < 0 || world < 1 || h_in < 1 || h_out < 1 || rank < 1 || elem_bytes < 1 || max_pieces < 0)
    return fail(LSG_EINVAL, "lsg_partition_segments: bad sizes");
  if (num_segments == 0) return LSG_OK;
  if (seg_starts == nullptr) return fail(LSG_EINVAL, "lsg_partition_segments: seg_starts is NULL");
  if (seg_starts[0] != 0) return fail(LSG_EINVAL, "lsg_partition_segments: seg_starts[0] must be 0");
  for (int s = 0; s < num_segments; ++s) {
    if (seg_starts[s + 1] < seg_starts[s]) return fail(LSG_EINVAL, "lsg_partition_segments: seg_starts decreasing");
    if (seg_owner != nullptr && seg_owner[s] >= world)
      return fail(LSG_EINVAL, "lsg_partition_segments: seg_owner names a rank >= world");
  }

  const int64_t row_bytes = static_cast<int64_t>(h_in + h_out) * elem_bytes;
  const int64_t adapter_bytes = (static_cast<int64_t>(h_in) * rank + static_cast<int64_t>(rank) * h_out) * elem_bytes;

  // Pinned segments (adapter on one rank only) load their owner first.
  std::vector<int64_t> base(world, 0);
  std::vector<lsg::Piece> pinned;
  std::vector<int32_t> pinned_owner, free_segs, parts;
  for (int s = 0; s < num_segments; ++s) {
    const int32_t len = seg_starts[s + 1] - seg_starts[s];
    if (len == 0) continue;
    if (seg_owner != nullptr && seg_owner[s] >= 0) {
      pinned.push_back({s, seg_starts[s], seg_starts[s + 1], len * row_bytes + adapter_bytes});
      pinned_owner.push_back(seg_owner[s]);
      base[seg_owner[s]] += pinned.back().bytes;
    } else {
      free_segs.push_back(s);
      parts.push_back(1);
    }
  }
  auto build = [&](std::vector<lsg::Piece>& pcs) {
    pcs.clear();
    for (size_t i = 0; i < free_segs.size(); ++i) {
      const int32_t s = free_segs[i];
      lsg::cut(pcs, s, seg_starts[s], seg_starts[s + 1] - seg_starts[s], parts[i], row_bytes, adapter_bytes);
    }
  };
  std::vector<lsg::Piece> pcs, best;
  std::vector<int32_t> owner, best_owner;
  build(pcs);
  int64_t best_span = lsg::lpt(pcs, base, owner);
  best = pcs;
  best_owner = owner;
  // Grow the part count of the free segment with the largest piece, up to world-1 extra pieces.
  for (int extra = 0; extra < world - 1 && !free_segs.empty(); ++extra) {
    int pick = -1;
    int64_t pick_bytes = -1;
    for (size_t i = 0; i < free_segs.size(); ++i) {
      const int32_t s = free_segs[i], len = seg_starts[s + 1] - seg_starts[s];
      if (parts[i] >= len || parts[i] >= world) continue;
      const int32_t biggest = (len + parts[i] - 1) / parts[i];
      const int64_t b = biggest * row_bytes + adapter_bytes;
      if (b > pick_bytes) {
        pick_bytes = b;
        pick = static_cast<int>(i);
      }
    }
    if (pick < 0) break;
    ++parts[pick];
    build(pcs);
    const int64_t span = lsg::lpt(pcs, base, owner);
    if (span < best_span) {
      best_span = span;
      best = pcs;
      best_owner = owner;
    }
  }
  const int64_t count = static_cast<int64_t>(pinned.size() + best.size());
  if (count > max_pieces || pieces == nullptr) {
    *num_pieces = static_cast<int32_t>(count);
    return fail(LSG_EINVAL, "lsg_partition_segments: max_pieces too small (num_pieces holds the count needed)");
  }
  // All pieces with their ranks, then output in (rank, segment, row) order: each
  // rank's pieces form its local batch.  Adjacent row ranges of one segment that
  // landed on one rank are merged (one local segment, the adapter read once).
  struct Placed {
    int32_t rank, seg, row0, row1;
  };
  std::vector<Placed> all;
  for (size_t i = 0; i < pinned.size(); ++i)
    all.push_back({pinned_owner[i], pinned[i].seg, pinned[i].row0, pinned[i].row1});
  for (size_t i = 0; i < best.size(); ++i) all.push_back({best_owner[i], best[i].seg, best[i].row0, best[i].row1});
  std::sort(all.begin(), all.end(), [](const Placed& a, const Placed& b) {
    return a.rank != b.rank ? a.rank < b.rank : a.seg != b.seg ? a.seg < b.seg : a.row0 < b.row0;
  });
  int32_t n = 0;
  for (const Placed& p : all) {
    if (n > 0 && pieces[n - 1].rank == p.rank && pieces[n - 1].seg == p.seg && pieces[n - 1].row1 == p.row0)
      pieces[n - 1].row1 = p.row1;
    else
      pieces[n++] = lsg_piece{p.rank, p.seg, p.row0, p.row1};
  }
  *num_pieces = n;
  return LSG_OK;
}
