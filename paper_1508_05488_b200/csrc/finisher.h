// Host finisher (see finisher.cpp).
#pragma once

#include <stddef.h>

#include <vector>

namespace chgpu {
namespace host {

struct Pt {
  double x, y;
};

enum { kOk = 0, kEmpty = 1, kDegenerate = 2, kInvalid = 3 };

int assemble_ring(const Pt* chains, const size_t kept_counts[4], const Pt corners[4],
                  std::vector<Pt>& ring);
void canonicalize(Pt* ring, size_t n);
int melkman(const Pt* poly, size_t n, std::vector<Pt>& hull);
// melkman() over a ring that is already free of consecutive and wrap
// duplicates (what assemble_ring returns).
int melkman_ring(const Pt* ring, size_t n, std::vector<Pt>& hull);
// assemble_ring + melkman_ring in one streaming pass (no ring copy).
int finish_chains(const Pt* chains, const size_t kept_counts[4], const Pt corners[4],
                  std::vector<Pt>& hull);
// finish_chains with the four chains run concurrently and verified; same result.
int finish_chains_split(const Pt* chains, const size_t kept_counts[4], const Pt corners[4],
                        std::vector<Pt>& hull);
// A call expecting about this many chain points is on its way to
// finish_chains_split: let the worker threads spin instead of parking.
void finisher_prewake(size_t expected_chain_points);
// The hull of the union of several runs of SPA chains (one run per shard:
// its 4 region chains concatenated, counts4[4 * k + r]), each region's runs
// merged in region order, then finish_chains_split over the merged chains.
int merge_chains_hull(const Pt* const* runs, const size_t* counts4, int nruns, const Pt corners[4],
                      std::vector<Pt>& hull);
int monotone_chain(const Pt* sorted_unique, size_t n, std::vector<Pt>& hull);
int sorted_hull(const Pt* pts, size_t n, std::vector<Pt>& hull);
void insert_sorted_unique(std::vector<Pt>& sorted, const Pt& p);

}  // namespace host
}  // namespace chgpu
