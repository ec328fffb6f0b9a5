// halo.h -- multi-GPU plan (host only, integer work): which GPU owns which global fine node, and which
// node values every pair of GPUs exchanges after the write-back (Algorithm 3 Step 4, followed
// by the overlap refresh that the lagged state of mode B needs, C2).
//
// Placement: subdomain *positions* (a porous box and a conduit box with the same grid index, C8) are the unit
// of work.  They are placed on the ranks by LPT (longest processing time first) on their cell counts (the
// extended porous box plus the extended conduit box): positions in decreasing weight, ties by index, each to
// the least-loaded rank, ties to the lowest rank.  For cfg4 at 2/4/8 ranks every rank receives
// the same mix of box shapes (18^3, 18^2 x 24, 18 x 24^2, 24^3), i.e. the octant balance of SURVEY 8(e);
// for cfg2 the imbalance is < 1% (contiguous blocks: 7%).  A global fine node is owned by the subdomain given
// by the core ownership rule C3 and hence by that subdomain's rank.  Every rank keeps the full composite
// arrays; after the write-back rank r needs, from each peer p, the values of the nodes that p owns and that
// lie in one of r's extended boxes Omega_j.  Lists are sorted, unique, and computed identically on every rank,
// so send and receive lists match without negotiation.
#pragma once
#include <algorithm>
#include <vector>

namespace lp {

struct RegionGrid {
  int d;
  int n[3];      // fine cells per axis
  int m[3];      // subdomain grid
  int ov;        // overlap in fine cells
};

// cells of the extended box of position s in one region (overlap clipped at the region box, C7)
inline long long box_cells(const RegionGrid& G, long long s) {
  long long rem = s, cells = 1;
  for (int a = 0; a < G.d; ++a) {
    const int pos = (int)(rem % G.m[a]);
    rem /= G.m[a];
    const int core = G.n[a] / G.m[a];
    cells *= std::min(G.n[a], (pos + 1) * core + G.ov) - std::max(0, pos * core - G.ov);
  }
  return cells;
}

// LPT placement of the positions over `world` ranks (weights: porous + conduit box cells); Gp and Gc share the
// subdomain grid m.  Returns rank_of_pos[s].
inline std::vector<int> placement(const RegionGrid& Gp, const RegionGrid& Gc, int world) {
  const int npos = Gp.m[0] * Gp.m[1] * (Gp.d > 2 ? Gp.m[2] : 1);
  std::vector<long long> w(npos);
  std::vector<int> order(npos), out(npos, 0);
  for (int s = 0; s < npos; ++s) {
    w[s] = box_cells(Gp, s) + box_cells(Gc, s);
    order[s] = s;
  }
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return w[a] > w[b]; });
  std::vector<long long> load(world, 0);
  for (int s : order) {
    int best = 0;
    for (int r = 1; r < world; ++r)
      if (load[r] < load[best]) best = r;
    out[s] = best;
    load[best] += w[s];
  }
  return out;
}

inline long long owner_position(const RegionGrid& G, const int g[3]) {
  long long idx = 0, stride = 1;
  for (int a = 0; a < G.d; ++a) {
    const int core = G.n[a] / G.m[a];
    const int o = std::min(g[a] / (2 * core), G.m[a] - 1);
    idx += o * stride;
    stride *= G.m[a];
  }
  return idx;
}

// half-grid extent of position s's extended box
inline void box_of(const RegionGrid& G, long long s, int lo[3], int hi[3]) {
  for (int a = 0; a < 3; ++a) lo[a] = hi[a] = 0;
  long long rem = s;
  for (int a = 0; a < G.d; ++a) {
    const int pos = (int)(rem % G.m[a]);
    rem /= G.m[a];
    const int core = G.n[a] / G.m[a];
    lo[a] = 2 * std::max(0, pos * core - G.ov);
    hi[a] = 2 * std::min(G.n[a], (pos + 1) * core + G.ov);
  }
}

// vertex_only: P1 vertices (even half-grid points), indexed in the vertex grid
struct HaloPlan {
  // per peer: global node indices (P2 half-grid lex, or P1 vertex lex)
  std::vector<std::vector<int>> need;  // need[p]: nodes owned by p that I read
  std::vector<std::vector<int>> give;  // give[p]: nodes I own that p reads
  std::vector<std::vector<int>> owned; // owned[p]: all nodes owned by rank p (for the gather to root)
};

inline void plan_region(const RegionGrid& G, const std::vector<int>& rank_of_pos, int rank, int world, bool vertex_only,
                        HaloPlan& P) {
  const int npos = G.m[0] * G.m[1] * (G.d > 2 ? G.m[2] : 1);
  P.need.assign(world, {});
  P.give.assign(world, {});
  P.owned.assign(world, {});
  int np[3] = {1, 1, 1};
  for (int a = 0; a < G.d; ++a) np[a] = 2 * G.n[a] + 1;
  const int step = vertex_only ? 2 : 1;
  auto gidx = [&](const int g[3]) {
    long long i = 0, s = 1;
    for (int a = 0; a < G.d; ++a) {
      const int v = vertex_only ? g[a] / 2 : g[a];
      i += v * s;
      s *= vertex_only ? (G.n[a] + 1) : np[a];
    }
    return (int)i;
  };
  // owned lists
  int g[3] = {0, 0, 0};
  for (g[2] = 0; g[2] < (G.d > 2 ? np[2] : 1); g[2] += step)
    for (g[1] = 0; g[1] < np[1]; g[1] += step)
      for (g[0] = 0; g[0] < np[0]; g[0] += step)
        P.owned[rank_of_pos[owner_position(G, g)]].push_back(gidx(g));
  // need / give: nodes of a rank's boxes owned by another rank
  for (long long s = 0; s < npos; ++s) {
    const int rs = rank_of_pos[s];
    int lo[3], hi[3];
    box_of(G, s, lo, hi);
    for (g[2] = lo[2]; g[2] <= (G.d > 2 ? hi[2] : 0); g[2] += step)
      for (g[1] = lo[1]; g[1] <= hi[1]; g[1] += step)
        for (g[0] = lo[0]; g[0] <= hi[0]; g[0] += step) {
          const int ro = rank_of_pos[owner_position(G, g)];
          if (ro == rs) continue;
          if (rs == rank) P.need[ro].push_back(gidx(g));
          if (ro == rank) P.give[rs].push_back(gidx(g));
        }
  }
  for (int p = 0; p < world; ++p) {
    for (auto* v : {&P.need[p], &P.give[p]}) {
      std::sort(v->begin(), v->end());
      v->erase(std::unique(v->begin(), v->end()), v->end());
    }
  }
}

}  // namespace lp
