// ORACLE TEST INFRASTRUCTURE ONLY.
//
// Periodic coupling for the UNMODIFIED reference kernels. The reference has
// no periodic boundary (BcKind is SlipWall/Farfield/Symmetry, euler.hpp:65),
// but compute_rhs / rk_step read the face coupling only through
// DgLevel::coupling(e, f) (solver.cpp:228,292,418): they run any face graph.
// This translation unit rewires a cube level's boundary faces to their
// translates on the opposite side of the box -- the node_map by the
// reference's own nearest-physical-point rule (solver.cpp:144-172), with the
// distance taken by minimum image -- so BASELINE config 1 (periodic
// isentropic vortex) can be checked against the reference's own arithmetic.
// Access to the private coupling table is the only liberty taken; the
// reference sources are compiled unchanged.
#include <array>
#include <atomic>
#include <cmath>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#define private public
#include "cdg/solver.hpp"
#undef private

namespace cdg_oracle {

void make_periodic(cdg::DgLevel& level, const double period[3]) {
  const int ne = level.n_elements();
  const int ng = level.re_->n_face_quad();
  auto wrap = [&](double x, int a) { return period[a] > 0.0 ? x - period[a] * std::floor(x / period[a] + 1e-9) : x; };
  // boundary faces keyed by the wrapped centroid (rounded): a face and its translate share the key
  std::map<std::array<long long, 3>, std::vector<std::pair<int, int>>> by_key;
  for (int e = 0; e < ne; ++e)
    for (int f = 0; f < 4; ++f) {
      if (level.coupling_[e][f].neighbor >= 0) continue;
      double c[3] = {0, 0, 0};
      for (int g = 0; g < ng; ++g) {
        const cdg::Vec3& x = level.geom_[e].face_phys[f * ng + g];
        c[0] += x.x / ng, c[1] += x.y / ng, c[2] += x.z / ng;
      }
      std::array<long long, 3> key;
      for (int a = 0; a < 3; ++a) key[a] = std::llround(wrap(c[a], a) * 1e7);
      for (int a = 0; a < 3; ++a)
        if (period[a] > 0.0 && key[a] == std::llround(period[a] * 1e7)) key[a] = 0;
      by_key[key].push_back({e, f});
    }
  for (auto& [key, faces] : by_key) {
    if (faces.size() != 2) throw std::runtime_error("make_periodic: unmatched boundary face");
    for (int side = 0; side < 2; ++side) {
      const auto [e, f] = faces[side];
      const auto [n, nf] = faces[1 - side];
      cdg::FaceCoupling fc;
      fc.neighbor = n;
      fc.neighbor_face = nf;
      fc.node_map.resize(ng);
      for (int g = 0; g < ng; ++g) {
        const cdg::Vec3 mine = level.geom_[e].face_phys[f * ng + g];
        int match = -1;
        double best = 1e300;
        for (int h = 0; h < ng; ++h) {
          const cdg::Vec3 theirs = level.geom_[n].face_phys[nf * ng + h];
          double d[3] = {mine.x - theirs.x, mine.y - theirs.y, mine.z - theirs.z};
          for (int a = 0; a < 3; ++a)
            if (period[a] > 0.0) d[a] -= period[a] * std::nearbyint(d[a] / period[a]);
          const double dist = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
          if (dist < best) best = dist, match = h;
        }
        fc.node_map[g] = match;
      }
      level.coupling_[e][f] = fc;
    }
  }
}

}  // namespace cdg_oracle
