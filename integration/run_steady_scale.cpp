// run_steady_scale.cpp -- the drop-in at the headline scale: the reference's
// own make_cube_mesh(n) + cdg::run_steady (solver.hpp:152-154), resolved to
// the GPU adapter (integration/cdg_gpu_adapter.cpp), whose straight-mesh
// levels come from cdg_gpu_level_create_from_mesh (no DgLevel). With the
// reference's DgLevel a 4.09M-element P=4 level needs ~570 GB of host memory
// (~140 KB per element); here the host side is the Mesh itself.
//
//   run_steady_scale N P ITERS   (prints one JSON line: setup / run seconds, rows)
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "cdg/meshgen.hpp"
#include "cdg/solver.hpp"

int main(int argc, char** argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 88;
  const int p = argc > 2 ? std::atoi(argv[2]) : 4;
  const int iters = argc > 3 ? std::atoi(argv[3]) : 20;
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  cdg::Mesh mesh = cdg::make_cube_mesh(n, "wall");
  cdg::CurvedMesh cmesh(mesh, 1);
  const double t_mesh = std::chrono::duration<double>(clk::now() - t0).count();
  cdg::RunConfig cfg;
  cfg.p_schedule = {p};
  cfg.fixed_iterations = {iters};
  cfg.check_interval = iters / 2 > 0 ? iters / 2 : 1;
  cfg.max_iterations_per_level = iters;
  const cdg::BcMap bcs = {{"wall", cdg::BcKind::SlipWall}};
  // a uniform flow along x (slip walls: the box holds it only approximately,
  // so the residual is non-zero and the rows are meaningful)
  cdg::ConservedState fs;
  fs.rho = 1.0;
  fs.mom = {0.3, 0.0, 0.0};
  fs.rhoE = 1.0 / 0.4 + 0.5 * 0.09;
  int rows = 0;
  double last_res = -1.0;
  const auto t1 = clk::now();
  const cdg::SteadyResult r = cdg::run_steady(cmesh, bcs, cfg, fs, [&](const cdg::ConvergenceRow& row) {
    ++rows;
    last_res = row.residual;
  });
  const double t_run = std::chrono::duration<double>(clk::now() - t1).count();
  std::printf("{\"n\": %d, \"elements\": %d, \"p\": %d, \"iterations\": %d, \"mesh_s\": %.2f, "
              "\"run_steady_s\": %.2f, \"rows\": %d, \"last_residual\": %.6e, \"solution_values\": %zu}\n",
              n, mesh.n_elements(), p, iters, t_mesh, t_run, rows, last_res, r.solution.raw().size());
  return rows > 0 && r.solution.raw().size() > 0 ? 0 : 1;
}
