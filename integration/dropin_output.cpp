// dropin_output.cpp -- the reference's output path (§8 f4) on a GPU-produced
// state: cdg::run_steady resolved to the GPU adapter, its SteadyResult written
// with the reference's own CDS1 writer (write_state, state_io.cpp:19-46),
// read back (read_state), exported with the reference's VTK writer
// (export_vtk_file, vtk.cpp:47-135) -- the sequence of the CLI's solve and
// export commands (cli_ops.cpp:119-171) -- and compared with the reference
// CPU run_steady (compiled alongside as run_steady_cpu) on the same case.
//
//   dropin_output OUT_DIR   (prints one JSON line)
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <functional>
#include <string>
#include <vector>

#include "cdg/meshgen.hpp"
#include "cdg/refelem.hpp"
#include "cdg/solver.hpp"
#include "cdg/state_io.hpp"
#include "cdg/vtk.hpp"

namespace cdg {
// the reference's run_steady with its CPU kernels (solver.cpp compiled with
// -Drun_steady=run_steady_cpu, oracle/Makefile target dropin)
SteadyResult run_steady_cpu(const CurvedMesh& cmesh, const BcMap& bc_map, const RunConfig& cfg,
                            const ConservedState& freestream,
                            const std::function<void(const ConvergenceRow&)>& on_row);
}  // namespace cdg

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : ".";
  cdg::Mesh mesh = cdg::make_cube_mesh(4, "wall");
  cdg::CurvedMesh cmesh(mesh, 2);
  cdg::RunConfig cfg;
  cfg.p_schedule = {1, 2};
  cfg.fixed_iterations = {40, 40};
  cfg.check_interval = 10;
  cfg.max_iterations_per_level = 40;
  const cdg::BcMap bcs = {{"wall", cdg::BcKind::SlipWall}};
  cdg::ConservedState fs;
  fs.rho = 1.0;
  fs.mom = {0.3, 0.05, 0.0};
  fs.rhoE = 1.0 / 0.4 + 0.5 * (0.09 + 0.0025);
  const cdg::SteadyResult gpu = cdg::run_steady(cmesh, bcs, cfg, fs, {});
  const cdg::SteadyResult cpu = cdg::run_steady_cpu(cmesh, bcs, cfg, fs, {});

  cdg::StateFile st;
  st.degree = gpu.final_degree;
  st.gamma = cfg.gas.gamma;
  st.store = gpu.solution;
  const std::string cds = dir + "/gpu_state.cds", vtk = dir + "/gpu_state.vtk";
  cdg::write_state(st, mesh, cds);
  const cdg::StateFile back = cdg::read_state(mesh, cds);
  const auto& a = gpu.solution.raw();
  const auto& b = back.store.raw();
  const bool roundtrip = a.size() == b.size() && std::equal(a.begin(), a.end(), b.begin()) &&
                         back.degree == gpu.final_degree && back.gamma == cfg.gas.gamma;
  std::vector<double> eps(mesh.n_elements(), 0.0);
  auto re = cdg::get_reference_element(back.degree);
  cdg::export_vtk_file(cmesh, *re, back.store, cdg::GasModel{back.gamma}, eps, vtk);
  std::ifstream vf(vtk, std::ios::binary | std::ios::ate);
  const long vtk_bytes = vf ? static_cast<long>(vf.tellg()) : -1;

  double state_diff = 0.0, state_max = 0.0, log_diff = 0.0;
  const auto& c = cpu.solution.raw();
  for (size_t i = 0; i < std::min(a.size(), c.size()); ++i) {
    state_diff = std::max(state_diff, std::abs(a[i] - c[i]));
    state_max = std::max(state_max, std::abs(c[i]));
  }
  const size_t nrows = std::min(gpu.log.size(), cpu.log.size());
  bool rows_match = gpu.log.size() == cpu.log.size();
  for (size_t i = 0; i < nrows; ++i) {
    rows_match = rows_match && gpu.log[i].level == cpu.log[i].level && gpu.log[i].iteration == cpu.log[i].iteration;
    log_diff = std::max(log_diff, std::abs(gpu.log[i].residual - cpu.log[i].residual) /
                                      std::max(std::abs(cpu.log[i].residual), 1e-300));
    log_diff = std::max(log_diff, std::abs(gpu.log[i].dt - cpu.log[i].dt) / std::abs(cpu.log[i].dt));
  }
  std::printf("{\"rows\": %zu, \"rows_match\": %s, \"log_rel_diff\": %.3e, \"state_rel_diff\": %.3e, "
              "\"cds1_roundtrip_bitwise\": %s, \"final_degree\": %d, \"vtk_bytes\": %ld}\n",
              gpu.log.size(), rows_match ? "true" : "false", log_diff, state_diff / state_max,
              roundtrip ? "true" : "false", gpu.final_degree, vtk_bytes);
  return roundtrip && rows_match && vtk_bytes > 0 ? 0 : 1;
}
