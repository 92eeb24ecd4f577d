"""The drop-in, run by the driver: the reference's OWN test and acceptance
programs linked against the GPU path.

oracle/Makefile (target `dropin`) compiles the unmodified reference sources
with solver.cpp's kernel entry points renamed (-Dcompute_rhs=compute_rhs_cpu
...) and links integration/cdg_gpu_adapter.cpp, which implements
cdg::make_workspace / compute_rhs / rk_step / interpolate_to_faces /
current_viscosity / aux_gradient / run_steady (solver.hpp:83-154) over the C
ABI (include/cdg_gpu.h). So every kernel call these programs make runs on the
B200:

  * oracle/_ref/test_solver_gpu  = /root/reference/proj/tests/test_solver.cpp
    (doctest; 19 test cases, the reference's solver unit suite);
  * oracle/_ref/acceptance_gpu   = tests/acceptance/acceptance_main.cpp with
    criteria C03 (free-stream preservation, straight + curved sphere), C04
    (discrete conservation), C06 (RK order), C11 (p-refinement), C12 (padded
    layout, bitwise paths, determinism).

Needs the prebuilt binaries (built here by __graft_entry__.build(); they travel
to the GPU box with the snapshot)."""
import os
import re
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

REF = Path(__file__).resolve().parent.parent / "oracle" / "_ref"


def _binary(name):
    b = REF / name
    if not b.exists():
        pytest.skip(f"{b} not built (reference sources absent when building)")
    return str(b)


def test_reference_solver_unit_suite_through_the_gpu_adapter():
    r = subprocess.run([_binary("test_solver_gpu")], capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    m = re.search(r"test cases:\s*(\d+)\s*\|\s*(\d+) passed\s*\|\s*(\d+) failed", out)
    assert m, out[-2000:]
    total, passed, failed = (int(x) for x in m.groups())
    assert r.returncode == 0 and failed == 0 and passed == total >= 19, out[-2000:]


def test_reference_acceptance_criteria_through_the_gpu_adapter(tmp_path):
    crit = ["3", "4", "6", "11", "12"]
    r = subprocess.run([_binary("acceptance_gpu"), "--fixture-dir", str(tmp_path)] + crit,
                       capture_output=True, text=True, timeout=1800, env=dict(os.environ, OMP_NUM_THREADS="8"))
    out = r.stdout + r.stderr
    passed = re.findall(r"^\[PASS\] C(\d+)", out, re.M)
    failed = re.findall(r"^\[FAIL\] C(\d+)", out, re.M)
    assert not failed, out[-3000:]
    assert sorted(int(c) for c in passed) == sorted(int(c) for c in crit), out[-3000:]


def test_run_steady_at_headline_scale_through_the_dropin():
    """The reference's make_cube_mesh(88) (4,088,832 tets) + cdg::run_steady at
    P=4, resolved to the GPU adapter: straight-mesh levels come from
    cdg_gpu_level_create_from_mesh, so the host never builds the ~570 GB
    DgLevel (integration/run_steady_scale.cpp)."""
    import json
    exe = REF / "run_steady_gpu"
    if not exe.exists():
        pytest.skip("oracle/_ref/run_steady_gpu not built")
    out = subprocess.run([str(exe), "88", "4", "10"], capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["elements"] == 6 * 88 ** 3 and d["rows"] == 2 and d["last_residual"] > 0
    assert d["solution_values"] == d["elements"] * 5 * 48


def test_output_path_from_a_gpu_run(tmp_path):
    """§8 f4: cdg::run_steady through the drop-in, the SteadyResult written with
    the reference's CDS1 writer, read back bit for bit, exported with its VTK
    writer (the CLI's solve + export sequence, cli_ops.cpp:119-171), and the
    log / state against the reference CPU run_steady on the same case
    (integration/dropin_output.cpp)."""
    import json
    exe = REF / "dropin_output"
    if not exe.exists():
        pytest.skip("oracle/_ref/dropin_output not built")
    out = subprocess.run([str(exe), str(tmp_path)], capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout + out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["cds1_roundtrip_bitwise"] and d["rows_match"] and d["rows"] == 8 and d["final_degree"] == 2
    assert d["log_rel_diff"] < 1e-10 and d["state_rel_diff"] < 1e-11
    assert d["vtk_bytes"] > 0 and (tmp_path / "gpu_state.vtk").read_text().startswith("# vtk DataFile")
