// cdg_gpu_adapter.hpp -- the one extension the GPU adapter adds to the
// reference solver API (proj/core/include/cdg/solver.hpp): which GPU the
// levels it creates live on. Everything else the adapter provides has the
// reference's own declarations (solver.hpp:83-154).
#pragma once

namespace cdg {

/// Device of the levels created after this call (one process per GPU). The
/// default is $CDG_GPU_DEVICE, else 0.
void gpu_select_device(int device);

}  // namespace cdg
