// Tensor-core product of the random-feature prior (family SAP_COSINE): CTA-pair
// kernel only, fp32 (tf32-split) features with ka = 32.
#include "krows_tc.cuh"
#include "krows_tc2.cuh"

namespace sap {
namespace tck {
bool launch_tc2_cos(const CUtensorMap &a, const CUtensorMap &c, const CUtensorMap &zh,
                    const CUtensorMap &zl, const Params &p, int nz, int ka, int grid,
                    cudaStream_t st) {
  if (ka != 32) return false;
  using tck2::launch_tc2_shape;
  switch (nz) {
    case 16: return launch_tc2_shape<SAP_COSINE, 16, 32, false>(a, c, zh, zl, p, grid, st);
    case 32: return launch_tc2_shape<SAP_COSINE, 32, 32, false>(a, c, zh, zl, p, grid, st);
    case 48: return launch_tc2_shape<SAP_COSINE, 48, 32, false>(a, c, zh, zl, p, grid, st);
    case 64: return launch_tc2_shape<SAP_COSINE, 64, 32, false>(a, c, zh, zl, p, grid, st);
    case 80: return launch_tc2_shape<SAP_COSINE, 80, 32, false>(a, c, zh, zl, p, grid, st);
    case 96: return launch_tc2_shape<SAP_COSINE, 96, 32, false>(a, c, zh, zl, p, grid, st);
    case 112: return launch_tc2_shape<SAP_COSINE, 112, 32, false>(a, c, zh, zl, p, grid, st);
    case 128: return launch_tc2_shape<SAP_COSINE, 128, 32, false>(a, c, zh, zl, p, grid, st);
    default: return false;
  }
}
}  // namespace tck
}  // namespace sap
