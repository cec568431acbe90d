// Tensor-core block-row kernel instantiated for one covariance family.
#include "krows_tc.cuh"
#include "krows_tc2.cuh"

namespace sap {
namespace tck {
bool launch_tc_m32(const CUtensorMap &a, const CUtensorMap &c, const CUtensorMap &zh,
                    const CUtensorMap &zl, const Params &p, int nz, int ka, int grid,
                    cudaStream_t st) {
  return launch_tc_family<SAP_MATERN32>(a, c, zh, zl, p, nz, ka, grid, st);
}
bool launch_tc2_m32(const CUtensorMap &a, const CUtensorMap &c, const CUtensorMap &zh,
                     const CUtensorMap &zl, const Params &p, int nz, int ka, int grid,
                     cudaStream_t st) {
  return tck2::launch_tc2_family<SAP_MATERN32>(a, c, zh, zl, p, nz, ka, grid, st);
}
}  // namespace tck
}  // namespace sap
