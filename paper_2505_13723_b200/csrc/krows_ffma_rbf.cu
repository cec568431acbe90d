// Instantiation of the FFMA block-row kernels for one family (split out of
// sapgp_b200.cu so the template instantiations compile in parallel).
#include "krows_ffma.cuh"

namespace sap {
int fail(int code, const char *fmt, ...);
int check_launch(const char *what);

template <int FAM, int DP>
int launch_dp(KrowsParams p, cudaStream_t st) {
  const int mt = (p.m + 15) / 16;
  dim3 grid(unsigned((p.b + kFfmaBM - 1) / kFfmaBM), unsigned(p.splits));
#define SAP_MT_CASE(MTV)                                                          \
  case MTV:                                                                       \
    krows_ffma_kernel<FAM, DP, MTV><<<grid, kFfmaThreads, 0, st>>>(p);            \
    break;
  switch (mt) {
    SAP_MT_CASE(1) SAP_MT_CASE(2) SAP_MT_CASE(3) SAP_MT_CASE(4)
    SAP_MT_CASE(5) SAP_MT_CASE(6) SAP_MT_CASE(7) SAP_MT_CASE(8)
    default: return fail(SAP_ERR_CONTRACT, "internal: bad column chunk %d", p.m);
  }
#undef SAP_MT_CASE
  return check_launch("krows_ffma_kernel");
}

template <int FAM>
int launch_fam(KrowsParams p, int dp, cudaStream_t st) {
  switch (dp) {
    case 4: return launch_dp<FAM, 4>(p, st);
    case 8: return launch_dp<FAM, 8>(p, st);
    case 12: return launch_dp<FAM, 12>(p, st);
    case 16: return launch_dp<FAM, 16>(p, st);
    case 32: return launch_dp<FAM, 32>(p, st);
    case 64: return launch_dp<FAM, 64>(p, st);
    default: return fail(SAP_ERR_CONTRACT, "unsupported padded dimension %d", dp);
  }
}


int launch_ffma_rbf(KrowsParams p, int dp, cudaStream_t st) { return launch_fam<SAP_RBF>(p, dp, st); }
}  // namespace sap
