// query_tc.cu -- tcgen05 fused query x user contraction + classify epilogue.
#include "internal.h"
namespace rmips {
cudaError_t query_filter_tc(QueryCtx&, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace rmips
