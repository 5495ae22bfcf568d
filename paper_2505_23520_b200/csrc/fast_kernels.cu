// Fast path placeholder — replaced by the tcgen05 kernels.
#include "fast.h"

namespace aa {
cudaError_t fast_anchor(const FastArgs&, const void*, const void*, const void*, float*, float*,
                        float*, float*, double*, cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t fast_pool(const FastArgs&, const void*, const float*, const float*, const double*,
                      double*, float*, cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t fast_identify(const FastArgs&, const void*, const float*, const double*, uint32_t*,
                          int64_t, cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t fast_sparse(const FastArgs&, const void*, const void*, const void*, const float*,
                        const float*, const float*, const uint32_t*, const int32_t*,
                        const int64_t*, int64_t, bool, void*, aa_dtype, void*, cudaStream_t) {
    return cudaErrorNotSupported;
}
cudaError_t fast_finalize(const FastArgs&, const float*, const float*, void*, aa_dtype,
                          cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t fast_dense(const FastArgs&, const void*, const void*, const void*, void*, aa_dtype,
                       cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t fast_recall(const FastArgs&, const void*, const void*, const uint32_t*, const int32_t*,
                        const int64_t*, int64_t, double*, double*, cudaStream_t) {
    return cudaErrorNotSupported;
}
}  // namespace aa
