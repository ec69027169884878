// tcgen05 (5th-gen tensor core) TF32 GEMMs for the dense transform.
// Placeholder until the tcgen05 path lands: the TF32 precision mode reports
// an error instead of silently running something else.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "ht_common.h"

namespace ht {

inline int tc_gemm_fwd(cudaStream_t, const float*, const float*, float*, int64_t, int, int) {
  return fail(HT_EINVAL, "precision 'tf32' (tcgen05) is not built yet; use 'fp32'");
}

inline int tc_gemm_bwd(cudaStream_t, const float*, const float*, const float*, float*, float*,
                       float*, float*, int64_t, int, int) {
  return fail(HT_EINVAL, "precision 'tf32' (tcgen05) is not built yet; use 'fp32'");
}

}  // namespace ht
