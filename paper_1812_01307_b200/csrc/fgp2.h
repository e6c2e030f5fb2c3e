// Row-walk 2-D TV prox (fgp2.cu): host-side entry points used by bsgd_abi.cu.
#pragma once

#include <cuda_runtime.h>

#include "prox_args.cuh"

namespace bsgd {

// Power-of-two images, 128 <= width <= 1024, height <= 16384, 16-byte aligned fields.
bool fgp2_rows_supported(const ProxArgs &a);
// Cooperative launch of fgp2_rows_kernel (a.ds must be set); cudaErrorCooperativeLaunchTooLarge
// when the grid cannot be co-resident.
cudaError_t fgp2_rows_launch(const ProxArgs &a, int num_sms, cudaStream_t st);

}  // namespace bsgd
