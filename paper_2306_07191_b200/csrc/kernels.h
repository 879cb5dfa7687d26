// Internal cross-translation-unit declarations.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "nif_b200.h"

namespace nif {
size_t gather_two_pass_workspace(int64_t n);
int gather_two_pass(const nif_scene_view* s, const uint8_t* route, const double* origins,
                    const double* dirs, const double* tmaxs, int64_t n, const nif_gather_out* out,
                    void* workspace, size_t workspace_bytes, cudaStream_t st);
int sm_count();
}  // namespace nif
