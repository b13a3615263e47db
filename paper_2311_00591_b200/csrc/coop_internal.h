// coop_internal.h -- declarations shared by libcoop's translation units (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "coop.h"

namespace coop {

// Launches the batched search (coop_search.cu). Arguments already validated.
int launch_window_search(const coop_tables_soa *t, const uint64_t *requests, coop_window *out,
                         cudaStream_t st);

// Test hook: COOP_FORCE_PLAIN_STAGING=1 disables the TMA staging path.
inline bool coop_force_plain_staging() {
  const char *v = getenv("COOP_FORCE_PLAIN_STAGING");
  return v && v[0] == '1';
}

// true if p is a device (or managed) pointer usable by kernels of the current device
inline bool is_device_ptr(const void *p) {
  if (!p) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

}  // namespace coop
