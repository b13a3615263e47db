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
// The two kernels behind it: the warp-per-pool stream (coop_search_stream.cu), which marks
// the pools it cannot finish with COOP_PENDING_, and the CTA-per-pool kernel (all pools, or
// with pending = true only the marked ones).
int launch_window_search_stream(const coop_tables_soa *t, const uint64_t *requests, coop_window *out,
                                 cudaStream_t st);
int launch_window_search_cta(const coop_tables_soa *t, const uint64_t *requests, coop_window *out,
                             cudaStream_t st, bool pending);
bool stream_search_enabled(int n_blocks);
// internal status of a pool result between the two kernels (never returned)
constexpr int32_t COOP_PENDING_ = 0x7fff0001;

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
