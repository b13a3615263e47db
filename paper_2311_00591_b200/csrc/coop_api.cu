// coop_api.cu -- the extern "C" boundary of libcoop (include/coop.h): argument checks,
// status codes, and the host-buffer streaming entry point.  All compute is in kernels.
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#include "coop.h"
#include "coop_internal.h"

using namespace coop;

extern "C" const char *coop_status_string(int s) {
  switch (s) {
    case COOP_OK: return "COOP_OK";
    case COOP_INFEASIBLE: return "COOP_INFEASIBLE";
    case COOP_ERR_INVALID_ARG: return "COOP_ERR_INVALID_ARG";
    case COOP_ERR_UNKNOWN_ID: return "COOP_ERR_UNKNOWN_ID";
    case COOP_ERR_UNSATISFIABLE: return "COOP_ERR_UNSATISFIABLE";
    case COOP_ERR_THRASHED: return "COOP_ERR_THRASHED";
    case COOP_ERR_CUDA: return "COOP_ERR_CUDA";
    case COOP_ERR_NOMEM: return "COOP_ERR_NOMEM";
    case COOP_ERR_BAD_STATE: return "COOP_ERR_BAD_STATE";
    case COOP_ERR_UNIMPLEMENTED: return "COOP_ERR_UNIMPLEMENTED";
    default: return "COOP_ERR_UNKNOWN_STATUS";
  }
}

extern "C" const char *coop_version(void) { return "coop-b200 0.1 sm_100a"; }

static int check_tables(const coop_tables_soa *t) {
  if (!t) return COOP_ERR_INVALID_ARG;
  if (t->n_pools < 0 || t->n_blocks < 1 || t->n_blocks > COOP_MAX_BLOCKS ||
      t->pool_stride < t->n_blocks || t->reserved != 0)
    return COOP_ERR_INVALID_ARG;
  if (t->n_pools > 0 && (!t->size_state || !t->cost || !t->stale)) return COOP_ERR_INVALID_ARG;
  return COOP_OK;
}

extern "C" int coop_window_search_batched(const coop_tables_soa *t, const uint64_t *requests,
                                          coop_window *out, coop_stream_t stream) {
  int rc = check_tables(t);
  if (rc != COOP_OK) return rc;
  if (t->n_pools == 0) return COOP_OK;
  if (!is_device_ptr(t->size_state) || !is_device_ptr(t->cost) || !is_device_ptr(t->stale) ||
      !is_device_ptr(requests) || !is_device_ptr(out))
    return COOP_ERR_INVALID_ARG;
  return launch_window_search(t, requests, out, (cudaStream_t)stream);
}

// Host-buffer entry: chunks of pools are copied H2D (re-pitched to a TMA-friendly stride),
// searched, and the results copied D2H; two streams alternate so that the copy of chunk
// c+1 overlaps the search of chunk c.
extern "C" int coop_window_search_batched_host(const coop_tables_soa *ht,
                                               const uint64_t *host_requests,
                                               coop_window *host_out, int64_t chunk_pools) {
  int rc = check_tables(ht);
  if (rc != COOP_OK) return rc;
  if (ht->n_pools == 0) return COOP_OK;
  if (!host_requests || !host_out) return COOP_ERR_INVALID_ARG;
  const int64_t P = ht->n_pools;
  const int32_t n = ht->n_blocks;
  const int64_t dstride = (n + 15) / 16 * 16;
  if (chunk_pools <= 0) chunk_pools = 16384;
  if (chunk_pools > P) chunk_pools = P;

  const size_t arr_bytes = (size_t)chunk_pools * dstride * 8;
  // staging workspace: per device, grown on demand and reused by later calls (no device
  // allocation on the steady-state path); one caller at a time per process
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  struct Staging {
    void *buf[2][5] = {{nullptr}};
    cudaStream_t st[2] = {nullptr, nullptr};
    size_t arr_bytes = 0, pools = 0;
  };
  static Staging ws[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return COOP_ERR_CUDA;
  Staging &W = ws[dev];
  int status = COOP_OK;
  if (W.arr_bytes < arr_bytes || W.pools < (size_t)chunk_pools) {
    for (int b = 0; b < 2; ++b)
      for (int a = 0; a < 5; ++a)
        if (W.buf[b][a]) {
          cudaFree(W.buf[b][a]);
          W.buf[b][a] = nullptr;
        }
    W.arr_bytes = W.pools = 0;
    for (int b = 0; b < 2 && status == COOP_OK; ++b) {
      if (!W.st[b] && cudaStreamCreateWithFlags(&W.st[b], cudaStreamNonBlocking) != cudaSuccess)
        status = COOP_ERR_CUDA;
      for (int a = 0; a < 3 && status == COOP_OK; ++a)
        if (cudaMalloc(&W.buf[b][a], arr_bytes) != cudaSuccess) status = COOP_ERR_NOMEM;
      if (status == COOP_OK && cudaMalloc(&W.buf[b][3], (size_t)chunk_pools * 8) != cudaSuccess)
        status = COOP_ERR_NOMEM;
      if (status == COOP_OK &&
          cudaMalloc(&W.buf[b][4], (size_t)chunk_pools * sizeof(coop_window)) != cudaSuccess)
        status = COOP_ERR_NOMEM;
    }
    if (status != COOP_OK) {
      for (int b = 0; b < 2; ++b)
        for (int a = 0; a < 5; ++a)
          if (W.buf[b][a]) {
            cudaFree(W.buf[b][a]);
            W.buf[b][a] = nullptr;
          }
      return status;
    }
    W.arr_bytes = arr_bytes;
    W.pools = (size_t)chunk_pools;
  }
  void *(&buf)[2][5] = W.buf;
  cudaStream_t *st = W.st;
  const void *src[3] = {ht->size_state, ht->cost, ht->stale};
  for (int64_t c0 = 0, ci = 0; c0 < P && status == COOP_OK; c0 += chunk_pools, ++ci) {
    const int b = (int)(ci & 1);
    const int64_t cp = (P - c0 < chunk_pools) ? (P - c0) : chunk_pools;
    for (int a = 0; a < 3 && status == COOP_OK; ++a) {
      const char *s = (const char *)src[a] + (size_t)c0 * ht->pool_stride * 8;
      if (cudaMemcpy2DAsync(buf[b][a], dstride * 8, s, ht->pool_stride * 8, (size_t)n * 8,
                            (size_t)cp, cudaMemcpyHostToDevice, st[b]) != cudaSuccess)
        status = COOP_ERR_CUDA;
    }
    if (status != COOP_OK) break;
    if (cudaMemcpyAsync(buf[b][3], host_requests + c0, (size_t)cp * 8, cudaMemcpyHostToDevice,
                        st[b]) != cudaSuccess) {
      status = COOP_ERR_CUDA;
      break;
    }
    coop_tables_soa dt;
    dt.size_state = (const uint64_t *)buf[b][0];
    dt.cost = (const double *)buf[b][1];
    dt.stale = (const double *)buf[b][2];
    dt.n_pools = cp;
    dt.n_blocks = n;
    dt.reserved = 0;
    dt.pool_stride = dstride;
    status = launch_window_search(&dt, (const uint64_t *)buf[b][3], (coop_window *)buf[b][4], st[b]);
    if (status != COOP_OK) break;
    if (cudaMemcpyAsync(host_out + c0, buf[b][4], (size_t)cp * sizeof(coop_window),
                        cudaMemcpyDeviceToHost, st[b]) != cudaSuccess)
      status = COOP_ERR_CUDA;
  }
  for (int b = 0; b < 2; ++b)
    if (cudaStreamSynchronize(st[b]) != cudaSuccess && status == COOP_OK) status = COOP_ERR_CUDA;
  return status;
}

// ---- test hook (not part of the ABI): the CUDA path's exact-sum arithmetic, compiled for
// the host, so the fixed-point rounding can be checked without a GPU.
#include "fixed192.cuh"
extern "C" double coop__fixed_round_sum_host(const double *h, int64_t n) {
  U192 acc = u192_zero();
  for (int64_t k = 0; k < n; ++k) acc = u192_add(acc, u192_from_double(h[k]));
  return u192_round_to_double(acc);
}
