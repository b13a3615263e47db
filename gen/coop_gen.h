/*
 * coop_gen.h -- seeded synthetic INPUT generators (a module of their own).
 *
 * Shared by the CUDA path (device-side generation for the benchmark) and the tests /
 * oracle side (host-side generation of the same pools).  Holds none of the method's
 * arithmetic: it only draws block tables and requests with the shapes of DESIGN.md
 * "Input recipe"; the host and device functions evaluate the same
 * __host__ __device__ item function, so the two are bit-identical by construction
 * (checked by tests/test_gen.py on the GPU).
 */
#ifndef COOP_GEN_H
#define COOP_GEN_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define COOPGEN_MODE_BENCH 0  /* config 4: 4096-block pools, pinned ends, short/long R  */
#define COOPGEN_MODE_SMALL 1  /* config 1: 32-block pools, sizes U[1,2^20], R U[1, S/2] */

/* Pools [p0, p0 + n_pools) of the global sequence, written at local index p - p0.
 * Arrays are SoA pool-major with pool_stride elements between pools.  Returns 0, or -1
 * on bad arguments. Host version: host pointers. */
int coopgen_pools_host(int mode, uint64_t seed, int64_t p0, int64_t n_pools, int32_t n,
                       int64_t pool_stride, uint64_t *size_state, double *cost,
                       double *stale, uint64_t *requests);

/* Device version: device pointers, asynchronous on `stream` (a cudaStream_t). */
int coopgen_pools_device(int mode, uint64_t seed, int64_t p0, int64_t n_pools, int32_t n,
                         int64_t pool_stride, uint64_t *size_state, double *cost,
                         double *stale, uint64_t *requests, void *stream);

#ifdef __cplusplus
}
#endif
#endif
