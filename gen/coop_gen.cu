// coop_gen.cu -- seeded synthetic block-table generator (input generation only).
// Compiled with --fmad=false / -ffp-contract=off so host and device agree bit-for-bit.
// Recipe: DESIGN.md "Input recipe" (Table 1 densities PAPER.md:185-187).
#include <cuda_runtime.h>

#include "coop_gen.h"

namespace {

__host__ __device__ inline uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// per-item draw: lane 0 free, 1 size, 2 class/cost, 3 staleness
__host__ __device__ inline uint64_t item_draw(uint64_t seed, int64_t p, int32_t n, int32_t k,
                                              int lane) {
  uint64_t ctr = ((uint64_t)p * (uint64_t)n + (uint64_t)k) * 4ull + (uint64_t)lane;
  return splitmix64(splitmix64(seed) ^ ctr);
}

// per-pool draw: m 0..2 interior pins, 3 pin count, 4..6 request, 7 spare
__host__ __device__ inline uint64_t pool_draw(uint64_t seed, int64_t p, int m) {
  return splitmix64(splitmix64(seed ^ 0xD1B54A32D192ED03ull) ^ ((uint64_t)p * 8ull + (uint64_t)m));
}

__host__ __device__ inline bool raw_free(uint64_t seed, int64_t p, int32_t n, int32_t k) {
  return (item_draw(seed, p, n, k, 0) % 100ull) < 12ull;  // 12 % raw free rate
}

__host__ __device__ inline bool is_pinned(int mode, uint64_t seed, int64_t p, int32_t n,
                                          int32_t k) {
  if (mode == COOPGEN_MODE_BENCH) {
    int32_t end = n / 32;  // parameter regions at both pool ends
    if (k < end || k >= n - end) return true;
    int32_t inner = n - 2 * end;
    if (inner <= 0) return false;
    for (int m = 0; m < 3; ++m)  // the executing op's inputs: 3 interior pins
      if (k == end + (int32_t)(pool_draw(seed, p, m) % (uint64_t)inner)) return true;
    return false;
  }
  int cnt = (int)(pool_draw(seed, p, 3) % 4ull);  // 0..3 interior pins
  for (int m = 0; m < cnt; ++m)
    if (k == (int32_t)(pool_draw(seed, p, m) % (uint64_t)n)) return true;
  return false;
}

__host__ __device__ inline void gen_item(int mode, uint64_t seed, int64_t p, int32_t n,
                                         int32_t k, uint64_t *ss, double *c, double *s) {
  uint64_t state;
  if (is_pinned(mode, seed, p, n, k))
    state = 2;  // PINNED
  else if (raw_free(seed, p, n, k) && !(k > 0 && raw_free(seed, p, n, k - 1)))
    state = 0;  // FREE (never two adjacent FREE items)
  else
    state = 1;  // EVICTABLE
  uint64_t x1 = item_draw(seed, p, n, k, 1);
  uint64_t size;
  if (mode == COOPGEN_MODE_BENCH) {
    uint64_t e = x1 % 19ull;  // log-uniform-ish: 512 B .. 256 MiB
    size = 512ull * ((1ull << e) + ((x1 >> 8) & ((1ull << e) - 1ull)));
  } else {
    size = 1ull + ((x1 >> 8) & ((1ull << 20) - 1ull));  // uniform int [1, 2^20]
  }
  uint64_t x2 = item_draw(seed, p, n, k, 2);
  double density;
  if (x2 % 100ull < 40ull)
    density = 35.6;  // C1 conv/matmul, Table 1 ResNet-50 column
  else
    density = ((x2 >> 8) & 1ull) ? 5.0 : 3.9;  // C2 norm / activation
  double mult = (double)(1ull + ((x2 >> 16) & 3ull));  // neighbourhood multiplier 1..4
  double cost = ((density * (double)size) / 1048576.0) * mult;
  double stale = (double)(1ull + item_draw(seed, p, n, k, 3) % 1000000ull);
  *ss = size | (state << 62);
  *c = cost;
  *s = stale;
}

__host__ __device__ inline uint64_t gen_request(int mode, uint64_t seed, int64_t p,
                                                uint64_t pool_total) {
  if (mode == COOPGEN_MODE_BENCH) {
    if (p % 64 == 63) return (1ull << 62) - 1ull;  // forced infeasible
    if (p % 2 == 0) {                              // short request: law of sizes
      uint64_t x = pool_draw(seed, p, 5);
      uint64_t e = x % 19ull;
      return 512ull * ((1ull << e) + ((x >> 8) & ((1ull << e) - 1ull)));
    }
    const uint64_t lo = 256ull << 20, hi = 8ull << 30;  // long request U[256 MiB, 8 GiB)
    return lo + pool_draw(seed, p, 6) % (hi - lo);
  }
  uint64_t half = pool_total / 2;
  if (half < 1) half = 1;
  return 1ull + pool_draw(seed, p, 4) % half;
}

__global__ void gen_items_kernel(int mode, uint64_t seed, int64_t p0, int64_t n_pools, int32_t n,
                                 int64_t stride, uint64_t *ss, double *c, double *s) {
  int64_t total = n_pools * (int64_t)n;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t lp = idx / n;
    int32_t k = (int32_t)(idx - lp * n);
    int64_t o = lp * stride + k;
    gen_item(mode, seed, p0 + lp, n, k, ss + o, c + o, s + o);
  }
}

__global__ void gen_requests_kernel(int mode, uint64_t seed, int64_t p0, int64_t n_pools,
                                    int32_t n, int64_t stride, const uint64_t *ss,
                                    uint64_t *req) {
  for (int64_t lp = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; lp < n_pools;
       lp += (int64_t)gridDim.x * blockDim.x) {
    uint64_t tot = 0;
    if (mode != COOPGEN_MODE_BENCH)
      for (int32_t k = 0; k < n; ++k) tot += ss[lp * stride + k] & ((1ull << 62) - 1ull);
    req[lp] = gen_request(mode, seed, p0 + lp, tot);
  }
}

bool bad_args(int mode, int64_t p0, int64_t n_pools, int32_t n, int64_t stride) {
  return (mode != COOPGEN_MODE_BENCH && mode != COOPGEN_MODE_SMALL) || p0 < 0 || n_pools < 0 ||
         n < 1 || stride < n;
}

}  // namespace

extern "C" int coopgen_pools_host(int mode, uint64_t seed, int64_t p0, int64_t n_pools,
                                  int32_t n, int64_t stride, uint64_t *ss, double *c,
                                  double *s, uint64_t *req) {
  if (bad_args(mode, p0, n_pools, n, stride) || !ss || !c || !s || !req) return -1;
  for (int64_t lp = 0; lp < n_pools; ++lp) {
    uint64_t tot = 0;
    for (int32_t k = 0; k < n; ++k) {
      int64_t o = lp * stride + k;
      gen_item(mode, seed, p0 + lp, n, k, ss + o, c + o, s + o);
      tot += ss[o] & ((1ull << 62) - 1ull);
    }
    req[lp] = gen_request(mode, seed, p0 + lp, tot);
  }
  return 0;
}

extern "C" int coopgen_pools_device(int mode, uint64_t seed, int64_t p0, int64_t n_pools,
                                    int32_t n, int64_t stride, uint64_t *ss, double *c,
                                    double *s, uint64_t *req, void *stream) {
  if (bad_args(mode, p0, n_pools, n, stride) || !ss || !c || !s || !req) return -1;
  if (n_pools == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  gen_items_kernel<<<sms * 8, 256, 0, st>>>(mode, seed, p0, n_pools, n, stride, ss, c, s);
  int64_t rb = (n_pools + 255) / 256;
  if (rb > sms * 8) rb = sms * 8;
  gen_requests_kernel<<<(unsigned)rb, 256, 0, st>>>(mode, seed, p0, n_pools, n, stride, ss, req);
  return cudaGetLastError() == cudaSuccess ? 0 : -5;
}
