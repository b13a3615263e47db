// coop_pool.cu -- the online single-pool calls of include/coop.h (coop_pool_init, coop_alloc,
// coop_free, coop_access, coop_rematerialize, coop_pool_stats, coop_pool_layout).
//
// The pool is DEVICE-resident: the address-ordered block table, the growing tensor graph
// (one op per coop_alloc: cost, inputs = parents, output = the new tensor), residency
// flags, pins, last accesses, the clock and the counters persist in global memory between
// calls.  Each call is ONE launch of a 256-thread CTA that loads the block table and the
// tensor flags into shared memory, runs the same Alg. 1 engine as the trace replay
// (replay_core.cuh: first fit by class side, Sec. 3.3 window search with projected costs
// and the exact 192-bit scans, eviction, coalescing, in-place transfer) and stores the
// state back.  Arguments (the parents) and results (status, coop_alloc_result, evicted
// ids) travel through mapped pinned host memory, so a call is launch + one stream sync.
// Readings R38-R44; bit-exact with the oracle O3.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <new>
#include <vector>

#include "replay_core.cuh"

namespace coop {
namespace {

enum : int32_t { PK_ALLOC = 0, PK_FREE = 1, PK_ACCESS = 2, PK_REMAT = 3 };

// persistent pool scalars + block table (global memory)
struct PoolState {
  uint64_t addr[kCap + 2], size[kCap + 2];
  int32_t owner[kCap + 2];
  int32_t nb, n_tensors, n_edges;
  uint64_t bytes_free;
  int64_t clock;
  coop_replay_result res;
};

// writable view of the graph arrays that TraceDev reads
struct GraphMut {
  uint64_t *size;
  int32_t *producer;
  uint8_t *unevict;
  int64_t *cost;
  int32_t *out, *src;
  uint8_t *phase, *cls;
  int32_t *in_ptr, *in_idx;
  int32_t *cons_head, *cons_next, *cons_out;
  int4 *rec;
};

// mapped pinned host memory shared by the host and the call's CTA
struct HostIO {
  int32_t status, n_victims;
  int64_t need_parent;
  coop_alloc_result r;
};

struct PArgs {
  KArgs k;
  GraphMut g;
  PoolState *ps;
  int32_t kind, t, src, n_parents;
  uint64_t size, adv;
  int64_t cost;
  uint32_t op_flags;
  HostIO *io;
  const int32_t *io_parents;
  int32_t *io_victims;
};

// The persistent state moves between global memory and the CTA's shared memory:
// pool_load before a call (or once, when the service kernel starts), pool_store after it
// (or when the service kernel flushes / exits).
__device__ __forceinline__ void pool_load(const PArgs &pa, Shared &sh) {
  PoolState &P = *pa.ps;
  const int tid = threadIdx.x;
  const int nb0 = P.nb, nt = P.n_tensors;
  const int nflag = min(nt + 1, pa.k.tr.T);
  uint8_t *tflags = pa.k.ws + pa.k.lay.tflags;  // CTA slot 0 (Cell's layout)
  for (int b = tid; b < nb0; b += kThreads) {
    sh.addr[b] = P.addr[b];
    sh.size[b] = P.size[b];
    sh.owner[b] = P.owner[b];
  }
  for (int x = tid; x < nflag; x += kThreads) sh.tfl[x] = tflags[x];
  if (tid == 0) {
    sh.nb = nb0;
    sh.bytes_free = P.bytes_free;
    sh.clock = P.clock;
    sh.res = P.res;
  }
  __syncthreads();
}

__device__ __forceinline__ void pool_store(const PArgs &pa, Shared &sh) {
  PoolState &P = *pa.ps;
  const int tid = threadIdx.x;
  const int nflag = min(P.n_tensors + 1, pa.k.tr.T);
  uint8_t *tflags = pa.k.ws + pa.k.lay.tflags;
  const int nb1 = sh.nb;
  for (int b = tid; b < nb1; b += kThreads) {
    P.addr[b] = sh.addr[b];
    P.size[b] = sh.size[b];
    P.owner[b] = sh.owner[b];
  }
  for (int x = tid; x < nflag; x += kThreads) tflags[x] = sh.tfl[x];
  if (tid == 0) {
    P.nb = nb1;
    P.bytes_free = sh.bytes_free;
    P.clock = sh.clock;
    P.res = sh.res;
  }
  __syncthreads();
}

// One online call on the state held in shared memory (loaded by pool_load).  Results go
// to the mapped HostIO; the caller orders them before its completion signal.
__device__ __forceinline__ void pool_call(const PArgs &pa, Shared &sh) {
  CellT<false> c(pa.k, sh, 0);  // coherent loads: the graph grows between calls
  PoolState &P = *pa.ps;
  const GraphMut &g = pa.g;
  const int tid = threadIdx.x, t = pa.t;
  if (tid == 0) {
    sh.status = COOP_OK;
    sh.cur_op = t;
    sh.redpar = 0;
    sh.win_first = sh.win_last = -1;
    sh.nvict = 0;
    sh.win_span = 0;
    sh.win_cost = 0;
  }
  c.epoch = c.w.epochs[tid];
  __syncthreads();

  int32_t st = COOP_OK;
  int64_t need = -1;
  bool fill = false;
  if (pa.kind == PK_ALLOC || pa.kind == PK_REMAT) {
    // the op's inputs: the call's parents (alloc) or the recorded ones (remat)
    const int np = pa.kind == PK_ALLOC ? pa.n_parents : g.in_ptr[t + 1] - g.in_ptr[t];
    // parents: copied once from mapped host memory (one PCIe round trip, all threads),
    // then read from the device copy in the graph's edge list
    const int32_t *par = g.in_idx + g.in_ptr[t];
    bool resident_now = false;
    if (pa.kind == PK_ALLOC) {
      const int32_t e0 = g.in_ptr[t];
      for (int j = tid; j < np; j += kThreads) g.in_idx[e0 + j] = pa.io_parents[j];
      if (tid == 0) {  // the new op / tensor t (read below with plain loads only)
        g.in_ptr[t + 1] = e0 + np;
        g.size[t] = pa.size;
        g.producer[t] = t;
        g.out[t] = t;
        g.cost[t] = pa.cost;
        g.src[t] = (pa.op_flags & COOP_OP_INPLACE) ? pa.src : -1;
        g.phase[t] = (pa.op_flags & COOP_OP_PHASE_FWD) ? COOP_PHASE_FWD : COOP_PHASE_BWD;
        g.cls[t] = (pa.op_flags & COOP_OP_EXPENSIVE) ? 1 : (pa.op_flags & COOP_OP_CHEAP) ? 2 : 0;
        g.rec[t] = make_int4((int)(uint32_t)(uint64_t)pa.cost, (int)(uint32_t)((uint64_t)pa.cost >> 32), e0, e0 + np);
        g.unevict[t] = ((pa.op_flags & COOP_OP_UNEVICTABLE) || (g.src[t] >= 0 && g.unevict[g.src[t]])) ? 1 : 0;
        sh.tfl[t] = 0;
        c.w.pins[t] = 0;
        c.w.last_access[t] = 0;
      }
      __syncthreads();
    } else {
      resident_now = sh.tfl[t] & TF_RES;
    }
    if (resident_now) {
      fill = true;  // remat of a resident tensor: nothing to do
    } else {
      int jbad = 0x7fffffff;
      for (int j = tid; j < np; j += kThreads)
        if (!(sh.tfl[par[j]] & TF_RES)) jbad = min(jbad, j);
      jbad = cta_min_i32(sh, jbad);
      if (jbad != 0x7fffffff) {
        st = COOP_NEEDS_REMAT;
        need = par[jbad];
      } else {
        for (int j = tid; j < np; j += kThreads) atomicAdd(&c.w.pins[par[j]], 1);  // R16
        __syncthreads();
        if (pa.kind == PK_ALLOC) c.allocate(t, t, true, 1);  // Alg. 1, in-place allowed
        else c.allocate(t, t, false, 5);                     // out of place (R21)
        const bool ok = c.ok();
        if (ok && tid == 0) {
          const int64_t cost = g.cost[t];
          sh.clock += cost;
          sh.res.total_us += cost;
          if (pa.kind == PK_ALLOC) {
            sh.tfl[t] |= TF_BORN;
            sh.res.base_us += cost;
            c.log_ev(6, t, t, c.w.taddr[t]);
          } else {
            sh.res.remat++;
            c.log_ev(7, t, t, c.w.taddr[t]);
          }
        }
        __syncthreads();
        const int64_t clk = sh.clock;
        for (int j = tid; j < np; j += kThreads) {
          if (ok) c.w.last_access[par[j]] = clk;
          atomicSub(&c.w.pins[par[j]], 1);
        }
        if (ok && tid == 0) c.w.last_access[t] = clk;
        __syncthreads();
        if (ok) {
          fill = true;
          if (pa.kind == PK_ALLOC && tid == 0) {  // link the op into its parents' consumer lists
            for (int j = 0; j < np; ++j) {
              const int e = P.n_edges + j;
              g.cons_out[e] = t;  // out[t] == t
              g.cons_next[e] = g.cons_head[par[j]];
              g.cons_head[par[j]] = e;
            }
            P.n_edges += np;
            P.n_tensors = t + 1;
          }
        } else {
          st = sh.status == COOP_OK ? COOP_ERR_UNSATISFIABLE : sh.status;
        }
      }
    }
  } else if (pa.kind == PK_FREE) {
    const uint8_t f = sh.tfl[t];
    if ((f & TF_DEAD) && !(f & TF_RES)) {
      st = COOP_ERR_BAD_STATE;  // double free
    } else {
      if (f & TF_RES) c.free_tensor(t);
      if (tid == 0) sh.tfl[t] |= TF_DEAD;
    }
  } else {  // PK_ACCESS
    const uint8_t f = sh.tfl[t];
    if ((f & TF_DEAD) && !(f & TF_RES)) {
      st = COOP_ERR_BAD_STATE;
    } else {
      if (tid == 0) {
        sh.clock += (int64_t)pa.adv;
        if (f & TF_RES) c.w.last_access[t] = sh.clock;  // staleness restarts (R17)
      }
      st = (f & TF_RES) ? COOP_OK : COOP_NEEDS_REMAT;
    }
  }
  __syncthreads();

  // ---- results to the host
  const int nv = sh.nvict;
  if (fill)
    for (int k = tid; k < nv; k += kThreads) pa.io_victims[k] = c.w.victims[k];
  if (tid == 0) {
    HostIO &io = *pa.io;
    io.status = st;
    io.n_victims = fill ? nv : 0;
    io.need_parent = need;
    if (fill) {
      coop_alloc_result r;
      r.tensor_id = t;
      r.addr = c.w.taddr[t];
      r.size = g.size[t];
      r.n_evicted = nv;
      r.window_first = sh.win_first;
      r.window_last = sh.win_last;
      r.reserved = 0;
      r.window_span = sh.win_first >= 0 ? sh.win_span : 0;
      r.window_cost = sh.win_first >= 0 ? __longlong_as_double((long long)sh.win_cost) : 0.0;
      io.r = r;
    }
  }
  c.w.epochs[tid] = c.epoch;
  __syncthreads();
}

__global__ void __launch_bounds__(kThreads, 1) pool_kernel(const PArgs pa) {
  extern __shared__ __align__(16) unsigned char smem[];
  Shared &sh = *reinterpret_cast<Shared *>(smem);
  pool_load(pa, sh);
  pool_call(pa, sh);
  pool_store(pa, sh);
  __threadfence_system();
}

// ---- persistent service (coop_pool_service) ----------------------------
// One resident CTA per pool polls a mailbox in mapped pinned host memory: the host writes
// a call's arguments, then bumps `seq`; thread 0 sees the new sequence number (acquire,
// system scope), the CTA runs pool_call, and thread 0 publishes `done = seq` after a
// system-scope fence.  A call therefore costs two PCIe crossings instead of a launch and
// a stream synchronisation.  The kernel exits on PK_STOP, or after `idle_ns` without a
// call (so a device-wide synchronisation elsewhere never waits longer than that); the
// host relaunches it on the next call.
enum : int32_t { PK_STOP = 4, PK_FLUSH = 5 };

struct alignas(64) Mailbox {  // mapped pinned host memory, written by the host (except done)
  int32_t kind, t, src, n_parents;  // arguments: bytes [0, 48), read as 3 x 16 bytes
  uint64_t size, adv;
  int64_t cost;
  uint32_t op_flags, pad0;
  int64_t seq;   // bumped by the host after the arguments
  int64_t pad1;
  int64_t done;  // written by the device (own 64-byte line)
  int64_t pad2[7];
};
static_assert(offsetof(Mailbox, size) == 16 && offsetof(Mailbox, op_flags) == 40 &&
              offsetof(Mailbox, seq) == 48 && offsetof(Mailbox, done) == 64, "mailbox layout");

__device__ __forceinline__ int64_t ld_acquire_sys(const int64_t *p) {
  int64_t v;
  asm volatile("ld.acquire.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(int64_t *p, int64_t v) {
  asm volatile("st.release.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void __launch_bounds__(kThreads, 1) pool_service_kernel(const PArgs base, Mailbox *mb,
                                                                   uint64_t idle_ns) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int64_t s_seq;
  __shared__ int32_t s_go;
  __shared__ PArgs s_pa;
  Shared &sh = *reinterpret_cast<Shared *>(smem);
  int64_t last = ld_acquire_sys(&mb->done);
  pool_load(base, sh);  // the state stays in shared memory while the kernel is resident
  for (;;) {
    if (threadIdx.x == 0) {
      const uint64_t t0 = gtimer();
      int64_t s;
      int go;
      for (;;) {
        s = ld_acquire_sys(&mb->seq);
        if (s != last) { go = 1; break; }
        if (gtimer() - t0 > idle_ns) { go = 0; break; }
      }
      s_seq = s;
      if (go) {
        // the 48 bytes of arguments after seq: three independent 16-byte loads in flight
        // together (one PCIe round trip), ordered after the acquire of seq
        uint64_t w[6];
        const uint64_t *f = reinterpret_cast<const uint64_t *>(mb);
#pragma unroll
        for (int q = 0; q < 3; ++q)
          asm volatile("ld.relaxed.sys.global.v2.b64 {%0, %1}, [%2];"
                       : "=l"(w[2 * q]), "=l"(w[2 * q + 1]) : "l"(f + 2 * q) : "memory");
        PArgs pa = base;
        pa.kind = (int32_t)(uint32_t)w[0];
        pa.t = (int32_t)(uint32_t)(w[0] >> 32);
        pa.src = (int32_t)(uint32_t)w[1];
        pa.n_parents = (int32_t)(uint32_t)(w[1] >> 32);
        pa.size = w[2];
        pa.adv = w[3];
        pa.cost = (int64_t)w[4];
        pa.op_flags = (uint32_t)w[5];
        if (pa.kind == PK_STOP) go = 2;
        s_pa = pa;
      }
      s_go = go;
    }
    __syncthreads();
    const int go = s_go;
    if (go == 1) {
      if (s_pa.kind == PK_FLUSH) pool_store(base, sh);
      else pool_call(s_pa, sh);
    } else {
      pool_store(base, sh);  // exit (idle or PK_STOP): the state back to global memory
    }
    __syncthreads();
    if (go == 0) {
      __threadfence_system();
      break;
    }
    last = s_seq;
    // the call's HostIO / victim writes (all threads, ordered by the barrier above) are
    // published by one release store at system scope
    if (threadIdx.x == 0) st_release_sys(&mb->done, last);
    if (go == 2) break;
  }
}

}  // namespace
}  // namespace coop

// =============================================================================== host
using namespace coop;

struct coop_pool_s {
  coop_pool_config cfg{};
  int device = 0;
  cudaStream_t stream = nullptr;
  PoolState *d_ps = nullptr;
  unsigned char *d_graph = nullptr;
  GraphMut g{};
  TraceDev td{};
  unsigned char *ws = nullptr;
  WsLayout lay{};
  unsigned char *io_host = nullptr;  // mapped pinned: HostIO | parents | victims
  unsigned char *io_dev = nullptr;
  int32_t n_tensors = 0, n_edges = 0;
  std::vector<uint64_t> sizes;  // host mirror for argument validation
  // persistent service (coop_pool_service): mailbox in mapped pinned memory
  Mailbox *mb_host = nullptr, *mb_dev = nullptr;
  int64_t seq = 0;
  uint64_t idle_ns = 0;  // 0: one launch per call
  bool launched = false;  // a service kernel may be resident on `stream`
  std::chrono::steady_clock::time_point last_call{};
};

namespace {

size_t io_bytes(const coop_pool_config &c) {
  return sizeof(HostIO) + (size_t)(c.max_edges + 1) * 4 + (size_t)(kCap + 2) * 4;
}

void service_stop(coop_pool_s *p);

void pool_release(coop_pool_s *p) {
  service_stop(p);
  if (p->mb_host) cudaFreeHost(p->mb_host);
  if (p->stream) cudaStreamDestroy(p->stream);
  if (p->d_ps) cudaFree(p->d_ps);
  if (p->d_graph) cudaFree(p->d_graph);
  if (p->ws) cudaFree(p->ws);
  if (p->io_host) cudaFreeHost(p->io_host);
  delete p;
}

// dynamic shared memory of the pool kernels: Shared plus one flag byte per tensor id
size_t pool_smem(const coop_pool_s *p) { return sizeof(Shared) + (size_t)(p->cfg.max_tensors + 15) / 16 * 16; }

PArgs base_args(coop_pool_s *p) {
  PArgs a{};
  a.k.tr = p->td;
  a.k.tfl_bytes = (p->cfg.max_tensors + 15) / 16 * 16;
  a.k.walkers = 0;  // the online pool's graph grows: generic closure walk
  a.k.flags = p->cfg.flags;
  a.k.thr = p->cfg.class_threshold;
  a.k.max_depth = 512;
  a.k.n_cells = 1;
  a.k.ws = p->ws;
  a.k.lay = p->lay;
  a.g = p->g;
  a.ps = p->d_ps;
  a.io = reinterpret_cast<HostIO *>(p->io_dev);
  a.io_parents = reinterpret_cast<const int32_t *>(p->io_dev + sizeof(HostIO));
  a.io_victims = reinterpret_cast<int32_t *>(p->io_dev + sizeof(HostIO) + (size_t)(p->cfg.max_edges + 1) * 4);
  return a;
}

// Launch the service kernel if none is resident (never launched, or it exited idle).
int service_ensure(coop_pool_s *p) {
  if (p->launched) {
    const cudaError_t q = cudaStreamQuery(p->stream);
    if (q == cudaErrorNotReady) return COOP_OK;
    if (q != cudaSuccess) return COOP_ERR_CUDA;
  }
  pool_service_kernel<<<1, kThreads, pool_smem(p), p->stream>>>(base_args(p), p->mb_dev, p->idle_ns);
  if (cudaGetLastError() != cudaSuccess) return COOP_ERR_CUDA;
  p->launched = true;
  return COOP_OK;
}

// Post one call to the mailbox and spin until the device acknowledges it.  A kernel that
// went idle between the post and its last poll is detected by cudaStreamQuery and
// relaunched (it then sees the pending sequence number).
int service_call(coop_pool_s *p, int32_t kind, int32_t t, uint64_t size, int64_t cost,
                 uint32_t op_flags, int32_t src, int32_t n_parents, uint64_t adv) {
  volatile Mailbox *m = p->mb_host;
  m->kind = kind;
  m->t = t;
  m->src = src;
  m->n_parents = n_parents;
  m->size = size;
  m->adv = adv;
  m->cost = cost;
  m->op_flags = op_flags;
  const int64_t s = ++p->seq;
  std::atomic_thread_fence(std::memory_order_release);
  m->seq = s;
  const auto t0 = std::chrono::steady_clock::now();
  // a kernel idle for about its timeout may have exited: check (and relaunch) up front
  if (!p->launched || (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(t0 - p->last_call).count() >= p->idle_ns / 2)
    if (service_ensure(p) != COOP_OK) return COOP_ERR_CUDA;
  for (uint32_t spin = 1; m->done != s; ++spin) {
    if ((spin & 0x3fffu) == 0) {
      const cudaError_t q = cudaStreamQuery(p->stream);
      if (q == cudaSuccess) {  // the kernel exited (idle) before seeing the call
        if (m->done == s) break;
        p->launched = false;
        if (service_ensure(p) != COOP_OK) return COOP_ERR_CUDA;
      } else if (q != cudaErrorNotReady) {
        return COOP_ERR_CUDA;
      }
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(60)) return COOP_ERR_CUDA;
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  p->last_call = std::chrono::steady_clock::now();
  return COOP_OK;
}

void service_stop(coop_pool_s *p) {
  if (!p->launched) return;
  if (cudaStreamQuery(p->stream) == cudaErrorNotReady) service_call(p, PK_STOP, 0, 0, 0, 0, -1, 0, 0);
  cudaStreamSynchronize(p->stream);
  p->launched = false;
}

int launch_call(coop_pool_s *p, int32_t kind, int32_t t, uint64_t size, int64_t cost,
                uint32_t op_flags, int32_t src, int32_t n_parents, uint64_t adv) {
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != p->device) cudaSetDevice(p->device);
  if (p->idle_ns) {
    const int rc = service_call(p, kind, t, size, cost, op_flags, src, n_parents, adv);
    if (prev != p->device) cudaSetDevice(prev);
    return rc;
  }
  PArgs a = base_args(p);
  a.kind = kind;
  a.t = t;
  a.src = src;
  a.n_parents = n_parents;
  a.size = size;
  a.adv = adv;
  a.cost = cost;
  a.op_flags = op_flags;
  pool_kernel<<<1, kThreads, pool_smem(p), p->stream>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(p->stream);
  if (prev != p->device) cudaSetDevice(prev);
  return e == cudaSuccess ? COOP_OK : COOP_ERR_CUDA;
}

HostIO &io_of(coop_pool_s *p) { return *reinterpret_cast<HostIO *>(p->io_host); }

int finish(coop_pool_s *p, coop_alloc_result *out, int64_t *evicted, int32_t cap) {
  HostIO &io = io_of(p);
  const int st = io.status;
  if (st == COOP_OK && out) *out = io.r;
  if (st == COOP_NEEDS_REMAT && out) {
    memset(out, 0, sizeof(*out));
    out->tensor_id = io.need_parent;
    out->window_first = out->window_last = -1;
  }
  if (st == COOP_OK && evicted) {
    const int32_t *v = reinterpret_cast<const int32_t *>(p->io_host + sizeof(HostIO) +
                                                         (size_t)(p->cfg.max_edges + 1) * 4);
    for (int k = 0; k < std::min(io.n_victims, cap); ++k) evicted[k] = v[k];
  }
  return st;
}

}  // namespace

extern "C" int coop_pool_init(const coop_pool_config *cfg, coop_pool_t *out) {
  if (!cfg || !out || cfg->budget < 1 || bad_flags(cfg->flags) || cfg->max_tensors < 1 ||
      cfg->max_tensors > kMaxT || cfg->max_edges < 0)
    return COOP_ERR_INVALID_ARG;
  coop_pool_s *p = new (std::nothrow) coop_pool_s();
  if (!p) return COOP_ERR_NOMEM;
  p->cfg = *cfg;
  if (!p->cfg.class_threshold) p->cfg.class_threshold = 15;
  cudaGetDevice(&p->device);
  const int T = cfg->max_tensors, E = cfg->max_edges;
  // graph arrays: one allocation, 256-byte aligned pieces
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t r = off;
    off = (off + bytes + 255) / 256 * 256;
    return r;
  };
  const size_t o_size = take((size_t)T * 8), o_prod = take((size_t)T * 4), o_unev = take((size_t)T),
               o_cost = take((size_t)T * 8), o_out = take((size_t)T * 4), o_src = take((size_t)T * 4),
               o_phase = take((size_t)T), o_cls = take((size_t)T), o_inp = take((size_t)(T + 1) * 4),
               o_ini = take((size_t)(E + 1) * 4), o_ch = take((size_t)T * 4),
               o_cn = take((size_t)(E + 1) * 4), o_co = take((size_t)(E + 1) * 4),
               o_rec = take((size_t)T * 16);
  int rc = COOP_OK;
  if (cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMalloc(&p->d_ps, sizeof(PoolState)) != cudaSuccess || cudaMalloc(&p->d_graph, off) != cudaSuccess) {
    rc = COOP_ERR_NOMEM;
  }
  p->lay = make_layout(T);
  if (rc == COOP_OK && cudaMalloc(&p->ws, p->lay.bytes) != cudaSuccess) rc = COOP_ERR_NOMEM;
  if (rc == COOP_OK && cudaHostAlloc(&p->io_host, io_bytes(p->cfg), cudaHostAllocMapped) != cudaSuccess) {
    p->io_host = nullptr;
    rc = COOP_ERR_NOMEM;
  }
  if (rc == COOP_OK && cudaHostGetDevicePointer((void **)&p->io_dev, p->io_host, 0) != cudaSuccess) rc = COOP_ERR_CUDA;
  if (rc == COOP_OK && cudaHostAlloc((void **)&p->mb_host, sizeof(Mailbox), cudaHostAllocMapped) != cudaSuccess) {
    p->mb_host = nullptr;
    rc = COOP_ERR_NOMEM;
  }
  if (rc == COOP_OK) {
    memset(p->mb_host, 0, sizeof(Mailbox));
    if (cudaHostGetDevicePointer((void **)&p->mb_dev, p->mb_host, 0) != cudaSuccess) rc = COOP_ERR_CUDA;
  }
  if (rc == COOP_OK && cudaFuncSetAttribute(pool_service_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)pool_smem(p)) != cudaSuccess)
    rc = COOP_ERR_CUDA;
  if (rc == COOP_OK && cudaFuncSetAttribute(pool_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)pool_smem(p)) != cudaSuccess)
    rc = COOP_ERR_CUDA;
  if (rc != COOP_OK) {
    pool_release(p);
    return rc;
  }
  unsigned char *b = p->d_graph;
  GraphMut &g = p->g;
  g.size = (uint64_t *)(b + o_size);
  g.producer = (int32_t *)(b + o_prod);
  g.unevict = (uint8_t *)(b + o_unev);
  g.cost = (int64_t *)(b + o_cost);
  g.out = (int32_t *)(b + o_out);
  g.src = (int32_t *)(b + o_src);
  g.phase = (uint8_t *)(b + o_phase);
  g.cls = (uint8_t *)(b + o_cls);
  g.in_ptr = (int32_t *)(b + o_inp);
  g.in_idx = (int32_t *)(b + o_ini);
  g.cons_head = (int32_t *)(b + o_ch);
  g.cons_next = (int32_t *)(b + o_cn);
  g.cons_out = (int32_t *)(b + o_co);
  g.rec = (int4 *)(b + o_rec);
  TraceDev &td = p->td;
  td.T = T;
  td.M = T;
  td.n_params = 0;
  td.size = g.size;
  td.producer = g.producer;
  td.unevict = g.unevict;
  td.cost = g.cost;
  td.out = g.out;
  td.src = g.src;
  td.phase = g.phase;
  td.in_ptr = g.in_ptr;
  td.in_idx = g.in_idx;
  td.cons_head = g.cons_head;
  td.cons_next = g.cons_next;
  td.cons_out = g.cons_out;
  td.rec = g.rec;
  td.cls = g.cls;
  // initial state: one free block [0, budget)
  PoolState *h = new (std::nothrow) PoolState();
  if (!h) {
    pool_release(p);
    return COOP_ERR_NOMEM;
  }
  memset(h, 0, sizeof(*h));
  h->nb = 1;
  h->addr[0] = 0;
  h->size[0] = cfg->budget;
  h->owner[0] = kFree;
  h->bytes_free = cfg->budget;
  h->res.fail_op = -1;
  h->res.digest = 0x9E3779B97F4A7C15ull;
  h->res.budget = cfg->budget;
  h->res.max_blocks = 1;
  // every initialisation is ordered on the pool's (non-blocking) stream, on which all of
  // its kernels run, and completed before the handle is returned
  bool ok = cudaMemcpyAsync(p->d_ps, h, sizeof(PoolState), cudaMemcpyHostToDevice, p->stream) == cudaSuccess &&
            cudaMemsetAsync(p->d_graph, 0, off, p->stream) == cudaSuccess &&
            cudaMemsetAsync(g.cons_head, 0xff, (size_t)T * 4, p->stream) == cudaSuccess &&
            cudaMemsetAsync(p->ws, 0, p->lay.bytes, p->stream) == cudaSuccess &&
            cudaStreamSynchronize(p->stream) == cudaSuccess;
  delete h;
  if (!ok) {
    pool_release(p);
    return COOP_ERR_CUDA;
  }
  memset(p->io_host, 0, io_bytes(p->cfg));
  p->sizes.reserve((size_t)T);
  *out = p;
  return COOP_OK;
}

extern "C" int coop_pool_destroy(coop_pool_t p) {
  if (!p) return COOP_ERR_INVALID_ARG;
  pool_release(p);
  return COOP_OK;
}

extern "C" int coop_alloc(coop_pool_t p, uint64_t size, uint64_t cost_us, uint32_t op_flags,
                          int64_t inplace_src, const int64_t *parents, int32_t n_parents,
                          coop_alloc_result *out, int64_t *evicted_ids, int32_t evicted_cap) {
  if (!p) return COOP_ERR_INVALID_ARG;
  if (size < 1 || size >= (1ull << 48) || cost_us >= (1ull << 40)) return COOP_ERR_INVALID_ARG;
  if ((op_flags & ~31u) || ((op_flags & COOP_OP_EXPENSIVE) && (op_flags & COOP_OP_CHEAP)))
    return COOP_ERR_INVALID_ARG;
  if (n_parents < 0 || (n_parents > 0 && !parents) || evicted_cap < 0 || (evicted_cap > 0 && !evicted_ids))
    return COOP_ERR_INVALID_ARG;
  for (int j = 0; j < n_parents; ++j)
    if (parents[j] < 0 || parents[j] >= p->n_tensors) return COOP_ERR_UNKNOWN_ID;
  if (op_flags & COOP_OP_INPLACE) {
    bool seen = false;
    for (int j = 0; j < n_parents; ++j) seen |= parents[j] == inplace_src;
    if (!seen || p->sizes[(size_t)inplace_src] != size) return COOP_ERR_INVALID_ARG;
  } else if (inplace_src != -1) {
    return COOP_ERR_INVALID_ARG;
  }
  if (p->n_tensors >= p->cfg.max_tensors || (int64_t)p->n_edges + n_parents > p->cfg.max_edges)
    return COOP_ERR_NOMEM;
  int32_t *par = reinterpret_cast<int32_t *>(p->io_host + sizeof(HostIO));
  for (int j = 0; j < n_parents; ++j) par[j] = (int32_t)parents[j];
  const int32_t t = p->n_tensors;
  const int rc = launch_call(p, PK_ALLOC, t, size, (int64_t)cost_us, op_flags,
                             (op_flags & COOP_OP_INPLACE) ? (int32_t)inplace_src : -1, n_parents, 0);
  if (rc != COOP_OK) return rc;
  const int st = finish(p, out, evicted_ids, evicted_cap);
  if (st == COOP_OK) {
    p->n_tensors = t + 1;
    p->n_edges += n_parents;
    p->sizes.push_back(size);
  }
  return st;
}

extern "C" int coop_free(coop_pool_t p, int64_t t) {
  if (!p) return COOP_ERR_INVALID_ARG;
  if (t < 0 || t >= p->n_tensors) return COOP_ERR_UNKNOWN_ID;
  const int rc = launch_call(p, PK_FREE, (int32_t)t, 0, 0, 0, -1, 0, 0);
  return rc != COOP_OK ? rc : io_of(p).status;
}

extern "C" int coop_access(coop_pool_t p, int64_t t, uint64_t advance_clock_us) {
  if (!p) return COOP_ERR_INVALID_ARG;
  if (t < 0 || t >= p->n_tensors) return COOP_ERR_UNKNOWN_ID;
  if (advance_clock_us >= (1ull << 40)) return COOP_ERR_INVALID_ARG;
  const int rc = launch_call(p, PK_ACCESS, (int32_t)t, 0, 0, 0, -1, 0, advance_clock_us);
  return rc != COOP_OK ? rc : io_of(p).status;
}

extern "C" int coop_rematerialize(coop_pool_t p, int64_t t, coop_alloc_result *out,
                                  int64_t *evicted_ids, int32_t evicted_cap) {
  if (!p) return COOP_ERR_INVALID_ARG;
  if (t < 0 || t >= p->n_tensors) return COOP_ERR_UNKNOWN_ID;
  if (evicted_cap < 0 || (evicted_cap > 0 && !evicted_ids)) return COOP_ERR_INVALID_ARG;
  const int rc = launch_call(p, PK_REMAT, (int32_t)t, 0, 0, 0, -1, 0, 0);
  if (rc != COOP_OK) return rc;
  return finish(p, out, evicted_ids, evicted_cap);
}

// With a resident service kernel the live state is in its shared memory: flush it first.
static int service_flush(coop_pool_t p) {
  if (!p->idle_ns || !p->launched || cudaStreamQuery(p->stream) != cudaErrorNotReady) return COOP_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != p->device) cudaSetDevice(p->device);
  const int rc = service_call(p, PK_FLUSH, 0, 0, 0, 0, -1, 0, 0);
  if (prev != p->device) cudaSetDevice(prev);
  return rc;
}

extern "C" int coop_pool_stats(coop_pool_t p, coop_replay_result *out) {
  if (!p || !out) return COOP_ERR_INVALID_ARG;
  if (service_flush(p) != COOP_OK) return COOP_ERR_CUDA;
  if (cudaMemcpy(out, &p->d_ps->res, sizeof(*out), cudaMemcpyDeviceToHost) != cudaSuccess)
    return COOP_ERR_CUDA;
  out->status = COOP_OK;
  return COOP_OK;
}

extern "C" int coop_pool_layout(coop_pool_t p, uint64_t *addr, uint64_t *size, int64_t *owner,
                                int32_t cap, int32_t *n_blocks) {
  if (!p || !n_blocks || cap < 0 || (cap > 0 && (!addr || !size || !owner))) return COOP_ERR_INVALID_ARG;
  if (service_flush(p) != COOP_OK) return COOP_ERR_CUDA;
  int32_t nb = 0;
  if (cudaMemcpy(&nb, &p->d_ps->nb, 4, cudaMemcpyDeviceToHost) != cudaSuccess) return COOP_ERR_CUDA;
  const int n = std::min(nb, cap);
  std::vector<int32_t> ow((size_t)std::max(n, 1));
  if (n > 0 && (cudaMemcpy(addr, p->d_ps->addr, (size_t)n * 8, cudaMemcpyDeviceToHost) != cudaSuccess ||
                cudaMemcpy(size, p->d_ps->size, (size_t)n * 8, cudaMemcpyDeviceToHost) != cudaSuccess ||
                cudaMemcpy(ow.data(), p->d_ps->owner, (size_t)n * 4, cudaMemcpyDeviceToHost) != cudaSuccess))
    return COOP_ERR_CUDA;
  for (int i = 0; i < n; ++i) owner[i] = ow[(size_t)i];
  *n_blocks = nb;
  return COOP_OK;
}

extern "C" int coop_pool_service(coop_pool_t p, uint32_t idle_timeout_us) {
  if (!p || idle_timeout_us > 10000000u) return COOP_ERR_INVALID_ARG;
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != p->device) cudaSetDevice(p->device);
  if (idle_timeout_us == 0) service_stop(p);
  p->idle_ns = (uint64_t)idle_timeout_us * 1000ull;
  const int rc = (idle_timeout_us && !p->launched) ? service_ensure(p) : COOP_OK;
  if (prev != p->device) cudaSetDevice(prev);
  return rc;
}
