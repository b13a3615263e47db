// coop_replay.cu -- trace replay under memory budgets: one CTA per (trace, budget) cell.
//
// Replays Alg. 1 Allocate(op, size) with the sliding-window eviction of
// Sec. 3.3, cheap tensor partitioning (Sec. 3.4),
// recomputable in-place (Sec. 3.5) and on-demand rematerialization
// (PAPER.md:22, 219-220), with the readings R10-R36 of DESIGN.md.  Bit-exact with the oracle
// O2 (same events, counters and eviction digest).
//
// Layout:
//   * the pool's address-ordered block table (addr, size, owner) lives in SHARED memory,
//     double-buffered so an insert / erase is one parallel copy + one barrier;
//   * per-tensor state (residency flags, pins, last access, address) and the scratch of
//     the window search live in a per-cell GLOBAL workspace (L2-resident);
//   * control flow is CTA-uniform: every thread walks the same op loop and the same
//     explicit rematerialization stack; scalar state changes are made by thread 0 and
//     published by __syncthreads; the parallel steps are the free-block scans, the shifts,
//     and on every pressure event the item view with projected costs (one DFS per thread
//     per candidate), the exact 192-bit span/cost scans, the per-start window ends and
//     the lexicographic argmin.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <new>
#include <vector>

#include <cooperative_groups.h>

#include "replay_core.cuh"

namespace coop {
namespace {

// a cluster's helper CTA (rank >= 1): its own CellT
__device__ __forceinline__ void helper_entry(const KArgs &a, Shared &sh, int slot, int rank) {
  CellT<true> c(a, sh, -1, slot, rank);
  c.cluster_helper();
}

__global__ void __launch_bounds__(kThreads, 1) replay_kernel(const KArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  Shared &sh = *reinterpret_cast<Shared *>(smem);
  if (a.g_smem) {  // the compact graph of the fast closure walk, once per CTA
    const uint4 *src = reinterpret_cast<const uint4 *>(a.tr.cg_cost);
    uint4 *dst = reinterpret_cast<uint4 *>(sh.tfl + a.tfl_bytes);
    for (int i = threadIdx.x; i < a.g_bytes / 16; i += kThreads) dst[i] = __ldg(src + i);
    __syncthreads();
  }
  if (a.warp_bfs) {  // the warps' / groups' visited bitmaps start (and stay, between items) all zero
    uint32_t *v = reinterpret_cast<uint32_t *>(sh.tfl + a.tfl_bytes + (a.g_smem ? a.g_bytes : 0));
    const int nbm = a.warp_bfs == 2 ? kGroups : kWarps;
    for (int i = threadIdx.x; i < nbm * a.vis_words; i += kThreads) v[i] = 0u;
    __syncthreads();
  }
  // clusters (a.helper > 0): rank 0 replays the cells of the cluster, the other ranks help
  // with the projected-cost closures of every pressure event (CellT::cluster_helper).  ONE
  // call site of CellT::run, so that it is inlined and the cell's state stays in registers
  // (two call sites made it a real call: the whole CellT on the stack, every member access
  // a local load -- config 2 10.4 -> 13.4 ms)
  const int csize = a.helper + 1;
  int slot = (int)blockIdx.x, nslots = (int)gridDim.x;
  if (a.helper) {
    const int rank = (int)cooperative_groups::this_cluster().block_rank();
    slot = (int)blockIdx.x / csize;
    nslots = (int)gridDim.x / csize;
    if (rank != 0) {
      helper_entry(a, sh, slot, rank);
      return;
    }
  }
  for (int cell = slot; cell < a.n_cells; cell += nslots) {
    CellT<true> c(a, sh, cell, a.helper ? slot : -1);
    c.run(a.budgets[cell]);
    if (threadIdx.x == 0) a.out[cell] = sh.res;
    __syncthreads();
  }
  if (a.helper) {
    cooperative_groups::cluster_group cl = cooperative_groups::this_cluster();
    if (threadIdx.x == 0) sh.helper_cmd = 2;  // exit
    cl.sync();  // A
    cl.sync();  // the helpers have read the command
  }
}

}  // namespace
}  // namespace coop

// =============================================================================== host
using namespace coop;

struct coop_trace_s {
  int32_t T = 0, M = 0, n_params = 0;
  std::vector<uint64_t> size;
  std::vector<uint8_t> is_param, unevict;
  std::vector<int32_t> producer, out, src, in_ptr, in_idx, last_use, params;
  std::vector<int64_t> cost;
  std::vector<uint8_t> phase;
  std::vector<int32_t> cons_ptr, cons_idx, lock_ptr, lock_idx, die_ptr, die_idx;
  std::vector<int32_t> cons_head, cons_next, cons_out;  // the CSR as linked lists (device layout)
  std::vector<int32_t> rec;  // per tensor {cost lo, cost hi, in_beg, in_end} (device layout)
  std::vector<unsigned char> cg;  // the compact graph of the fast closure walk (cg_offsets), or empty
  int32_t cg_nnz = 0;
  void *dev = nullptr;
  TraceDev td{};
  unsigned char *ws = nullptr;
  size_t ws_cells = 0;
  WsLayout lay{};
  uint64_t *d_budgets = nullptr;
  size_t budgets_cap = 0;
  coop_replay_result *d_wave = nullptr;  // coop_budget_search's result buffer (grows on demand)
  size_t wave_cap = 0;
  // completion of the last replay launched on this handle: the next call's stream waits on
  // it before reusing the workspace and the budget buffer (calls on one handle serialise,
  // whatever streams they are issued on)
  cudaEvent_t done = nullptr;
  int device = 0;
};

namespace {

// independent validation (R19, R30) -- not shared with the oracle
int validate_and_prepare(coop_trace_s &t) {
  const int T = t.T, M = t.M;
  if (T < 1 || M < 0 || t.in_ptr[0] != 0) return COOP_ERR_INVALID_ARG;
  t.last_use.assign(T, -1);
  for (int i = 0; i < T; ++i) {
    if (t.size[i] < 1 || t.size[i] >= (1ull << 48)) return COOP_ERR_INVALID_ARG;
    if (t.is_param[i]) {
      if (t.producer[i] != -1) return COOP_ERR_INVALID_ARG;
    } else if (t.producer[i] < 0 || t.producer[i] >= M || t.out[t.producer[i]] != i) {
      return COOP_ERR_INVALID_ARG;
    }
  }
  for (int k = 0; k < M; ++k) {
    if (t.cost[k] < 0 || t.cost[k] >= (1ll << 40) || t.phase[k] > COOP_PHASE_UPD) return COOP_ERR_INVALID_ARG;
    const int o = t.out[k];
    if (o < 0 || o >= T || t.producer[o] != k || t.in_ptr[k + 1] < t.in_ptr[k]) return COOP_ERR_INVALID_ARG;
    bool seen = false;
    for (int j = t.in_ptr[k]; j < t.in_ptr[k + 1]; ++j) {
      const int u = t.in_idx[j];
      if (u < 0 || u >= T) return COOP_ERR_INVALID_ARG;
      if (!t.is_param[u] && t.producer[u] >= k) return COOP_ERR_INVALID_ARG;
      if (u == t.src[k]) seen = true;
      t.last_use[u] = k;
    }
    if (t.src[k] >= 0 && (t.src[k] >= T || !seen || t.size[t.src[k]] != t.size[o])) return COOP_ERR_INVALID_ARG;
  }
  for (int k = 0; k < M; ++k)
    if (t.src[k] >= 0 && t.last_use[t.src[k]] != k) return COOP_ERR_INVALID_ARG;
  for (int i = 0; i < T; ++i)
    if (t.last_use[i] < 0 && !t.is_param[i]) t.last_use[i] = t.producer[i];
  // unevictable: parameters and in-place results of unevictable inputs (R19)
  t.unevict.assign(T, 0);
  for (int i = 0; i < T; ++i) t.unevict[i] = t.is_param[i] ? 1 : 0;
  for (int k = 0; k < M; ++k)
    if (t.src[k] >= 0 && t.unevict[t.src[k]]) t.unevict[t.out[k]] = 1;
  t.params.clear();
  for (int i = 0; i < T; ++i)
    if (t.is_param[i]) t.params.push_back(i);
  t.n_params = (int32_t)t.params.size();
  // consumers (ops reading each tensor, in op order)
  t.cons_ptr.assign(T + 1, 0);
  for (int32_t u : t.in_idx) t.cons_ptr[u + 1]++;
  for (int i = 0; i < T; ++i) t.cons_ptr[i + 1] += t.cons_ptr[i];
  t.cons_idx.assign(t.in_idx.size(), 0);
  {
    std::vector<int32_t> fill(T, 0);
    for (int k = 0; k < M; ++k)
      for (int j = t.in_ptr[k]; j < t.in_ptr[k + 1]; ++j) {
        const int u = t.in_idx[j];
        t.cons_idx[t.cons_ptr[u] + fill[u]++] = k;
      }
  }
  t.cons_head.assign(T, -1);
  t.cons_next.assign(t.cons_idx.size(), -1);
  t.cons_out.assign(t.cons_idx.size(), 0);
  for (size_t e = 0; e < t.cons_idx.size(); ++e) t.cons_out[e] = t.out[t.cons_idx[e]];
  t.rec.assign((size_t)T * 4, 0);
  for (int i = 0; i < T; ++i) {
    const int p = t.producer[i];
    const uint64_t c = p >= 0 ? (uint64_t)t.cost[p] : 0ull;
    t.rec[(size_t)i * 4 + 0] = (int32_t)(uint32_t)c;
    t.rec[(size_t)i * 4 + 1] = (int32_t)(uint32_t)(c >> 32);
    t.rec[(size_t)i * 4 + 2] = p >= 0 ? t.in_ptr[p] : -1;
    t.rec[(size_t)i * 4 + 3] = p >= 0 ? t.in_ptr[p + 1] : -1;
  }
  for (int i = 0; i < T; ++i) {
    if (t.cons_ptr[i + 1] > t.cons_ptr[i]) t.cons_head[i] = t.cons_ptr[i];
    for (int j = t.cons_ptr[i]; j + 1 < t.cons_ptr[i + 1]; ++j) t.cons_next[j] = j + 1;
  }
  // deaths per op, ascending tensor id (R20): last use here, unless unevictable (except
  // the op's mutated input)
  t.die_ptr.assign(M + 1, 0);
  {
    std::vector<std::vector<int32_t>> d(M);
    for (int i = 0; i < T; ++i) {
      const int k = t.last_use[i];
      if (k < 0) continue;
      if (t.unevict[i] && t.src[k] != i) continue;
      d[k].push_back(i);
    }
    t.die_idx.clear();
    for (int k = 0; k < M; ++k) {
      t.die_idx.insert(t.die_idx.end(), d[k].begin(), d[k].end());
      t.die_ptr[k + 1] = (int32_t)t.die_idx.size();
    }
  }
  // R36 lock lists: need(t) = unevictable tensors read by t's recompute closure
  {
    std::vector<int32_t> uid(T, -1);
    int nu = 0;
    for (int i = 0; i < T; ++i)
      if (t.unevict[i]) uid[i] = nu++;
    const int words = std::max(1, (nu + 63) / 64);
    std::vector<uint64_t> need((size_t)T * words, 0);
    for (int k = 0; k < M; ++k) {
      uint64_t *no = &need[(size_t)t.out[k] * words];
      for (int j = t.in_ptr[k]; j < t.in_ptr[k + 1]; ++j) {
        const int u = t.in_idx[j];
        if (t.unevict[u]) no[uid[u] >> 6] |= 1ull << (uid[u] & 63);
        else {
          const uint64_t *nu_ = &need[(size_t)u * words];
          for (int x = 0; x < words; ++x) no[x] |= nu_[x];
        }
      }
    }
    t.lock_ptr.assign(M + 1, 0);
    t.lock_idx.clear();
    for (int k = 0; k < M; ++k) {
      const int s = t.src[k];
      if (s >= 0 && t.unevict[s]) {
        for (int i = 0; i < T; ++i) {
          if (t.unevict[i] || t.is_param[i] || t.producer[i] >= k || t.last_use[i] <= k) continue;
          if ((need[(size_t)i * words + (uid[s] >> 6)] >> (uid[s] & 63)) & 1ull) t.lock_idx.push_back(i);
        }
      }
      t.lock_ptr[k + 1] = (int32_t)t.lock_idx.size();
    }
  }
  // compact graph for the replay's fast closure walk (16-bit ids / offsets, 32-bit costs)
  {
    const int nnz = (int)t.in_idx.size();
    bool ok = T < 65535 && nnz < 65535;
    for (int k = 0; k < M && ok; ++k) ok = t.cost[k] < (1ll << 31);
    t.cg.clear();
    t.cg_nnz = 0;
    if (ok) {
      size_t off[6];
      cg_offsets(T, nnz, off);
      t.cg.assign(off[5], 0);
      int32_t *cost = reinterpret_cast<int32_t *>(t.cg.data() + off[0]);
      uint16_t *iptr = reinterpret_cast<uint16_t *>(t.cg.data() + off[1]);
      uint16_t *cptr = reinterpret_cast<uint16_t *>(t.cg.data() + off[2]);
      uint16_t *iidx = reinterpret_cast<uint16_t *>(t.cg.data() + off[3]);
      uint16_t *cout = reinterpret_cast<uint16_t *>(t.cg.data() + off[4]);
      int ni = 0;
      for (int x = 0; x < T; ++x) {
        const int p = t.producer[x];
        cost[x] = p >= 0 ? (int32_t)t.cost[p] : -1;
        iptr[x] = (uint16_t)ni;
        if (p >= 0)
          for (int j = t.in_ptr[p]; j < t.in_ptr[p + 1]; ++j) iidx[ni++] = (uint16_t)t.in_idx[j];
      }
      iptr[T] = (uint16_t)ni;
      int nc = 0;
      for (int x = 0; x < T; ++x) {
        cptr[x] = (uint16_t)nc;
        for (int j = t.cons_ptr[x]; j < t.cons_ptr[x + 1]; ++j) cout[nc++] = (uint16_t)t.out[t.cons_idx[j]];
      }
      cptr[T] = (uint16_t)nc;
      t.cg_nnz = nnz;
    }
  }
  return COOP_OK;
}

template <class V>
size_t put(std::vector<unsigned char> &blob, const V &v) {
  size_t off = (blob.size() + 15) / 16 * 16;
  const size_t bytes = v.size() * sizeof(typename V::value_type);
  blob.resize(off + bytes + 16);
  if (bytes) memcpy(blob.data() + off, v.data(), bytes);
  return off;
}


}  // namespace


// Device mirror of the preprocessed trace, uploaded on first use (so creation, validation
// and peak computation work without a GPU).
static int upload_trace(coop_trace_s *t) {
  if (t->dev) return COOP_OK;
  const int T = t->T, M = t->M;
  std::vector<unsigned char> blob;
  const size_t o_size = put(blob, t->size), o_prod = put(blob, t->producer), o_unev = put(blob, t->unevict),
               o_cost = put(blob, t->cost), o_out = put(blob, t->out), o_src = put(blob, t->src),
               o_phase = put(blob, t->phase), o_inp = put(blob, t->in_ptr), o_ini = put(blob, t->in_idx),
               o_cp = put(blob, t->cons_head), o_cn = put(blob, t->cons_next), o_ci = put(blob, t->cons_out), o_rec = put(blob, t->rec), o_lp = put(blob, t->lock_ptr),
               o_li = put(blob, t->lock_idx), o_dp = put(blob, t->die_ptr), o_di = put(blob, t->die_idx),
               o_par = put(blob, t->params), o_cg = put(blob, t->cg);
  cudaGetDevice(&t->device);
  if (cudaMalloc(&t->dev, blob.size()) != cudaSuccess) {
    t->dev = nullptr;
    return COOP_ERR_NOMEM;
  }
  if (cudaMemcpy(t->dev, blob.data(), blob.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaFree(t->dev);
    t->dev = nullptr;
    return COOP_ERR_CUDA;
  }
  unsigned char *b = (unsigned char *)t->dev;
  TraceDev &td = t->td;
  td.T = T;
  td.M = M;
  td.n_params = t->n_params;
  td.size = (const uint64_t *)(b + o_size);
  td.producer = (const int32_t *)(b + o_prod);
  td.unevict = (const uint8_t *)(b + o_unev);
  td.cost = (const int64_t *)(b + o_cost);
  td.out = (const int32_t *)(b + o_out);
  td.src = (const int32_t *)(b + o_src);
  td.phase = (const uint8_t *)(b + o_phase);
  td.in_ptr = (const int32_t *)(b + o_inp);
  td.in_idx = (const int32_t *)(b + o_ini);
  td.cons_head = (const int32_t *)(b + o_cp);
  td.cons_next = (const int32_t *)(b + o_cn);
  td.cons_out = (const int32_t *)(b + o_ci);
  td.rec = (const int4 *)(b + o_rec);
  td.cls = nullptr;
  td.lock_ptr = (const int32_t *)(b + o_lp);
  td.lock_idx = (const int32_t *)(b + o_li);
  td.die_ptr = (const int32_t *)(b + o_dp);
  td.die_idx = (const int32_t *)(b + o_di);
  td.params = (const int32_t *)(b + o_par);
  td.cg_nnz = t->cg_nnz;
  td.cg_cost = t->cg.empty() ? nullptr : (const int32_t *)(b + o_cg);
  td.cg_iptr = td.cg_cptr = td.cg_iidx = td.cg_cout = nullptr;  // carved from cg_cost by cg_offsets
  return COOP_OK;
}

extern "C" int coop_trace_create(const coop_trace_desc *d, coop_trace_t *out) {
  if (!d || !out || d->n_tensors < 1 || d->n_ops < 0 || !d->size || !d->is_param || !d->producer ||
      (d->n_ops > 0 && (!d->cost_us || !d->out || !d->inplace_src || !d->phase || !d->in_ptr)))
    return COOP_ERR_INVALID_ARG;
  coop_trace_s *t = new (std::nothrow) coop_trace_s();
  if (!t) return COOP_ERR_NOMEM;
  const int T = d->n_tensors, M = d->n_ops;
  t->T = T;
  t->M = M;
  t->size.assign(d->size, d->size + T);
  t->is_param.assign(d->is_param, d->is_param + T);
  t->producer.assign(d->producer, d->producer + T);
  t->cost.assign(d->cost_us, d->cost_us + M);
  t->out.assign(d->out, d->out + M);
  t->src.assign(d->inplace_src, d->inplace_src + M);
  t->phase.assign(d->phase, d->phase + M);
  t->in_ptr.assign(d->in_ptr, d->in_ptr + M + 1);
  if (M == 0) t->in_ptr.assign(1, 0);
  const int nnz = t->in_ptr[M];
  if (nnz < 0 || (nnz > 0 && !d->in_idx)) {
    delete t;
    return COOP_ERR_INVALID_ARG;
  }
  t->in_idx.assign(d->in_idx, d->in_idx + nnz);
  int rc = validate_and_prepare(*t);
  if (rc != COOP_OK) {
    delete t;
    return rc;
  }
  t->lay = make_layout(T);
  *out = t;
  return COOP_OK;
}

extern "C" int coop_trace_destroy(coop_trace_t t) {
  if (!t) return COOP_ERR_INVALID_ARG;
  if (t->dev) {
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != t->device) cudaSetDevice(t->device);
    if (t->done) cudaEventSynchronize(t->done);
    cudaFree(t->dev);
    if (t->ws) cudaFree(t->ws);
    if (t->d_budgets) cudaFree(t->d_budgets);
    if (t->d_wave) cudaFree(t->d_wave);
    if (t->done) cudaEventDestroy(t->done);
    if (prev != t->device) cudaSetDevice(prev);
  }
  delete t;
  return COOP_OK;
}

// Peak resident bytes without eviction (R25): host-side sweep of the liveness intervals.
extern "C" int coop_trace_peak_live(coop_trace_t t, uint32_t flags, uint64_t *out) {
  if (!t || !out) return COOP_ERR_INVALID_ARG;
  uint64_t live = 0, peak = 0;
  for (int i = 0; i < t->T; ++i)
    if (t->is_param[i]) live += t->size[i];
  peak = live;
  for (int k = 0; k < t->M; ++k) {
    const int s = t->src[k];
    const bool inplace = s >= 0 && (flags & COOP_F_INPLACE);
    if (!inplace) live += t->size[t->out[k]];
    peak = std::max(peak, live);
    for (int j = t->die_ptr[k]; j < t->die_ptr[k + 1]; ++j) {
      const int i = t->die_idx[j];
      if (inplace && i == s) continue;  // its bytes now belong to the output
      live -= t->size[i];
    }
  }
  *out = peak;
  return COOP_OK;
}

static int64_t *coop__last_phase_buf = nullptr;
// test / profiling hook (not part of the ABI): copy the last replay's phase times (8 per cell)
extern "C" int coop__replay_phase_ns(int64_t *host, int32_t n_cells) {
  if (!coop__last_phase_buf) return COOP_ERR_INVALID_ARG;
  return cudaMemcpy(host, coop__last_phase_buf, (size_t)n_cells * 64, cudaMemcpyDeviceToHost) == cudaSuccess
             ? COOP_OK : COOP_ERR_CUDA;
}

struct SnapSink {
  uint64_t *ss;
  double *c, *s;
  uint64_t *req;
  coop_window *win;
  int64_t *count;
  int64_t cap;
  int32_t n;
};

static int replay_on_device(coop_trace_t t, const uint64_t *budgets, int32_t n_budgets, uint32_t flags,
                            uint32_t class_threshold, int32_t max_depth, coop_replay_result *out,
                            coop_event *log, int64_t log_cap, cudaStream_t st, const SnapSink *snap = nullptr);

extern "C" int coop_replay_trace(coop_trace_t t, const uint64_t *budgets, int32_t n_budgets,
                                 uint32_t flags, uint32_t class_threshold, int32_t max_depth,
                                 coop_replay_result *out, coop_event *log, int64_t log_cap,
                                 coop_stream_t stream) {
  if (!t || n_budgets < 0 || (n_budgets > 0 && (!budgets || !out)) || log_cap < 0 ||
      bad_flags(flags) || max_depth > 1024)
    return COOP_ERR_INVALID_ARG;
  if (n_budgets == 0) return COOP_OK;
  for (int i = 0; i < n_budgets; ++i)
    if (budgets[i] < 1) return COOP_ERR_INVALID_ARG;
  if (!is_device_ptr(out) || (log && !is_device_ptr(log))) return COOP_ERR_INVALID_ARG;
  if (t->T > kMaxT) return COOP_ERR_NOMEM;  // per-tensor flags / pins live in shared memory
  int prev = 0;
  cudaGetDevice(&prev);
  if (t->dev && prev != t->device) cudaSetDevice(t->device);  // launch where the mirror lives
  const int rc = replay_on_device(t, budgets, n_budgets, flags, class_threshold, max_depth, out, log,
                                  log_cap, (cudaStream_t)stream);
  if (prev != t->device) cudaSetDevice(prev);
  return rc;
}

static int replay_on_device(coop_trace_t t, const uint64_t *budgets, int32_t n_budgets, uint32_t flags,
                            uint32_t class_threshold, int32_t max_depth, coop_replay_result *out,
                            coop_event *log, int64_t log_cap, cudaStream_t st, const SnapSink *snap) {
  const int up = upload_trace(t);
  if (up != COOP_OK) return up;
  if (!t->done && cudaEventCreateWithFlags(&t->done, cudaEventDisableTiming) != cudaSuccess) return COOP_ERR_CUDA;
  // the previous call on this handle (possibly on another stream) still owns ws / d_budgets
  if (cudaStreamWaitEvent(st, t->done, 0) != cudaSuccess) return COOP_ERR_CUDA;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, t->device);
  // dynamic shared memory: Shared, the tensor flags, then (fast closure walk) the compact
  // graph if it fits and as many walker bitmaps as fit (at least 32, at most kThreads)
  int max_smem = 0;
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, t->device);
  const int tfl_bytes = (t->T + 15) / 16 * 16;
  const int vis_words = (t->T + 127) / 128 * 4;
  const size_t base = sizeof(Shared) + (size_t)tfl_bytes;
  int g_smem = 0, walkers = 0, warp_bfs = 0;
  const int g_bytes = (int)t->cg.size();
  // profiling hooks: COOP_REPLAY_WALK = "generic" (round 1's per-thread walk over the global
  // graph), "lane" (per-thread walkers with shared-memory bitmaps), "warp" (one closure per
  // warp, edge-parallel BFS); COOP_REPLAY_GSMEM=0 keeps the compact graph in global memory.
  // Default: per-thread walkers when at least 128 of them fit, else the warp BFS (large T:
  // few bitmaps fit, and those traces -- BiLSTM, GPT-3 -- have long closures).
  const char *wenv = getenv("COOP_REPLAY_WALK");
  const char *genv = getenv("COOP_REPLAY_GSMEM");
  const bool gsm_ok = !(genv && genv[0] == '0');
  const size_t warp_extra = (size_t)kWarps * ((size_t)vis_words * 4 + (size_t)kRing * 2);
  const size_t group_extra = (size_t)kGroups * ((size_t)vis_words * 4 + (size_t)kGRing * 2);
  if (!t->cg.empty() && !(wenv && wenv[0] == 'g')) {
    const size_t per = (size_t)vis_words * 4;  // one visited bitmap per walker
    if (gsm_ok && base + (size_t)g_bytes + 32 * per <= (size_t)max_smem) {
      g_smem = 1;
      walkers = (int)std::min<size_t>(kThreads, ((size_t)max_smem - base - g_bytes) / per);
    } else if (base + 32 * per <= (size_t)max_smem) {
      walkers = (int)std::min<size_t>(kThreads, ((size_t)max_smem - base) / per);
    }
    walkers = walkers / 32 * 32;  // whole warps
    const bool want_group = wenv && wenv[0] == 'G';
    const bool want_warp = wenv ? wenv[0] == 'w' : walkers < 128;
    if (want_group) {
      const int gs = gsm_ok && base + (size_t)g_bytes + group_extra <= (size_t)max_smem;
      if (gs || base + group_extra <= (size_t)max_smem) {
        g_smem = gs;
        walkers = kThreads;
        warp_bfs = 2;
      }
    }
    if (want_warp) {
      const int gs = gsm_ok && base + (size_t)g_bytes + warp_extra <= (size_t)max_smem;
      if (gs || base + warp_extra <= (size_t)max_smem) {
        g_smem = gs;
        walkers = kThreads;
        warp_bfs = 1;
      }
    }
  }
  const size_t smem = base + (g_smem ? (size_t)g_bytes : 0) +
                      (warp_bfs == 2 ? group_extra : warp_bfs ? warp_extra : (size_t)walkers * vis_words * 4);
  if (cudaFuncSetAttribute(replay_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return COOP_ERR_CUDA;
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, replay_kernel, kThreads, smem);
  if (per_sm < 1) per_sm = 1;
  // cluster helpers: more SMs walking the closures of each cell (COOP_REPLAY_HELPER=0..3
  // overrides the default below)
  int helper = 0;
  if (walkers > 0) {
    const char *henv = getenv("COOP_REPLAY_HELPER");
    // helpers per cell, 0..7.  Default (measured on B200): none for traces below 4096
    // tensors (their closures are short: ResNet-50 loses more to the per-event cluster
    // barriers than it gains); for larger traces 1 when the cells fill a quarter to half of
    // the SMs (all of them then still run at once: config 3, 64 GPT-3 cells on 128 SMs), else
    // 7 (a sweep's time is its slowest cell: the BiLSTM 256-cell sweep 50 -> 31 / 23 / 20 /
    // 18.5 / 18.1 s with 1 / 2 / 3 / 5 / 7 helpers; a GPT-3 256-cell sweep alone pays for the
    // extra waves, 446 -> 733 ms, hidden under BiLSTM in config 5)
    if (henv) helper = std::max(0, std::min(kMaxCluster - 1, atoi(henv)));
    else if (t->T >= 4096)
      helper = ((int64_t)n_budgets * 4 > (int64_t)sms && (int64_t)n_budgets * 2 <= (int64_t)sms) ? 1 : 7;
  }
  int max_clusters = 0;
  if (helper) {
    cudaLaunchConfig_t qc = {};
    cudaLaunchAttribute qa[1];
    qa[0].id = cudaLaunchAttributeClusterDimension;
    qa[0].val.clusterDim.x = (unsigned)(helper + 1);
    qa[0].val.clusterDim.y = 1;
    qa[0].val.clusterDim.z = 1;
    qc.gridDim = dim3((unsigned)(helper + 1) * (unsigned)(sms / (helper + 1)), 1, 1);
    qc.blockDim = dim3(kThreads, 1, 1);
    qc.dynamicSmemBytes = smem;
    qc.attrs = qa;
    qc.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&max_clusters, replay_kernel, &qc) != cudaSuccess || max_clusters < 1) {
      cudaGetLastError();
      helper = 0;
    }
  }
  // concurrent cells = min(n_budgets, resident CTAs or clusters); the workspace holds that many
  const size_t cells = (size_t)std::min<int64_t>(n_budgets, helper ? (int64_t)max_clusters : (int64_t)sms * per_sm);
  if (cells > t->ws_cells) {
    if (t->ws) cudaFree(t->ws);
    t->ws = nullptr;
    t->ws_cells = 0;
    if (cudaMalloc(&t->ws, cells * t->lay.bytes) != cudaSuccess) return COOP_ERR_NOMEM;
    // DFS epochs start at 0; ordered before the kernel on the launch stream
    if (cudaMemsetAsync(t->ws, 0, cells * t->lay.bytes, st) != cudaSuccess) return COOP_ERR_CUDA;
    t->ws_cells = cells;
  }
  if ((size_t)n_budgets > t->budgets_cap) {
    if (t->d_budgets) cudaFree(t->d_budgets);
    if (cudaMalloc(&t->d_budgets, (size_t)n_budgets * 8) != cudaSuccess) return COOP_ERR_NOMEM;
    t->budgets_cap = (size_t)n_budgets;
  }
  cudaMemcpyAsync(t->d_budgets, budgets, (size_t)n_budgets * 8, cudaMemcpyHostToDevice, st);
  KArgs a{};
  a.tr = t->td;
  a.budgets = t->d_budgets;
  a.flags = flags;
  a.thr = class_threshold ? class_threshold : 15;
  a.max_depth = max_depth > 0 ? max_depth : 512;
  a.n_cells = n_budgets;
  a.out = out;
  a.log = log;
  a.log_cap = log ? log_cap : 0;
  a.ws = t->ws;
  a.lay = t->lay;
  a.tfl_bytes = tfl_bytes;
  a.g_smem = g_smem;
  a.g_bytes = g_bytes;
  a.walkers = walkers;
  a.warp_bfs = warp_bfs;
  a.vis_words = vis_words;
  {  // profiling hook: COOP_REPLAY_PHASES=1 accumulates per-phase pressure-event times per cell
    static int64_t *pbuf = nullptr;
    static size_t pcap = 0;
    const char *pe = getenv("COOP_REPLAY_PHASES");
    if (pe && pe[0] == '1') {
      if ((size_t)n_budgets * 8 > pcap) {
        if (pbuf) cudaFree(pbuf);
        pcap = (size_t)n_budgets * 8;
        if (cudaMalloc(&pbuf, pcap * 8) != cudaSuccess) return COOP_ERR_NOMEM;
      }
      cudaMemsetAsync(pbuf, 0, (size_t)n_budgets * 64, st);
      a.phase_ns = pbuf;
      coop__last_phase_buf = pbuf;
    }
  }
  if (snap) {
    if (cudaMemsetAsync(snap->count, 0, sizeof(int64_t), st) != cudaSuccess) return COOP_ERR_CUDA;
    a.snap_ss = snap->ss;
    a.snap_c = snap->c;
    a.snap_s = snap->s;
    a.snap_req = snap->req;
    a.snap_win = snap->win;
    a.snap_count = snap->count;
    a.snap_cap = snap->cap;
    a.snap_n = snap->n;
  }
  // each CTA (cluster) owns a workspace slot: cells are assigned cyclically, slot b takes
  // cells b, b + slots, ...
  a.helper = helper;
  if (helper) {
    cudaLaunchConfig_t lc = {};
    cudaLaunchAttribute la[1];
    la[0].id = cudaLaunchAttributeClusterDimension;
    la[0].val.clusterDim.x = (unsigned)(helper + 1);
    la[0].val.clusterDim.y = 1;
    la[0].val.clusterDim.z = 1;
    lc.gridDim = dim3((unsigned)(helper + 1) * (unsigned)cells, 1, 1);
    lc.blockDim = dim3(kThreads, 1, 1);
    lc.dynamicSmemBytes = smem;
    lc.stream = st;
    lc.attrs = la;
    lc.numAttrs = 1;
    if (cudaLaunchKernelEx(&lc, replay_kernel, a) != cudaSuccess) return COOP_ERR_CUDA;
  } else {
    replay_kernel<<<(unsigned)cells, kThreads, smem, st>>>(a);
  }
  if (cudaGetLastError() != cudaSuccess) return COOP_ERR_CUDA;
  return cudaEventRecord(t->done, st) == cudaSuccess ? COOP_OK : COOP_ERR_CUDA;
}

extern "C" int coop_replay_snapshots(coop_trace_t t, uint64_t budget, uint32_t flags, uint32_t class_threshold,
                                     int32_t max_depth, int32_t n_max, int64_t cap, uint64_t *size_state,
                                     double *cost, double *stale, uint64_t *requests, coop_window *windows,
                                     int64_t *count, coop_replay_result *out, coop_stream_t stream) {
  if (!t || budget < 1 || bad_flags(flags) || (flags & (COOP_F_POLICY_DTR | COOP_F_POLICY_DTE)) ||
      max_depth > 1024 || n_max < 1 || n_max > COOP_MAX_BLOCKS || cap < 0 || !out || !count)
    return COOP_ERR_INVALID_ARG;
  if (cap > 0 && (!size_state || !cost || !stale || !requests || !windows)) return COOP_ERR_INVALID_ARG;
  if (!is_device_ptr(out) || !is_device_ptr(count) ||
      (cap > 0 && (!is_device_ptr(size_state) || !is_device_ptr(cost) || !is_device_ptr(stale) ||
                   !is_device_ptr(requests) || !is_device_ptr(windows))))
    return COOP_ERR_INVALID_ARG;
  if (t->T > kMaxT) return COOP_ERR_NOMEM;
  SnapSink snap{size_state, cost, stale, requests, windows, count, cap, n_max};
  int prev = 0;
  cudaGetDevice(&prev);
  if (t->dev && prev != t->device) cudaSetDevice(t->device);
  const int rc = replay_on_device(t, &budget, 1, flags, class_threshold, max_depth, out, nullptr, 0,
                                  (cudaStream_t)stream, &snap);
  if (prev != t->device) cudaSetDevice(prev);
  return rc;
}

// ------------------------------------------------------------------ budget searches (R45)
namespace {

uint64_t grid_budget(uint64_t lo, uint64_t hi, int64_t j, int64_t steps) {
  const unsigned __int128 d = (unsigned __int128)(hi - lo) * (unsigned __int128)j / (unsigned __int128)steps;
  const uint64_t b = lo + (uint64_t)d;
  return b < 1 ? 1 : b;
}

// one wave of replays on the default stream; results copied to the host
int run_wave(coop_trace_t t, const std::vector<uint64_t> &budgets, uint32_t flags, uint32_t thr,
             int32_t depth, std::vector<coop_replay_result> &res) {
  res.assign(budgets.size(), coop_replay_result{});
  if (budgets.empty()) return COOP_OK;
  if (budgets.size() > t->wave_cap) {  // grows once per handle, not per wave
    if (t->d_wave) cudaFree(t->d_wave);
    t->d_wave = nullptr;
    t->wave_cap = 0;
    if (cudaMalloc(&t->d_wave, budgets.size() * sizeof(coop_replay_result)) != cudaSuccess) return COOP_ERR_NOMEM;
    t->wave_cap = budgets.size();
  }
  int rc = coop_replay_trace(t, budgets.data(), (int32_t)budgets.size(), flags, thr, depth, t->d_wave, nullptr, 0,
                             nullptr);
  if (rc == COOP_OK &&
      cudaMemcpy(res.data(), t->d_wave, budgets.size() * sizeof(coop_replay_result), cudaMemcpyDeviceToHost) !=
          cudaSuccess)
    rc = COOP_ERR_CUDA;
  return rc;
}

bool meets(const coop_replay_result &r, int metric) {  // 0: completes, 1: completes without eviction
  return r.status == COOP_OK && (metric == 0 || r.evictions == 0);
}

}  // namespace

extern "C" int coop_budget_search(coop_trace_t t, uint32_t flags, uint32_t thr, int32_t depth,
                                  int32_t kc, int32_t kf, coop_budget_result *out) {
  if (!t || !out || kc < 1 || kc > 4096 || kf < 1 || kf > 4096 || bad_flags(flags) || depth > 1024)
    return COOP_ERR_INVALID_ARG;
  uint64_t peak = 0;
  int rc = coop_trace_peak_live(t, flags, &peak);
  if (rc != COOP_OK) return rc;
  coop_budget_result r{};
  r.peak = peak;
  // Z = the bytes of every tensor: a pool that large never evicts (R45)
  uint64_t zsum = 0;
  for (int i = 0; i < t->T; ++i) zsum += t->size[i];
  if (zsum < peak) zsum = peak;
  // coarse waves on the brackets (0, P], (P, 2P], ... until every metric has a satisfying
  // grid point or the bracket reaches Z; both metrics share a bracket's wave
  uint64_t blo = 0, bhi = peak > 0 ? peak : 1;
  uint64_t mlo[2] = {0, 0}, mhi[2] = {0, 0};
  int kstar[2] = {-1, -1};
  std::vector<uint64_t> coarse((size_t)kc);
  std::vector<coop_replay_result> cres;
  for (;;) {
    for (int k = 1; k <= kc; ++k) coarse[(size_t)k - 1] = grid_budget(blo, bhi, k, kc);
    rc = run_wave(t, coarse, flags, thr, depth, cres);
    if (rc != COOP_OK) return rc;
    r.replays += kc;
    for (int m = 0; m < 2; ++m) {
      if (kstar[m] >= 0) continue;
      for (int k = 0; k < kc && kstar[m] < 0; ++k)
        if (meets(cres[(size_t)k], m)) {
          kstar[m] = k + 1;
          mlo[m] = blo;
          mhi[m] = bhi;
        }
    }
    if ((kstar[0] >= 0 && kstar[1] >= 0) || bhi >= zsum) break;
    blo = bhi;
    bhi = bhi > (UINT64_MAX >> 1) ? UINT64_MAX : 2 * bhi;
  }
  // both metrics' fine grids inside (B_{k*-1}, B_{k*}] of their brackets, in one wave
  std::vector<uint64_t> fine;
  uint64_t flo[2] = {0, 0}, fhi[2] = {0, 0};
  for (int m = 0; m < 2; ++m) {
    if (kstar[m] < 0) continue;
    flo[m] = kstar[m] > 1 ? grid_budget(mlo[m], mhi[m], kstar[m] - 1, kc) : mlo[m];
    fhi[m] = grid_budget(mlo[m], mhi[m], kstar[m], kc);
    for (int j = 1; j <= kf; ++j) fine.push_back(grid_budget(flo[m], fhi[m], j, kf));
  }
  std::vector<coop_replay_result> fres;
  rc = run_wave(t, fine, flags, thr, depth, fres);
  if (rc != COOP_OK) return rc;
  r.replays += (int32_t)fine.size();
  size_t base = 0;
  for (int m = 0; m < 2; ++m) {
    uint64_t *dst = m == 0 ? &r.min_budget : &r.cutoff_budget;
    int32_t *st = m == 0 ? &r.min_status : &r.cutoff_status;
    if (kstar[m] < 0) {
      *dst = 0;
      *st = COOP_INFEASIBLE;
      continue;
    }
    *st = COOP_OK;
    *dst = fhi[m];
    for (int j = 0; j < kf; ++j)
      if (meets(fres[base + (size_t)j], m)) {
        *dst = fine[base + (size_t)j];
        break;
      }
    base += (size_t)kf;
  }
  *out = r;
  return COOP_OK;
}
