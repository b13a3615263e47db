/*
 * oracle_replay.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * O2: replay of an allocation trace under one memory budget with Coop's allocator,
 * written step by step in the paper's order:
 *   Alg. 1 Allocate(op, size)
 *   sliding-window eviction, h = c/s    PAPER.md:141-153 (Sec. 3.3) -> orc_window_search
 *   cheap tensor partitioning           PAPER.md:157-173 (Sec. 3.4), Table 1 (185-187)
 *   recomputable in-place, parameters at the two pool ends    PAPER.md:206-222 (Sec. 3.5)
 *   conventional allocator (first fit, coalescing free list)  PAPER.md:65-67 (Sec. 2.1)
 *   rematerialization on demand
 * with the readings R10-R35 of DESIGN.md where the paper is silent.  Plain data
 * structures: a sorted array of blocks scanned linearly, recursion for
 * rematerialization, a DFS with visited marks for projected costs.  Slow and simple.
 */
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

#define NO_OWNER (-1)

typedef struct {
  uint64_t addr, size;
  int32_t owner; /* tensor id, NO_OWNER = free */
} blk;

typedef struct {
  const orc_trace *tr;
  orc_cfg cfg;
  blk *b;
  int nb, cap;
  uint64_t bytes_free;
  /* tensor state */
  uint8_t *born, *resident, *dead, *unevict;
  int32_t *pins, *last_use;
  int64_t *last_access;
  uint64_t *addr;
  int32_t *cons_ptr, *cons_idx; /* ops reading each tensor */
  int32_t *lock_ptr, *lock_idx; /* per op: live tensors that need the replaced value (R36) */
  uint8_t *locked;
  uint32_t *mark;
  uint32_t epoch;
  int32_t *stack;
  /* search scratch */
  uint64_t *v_ss;
  double *v_c, *v_s;
  int64_t clock;
  int32_t cur_op;
  orc_replay_result *res;
  orc_event *log;
  int64_t log_cap;
  int status;
  /* O3 (online calls) only */
  const uint8_t *cls;       /* per op: 0 = class by threshold, 1 = C1, 2 = C2; NULL = all 0 */
  int32_t win_first, win_last, nvict;
  uint64_t win_span;
  double win_cost;
  int32_t *victims;         /* the last window's tensors, ascending address; NULL = off */
} R;

static uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static void log_ev(R *r, int kind, int op, int tensor, uint64_t addr) {
  int64_t i = r->res->n_events++;
  if (r->log && i < r->log_cap) {
    r->log[i].kind = kind;
    r->log[i].op = op;
    r->log[i].tensor = tensor;
    r->log[i].pad = 0;
    r->log[i].addr = addr;
  }
}

/* ------------------------------------------------------------------ the pool (Sec. 2.1) */
static int find_block_of(R *r, int32_t t) {
  for (int i = 0; i < r->nb; ++i)
    if (r->b[i].owner == t) return i;
  return -1;
}

/* lowest-addressed (right = 0) or highest-addressed (right = 1) free block >= size (R12) */
static int find_fit(R *r, uint64_t size, int right) {
  int found = -1;
  for (int i = 0; i < r->nb; ++i) {
    if (r->b[i].owner == NO_OWNER && r->b[i].size >= size) {
      found = i;
      if (!right) break;
    }
  }
  return found;
}

static void insert_blk(R *r, int at, blk v) {
  if (r->nb == r->cap) {
    r->cap *= 2;
    r->b = (blk *)realloc(r->b, sizeof(blk) * (size_t)r->cap);
  }
  memmove(&r->b[at + 1], &r->b[at], sizeof(blk) * (size_t)(r->nb - at));
  r->b[at] = v;
  r->nb++;
  if (r->nb > r->res->max_blocks) r->res->max_blocks = r->nb;
}

static void erase_blk(R *r, int at) {
  memmove(&r->b[at], &r->b[at + 1], sizeof(blk) * (size_t)(r->nb - at - 1));
  r->nb--;
}

/* place `size` bytes for tensor t in free block i: "leftmost side of a free chunk"
 * (Alg. 1 block.left_addr) or block.right_addr - size (Alg. 1). */
static uint64_t place(R *r, int i, uint64_t size, int right, int32_t t) {
  blk f = r->b[i];
  uint64_t a;
  if (f.size == size) {
    r->b[i].owner = t;
    a = f.addr;
  } else if (!right) {
    blk live = {f.addr, size, t};
    r->b[i].addr = f.addr + size;
    r->b[i].size = f.size - size;
    insert_blk(r, i, live);
    a = f.addr;
  } else {
    blk live = {f.addr + f.size - size, size, t};
    r->b[i].size = f.size - size;
    insert_blk(r, i + 1, live);
    a = live.addr;
  }
  r->bytes_free -= size;
  return a;
}

/* free block i and merge with free neighbours ("merged with other chunks with adjacent
 * memory addresses") */
static void release(R *r, int i) {
  r->b[i].owner = NO_OWNER;
  r->bytes_free += r->b[i].size;
  if (i + 1 < r->nb && r->b[i + 1].owner == NO_OWNER) {
    r->b[i].size += r->b[i + 1].size;
    erase_blk(r, i + 1);
  }
  if (i > 0 && r->b[i - 1].owner == NO_OWNER) {
    r->b[i - 1].size += r->b[i].size;
    erase_blk(r, i);
  }
}

static int n_free_blocks(R *r) {
  int k = 0;
  for (int i = 0; i < r->nb; ++i) k += (r->b[i].owner == NO_OWNER);
  return k;
}

/* ------------------------------------------------------------------ trace helpers */
static int32_t n_in(const orc_trace *tr, int op) { return tr->in_ptr[op + 1] - tr->in_ptr[op]; }
static int32_t in_at(const orc_trace *tr, int op, int k) { return tr->in_idx[tr->in_ptr[op] + k]; }

/* C1 ("expensive", super-linear) iff cost density >= threshold us/MiB (R14, Table 1) */
static int is_c1(R *r, int op) {
  if (r->cls && r->cls[op]) return r->cls[op] == 1; /* O3: class given by the caller */
  uint64_t bytes = r->tr->size[r->tr->out[op]];
  return (uint64_t)r->tr->cost_us[op] * 1048576ull >= (uint64_t)r->cfg.class_threshold * bytes;
}

/* cheap tensors go to the right end during forward propagation (R12-R13) */
static int goes_right(R *r, int op) {
  if (!(r->cfg.flags & ORC_F_PARTITION)) return 0;
  int ph = r->tr->phase[op];
  if (ph != ORC_PHASE_FWD && !(r->cfg.flags & ORC_F_PARTITION_ALL_PHASES)) return 0;
  return !is_c1(r, op);
}

/* ------------------------------------------------------------------ projected cost */
/* c(t) = cost of t's producer + its evicted neighbourhood (R18):
 * the SET of non-resident ancestors reachable through non-resident tensors, plus the
 * SET of evicted (not dead) descendants reachable through evicted tensors. */
static int64_t projected_cost(R *r, int32_t t) {
  const orc_trace *tr = r->tr;
  int64_t c = tr->cost_us[tr->producer[t]];
  r->epoch++;
  r->mark[t] = r->epoch;
  int sp = 0;
  int op = tr->producer[t];
  for (int k = 0; k < n_in(tr, op); ++k) r->stack[sp++] = in_at(tr, op, k);
  while (sp > 0) {
    int32_t u = r->stack[--sp];
    if (r->mark[u] == r->epoch) continue;
    r->mark[u] = r->epoch;
    if (r->resident[u] || tr->producer[u] < 0) continue;
    c += tr->cost_us[tr->producer[u]];
    int pu = tr->producer[u];
    for (int k = 0; k < n_in(tr, pu); ++k) r->stack[sp++] = in_at(tr, pu, k);
  }
  for (int k = r->cons_ptr[t]; k < r->cons_ptr[t + 1]; ++k) r->stack[sp++] = tr->out[r->cons_idx[k]];
  while (sp > 0) {
    int32_t d = r->stack[--sp];
    if (r->mark[d] == r->epoch) continue;
    r->mark[d] = r->epoch;
    if (!r->born[d] || r->resident[d] || r->dead[d]) continue; /* only evicted tensors */
    c += tr->cost_us[tr->producer[d]];
    for (int k = r->cons_ptr[d]; k < r->cons_ptr[d + 1]; ++k) r->stack[sp++] = tr->out[r->cons_idx[k]];
  }
  return c;
}

/* ------------------------------------------------------------------ eviction */
static void evict(R *r, int32_t t) {
  int i = find_block_of(r, t);
  uint64_t a = r->b[i].addr;
  release(r, i);
  r->resident[t] = 0;
  r->res->evictions++;
  log_ev(r, ORC_EV_EVICT, r->cur_op, t, a);
  uint64_t d = r->res->digest; /* R29 */
  d = splitmix64(d ^ (((uint64_t)(uint32_t)r->cur_op << 32) | (uint32_t)t));
  d = splitmix64(d ^ a);
  r->res->digest = d;
}

/* The baselines the paper compares against (R46):
 * repeat { h(t) for every resident evictable tensor -- DTR: c / (m s); DTE: c / ((m + the
 * free bytes adjacent to t's block) s) -- and evict the argmin (ties: lowest address) }
 * until some free block can hold `size` ("This process runs several times until the
 * released memory is sufficient for the new tensor"). */
static int evict_loop(R *r, uint64_t size) {
  int dte = (r->cfg.flags & ORC_F_DTE) != 0;
  r->win_first = r->win_last = -1;
  r->win_span = 0;
  r->win_cost = 0.0;
  r->nvict = 0;
  while (find_fit(r, size, 0) < 0) {
    int best = -1;
    double bh = 0.0;
    for (int i = 0; i < r->nb; ++i) {
      int32_t o = r->b[i].owner;
      if (o == NO_OWNER || r->unevict[o] || r->pins[o] > 0 || r->locked[o]) continue;
      int64_t s = r->clock - r->last_access[o]; /* staleness (R17) */
      if (s < 1) s = 1;
      uint64_t m = r->b[i].size;
      if (dte) {
        if (i > 0 && r->b[i - 1].owner == NO_OWNER) m += r->b[i - 1].size;
        if (i + 1 < r->nb && r->b[i + 1].owner == NO_OWNER) m += r->b[i + 1].size;
      }
      double h = (double)projected_cost(r, o) / ((double)m * (double)s);
      r->res->heuristic_evals++;
      if (best < 0 || h < bh) {
        best = i;
        bh = h;
      }
    }
    if (best < 0) {
      r->status = ORC_UNSATISFIABLE; /* nothing left to evict */
      return -1;
    }
    int32_t v = r->b[best].owner;
    if (r->victims && r->nvict < 8192) r->victims[r->nvict] = v;
    r->nvict++;
    evict(r, v);
  }
  return 0;
}

/* sliding-window search over the address-ordered item list and eviction of the window
 * (Alg. 1 line "evict(sliding_window_search(size))"); returns 0 on success. */
static int evict_window(R *r, uint64_t size) {
  const orc_trace *tr = r->tr;
  if (r->cfg.flags & (ORC_F_DTR | ORC_F_DTE)) return evict_loop(r, size);
  int n = r->nb;
  if (n > 8192) {
    r->status = ORC_UNSATISFIABLE; /* beyond the search domain (R7) */
    return -1;
  }
  for (int i = 0; i < n; ++i) {
    int32_t o = r->b[i].owner;
    uint64_t st;
    r->v_c[i] = 0.0;
    r->v_s[i] = 1.0;
    if (o == NO_OWNER) {
      st = ORC_FREE; /* free chunk: a special tensor with h = 0 */
    } else if (r->unevict[o] || r->pins[o] > 0 || r->locked[o]) {
      st = ORC_PINNED; /* unevictable / in use (R16) */
    } else {
      st = ORC_EVICTABLE;
      int64_t s = r->clock - r->last_access[o]; /* staleness (R17) */
      if (s < 1) s = 1;
      r->v_c[i] = (double)projected_cost(r, o);
      r->v_s[i] = (double)s;
      r->res->heuristic_evals++;
    }
    (void)tr;
    r->v_ss[i] = r->b[i].size | (st << 62);
  }
  orc_window w;
  orc_window_search(n, r->v_ss, r->v_c, r->v_s, size, &w);
  if (w.status != ORC_OK) {
    r->status = ORC_UNSATISFIABLE; /* R24 */
    return -1;
  }
  /* evict the window's tensors in ascending address order (R10) */
  int32_t victims[8192];
  int nv = 0;
  for (int i = w.first; i <= w.last; ++i)
    if (r->b[i].owner != NO_OWNER) victims[nv++] = r->b[i].owner;
  r->win_first = w.first;
  r->win_last = w.last;
  r->win_span = w.span;
  r->win_cost = w.cost;
  r->nvict = nv;
  if (r->victims)
    for (int k = 0; k < nv; ++k) r->victims[k] = victims[k];
  for (int k = 0; k < nv; ++k) evict(r, victims[k]);
  return 0;
}

/* Alg. 1 Allocate(op, size) for tensor t.  allow_inplace: original
 * execution of an in-place op with recomputable in-place on (R19); recomputes of an
 * in-place op run out-of-place (R21). */
static int allocate(R *r, int op, int32_t t, int allow_inplace, int ev_kind) {
  const orc_trace *tr = r->tr;
  uint64_t size = tr->size[t];
  int32_t src = tr->inplace_src[op];
  if (allow_inplace && src >= 0 && (r->cfg.flags & ORC_F_INPLACE)) {
    int i = find_block_of(r, src); /* addr <- input.addr */
    r->b[i].owner = t;
    r->addr[t] = r->b[i].addr;
    r->resident[src] = 0;
    r->resident[t] = 1;
    r->res->inplace_reuse++;
    log_ev(r, ORC_EV_INPLACE, op, t, r->addr[t]);
    return 0;
  }
  int right = goes_right(r, op);
  int i = find_fit(r, size, right);
  if (i < 0) {
    r->res->pressure++;
    if (r->bytes_free >= size) r->res->frag_fail++;
    if (evict_window(r, size) != 0) {
      r->res->fail_op = r->cur_op;
      return -1;
    }
    i = find_fit(r, size, right); /* the unique coalesced block >= size */
    r->addr[t] = place(r, i, size, right, t);
    r->res->sum_free_bytes_after += r->bytes_free; /* R27 */
    r->res->sum_free_blocks_after += n_free_blocks(r);
  } else {
    r->addr[t] = place(r, i, size, right, t);
  }
  r->resident[t] = 1;
  log_ev(r, ev_kind, op, t, r->addr[t]);
  return 0;
}

static void free_tensor(R *r, int32_t t) {
  int i = find_block_of(r, t);
  uint64_t a = r->b[i].addr;
  release(r, i);
  r->resident[t] = 0;
  log_ev(r, ORC_EV_FREE, r->cur_op, t, a);
}

/* ------------------------------------------------------------------ rematerialization */
/* M(t, d): recompute evicted (or dead, R22) tensor t via its producer */
static int materialize(R *r, int32_t t, int depth) {
  const orc_trace *tr = r->tr;
  if (depth > r->cfg.max_depth) {
    r->status = ORC_THRASHED; /* R23 */
    r->res->fail_op = r->cur_op;
    return -1;
  }
  if (depth > r->res->max_depth) r->res->max_depth = depth;
  int op = tr->producer[t];
  if (op < 0) { /* a replaced parameter version cannot be recomputed */
    r->status = ORC_UNSATISFIABLE;
    r->res->fail_op = r->cur_op;
    return -1;
  }
  int ni = n_in(tr, op);
  for (int k = 0; k < ni; ++k) r->pins[in_at(tr, op, k)]++; /* held by the stack (R16) */
  for (int k = 0; k < ni; ++k) {
    int32_t u = in_at(tr, op, k);
    if (!r->resident[u] && materialize(r, u, depth + 1) != 0) return -1;
  }
  if (allocate(r, op, t, 0, ORC_EV_REMAT) != 0) {
    if (r->status == ORC_OK) r->status = ORC_UNSATISFIABLE;
    return -1;
  }
  r->clock += tr->cost_us[op];
  r->res->total_us += tr->cost_us[op];
  r->res->remat++;
  log_ev(r, ORC_EV_REXEC, op, t, r->addr[t]);
  for (int k = 0; k < ni; ++k) r->last_access[in_at(tr, op, k)] = r->clock;
  r->last_access[t] = r->clock;
  for (int k = 0; k < ni; ++k) r->pins[in_at(tr, op, k)]--;
  /* a dead input materialized for this recompute stays resident (evictable) until the
   * end of the current trace op (R22) */
  return 0;
}

/* ------------------------------------------------------------------ validation */
static int validate(const orc_trace *tr, int32_t *last_use) {
  int T = tr->n_tensors, M = tr->n_ops;
  if (T < 1 || M < 0) return -1;
  for (int t = 0; t < T; ++t) {
    if (tr->size[t] < 1 || tr->size[t] >= (1ull << 48)) return -1;
    if (tr->is_param[t]) {
      if (tr->producer[t] != -1) return -1;
    } else {
      int p = tr->producer[t];
      if (p < 0 || p >= M || tr->out[p] != t) return -1;
    }
    last_use[t] = -1;
  }
  if (tr->in_ptr[0] != 0) return -1;
  for (int k = 0; k < M; ++k) {
    if (tr->cost_us[k] < 0 || tr->cost_us[k] >= (1ll << 40)) return -1;
    if (tr->phase[k] > ORC_PHASE_UPD) return -1;
    int o = tr->out[k];
    if (o < 0 || o >= T || tr->producer[o] != k) return -1;
    if (tr->in_ptr[k + 1] < tr->in_ptr[k]) return -1;
    int src_seen = 0;
    for (int j = tr->in_ptr[k]; j < tr->in_ptr[k + 1]; ++j) {
      int u = tr->in_idx[j];
      if (u < 0 || u >= T) return -1;
      if (!tr->is_param[u] && tr->producer[u] >= k) return -1; /* DAG in trace order */
      if (u == tr->inplace_src[k]) src_seen = 1;
      last_use[u] = k;
    }
    if (tr->inplace_src[k] >= 0) {
      int s = tr->inplace_src[k];
      if (s >= T || !src_seen || tr->size[s] != tr->size[o]) return -1;
    }
  }
  for (int k = 0; k < M; ++k) { /* the mutated input is never read again (R19) */
    int s = tr->inplace_src[k];
    if (s >= 0 && last_use[s] != k) return -1;
  }
  for (int t = 0; t < T; ++t) /* outputs that are never read die at production (R20) */
    if (last_use[t] < 0 && !tr->is_param[t]) last_use[t] = tr->producer[t];
  return 0;
}

/* unevictable-ness: parameters, and outputs of in-place ops on unevictable tensors (R19) */
static void compute_unevict(const orc_trace *tr, uint8_t *u) {
  for (int t = 0; t < tr->n_tensors; ++t) u[t] = tr->is_param[t] ? 1 : 0;
  for (int k = 0; k < tr->n_ops; ++k) {
    int s = tr->inplace_src[k];
    if (s >= 0 && u[s]) u[tr->out[k]] = 1;
  }
}

/* R36: an in-place op that overwrites an UNEVICTABLE tensor (a parameter update) destroys
 * the only copy of its old value.  Every tensor that is alive after the op and whose
 * recomputation would read that value (through producers of evictable tensors) is made
 * resident before the op and locked (never evicted) until it dies.  need(t) = the set of
 * unevictable tensors read by the recompute closure of t; L_k = {t alive across k, t not
 * unevictable, src(k) in need(t)}.  Static: computed once from the trace. */
static void build_lock_lists(const orc_trace *tr, const uint8_t *unevict, const int32_t *last_use,
                             int32_t **ptr_out, int32_t **idx_out) {
  int T = tr->n_tensors, M = tr->n_ops;
  int32_t *uid = (int32_t *)malloc(sizeof(int32_t) * (size_t)T);
  int nu = 0;
  for (int t = 0; t < T; ++t) uid[t] = unevict[t] ? nu++ : -1;
  int words = (nu + 63) / 64;
  if (words == 0) words = 1;
  uint64_t *need = (uint64_t *)calloc((size_t)T * (size_t)words, sizeof(uint64_t));
  for (int k = 0; k < M; ++k) { /* tensors are produced in op order */
    int o = tr->out[k];
    uint64_t *no = need + (size_t)o * words;
    for (int j = tr->in_ptr[k]; j < tr->in_ptr[k + 1]; ++j) {
      int u = tr->in_idx[j];
      if (unevict[u]) {
        no[uid[u] / 64] |= 1ull << (uid[u] % 64);
      } else {
        uint64_t *nu_ = need + (size_t)u * words;
        for (int w = 0; w < words; ++w) no[w] |= nu_[w];
      }
    }
  }
  int32_t *ptr = (int32_t *)calloc((size_t)M + 1, sizeof(int32_t));
  int cap = 1024, cnt = 0;
  int32_t *idx = (int32_t *)malloc(sizeof(int32_t) * (size_t)cap);
  for (int k = 0; k < M; ++k) {
    int s = tr->inplace_src[k];
    if (s >= 0 && unevict[s]) {
      for (int t = 0; t < T; ++t) {
        if (unevict[t] || tr->is_param[t]) continue;
        if (tr->producer[t] >= k || last_use[t] <= k) continue;
        if (!(need[(size_t)t * words + uid[s] / 64] >> (uid[s] % 64) & 1ull)) continue;
        if (cnt == cap) {
          cap *= 2;
          idx = (int32_t *)realloc(idx, sizeof(int32_t) * (size_t)cap);
        }
        idx[cnt++] = t;
      }
    }
    ptr[k + 1] = cnt;
  }
  free(uid);
  free(need);
  *ptr_out = ptr;
  *idx_out = idx;
}

uint64_t orc_peak_live(const orc_trace *tr, uint32_t flags) {
  int T = tr->n_tensors, M = tr->n_ops;
  int32_t *lu = (int32_t *)malloc(sizeof(int32_t) * (size_t)T);
  uint8_t *ue = (uint8_t *)malloc((size_t)T);
  if (validate(tr, lu) != 0) {
    free(lu);
    free(ue);
    return 0;
  }
  compute_unevict(tr, ue);
  uint64_t live = 0, peak = 0;
  for (int t = 0; t < T; ++t)
    if (tr->is_param[t]) live += tr->size[t];
  peak = live;
  for (int k = 0; k < M; ++k) {
    int o = tr->out[k], s = tr->inplace_src[k];
    int inplace = (s >= 0 && (flags & ORC_F_INPLACE));
    if (!inplace) live += tr->size[o];
    if (live > peak) peak = live;
    for (int t = 0; t < T; ++t) { /* deaths after op k (R20): plain scan */
      if (lu[t] != k) continue;
      if (ue[t] && t != s) continue;
      if (inplace && t == s) continue; /* its bytes now belong to the output */
      live -= tr->size[t];
    }
  }
  free(lu);
  free(ue);
  return peak;
}

/* ------------------------------------------------------------------ the replay */
int orc_replay(const orc_trace *tr, const orc_cfg *cfg_in, orc_replay_result *res,
               orc_event *log, int64_t log_cap) {
  if (!tr || !cfg_in || !res) return ORC_INVALID_ARG;
  memset(res, 0, sizeof(*res));
  res->fail_op = -1;
  res->digest = 0x9E3779B97F4A7C15ull;
  res->budget = cfg_in->budget;
  int T = tr->n_tensors, M = tr->n_ops;
  R r;
  memset(&r, 0, sizeof(r));
  r.tr = tr;
  r.cfg = *cfg_in;
  if (r.cfg.class_threshold == 0) r.cfg.class_threshold = 15;
  if (r.cfg.max_depth <= 0) r.cfg.max_depth = 512;
  r.res = res;
  r.log = log;
  r.log_cap = log_cap;
  r.last_use = (int32_t *)calloc((size_t)T, sizeof(int32_t));
  if (validate(tr, r.last_use) != 0 || cfg_in->budget < 1) {
    free(r.last_use);
    res->status = ORC_INVALID_ARG;
    return ORC_INVALID_ARG;
  }
  r.born = (uint8_t *)calloc((size_t)T, 1);
  r.resident = (uint8_t *)calloc((size_t)T, 1);
  r.dead = (uint8_t *)calloc((size_t)T, 1);
  r.unevict = (uint8_t *)calloc((size_t)T, 1);
  r.pins = (int32_t *)calloc((size_t)T, sizeof(int32_t));
  r.last_access = (int64_t *)calloc((size_t)T, sizeof(int64_t));
  r.addr = (uint64_t *)calloc((size_t)T, sizeof(uint64_t));
  r.mark = (uint32_t *)calloc((size_t)T, sizeof(uint32_t));
  int nnz = tr->in_ptr[M];
  r.stack = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nnz + T + 16) * 2);
  r.cons_ptr = (int32_t *)calloc((size_t)T + 1, sizeof(int32_t));
  r.cons_idx = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nnz + 1));
  r.cap = 64;
  r.b = (blk *)malloc(sizeof(blk) * (size_t)r.cap);
  r.v_ss = (uint64_t *)malloc(sizeof(uint64_t) * 8192);
  r.v_c = (double *)malloc(sizeof(double) * 8192);
  r.v_s = (double *)malloc(sizeof(double) * 8192);
  compute_unevict(tr, r.unevict);
  r.locked = (uint8_t *)calloc((size_t)T, 1);
  build_lock_lists(tr, r.unevict, r.last_use, &r.lock_ptr, &r.lock_idx);
  /* consumers CSR: ops reading each tensor, in op order */
  for (int j = 0; j < nnz; ++j) r.cons_ptr[tr->in_idx[j] + 1]++;
  for (int t = 0; t < T; ++t) r.cons_ptr[t + 1] += r.cons_ptr[t];
  {
    int32_t *fill = (int32_t *)calloc((size_t)T, sizeof(int32_t));
    for (int k = 0; k < M; ++k)
      for (int j = tr->in_ptr[k]; j < tr->in_ptr[k + 1]; ++j) {
        int u = tr->in_idx[j];
        r.cons_idx[r.cons_ptr[u] + fill[u]++] = k;
      }
    free(fill);
  }
  /* the pool: one free block [0, budget) held by the allocator */
  r.b[0].addr = 0;
  r.b[0].size = cfg_in->budget;
  r.b[0].owner = NO_OWNER;
  r.nb = 1;
  r.bytes_free = cfg_in->budget;
  res->max_blocks = 1;
  r.status = ORC_OK;
  r.cur_op = -1;

  /* parameters first: to the two ends of the pool with recomputable in-place (
   * R15: each to the end holding fewer parameter bytes, ties left); leftmost otherwise */
  uint64_t left_bytes = 0, right_bytes = 0;
  for (int t = 0; t < T && r.status == ORC_OK; ++t) {
    if (!tr->is_param[t]) continue;
    int right = (cfg_in->flags & ORC_F_INPLACE) ? (right_bytes < left_bytes) : 0;
    int i = find_fit(&r, tr->size[t], right);
    if (i < 0) {
      r.status = ORC_UNSATISFIABLE;
      break;
    }
    r.addr[t] = place(&r, i, tr->size[t], right, t);
    if (right) right_bytes += tr->size[t];
    else left_bytes += tr->size[t];
    r.born[t] = r.resident[t] = 1;
    log_ev(&r, ORC_EV_PARAM, -1, t, r.addr[t]);
  }

  for (int k = 0; k < M && r.status == ORC_OK; ++k) {
    r.cur_op = k;
    int ni = n_in(tr, k);
    int32_t o = tr->out[k];
    for (int j = 0; j < ni; ++j) r.pins[in_at(tr, k, j)]++; /* the op's inputs (R16) */
    for (int j = r.lock_ptr[k]; j < r.lock_ptr[k + 1]; ++j) r.locked[r.lock_idx[j]] = 1;
    for (int j = 0; j < ni && r.status == ORC_OK; ++j) {
      int32_t u = in_at(tr, k, j);
      if (!r.resident[u]) materialize(&r, u, 0);
    }
    for (int j = r.lock_ptr[k]; j < r.lock_ptr[k + 1] && r.status == ORC_OK; ++j) {
      int32_t u = r.lock_idx[j]; /* R36: materialize before the old value is overwritten */
      if (!r.resident[u]) materialize(&r, u, 0);
    }
    if (r.status != ORC_OK) break;
    if (allocate(&r, k, o, 1, ORC_EV_ALLOC) != 0) {
      if (r.status == ORC_OK) r.status = ORC_UNSATISFIABLE;
      break;
    }
    r.born[o] = 1;
    r.clock += tr->cost_us[k];
    res->base_us += tr->cost_us[k];
    res->total_us += tr->cost_us[k];
    log_ev(&r, ORC_EV_EXEC, k, o, r.addr[o]);
    for (int j = 0; j < ni; ++j) r.last_access[in_at(tr, k, j)] = r.clock;
    r.last_access[o] = r.clock;
    for (int j = 0; j < ni; ++j) r.pins[in_at(tr, k, j)]--;
    /* deaths after op k, ascending tensor id (R20; the mutated input always dies here),
     * together with dead tensors rematerialized transiently during this op (R22) */
    int32_t src = tr->inplace_src[k];
    for (int t = 0; t < T; ++t) {
      if (r.last_use[t] == k && (!r.unevict[t] || t == src)) r.dead[t] = 1;
      if (r.dead[t] && r.resident[t] && (!r.unevict[t] || t == src)) free_tensor(&r, t);
    }
  }
  res->status = r.status;
  free(r.last_use); free(r.born); free(r.resident); free(r.dead); free(r.unevict);
  free(r.pins); free(r.last_access); free(r.addr); free(r.mark); free(r.stack);
  free(r.cons_ptr); free(r.cons_idx); free(r.lock_ptr); free(r.lock_idx); free(r.locked); free(r.b); free(r.v_ss); free(r.v_c); free(r.v_s);
  return r.status;
}

/* ======================================================================= O3: online calls
 * One pool [0, budget) driven call by call (the framework side of Alg. 1): every
 * orc_pool_alloc is one op producing one new tensor (op id = tensor id), its parents are
 * the op's inputs.  The same Alg. 1 / Sec. 3.3-3.5 steps as O2 (allocate, evict_window,
 * projected_cost, place, release); readings R38-R44 of DESIGN.md.  Plain arrays with a
 * fixed capacity; the consumer lists are rebuilt from scratch on every call. */
struct orc_pool_s {
  R r;
  orc_trace tr;
  orc_replay_result res;
  int32_t T, nnz, max_tensors, max_edges;
  uint64_t *size;
  uint8_t *is_param, *phase, *cls;
  int32_t *producer, *out, *src, *in_ptr, *in_idx;
  int64_t *cost;
};

orc_pool *orc_pool_create(uint64_t budget, uint32_t flags, uint32_t class_threshold,
                          int32_t max_tensors, int32_t max_edges) {
  if (budget < 1 || (flags & ~31u) || ((flags & ORC_F_DTR) && (flags & ORC_F_DTE)) || max_tensors < 1 ||
      max_edges < 0)
    return NULL;
  orc_pool *p = (orc_pool *)calloc(1, sizeof(orc_pool));
  int T = max_tensors, E = max_edges;
  p->max_tensors = T;
  p->max_edges = E;
  p->size = (uint64_t *)calloc((size_t)T, sizeof(uint64_t));
  p->is_param = (uint8_t *)calloc((size_t)T, 1);
  p->phase = (uint8_t *)calloc((size_t)T, 1);
  p->cls = (uint8_t *)calloc((size_t)T, 1);
  p->producer = (int32_t *)calloc((size_t)T, sizeof(int32_t));
  p->out = (int32_t *)calloc((size_t)T, sizeof(int32_t));
  p->src = (int32_t *)calloc((size_t)T, sizeof(int32_t));
  p->in_ptr = (int32_t *)calloc((size_t)T + 1, sizeof(int32_t));
  p->in_idx = (int32_t *)calloc((size_t)E + 1, sizeof(int32_t));
  p->cost = (int64_t *)calloc((size_t)T, sizeof(int64_t));
  p->tr.size = p->size;
  p->tr.is_param = p->is_param;
  p->tr.producer = p->producer;
  p->tr.cost_us = p->cost;
  p->tr.out = p->out;
  p->tr.inplace_src = p->src;
  p->tr.phase = p->phase;
  p->tr.in_ptr = p->in_ptr;
  p->tr.in_idx = p->in_idx;
  R *r = &p->r;
  r->tr = &p->tr;
  r->cfg.budget = budget;
  r->cfg.flags = flags;
  r->cfg.class_threshold = class_threshold ? class_threshold : 15;
  r->cfg.max_depth = 512;
  r->cls = p->cls;
  r->res = &p->res;
  r->born = (uint8_t *)calloc((size_t)T, 1);
  r->resident = (uint8_t *)calloc((size_t)T, 1);
  r->dead = (uint8_t *)calloc((size_t)T, 1);
  r->unevict = (uint8_t *)calloc((size_t)T, 1);
  r->locked = (uint8_t *)calloc((size_t)T, 1);
  r->pins = (int32_t *)calloc((size_t)T, sizeof(int32_t));
  r->last_access = (int64_t *)calloc((size_t)T, sizeof(int64_t));
  r->addr = (uint64_t *)calloc((size_t)T, sizeof(uint64_t));
  r->mark = (uint32_t *)calloc((size_t)T, sizeof(uint32_t));
  r->stack = (int32_t *)malloc(sizeof(int32_t) * ((size_t)E + (size_t)T + 16) * 2);
  r->cons_ptr = (int32_t *)calloc((size_t)T + 1, sizeof(int32_t));
  r->cons_idx = (int32_t *)calloc((size_t)E + 1, sizeof(int32_t));
  r->victims = (int32_t *)calloc(8192, sizeof(int32_t));
  r->cap = 64;
  r->b = (blk *)malloc(sizeof(blk) * (size_t)r->cap);
  r->v_ss = (uint64_t *)malloc(sizeof(uint64_t) * 8192);
  r->v_c = (double *)malloc(sizeof(double) * 8192);
  r->v_s = (double *)malloc(sizeof(double) * 8192);
  /* the pool: one free block [0, budget) */
  r->b[0].addr = 0;
  r->b[0].size = budget;
  r->b[0].owner = NO_OWNER;
  r->nb = 1;
  r->bytes_free = budget;
  p->res.fail_op = -1;
  p->res.digest = 0x9E3779B97F4A7C15ull;
  p->res.budget = budget;
  p->res.max_blocks = 1;
  r->status = ORC_OK;
  r->cur_op = -1;
  return p;
}

void orc_pool_destroy(orc_pool *p) {
  if (!p) return;
  R *r = &p->r;
  free(r->born); free(r->resident); free(r->dead); free(r->unevict); free(r->locked);
  free(r->pins); free(r->last_access); free(r->addr); free(r->mark); free(r->stack);
  free(r->cons_ptr); free(r->cons_idx); free(r->victims); free(r->b);
  free(r->v_ss); free(r->v_c); free(r->v_s);
  free(p->size); free(p->is_param); free(p->phase); free(p->cls); free(p->producer);
  free(p->out); free(p->src); free(p->in_ptr); free(p->in_idx); free(p->cost);
  free(p);
}

/* consumers CSR over ops [0, n): rebuilt from scratch (plain) */
static void o3_consumers(orc_pool *p, int n) {
  R *r = &p->r;
  for (int t = 0; t <= p->max_tensors; ++t) r->cons_ptr[t] = 0;
  for (int j = 0; j < p->in_ptr[n]; ++j) r->cons_ptr[p->in_idx[j] + 1]++;
  for (int t = 0; t < p->max_tensors; ++t) r->cons_ptr[t + 1] += r->cons_ptr[t];
  int32_t *fill = (int32_t *)calloc((size_t)p->max_tensors, sizeof(int32_t));
  for (int k = 0; k < n; ++k)
    for (int j = p->in_ptr[k]; j < p->in_ptr[k + 1]; ++j) {
      int u = p->in_idx[j];
      r->cons_idx[r->cons_ptr[u] + fill[u]++] = k;
    }
  free(fill);
}

static void o3_fill(orc_pool *p, int32_t t, orc_alloc_result *out, int32_t *evicted, int32_t cap) {
  R *r = &p->r;
  if (!out) return;
  out->tensor_id = t;
  out->addr = r->addr[t];
  out->size = p->size[t];
  out->n_evicted = r->nvict;
  out->window_first = r->win_first;
  out->window_last = r->win_last;
  out->reserved = 0;
  out->window_span = r->nvict || r->win_first >= 0 ? r->win_span : 0;
  out->window_cost = r->win_first >= 0 ? r->win_cost : 0.0;
  for (int k = 0; k < r->nvict && k < cap; ++k) evicted[k] = r->victims[k];
}

/* Alg. 1 for one new tensor (R38-R41): validation, parents resident, allocate (in-place
 * when the op mutates a parent and recomputable in-place is on), then the op runs */
int orc_pool_alloc(orc_pool *p, uint64_t size, uint64_t cost_us, uint32_t op_flags,
                   int32_t inplace_src, const int32_t *parents, int32_t n_parents,
                   orc_alloc_result *out, int32_t *evicted, int32_t evicted_cap) {
  R *r = &p->r;
  if (size < 1 || size >= (1ull << 48) || cost_us >= (1ull << 40)) return ORC_INVALID_ARG;
  if ((op_flags & ~31u) || ((op_flags & ORC_OP_EXPENSIVE) && (op_flags & ORC_OP_CHEAP)))
    return ORC_INVALID_ARG;
  if (n_parents < 0 || (n_parents > 0 && !parents) || evicted_cap < 0) return ORC_INVALID_ARG;
  for (int j = 0; j < n_parents; ++j)
    if (parents[j] < 0 || parents[j] >= p->T) return ORC_UNKNOWN_ID;
  if (op_flags & ORC_OP_INPLACE) {
    int seen = 0;
    for (int j = 0; j < n_parents; ++j) seen |= (parents[j] == inplace_src);
    if (!seen || p->size[inplace_src] != size) return ORC_INVALID_ARG;
  } else if (inplace_src != -1) {
    return ORC_INVALID_ARG;
  }
  if (p->T >= p->max_tensors || p->nnz + n_parents > p->max_edges) return ORC_NOMEM;
  for (int j = 0; j < n_parents; ++j)
    if (!r->resident[parents[j]]) {
      if (out) out->tensor_id = parents[j];
      return ORC_NEEDS_REMAT;
    }
  int32_t t = p->T;
  p->size[t] = size;
  p->producer[t] = t;
  p->out[t] = t;
  p->cost[t] = (int64_t)cost_us;
  p->src[t] = (op_flags & ORC_OP_INPLACE) ? inplace_src : -1;
  p->phase[t] = (op_flags & ORC_OP_PHASE_FWD) ? ORC_PHASE_FWD : ORC_PHASE_BWD;
  p->cls[t] = (op_flags & ORC_OP_EXPENSIVE) ? 1 : (op_flags & ORC_OP_CHEAP) ? 2 : 0;
  for (int j = 0; j < n_parents; ++j) p->in_idx[p->nnz + j] = parents[j];
  p->in_ptr[t + 1] = p->nnz + n_parents;
  r->unevict[t] = (op_flags & ORC_OP_UNEVICTABLE) || (p->src[t] >= 0 && r->unevict[p->src[t]]);
  p->tr.n_tensors = p->tr.n_ops = t + 1;
  o3_consumers(p, t);
  r->cur_op = t;
  r->win_first = r->win_last = -1;
  r->nvict = 0;
  r->win_span = 0;
  for (int j = 0; j < n_parents; ++j) r->pins[parents[j]]++; /* the op's inputs (R16) */
  int rc = allocate(r, t, t, 1, ORC_EV_ALLOC);
  for (int j = 0; j < n_parents; ++j) r->pins[parents[j]]--;
  if (rc != 0) {
    int st = r->status == ORC_OK ? ORC_UNSATISFIABLE : r->status;
    r->status = ORC_OK; /* the pool stays usable; the tensor is not created */
    p->tr.n_tensors = p->tr.n_ops = t;
    r->unevict[t] = 0;
    return st;
  }
  r->born[t] = 1;
  r->clock += (int64_t)cost_us;
  p->res.base_us += (int64_t)cost_us;
  p->res.total_us += (int64_t)cost_us;
  log_ev(r, ORC_EV_EXEC, t, t, r->addr[t]);
  for (int j = 0; j < n_parents; ++j) r->last_access[parents[j]] = r->clock;
  r->last_access[t] = r->clock;
  p->nnz += n_parents;
  p->T = t + 1;
  o3_fill(p, t, out, evicted, evicted_cap);
  return ORC_OK;
}

/* the caller frees a tensor (R42): a resident block is released and coalesced */
int orc_pool_free(orc_pool *p, int32_t t) {
  R *r = &p->r;
  if (t < 0 || t >= p->T) return ORC_UNKNOWN_ID;
  if (r->dead[t] && !r->resident[t]) return ORC_BAD_STATE;
  r->cur_op = t;
  if (r->resident[t]) free_tensor(r, t);
  r->dead[t] = 1;
  return ORC_OK;
}

/* the caller reads a tensor (R43): the clock advances; staleness restarts if resident */
int orc_pool_access(orc_pool *p, int32_t t, uint64_t advance_us) {
  R *r = &p->r;
  if (t < 0 || t >= p->T) return ORC_UNKNOWN_ID;
  if (advance_us >= (1ull << 40)) return ORC_INVALID_ARG;
  if (r->dead[t] && !r->resident[t]) return ORC_BAD_STATE;
  r->clock += (int64_t)advance_us;
  if (!r->resident[t]) return ORC_NEEDS_REMAT;
  r->last_access[t] = r->clock;
  return ORC_OK;
}

/* re-allocate an evicted (or freed) tensor whose parents are resident (R44): Alg. 1
 * out-of-place (R21), then its producer runs again */
int orc_pool_remat(orc_pool *p, int32_t t, orc_alloc_result *out, int32_t *evicted,
                   int32_t evicted_cap) {
  R *r = &p->r;
  if (t < 0 || t >= p->T) return ORC_UNKNOWN_ID;
  if (evicted_cap < 0) return ORC_INVALID_ARG;
  r->win_first = r->win_last = -1;
  r->nvict = 0;
  r->win_span = 0;
  if (r->resident[t]) {
    o3_fill(p, t, out, evicted, evicted_cap);
    return ORC_OK;
  }
  for (int j = p->in_ptr[t]; j < p->in_ptr[t + 1]; ++j)
    if (!r->resident[p->in_idx[j]]) {
      if (out) out->tensor_id = p->in_idx[j];
      return ORC_NEEDS_REMAT;
    }
  o3_consumers(p, p->T);
  r->cur_op = t;
  for (int j = p->in_ptr[t]; j < p->in_ptr[t + 1]; ++j) r->pins[p->in_idx[j]]++;
  int rc = allocate(r, t, t, 0, ORC_EV_REMAT);
  for (int j = p->in_ptr[t]; j < p->in_ptr[t + 1]; ++j) r->pins[p->in_idx[j]]--;
  if (rc != 0) {
    int st = r->status == ORC_OK ? ORC_UNSATISFIABLE : r->status;
    r->status = ORC_OK;
    return st;
  }
  r->clock += p->cost[t];
  p->res.total_us += p->cost[t];
  p->res.remat++;
  log_ev(r, ORC_EV_REXEC, t, t, r->addr[t]);
  for (int j = p->in_ptr[t]; j < p->in_ptr[t + 1]; ++j) r->last_access[p->in_idx[j]] = r->clock;
  r->last_access[t] = r->clock;
  o3_fill(p, t, out, evicted, evicted_cap);
  return ORC_OK;
}

int orc_pool_stats(orc_pool *p, orc_replay_result *out) {
  *out = p->res;
  out->status = ORC_OK;
  return ORC_OK;
}

/* the block table, address order: owner -1 = free */
int32_t orc_pool_layout(orc_pool *p, uint64_t *addr, uint64_t *size, int32_t *owner, int32_t cap) {
  R *r = &p->r;
  for (int i = 0; i < r->nb && i < cap; ++i) {
    addr[i] = r->b[i].addr;
    size[i] = r->b[i].size;
    owner[i] = r->b[i].owner;
  }
  return r->nb;
}

/* ======================================================================= O4: budget searches
 * Sec. 4.2 minimum budget and App. C cutoff budget on
 * the grid of DESIGN.md R45, every grid point replayed by O2 (plain loops). */
static uint64_t o4_grid(uint64_t lo, uint64_t hi, int64_t j, int64_t steps) {
  unsigned __int128 d = (unsigned __int128)(hi - lo) * (unsigned __int128)j / (unsigned __int128)steps;
  uint64_t b = lo + (uint64_t)d;
  return b < 1 ? 1 : b;
}

static int o4_meets(const orc_replay_result *r, int metric) {
  return r->status == ORC_OK && (metric == 0 || r->evictions == 0);
}

int orc_budget_search(const orc_trace *tr, uint32_t flags, uint32_t class_threshold, int32_t max_depth,
                      int32_t kc, int32_t kf, orc_budget_result *out) {
  if (!tr || !out || kc < 1 || kf < 1) return ORC_INVALID_ARG;
  memset(out, 0, sizeof(*out));
  uint64_t peak = orc_peak_live(tr, flags);
  out->peak = peak;
  /* Z = the bytes of every tensor of the trace: a pool that large never evicts, so the
   * brackets below stop there (R45) */
  uint64_t zsum = 0;
  for (int i = 0; i < tr->n_tensors; ++i) zsum += tr->size[i];
  if (zsum < peak) zsum = peak;
  orc_cfg cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.flags = flags;
  cfg.class_threshold = class_threshold;
  cfg.max_depth = max_depth;
  for (int m = 0; m < 2; ++m) {
    uint64_t *dst = m == 0 ? &out->min_budget : &out->cutoff_budget;
    int32_t *st = m == 0 ? &out->min_status : &out->cutoff_status;
    /* coarse grid on the brackets (0, P], (P, 2P], (2P, 4P], ... until the bracket's upper
     * end reaches Z: the smallest k of the first bracket that has one */
    int kstar = -1;
    uint64_t blo = 0, bhi = peak > 0 ? peak : 1;
    orc_replay_result r;
    for (;;) {
      for (int k = 1; k <= kc && kstar < 0; ++k) {
        cfg.budget = o4_grid(blo, bhi, k, kc);
        orc_replay(tr, &cfg, &r, NULL, 0);
        if (o4_meets(&r, m)) kstar = k;
      }
      if (kstar >= 0 || bhi >= zsum) break;
      blo = bhi;
      bhi = bhi > (UINT64_MAX >> 1) ? UINT64_MAX : 2 * bhi;
    }
    if (kstar < 0) {
      *st = ORC_INFEASIBLE;
      *dst = 0;
      continue;
    }
    /* fine grid inside (B_{k*-1}, B_{k*}] of that bracket */
    uint64_t lo = kstar > 1 ? o4_grid(blo, bhi, kstar - 1, kc) : blo, hi = o4_grid(blo, bhi, kstar, kc);
    *st = ORC_OK;
    *dst = hi;
    for (int j = 1; j <= kf; ++j) {
      cfg.budget = o4_grid(lo, hi, j, kf);
      orc_replay(tr, &cfg, &r, NULL, 0);
      if (o4_meets(&r, m)) {
        *dst = cfg.budget;
        break;
      }
    }
  }
  return ORC_OK;
}
