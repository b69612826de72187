// api.cu -- the C ABI of libdmk (include/dmk.h): argument checking, memory
// placement (host <-> device), plan lifetime, introspection.
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <exception>

#include "common.cuh"

namespace dmk {
bool pw64_group_env();
void build_tree(dmk_plan_s* P, const double* dpts);
void eval_plan(dmk_plan_s* P, const double* dcharges, double* dout);

static thread_local std::string g_err;
int64_t g_launches = 0, g_cub_launches = 0;
thread_local int64_t g_alloc_bytes = 0;
void set_error(const std::string& m) { g_err = m; }
void fail(int code, const std::string& m) { throw Error{code, m}; }

template <class F>
static int guard(F f) {
  try {
    f();
    g_err.clear();
    return DMK_OK;
  } catch (const Error& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return DMK_ERR_CUDA;
  }
}

static void require_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) fail(DMK_ERR_CUDA, "no CUDA device available (libdmk has no CPU path)");
  // Plans allocate and free ~1 GB per evaluation cycle through the stream-ordered
  // allocator; keep freed memory in the device pool instead of returning it to the
  // driver at every synchronisation (which would re-map pages on every plan).
  int dev = 0;
  DMK_CUDA(cudaGetDevice(&dev));
  cudaMemPool_t pool;
  DMK_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t thr = UINT64_MAX;
  DMK_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
}

// ---- stream-ordered pool reservation.  Plans allocate and free their buffers through the
// device's default pool (release threshold: never).  When a plan needs more than the pool
// holds, cudaMallocAsync maps new physical memory -- tens to hundreds of ms, at random
// steps of a repeated evaluation (measured on config 2: 60-190 ms outliers in 24 steps,
// none after a pre-grown pool, profiles/r02_repeat_c2c.json).  So the pool is grown
// ahead, once per size class: to twice the bytes the largest plan so far requested.
namespace {
std::mutex g_res_mu;
std::vector<std::pair<int, int64_t>> g_reserved;   // (device, bytes)
}
static void reserve_pool(int64_t bytes, cudaStream_t s) {
  int dev = 0;
  DMK_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_res_mu);
  int64_t* have = nullptr;
  for (auto& r : g_reserved)
    if (r.first == dev) have = &r.second;
  if (!have) {
    g_reserved.push_back({dev, 0});
    have = &g_reserved.back().second;
  }
  const int64_t want = 2 * bytes;
  if (want <= *have) return;
  void* p = nullptr;
  if (cudaMallocAsync(&p, (size_t)want, s) == cudaSuccess) {
    cudaFreeAsync(p, s);
    *have = want;
  } else {
    cudaGetLastError();   // not enough memory for the reserve: allocate on demand
  }
}

// ---- stream/event pool (per device, process-wide, thread-safe)
namespace {
struct StreamSet {
  int dev;
  cudaStream_t side, hi, root;
  cudaEvent_t fork, join, rootev;
};
std::mutex g_pool_mu;
std::vector<StreamSet> g_pool;
}  // namespace

static void acquire_streams(dmk_plan_s* P) {
  int dev = 0;
  DMK_CUDA(cudaGetDevice(&dev));
  StreamSet ss{};
  bool found = false;
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    for (size_t i = 0; i < g_pool.size(); ++i)
      if (g_pool[i].dev == dev) {
        ss = g_pool[i];
        g_pool.erase(g_pool.begin() + i);
        found = true;
        break;
      }
  }
  if (!found) {
    int prio_lo = 0, prio_hi = 0;
    ss.dev = dev;
    DMK_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    DMK_CUDA(cudaStreamCreateWithPriority(&ss.side, cudaStreamNonBlocking, prio_lo));
    DMK_CUDA(cudaStreamCreateWithPriority(&ss.hi, cudaStreamNonBlocking, prio_hi));
    DMK_CUDA(cudaStreamCreateWithPriority(&ss.root, cudaStreamNonBlocking, prio_hi));
    DMK_CUDA(cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming));
    DMK_CUDA(cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming));
    DMK_CUDA(cudaEventCreateWithFlags(&ss.rootev, cudaEventDisableTiming));
  }
  P->pool_dev = dev;
  P->side_stream = ss.side;
  P->hi_stream = ss.hi;
  P->root_stream = ss.root;
  P->ev_fork = ss.fork;
  P->ev_join = ss.join;
  P->ev_root = ss.rootev;
}

static void alloc_eval_buffers(dmk_plan_s* P) {
  const Tables& T = *P->tab;
  cudaStream_t s = P->stream;
  const int64_t p3 = (int64_t)T.p * T.p * T.p;
  P->q.alloc(P->n, s);
  P->ufar.alloc(P->n, s);
  P->unear.alloc(P->n, s);
  // outgoing expansions in the real parity-split layout (2^d parity classes over the
  // non-negative mode orthant, kernels.cu / kernels2d.cu)
  const int64_t h0 = T.nf0 + 1, h1 = T.nf + 1;
  const int64_t pd = P->dim == 2 ? (int64_t)T.p * T.p : p3;
  P->phi_size0 = P->dim == 2 ? 4 * h0 * h0 : 8 * h0 * h0 * h0;
  P->phi_size1 = P->dim == 2 ? 4 * h1 * h1 : 8 * h1 * h1 * h1;
  P->scalar.alloc(1, s);
  if (P->th.nlevels > 1) {
    P->mom.alloc(P->nfout * pd, s);
    P->phi_count = P->phi_size0 + (P->nfout - 1) * P->phi_size1;
    P->phi_f32 = P->dim == 3 && T.p <= 18;
    P->phi.alloc(P->phi_f32 ? (P->phi_count + 1) / 2 : P->phi_count, s);
    P->lam.alloc(P->nexp * pd, s);
    // fp32 tier (p <= 18, 3D): weighted incoming plane waves of every local box (k_pwshift)
    if (P->dim == 3 && T.p <= 18) P->pwt.alloc(P->nexp * P->phi_size1, s);
    // symmetric near field (fp32 tier): one partial sum per same-level entry and target
    if (P->dim == 3 && T.p <= 18) P->part.alloc(P->npart ? P->npart : 1, s);
    if (P->dim == 3 && T.p > 18 && pw64_group_env() && P->nexp > 1) P->pwt64.alloc(P->nexp * P->phi_size1, s);
  }
}

}  // namespace dmk

using namespace dmk;

// the streams go back to the pool once idle (dmk_destroy synchronises them first)
dmk_plan_s::~dmk_plan_s() {
  for (auto e : ev_pool) cudaEventDestroy(e);
  if (pool_dev >= 0 && side_stream) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    g_pool.push_back(StreamSet{pool_dev, side_stream, hi_stream, root_stream, ev_fork, ev_join, ev_root});
  }
}

extern "C" {

const char* dmk_last_error(void) { return g_err.c_str(); }
const char* dmk_version(void) { return "libdmk 0.2 (sm_100a; 3D Laplace, 3D Yukawa, 2D log; PSWF split; "
         "eps 1e-3/1e-6: fp32 tier with fp64 accumulation, eps 1e-9: fp64)"; }

int dmk_plan(int dim, int kernel, double eps, int64_t n, const double* points, int mem, const dmk_options* opt,
             dmk_plan_t* out) {
  return guard([&] {
    if (!out) fail(DMK_ERR_ARG, "out is NULL");
    *out = nullptr;
    if (!points) fail(DMK_ERR_ARG, "points is NULL");
    if (n < 1 || n >= (int64_t)1 << 31) fail(DMK_ERR_ARG, "n must be in [1, 2^31)");
    if (mem != DMK_MEM_DEVICE && mem != DMK_MEM_HOST) fail(DMK_ERR_ARG, "bad mem");
    if (!(eps > 0)) fail(DMK_ERR_ARG, "eps must be > 0");
    if (dim != 2 && dim != 3) fail(DMK_ERR_UNSUPPORTED, "dim must be 2 or 3");
    if (dim == 3 && kernel != DMK_KERNEL_LAPLACE && kernel != DMK_KERNEL_YUKAWA)
      fail(DMK_ERR_UNSUPPORTED, "kernel not implemented in 3D (DMK_KERNEL_LAPLACE, DMK_KERNEL_YUKAWA)");
    if (dim == 2 && kernel != DMK_KERNEL_LOG)
      fail(DMK_ERR_UNSUPPORTED, "kernel not implemented in 2D (DMK_KERNEL_LOG)");
    if (kernel == DMK_KERNEL_YUKAWA && !(opt && opt->lambda > 0))
      fail(DMK_ERR_ARG, "DMK_KERNEL_YUKAWA needs opt->lambda > 0");
    if (snap_eps(eps) == 0) fail(DMK_ERR_UNSUPPORTED, "eps tighter than 1e-9 is not supported");
    require_device();
    dmk_plan_s* P = new dmk_plan_s();
    try {
      P->dim = dim;
      P->kernel = kernel;
      P->n_targets = n;
      P->eps = eps;
      P->n = n;
      if (opt) {
        if (opt->leaf_capacity < 1) fail(DMK_ERR_ARG, "leaf_capacity must be >= 1");
        P->ns = opt->leaf_capacity;
        P->stream = (cudaStream_t)opt->stream;
        P->lambda = opt->lambda;
        if (opt->min_level < 0 || opt->min_level > 6) fail(DMK_ERR_ARG, "min_level must be in [0, 6]");
        P->min_level = opt->min_level;
        if (opt->n_targets < 0 || opt->n_targets > n) fail(DMK_ERR_ARG, "n_targets must be in [0, n]");
        if (opt->n_targets > 0) P->n_targets = opt->n_targets;
        if (opt->root) {
          P->root_fixed = true;
          for (int d = 0; d < dim; ++d) P->lo[d] = opt->root[d];
          P->side = opt->root[dim];
        }
      }
      acquire_streams(P);
      const char* ps = std::getenv("DMK_SERIAL");
      P->serial = ps && ps[0] == '1';
      const char* pe = std::getenv("DMK_PROFILE");
      P->profile = pe && pe[0] == '1';
      const char* pf = std::getenv("DMK_FULL_SORT");
      P->fast_sort = !(pf && pf[0] == '1');
      const char* pt = std::getenv("DMK_PROFILE_TREE");
      P->profile_tree = pt && pt[0] == '1';
      const int64_t bytes0 = g_alloc_bytes;
      const double* dpts = points;
      DevBuf<double> tmp;
      if (mem == DMK_MEM_HOST) {
        tmp.alloc(dim * n, P->stream);
        DMK_CUDA(cudaMemcpyAsync(tmp.p, points, dim * n * sizeof(double), cudaMemcpyHostToDevice, P->stream));
        dpts = tmp.p;
      }
      build_tree(P, dpts);
      // tables after the tree: the Yukawa split runs in unit-root-cube coordinates,
      // lambda' = lambda * side (K(side r') = exp(-lambda' r')/(side r'))
      P->tab_ref = get_tables(kernel, eps, kernel == DMK_KERNEL_YUKAWA ? P->lambda * P->side : 0.0);
      P->tab = P->tab_ref.get();
      alloc_eval_buffers(P);
      reserve_pool(g_alloc_bytes - bytes0, P->stream);
      // no synchronisation: the plan's device work is ordered on P->stream before any
      // evaluation or read-back (all of which run on P->stream)
      DMK_CUDA(cudaGetLastError());
    } catch (...) {
      delete P;
      throw;
    }
    *out = P;
  });
}

// Host charges: the H2D copy does not depend on the plan's build, so it goes to the
// plan's root-box stream (idle between evaluations) and overlaps whatever of the build
// the plan stream is still running when the caller gets here (dmk_plan returns without
// a final synchronisation); the plan stream waits for the copy before the gather.
static void upload_charges(dmk_plan_s* P, const double* charges, DevBuf<double>& dq) {
  cudaStream_t s = P->stream, cs = P->root_stream ? P->root_stream : s;
  dq.alloc(P->n, cs);
  DMK_CUDA(cudaMemcpyAsync(dq.p, charges, P->n * sizeof(double), cudaMemcpyHostToDevice, cs));
  if (cs != s) {
    DMK_CUDA(cudaEventRecord(P->ev_fork, cs));
    DMK_CUDA(cudaStreamWaitEvent(s, P->ev_fork, 0));
  }
}

int dmk_eval(dmk_plan_t P, const double* charges, double* potentials, int mem) {
  return guard([&] {
    if (!P) fail(DMK_ERR_ARG, "plan is NULL");
    if (!charges || !potentials) fail(DMK_ERR_ARG, "null buffer");
    if (mem != DMK_MEM_DEVICE && mem != DMK_MEM_HOST) fail(DMK_ERR_ARG, "bad mem");
    cudaStream_t s = P->stream;
    if (mem == DMK_MEM_HOST) {
      DevBuf<double> dq, du;
      du.alloc(P->n, s);
      upload_charges(P, charges, dq);
      eval_plan(P, dq.p, du.p);
      DMK_CUDA(cudaMemcpyAsync(potentials, du.p, P->n * sizeof(double), cudaMemcpyDeviceToHost, s));
      DMK_CUDA(cudaStreamSynchronize(s));
    } else {
      eval_plan(P, charges, potentials);
    }
    P->evaluated = true;
    P->upward_done = true;
  });
}

int dmk_upward(dmk_plan_t P, const double* charges, int mem) {
  return guard([&] {
    if (!P || !charges) fail(DMK_ERR_ARG, "null argument");
    if (mem != DMK_MEM_DEVICE && mem != DMK_MEM_HOST) fail(DMK_ERR_ARG, "bad mem");
    cudaStream_t s = P->stream;
    if (mem == DMK_MEM_HOST) {
      DevBuf<double> dq;
      upload_charges(P, charges, dq);
      eval_upward(P, dq.p);
      DMK_CUDA(cudaStreamSynchronize(s));
    } else {
      eval_upward(P, charges);
    }
    P->upward_done = true;
  });
}

int dmk_downward(dmk_plan_t P, double* potentials, int mem) {
  return guard([&] {
    if (!P || !potentials) fail(DMK_ERR_ARG, "null argument");
    if (mem != DMK_MEM_DEVICE && mem != DMK_MEM_HOST) fail(DMK_ERR_ARG, "bad mem");
    if (!P->upward_done) fail(DMK_ERR_STATE, "dmk_downward before dmk_upward");
    cudaStream_t s = P->stream;
    if (mem == DMK_MEM_HOST) {
      DevBuf<double> du;
      du.alloc(P->n, s);
      eval_downward(P, du.p);
      DMK_CUDA(cudaMemcpyAsync(potentials, du.p, P->n * sizeof(double), cudaMemcpyDeviceToHost, s));
      DMK_CUDA(cudaStreamSynchronize(s));
    } else {
      eval_downward(P, potentials);
    }
    P->evaluated = true;
  });
}

int dmk_level_moments(dmk_plan_t P, int level, double* dense, int64_t count, int mem, int set) {
  return guard([&] {
    if (!P || !dense) fail(DMK_ERR_ARG, "null argument");
    if (mem != DMK_MEM_DEVICE && mem != DMK_MEM_HOST) fail(DMK_ERR_ARG, "bad mem");
    if (!P->upward_done) fail(DMK_ERR_STATE, "dmk_level_moments before dmk_upward");
    if (level < 0 || level > 6) fail(DMK_ERR_ARG, "level out of range");
    const int64_t p3 = (int64_t)P->tab->p * P->tab->p * P->tab->p;
    const int64_t need = ((int64_t)1 << (3 * level)) * p3;
    if (count != need) fail(DMK_ERR_ARG, "count must be 8^level * p^3 = " + std::to_string(need));
    cudaStream_t s = P->stream;
    if (mem == DMK_MEM_HOST) {
      DevBuf<double> d;
      d.alloc(need, s);
      if (set) DMK_CUDA(cudaMemcpyAsync(d.p, dense, need * sizeof(double), cudaMemcpyHostToDevice, s));
      level_moments(P, level, d.p, set != 0);
      if (!set) DMK_CUDA(cudaMemcpyAsync(dense, d.p, need * sizeof(double), cudaMemcpyDeviceToHost, s));
      DMK_CUDA(cudaStreamSynchronize(s));
    } else {
      level_moments(P, level, dense, set != 0);
    }
  });
}

int dmk_box_moments(dmk_plan_t P, int level, const int64_t* codes, int64_t nbox, double* values, int mem, int set) {
  return guard([&] {
    if (!P || (nbox > 0 && (!codes || !values))) fail(DMK_ERR_ARG, "null argument");
    if (nbox < 0) fail(DMK_ERR_ARG, "nbox must be >= 0");
    if (mem != DMK_MEM_DEVICE && mem != DMK_MEM_HOST) fail(DMK_ERR_ARG, "bad mem");
    if (!P->upward_done) fail(DMK_ERR_STATE, "dmk_box_moments before dmk_upward");
    if (level < 0 || level > 6) fail(DMK_ERR_ARG, "level out of range");
    const int64_t nmax = (int64_t)1 << (3 * level);
    const int64_t p3 = (int64_t)P->tab->p * P->tab->p * P->tab->p;
    cudaStream_t s = P->stream;
    if (mem == DMK_MEM_HOST) {
      for (int64_t k = 0; k < nbox; ++k)
        if (codes[k] < 0 || codes[k] >= nmax) fail(DMK_ERR_ARG, "box code out of range for the level");
      DevBuf<int64_t> dc;
      DevBuf<double> d;
      dc.alloc(nbox, s);
      d.alloc(nbox * p3, s);
      if (nbox) DMK_CUDA(cudaMemcpyAsync(dc.p, codes, nbox * sizeof(int64_t), cudaMemcpyHostToDevice, s));
      if (set && nbox) DMK_CUDA(cudaMemcpyAsync(d.p, values, nbox * p3 * sizeof(double), cudaMemcpyHostToDevice, s));
      box_moments(P, level, dc.p, nbox, d.p, set != 0);
      if (!set && nbox) DMK_CUDA(cudaMemcpyAsync(values, d.p, nbox * p3 * sizeof(double), cudaMemcpyDeviceToHost, s));
      DMK_CUDA(cudaStreamSynchronize(s));
    } else {
      // device codes: stream-ordered, no synchronisation; codes outside the level are skipped
      box_moments(P, level, codes, nbox, values, set != 0);
    }
  });
}

int dmk_destroy(dmk_plan_t P) {
  return guard([&] {
    if (!P) return;
    cudaStream_t s = P->stream;
    if (P->p2p_pending) cudaStreamWaitEvent(s, P->ev_join, 0);   // near-field branch still running
    if (P->side_stream) cudaStreamSynchronize(P->side_stream);
    if (P->hi_stream) cudaStreamSynchronize(P->hi_stream);
    if (P->root_stream) cudaStreamSynchronize(P->root_stream);
    delete P;   // DevBuf destructors enqueue cudaFreeAsync on the plan stream
    cudaStreamSynchronize(s);
  });
}

int dmk_plan_info_get(dmk_plan_t P, dmk_plan_info* info) {
  return guard([&] {
    if (!P || !info) fail(DMK_ERR_ARG, "null argument");
    std::memset(info, 0, sizeof(*info));
    info->n = P->n;
    info->nbox = P->nbox;
    info->nlevels = P->th.nlevels;
    info->p = P->tab->p;
    info->nf = P->tab->nf;
    info->nf0 = P->tab->nf0;
    info->nfout = P->nfout;
    info->nexp = P->nexp;
    info->ndlist = P->ndlist;
    for (int d = 0; d < 3; ++d) info->lo[d] = P->lo[d];
    info->side = P->side;
    info->c = P->tab->c;
    info->respoly_degree = (int32_t)P->tab->respoly_deg;
    info->dim = P->dim;
  });
}

}  // extern "C"

namespace dmk {
template <class T>
static void copy_widen(cudaStream_t s, const T* d, int64_t cnt, int64_t* out) {
  std::vector<T> h(cnt);
  if (cnt) DMK_CUDA(cudaMemcpyAsync(h.data(), d, cnt * sizeof(T), cudaMemcpyDeviceToHost, s));
  DMK_CUDA(cudaStreamSynchronize(s));
  for (int64_t i = 0; i < cnt; ++i) out[i] = (int64_t)h[i];
}
}  // namespace dmk

extern "C" {

int dmk_tree_copy(dmk_plan_t P, int which, int64_t* out) {
  return guard([&] {
    if (!P || !out) fail(DMK_ERR_ARG, "null argument");
    cudaStream_t s = P->stream;
    const int64_t nb = P->nbox;
    switch (which) {
      case DMK_TREE_PERM: copy_widen(s, P->perm.p, P->n, out); break;
      case DMK_TREE_BOX_LEVEL: copy_widen(s, P->box_level.p, nb, out); break;
      case DMK_TREE_BOX_CODE: copy_widen(s, P->box_code.p, nb, out); break;
      case DMK_TREE_BOX_START: copy_widen(s, P->box_start.p, nb, out); break;
      case DMK_TREE_BOX_END: copy_widen(s, P->box_end.p, nb, out); break;
      case DMK_TREE_BOX_LEAF: {
        copy_widen(s, P->box_flags.p, nb, out);
        for (int64_t i = 0; i < nb; ++i) out[i] &= 1;
        break;
      }
      case DMK_TREE_BOX_PARENT: copy_widen(s, P->box_parent.p, nb, out); break;
      case DMK_TREE_COLLEAGUES: copy_widen(s, P->box_coll.p, (P->dim == 2 ? 9 : 27) * nb, out); break;
      case DMK_TREE_DLIST_OFF: copy_widen(s, P->dlist_off.p, nb + 1, out); break;
      case DMK_TREE_DLIST: copy_widen(s, P->dlist.p, P->ndlist, out); break;
      case DMK_TREE_FOUT: copy_widen(s, P->fout_rank.p, nb, out); break;
      case DMK_TREE_EXP: copy_widen(s, P->exp_rank.p, nb, out); break;
      default: fail(DMK_ERR_ARG, "unknown tree array");
    }
  });
}

int dmk_stage_copy(dmk_plan_t P, int which, double* out, int64_t count) {
  return guard([&] {
    if (!P || !out) fail(DMK_ERR_ARG, "null argument");
    if (!P->evaluated) fail(DMK_ERR_STATE, "no dmk_eval has run on this plan");
    const DevBuf<double>* b = nullptr;
    switch (which) {
      case DMK_STAGE_MOMENTS: b = &P->mom; break;
      case DMK_STAGE_OUTGOING:
        if (count != P->phi_count) fail(DMK_ERR_ARG, "count must equal the stage size " + std::to_string(P->phi_count));
        if (P->phi_f32) {   // stored in fp32 (reading R16): widen
          std::vector<float> h(count);
          DMK_CUDA(cudaMemcpyAsync(h.data(), P->phi.p, count * sizeof(float), cudaMemcpyDeviceToHost, P->stream));
          DMK_CUDA(cudaStreamSynchronize(P->stream));
          for (int64_t i = 0; i < count; ++i) out[i] = h[i];
          return;
        }
        b = &P->phi;
        break;
      case DMK_STAGE_LOCAL: b = &P->lam; break;
      case DMK_STAGE_UFAR: b = &P->ufar; break;
      case DMK_STAGE_UNEAR: b = &P->unear; break;
      default: fail(DMK_ERR_ARG, "unknown stage");
    }
    if (count != (int64_t)b->n) fail(DMK_ERR_ARG, "count must equal the stage size " + std::to_string(b->n));
    DMK_CUDA(cudaMemcpyAsync(out, b->p, count * sizeof(double), cudaMemcpyDeviceToHost, P->stream));
    DMK_CUDA(cudaStreamSynchronize(P->stream));
  });
}

int64_t dmk_stage_size(dmk_plan_t P, int which) {
  if (!P) return DMK_ERR_ARG;
  switch (which) {
    case DMK_STAGE_MOMENTS: return (int64_t)P->mom.n;
    case DMK_STAGE_OUTGOING: return P->phi_count;
    case DMK_STAGE_LOCAL: return (int64_t)P->lam.n;
    case DMK_STAGE_UFAR: return (int64_t)P->ufar.n;
    case DMK_STAGE_UNEAR: return (int64_t)P->unear.n;
    default: return DMK_ERR_ARG;
  }
}

int dmk_eval_timings(dmk_plan_t P, double* ms, const char** names, int cap) {
  if (!P) return DMK_ERR_ARG;
  int rc = guard([&] { resolve_timings(P); });
  if (rc != DMK_OK) return rc;
  int k = 0;
  std::vector<std::pair<const char*, double>> all(P->tree_timings);
  all.insert(all.end(), P->timings.begin(), P->timings.end());
  for (auto& pr : all) {
    if (k >= cap) break;
    if (ms) ms[k] = pr.second;
    if (names) names[k] = pr.first;
    ++k;
  }
  return k;
}

int64_t dmk_kernel_launches(int64_t* cub_calls) {
  if (cub_calls) *cub_calls = g_cub_launches;
  return g_launches;
}

}  // extern "C"
