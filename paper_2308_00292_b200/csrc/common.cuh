// common.cuh -- internal types of libdmk (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <memory>
#include <string>
#include <vector>

#include "../../include/dmk.h"

namespace dmk {
extern int64_t g_launches, g_cub_launches;
extern thread_local int64_t g_alloc_bytes;   // bytes requested through DevBuf on this thread

constexpr int NBITS = 21;  // bits per coordinate of the 63-bit Morton key
constexpr int LMAX = 20;   // deepest level a box may be refined into

// ---------------------------------------------------------------- errors
struct Error {
  int code;
  std::string msg;
};
void set_error(const std::string& m);
[[noreturn]] void fail(int code, const std::string& m);

#define DMK_CUDA(call)                                                                  \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      ::dmk::fail(DMK_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_) +   \
                                    " (" + __FILE__ + ":" + std::to_string(__LINE__) + ")"); \
  } while (0)
// placed directly after each of libdmk's own kernel launches: counts it, checks it
#define DMK_LAUNCH_CHECK()     \
  do {                         \
    ++::dmk::g_launches;       \
    DMK_CUDA(cudaGetLastError()); \
  } while (0)

// ---------------------------------------------------------------- device buffer
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void alloc(size_t count, cudaStream_t st) {
    release();
    s = st;
    n = count;
    if (count) DMK_CUDA(cudaMallocAsync((void**)&p, count * sizeof(T), st));
    g_alloc_bytes += (int64_t)(count * sizeof(T));
  }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  T* get() const { return p; }
  size_t bytes() const { return n * sizeof(T); }
};

// One same-level leaf pair (B, S) of the symmetric near field (kernels.cu k_p2p32s):
// point ranges, the partial-sum slots of B's entry for S and S's entry for B (int64),
// and c_B - c_S (exact fp32) with 1/r_L; S == B (nS < 0 marks it): one-sided
struct SymTask {
  int4 rng;         // bB, nB, bS, nS (nS = -nB: the leaf with itself)
  longlong2 slot;   // slotB, slotS
  float4 geo;       // c_B - c_S (x, y, z), 1/r_L
};

// ---------------------------------------------------------------- tables (Step 1)
// Per-precision tables, computed on the host once and kept on the device.
struct Tables {
  int dim = 3;
  int kernel = 0;
  double lam = 0;          // Yukawa parameter in unit-root-cube coordinates (0 for 1/r)
  double eps = 0, c = 0;
  int p = 0, nf = 0, nf0 = 0;
  double RT = 0, P0 = 0;   // root window truncation radius and Fourier period
  // host copies
  int pp = 0;                   // p rounded up to even (row length of Qr)
  std::vector<double> Qr1, Qr0; // [nf+1][pp] real parity-split plane-wave matrix, levels>=1 / root
  std::vector<double> Gr1, Gr0; // [p][hh] back transform, hh = nf+1 rounded up to even
  std::vector<double> A;        // [2][p][p]: A_s[n][k], T_n(x/2 + s/2) = sum_k A_s[n][k] T_k(x), s=-1,+1
  std::vector<double> W;        // [LMAX+1][nh][nh][nh] difference-kernel weights (|m1|,|m2|,|m3|)
  std::vector<double> W0;       // [nh0][nh0][nh0] root window weights
  std::vector<double> respoly;  // residual: M_L(r) r_L ~= sum_k a_k s^k, s = 2 r^2/r_L^2 - 1
  std::vector<double> respoly_lv;   // [LMAX+1][respoly_deg+1]: per-level coefficients
  int respoly_deg = 0;
  double m0 = 0;                // r_0 M_0(0) (1/r: psi(0)/c0 at every level)
  // device copies
  double *dQr1 = nullptr, *dQr0 = nullptr, *dGr1 = nullptr, *dGr0 = nullptr, *dA = nullptr, *dW = nullptr,
         *dW0 = nullptr, *dRespoly = nullptr;
  size_t wstride = 0;
  int dev = -1;   // device holding the d* arrays (freed with the last reference)
  Tables() = default;
  Tables(const Tables&) = delete;
  Tables& operator=(const Tables&) = delete;
  ~Tables();
};
// cached per (device, kernel, precision row, lambda'); throws via fail()
std::shared_ptr<const Tables> get_tables(int kernel, double eps, double lam);
size_t tables_cached();   // number of cached table sets (tests)
double snap_eps(double eps);

// ---------------------------------------------------------------- plan
struct TreeHost {
  int nlevels = 0;
  std::vector<int64_t> level_off;   // boxes of level l: [level_off[l], level_off[l+1])
  std::vector<int64_t> fout_off;    // F_out boxes (ranked by box index) per level
  std::vector<int64_t> exp_off;     // local-expansion boxes per level
};

}  // namespace dmk

struct dmk_plan_s {
  int dim = 3, kernel = 0, ns = 200;
  double eps = 0, lambda = 0;   // lambda: Yukawa parameter in the caller's units
  int64_t n = 0;
  cudaStream_t stream = 0;
  std::shared_ptr<const dmk::Tables> tab_ref;   // keeps the tables alive (cache may evict)
  const dmk::Tables* tab = nullptr;
  bool profile = false;        // DMK_PROFILE=1: per-phase CUDA events in dmk_eval (no host syncs)
  bool profile_tree = false;   // DMK_PROFILE_TREE=1: synchronising phase marks in dmk_plan
  bool evaluated = false;
  bool upward_done = false;

  // root cube
  double lo[3] = {0, 0, 0};
  double side = 1;
  bool root_fixed = false;   // lo/side given by the caller (dmk_options.root)
  int min_level = 0;         // levels < min_level fully refined (dmk_options.min_level)
  int64_t n_targets = 0;     // the first n_targets caller points are targets (= n by default)
  bool fast_sort = true;     // 3D: sort the top 24 key bits first (DMK_FULL_SORT=1: all 63)
  int sorted_from_bit = 0;   // 0: keys fully sorted; else only bits >= this are ordered

  // sorted points (normalised coordinates in [0,1]^3) and permutation
  dmk::DevBuf<uint64_t> keys;
  dmk::DevBuf<int32_t> perm;        // sorted -> caller index
  dmk::DevBuf<double> xs, ys, zs;

  // boxes
  int64_t nbox = 0;
  dmk::TreeHost th;
  dmk::DevBuf<uint64_t> box_code;
  dmk::DevBuf<int32_t> box_level, box_start, box_end, box_parent, box_child /*8*nbox*/,
      box_coll /*27*nbox*/;
  dmk::DevBuf<uint8_t> box_flags;   // bit0 leaf, bit1 F_out, bit2 F_in, bit3 local expansion
  dmk::DevBuf<int32_t> fout_rank, exp_rank;      // per box, -1 if none
  dmk::DevBuf<int32_t> fout_list, exp_list;      // box ids, ordered by box id (=> by level)
  int64_t nfout = 0, nexp = 0;
  // direct lists (CSR over boxes)
  dmk::DevBuf<int32_t> dlist_off, dlist;
  int64_t ndlist = 0;
  // symmetric near field (3D fp32 tier, kernels.cu k_p2p32s): per box the number of
  // same-level entries (the list's prefix) and the first of its (entry, target)
  // partial-sum slots; per box the first mixed-level entry (the queue form's range);
  // the partial sums (fp32, one per same-level entry and target); the number of
  // mixed-level entries
  dmk::DevBuf<int32_t> dlist_same, dlist_mbeg;
  dmk::DevBuf<uint32_t> dlist_cmask;   // per box: its non-empty leaf colleagues (bit = slot)
  dmk::DevBuf<int64_t> part_off;
  dmk::DevBuf<float> part;
  int64_t npart = 0, nmixed = 0;
  // the symmetric form's tasks (one per same-level leaf pair, S >= B), appended on the
  // device (the count stays there: the kernel is persistent), capacity = same-level entries
  dmk::DevBuf<dmk::SymTask> sym_tasks;
  dmk::DevBuf<int32_t> sym_ntask;
  int64_t sym_cap = 0;
  // work list for the P2P kernel: (leaf box, first target) items of <= 32 targets
  dmk::DevBuf<int32_t> p2p_items;
  int64_t np2p = 0;
  // Sec. 3.4 form (3D): octant offsets of every leaf, octant work items (leaf, octant,
  // t0, t1), number of target leaves (the form is chosen for big leaves)
  dmk::DevBuf<int32_t> leaf_oct;
  dmk::DevBuf<int4> p2p_items_o;
  int64_t np2p_o = 0, nleaf_t = 0;
  // fp32 P2P tier (p <= 18): leaf-local double-single source records, Morton order:
  // (x, y, z, rho) high parts and (x, y, z, 0) low parts
  dmk::DevBuf<float4> xl4, xl4lo;
  dmk::DevBuf<float4> box_c4;       // 3D: box centre and side in fp32 (exact, dyadic)
  // anterpolation / evaluation work: box ids
  dmk::DevBuf<int32_t> anterp_list, eval_list;
  int64_t nanterp = 0, neval = 0;
  std::vector<int64_t> c2p_off, p2c_off;   // per-level ranges into fout_list / exp_list

  // eval buffers
  dmk::DevBuf<double> q, mom, lam, ufar, unear;
  // outgoing plane waves: phi_count values, stored as fp32 (phi_f32, the 3D p <= 18 tier,
  // reading R16) or fp64; the buffer is sized in bytes for the stored type
  dmk::DevBuf<double> phi;
  int64_t phi_count = 0;
  bool phi_f32 = false;
  dmk::DevBuf<float> pwt;                 // fp32 tier: translated + weighted plane waves per local box
  dmk::DevBuf<double> pwt64;              // eps = 1e-9 (p = 28): the same in fp64
  dmk::DevBuf<double> scalar;             // device scratch scalar (2D: total charge)
  int64_t phi_size0 = 0, phi_size1 = 0;   // doubles per root / per other box

  // profiling
  std::vector<std::pair<const char*, double>> timings;
  std::vector<std::pair<const char*, double>> tree_timings;
  struct Mark {
    const char* name;
    cudaEvent_t e0, e1;
  };
  std::vector<Mark> ev_marks;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  // near-field branch: side stream + fork/join events (created with the plan)
  // streams and events from a process-wide pool (creating them costs more than a
  // small evaluation): near field (lowest priority), far field and the root-box chain
  // (highest priority), fork/join events
  cudaStream_t side_stream = nullptr, hi_stream = nullptr, root_stream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_root = nullptr;
  int pool_dev = -1;
  bool p2p_pending = false;   // a near-field branch was forked and not yet joined
  bool serial = false;        // DMK_SERIAL=1: near field on the plan stream (no overlap)
  ~dmk_plan_s();
};

namespace dmk {
void resolve_timings(dmk_plan_s* P);
void eval_plan_2d(dmk_plan_s* PL, double* dout);
void eval_upward(dmk_plan_s* PL, const double* dcharges);
void eval_downward(dmk_plan_s* PL, double* dout);
void level_moments(dmk_plan_s* PL, int level, double* ddense, bool set);
void box_moments(dmk_plan_s* PL, int level, const int64_t* dcodes, int64_t nb, double* dvals, bool set);
// cumulative number of libdmk kernel launches (this library's own kernels; the
// CUB sort/scan/select kernels compiled into the library are counted separately)
extern int64_t g_launches, g_cub_launches;
}  // namespace dmk
