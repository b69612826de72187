// tree.cu -- device-resident adaptive 2^D-tree (octree D = 3, quadtree D = 2) and
// interaction lists
// (Sec. 3.5 Step 0; Sec. 3.2; lists of
// Sec. 3.3 / Fig. 7).
//
// Everything point- or box-sized runs in CUDA kernels; the host only reads back
// counts to size the next level's arrays.  Conventions (readings R5-R8 of
// DESIGN.md) are identical to the oracle's, so the integer structure must match it
// bit for bit:
//   root cube lo = per-axis min, side = max extent; q = floor((x - lo) * (2^21/side))
//   (IEEE-rounded subtract, then multiply: no FMA contraction), 63-bit Morton keys
//   (x most significant), stable sort; refine a box iff it holds > n_s points and its
//   level is < LMAX; 2:1 balance over closed-box contact, built bottom-up; keep all
//   non-leaf boxes and all non-empty leaves, numbered by (level, Morton code).
#include <chrono>
#include <cstdlib>
#include <cstring>

#include <cub/cub.cuh>

#include "common.cuh"
#include "device.cuh"

namespace dmk {
namespace {

constexpr int TPB = 256;
inline int nblk(int64_t n, int t = TPB) { return (int)((n + t - 1) / t); }

template <class F>
void cub_run(cudaStream_t s, F f) {
  size_t bytes = 0;
  DMK_CUDA(f(nullptr, bytes));
  DevBuf<char> tmp;
  tmp.alloc(bytes ? bytes : 1, s);
  DMK_CUDA(f(tmp.p, bytes));
  ++g_cub_launches;
}

__device__ __forceinline__ uint64_t spread3(uint64_t x) {
  x &= 0x1fffffULL;
  x = (x | x << 32) & 0x1f00000000ffffULL;
  x = (x | x << 16) & 0x1f0000ff0000ffULL;
  x = (x | x << 8) & 0x100f00f00f00f00fULL;
  x = (x | x << 4) & 0x10c30c30c30c30c3ULL;
  x = (x | x << 2) & 0x1249249249249249ULL;
  return x;
}
__device__ __forceinline__ uint32_t compact3(uint64_t x) {
  x &= 0x1249249249249249ULL;
  x = (x ^ (x >> 2)) & 0x10c30c30c30c30c3ULL;
  x = (x ^ (x >> 4)) & 0x100f00f00f00f00fULL;
  x = (x ^ (x >> 8)) & 0x1f0000ff0000ffULL;
  x = (x ^ (x >> 16)) & 0x1f00000000ffffULL;
  x = (x ^ (x >> 32)) & 0x1fffffULL;
  return (uint32_t)x;
}
__device__ __forceinline__ uint64_t spread2(uint64_t x) {
  x &= 0x1fffffULL;
  x = (x | x << 16) & 0x0000ffff0000ffffULL;
  x = (x | x << 8) & 0x00ff00ff00ff00ffULL;
  x = (x | x << 4) & 0x0f0f0f0f0f0f0f0fULL;
  x = (x | x << 2) & 0x3333333333333333ULL;
  x = (x | x << 1) & 0x5555555555555555ULL;
  return x;
}
__device__ __forceinline__ uint32_t compact2(uint64_t x) {
  x &= 0x5555555555555555ULL;
  x = (x ^ (x >> 1)) & 0x3333333333333333ULL;
  x = (x ^ (x >> 2)) & 0x0f0f0f0f0f0f0f0fULL;
  x = (x ^ (x >> 4)) & 0x00ff00ff00ff00ffULL;
  x = (x ^ (x >> 8)) & 0x0000ffff0000ffffULL;
  x = (x ^ (x >> 16)) & 0x00000000ffffffffULL;
  return (uint32_t)x & 0x1fffff;
}
// Morton code of integer box coordinates c[0..D-1]; coordinate 0 most significant in
// each D-tuple of bits
template <int D>
__device__ __forceinline__ uint64_t encode(const int* c) {
  if (D == 3) return (spread3(c[0]) << 2) | (spread3(c[1]) << 1) | spread3(c[2]);
  return (spread2(c[0]) << 1) | spread2(c[1]);
}
template <int D>
__device__ __forceinline__ void decode(uint64_t code, int* c) {
  if (D == 3) {
    c[0] = (int)compact3(code >> 2);
    c[1] = (int)compact3(code >> 1);
    c[2] = (int)compact3(code);
  } else {
    c[0] = (int)compact2(code >> 1);
    c[1] = (int)compact2(code);
  }
}
template <int D>
struct Dim {
  static constexpr int NCH = 1 << D, NCOL = D == 3 ? 27 : 9;
};

// binary search for `v` in sorted a[0..n); returns index or -1
__device__ __forceinline__ int64_t bsearch_u64(const uint64_t* a, int64_t n, uint64_t v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return (lo < n && a[lo] == v) ? lo : -1;
}
__device__ __forceinline__ int64_t lower_bound_u64(const uint64_t* a, int64_t n, uint64_t v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// ---------------------------------------------------------------- kernels
template <int D>
__global__ void k_bbox_partial(const double* __restrict__ pts, int64_t n, double* out) {
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    for (int d = 0; d < D; ++d) {
      double v = pts[D * i + d];
      mn[d] = fmin(mn[d], v);
      mx[d] = fmax(mx[d], v);
    }
  __shared__ double s[6][TPB];
  for (int d = 0; d < 3; ++d) {
    s[d][threadIdx.x] = mn[d];
    s[3 + d][threadIdx.x] = mx[d];
  }
  __syncthreads();
  for (int w = TPB / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w)
      for (int d = 0; d < 3; ++d) {
        s[d][threadIdx.x] = fmin(s[d][threadIdx.x], s[d][threadIdx.x + w]);
        s[3 + d][threadIdx.x] = fmax(s[3 + d][threadIdx.x], s[3 + d][threadIdx.x + w]);
      }
    __syncthreads();
  }
  if (threadIdx.x < 6) out[blockIdx.x * 6 + threadIdx.x] = s[threadIdx.x][0];
}

// root cube on the device (reading R5): lo = per-axis minimum, side = max extent (1 if
// 0), scale = 2^21/side; bad = non-finite coordinates.  Read by the key and gather
// kernels without a host round trip; the host copy is read at the next synchronisation.
struct Geo {
  double lo[3], side, scale;
  int bad;
};
template <int D>
__global__ void __launch_bounds__(TPB) k_bbox_final(const double* __restrict__ part, int nb, Geo* g) {
  __shared__ double sm[6][TPB];
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int b = threadIdx.x; b < nb; b += TPB)
    for (int d = 0; d < D; ++d) {
      mn[d] = fmin(mn[d], part[6 * b + d]);
      mx[d] = fmax(mx[d], part[6 * b + 3 + d]);
    }
  for (int d = 0; d < 3; ++d) {
    sm[d][threadIdx.x] = mn[d];
    sm[3 + d][threadIdx.x] = mx[d];
  }
  __syncthreads();
  for (int w = TPB / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w)
      for (int d = 0; d < 3; ++d) {
        sm[d][threadIdx.x] = fmin(sm[d][threadIdx.x], sm[d][threadIdx.x + w]);
        sm[3 + d][threadIdx.x] = fmax(sm[3 + d][threadIdx.x], sm[3 + d][threadIdx.x + w]);
      }
    __syncthreads();
  }
  if (threadIdx.x != 0) return;
  for (int d = 0; d < 3; ++d) {
    mn[d] = sm[d][0];
    mx[d] = sm[3 + d][0];
  }
  double ext = 0;
  for (int d = 0; d < 3; ++d) g->lo[d] = d < D ? mn[d] : 0.0;
  for (int d = 0; d < D; ++d) ext = fmax(ext, mx[d] - mn[d]);
  g->bad = isfinite(ext) ? 0 : 1;
  g->side = ext > 0 ? ext : 1.0;
  g->scale = (double)(1 << NBITS) / g->side;
}

template <int D>
__global__ void k_keys(const double* __restrict__ pts, int64_t n, const Geo* __restrict__ g, uint64_t* keys,
                       int32_t* idx) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double lo[3] = {g->lo[0], g->lo[1], g->lo[2]}, scale = g->scale;
  int q[3];
  for (int d = 0; d < D; ++d) {
    double t = floor(__dmul_rn(__dsub_rn(pts[D * i + d], lo[d]), scale));
    t = fmin(fmax(t, 0.0), (double)((1 << NBITS) - 1));
    q[d] = (int)t;
  }
  keys[i] = encode<D>(q);
  idx[i] = (int32_t)i;
}

template <int D>
__global__ void k_gather_pts(const double* __restrict__ pts, const int32_t* __restrict__ perm, int64_t n,
                             const Geo* __restrict__ g, double* xs, double* ys, double* zs) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double lo0 = g->lo[0], lo1 = g->lo[1], lo2 = g->lo[2], side = g->side;
  int64_t j = perm[i];
  xs[i] = __ddiv_rn(__dsub_rn(pts[D * j + 0], lo0), side);
  ys[i] = __ddiv_rn(__dsub_rn(pts[D * j + 1], lo1), side);
  if (D == 3) zs[i] = __ddiv_rn(__dsub_rn(pts[D * j + 2], lo2), side);
}

// level-l box of point a is "big" (> ns points) and a is its first point
template <int D>
__global__ void k_big(const uint64_t* __restrict__ keys, int64_t n, int l, int ns, uint64_t* codes,
                      uint8_t* flags) {
  int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a >= n) return;
  int sh = D * (NBITS - l);
  uint64_t c = (sh >= 64) ? 0 : (keys[a] >> sh);
  bool start = (a == 0) || (((sh >= 64) ? 0 : (keys[a - 1] >> sh)) != c);
  bool big = (a + ns < n) && ((((sh >= 64) ? 0 : (keys[a + ns] >> sh))) == c);
  codes[a] = c;
  flags[a] = (start && big) ? 1 : 0;
}

// number of "big" level-l boxes (> ns points) for every level, one pass over the keys
template <int D>
__global__ void k_count_big(const uint64_t* __restrict__ keys, int64_t n, int ns, int l0, unsigned long long* cnt) {
  __shared__ unsigned int c[LMAX];
  for (int l = threadIdx.x; l < LMAX; l += blockDim.x) c[l] = 0;
  __syncthreads();
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < n; a += (int64_t)gridDim.x * blockDim.x) {
    for (int l = l0; l < LMAX; ++l) {
      const int sh = D * (NBITS - l);
      const uint64_t cd = (sh >= 64) ? 0 : (keys[a] >> sh);
      const bool big = (a + ns < n) && (((sh >= 64) ? 0 : (keys[a + ns] >> sh)) == cd);
      if (!big) break;   // the level-l box of a holds <= ns points from a on: so do its children
      const bool start = (a == 0) || (((sh >= 64) ? 0 : (keys[a - 1] >> sh)) != cd);
      if (start) atomicAdd(&c[l], 1u);
    }
  }
  __syncthreads();
  for (int l = threadIdx.x; l < LMAX; l += blockDim.x)
    if (c[l]) atomicAdd(&cnt[l], (unsigned long long)c[l]);
}

// the level-l boxes touching each level-(l+1) box q (2^D candidates, clipped)
template <int D>
__global__ void k_touch(const uint64_t* __restrict__ Bq, int64_t nq, int l, uint64_t* out, uint8_t* flags,
                        uint64_t sentinel = 0) {
  constexpr int NCH = Dim<D>::NCH;
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nq * NCH) return;
  int64_t i = t / NCH;
  int o = (int)(t % NCH);
  int q[3], c[3];
  decode<D>(Bq[i], q);
  int n1 = 1 << l;
  bool ok = true;
  for (int d = 0; d < D; ++d) {
    int lo = (q[d] % 2 == 0) ? q[d] / 2 - 1 : q[d] / 2;
    c[d] = lo + ((o >> (D - 1 - d)) & 1);
    ok = ok && c[d] >= 0 && c[d] < n1;
  }
  out[t] = ok ? encode<D>(c) : sentinel;
  if (flags) flags[t] = ok ? 1 : 0;
}


// box set of level l: children of the level-(l-1) non-leaf boxes that hold points or are
// themselves non-leaf (candidates enumerated in Morton order, so the selection is sorted)
template <int D>
__global__ void k_child_cand(const uint64_t* __restrict__ Bp, int64_t nBp, const uint64_t* __restrict__ Bl,
                             int64_t nBl, const uint64_t* __restrict__ keys, int64_t n, int l, uint64_t* codes,
                             uint8_t* flags) {
  constexpr int NCH = 1 << D;
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nBp * NCH) return;
  const uint64_t c = (Bp[t / NCH] << D) | (uint64_t)(t % NCH);
  const int sh = D * (NBITS - l);
  const int64_t lb = lower_bound_u64(keys, n, c << sh);
  const bool nonempty = lb < n && (keys[lb] >> sh) == c;
  const bool nonleaf = nBl > 0 && bsearch_u64(Bl, nBl, c) >= 0;
  codes[t] = c;
  flags[t] = (nonempty || nonleaf) ? 1 : 0;
}

// ---- coarse levels as dense bitmaps (levels 0..LBC: 2^{D l} bits each), so that the
// balance and the box sets of these levels need no sort and no host round trip.
template <int D>
struct Coarse {
  static constexpr int LBC = D == 3 ? 7 : 10;   // 2^21 bits at the finest coarse level
  int64_t woff[LBC + 2];                        // word offset of each level
};
__device__ __forceinline__ void bm_set(uint32_t* bm, uint64_t bit) { atomicOr(bm + (bit >> 5), 1u << (bit & 31)); }
__device__ __forceinline__ bool bm_get(const uint32_t* bm, uint64_t bit) { return (bm[bit >> 5] >> (bit & 31)) & 1u; }

// per point: non-empty boxes (NE) and big boxes (U, > ns points, level >= l0) of every
// coarse level whose first point it is
template <int D>
__global__ void k_mark_coarse(const uint64_t* __restrict__ keys, int64_t n, int ns, int l0, Coarse<D> cs,
                              uint32_t* bmU, uint32_t* bmNE) {
  const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a >= n) return;
  const uint64_t k = keys[a], kp = a > 0 ? keys[a - 1] : 0, kb = a + ns < n ? keys[a + ns] : 0;
  for (int l = 0; l <= Coarse<D>::LBC; ++l) {
    const int sh = D * (NBITS - l);
    const uint64_t c = k >> sh;
    if (a > 0 && (kp >> sh) == c) continue;   // not the first point of its level-l box
    bm_set(bmNE + cs.woff[l], c);
    if (l >= l0 && l < LMAX && a + ns < n && (kb >> sh) == c) bm_set(bmU + cs.woff[l], c);
  }
}
// every bit of a level (forced refinement of the levels above min_level)
__global__ void k_bm_all(uint32_t* bm, int64_t nbits) {
  const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (w * 32 >= nbits) return;
  const int64_t r = nbits - w * 32;
  bm[w] = r >= 32 ? 0xffffffffu : ((1u << r) - 1u);
}
// balance: the level-l boxes touching each level-(l+1) box of B_{l+1} (list or bitmap),
// set in the level-l bitmap (R7, closed contact; see k_touch)
template <int D>
__device__ __forceinline__ void touch_set(uint64_t q, int l, uint32_t* out) {
  constexpr int NCH = Dim<D>::NCH;
  int x[3], c[3];
  decode<D>(q, x);
  const int n1 = 1 << l;
  for (int o = 0; o < NCH; ++o) {
    bool ok = true;
    for (int d = 0; d < D; ++d) {
      const int lo = (x[d] % 2 == 0) ? x[d] / 2 - 1 : x[d] / 2;
      c[d] = lo + ((o >> (D - 1 - d)) & 1);
      ok = ok && c[d] >= 0 && c[d] < n1;
    }
    if (ok) bm_set(out, encode<D>(c));
  }
}
template <int D>
__global__ void k_touch_list_bm(const uint64_t* __restrict__ Bq, int64_t nq, int l, uint32_t* out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < nq) touch_set<D>(Bq[i], l, out);
}
template <int D>
__global__ void k_touch_bm(const uint32_t* __restrict__ in, int64_t nbits_in, int l, uint32_t* out) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b < nbits_in && bm_get(in, b)) touch_set<D>((uint64_t)b, l, out);
}
// E_l = B_l + non-empty children of B_{l-1}, word by word
template <int D>
__global__ void k_E_bm(const uint32_t* __restrict__ Bl, const uint32_t* __restrict__ NEl,
                       const uint32_t* __restrict__ Bp, int64_t nbits, uint32_t* El) {
  const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (w * 32 >= nbits) return;
  uint32_t e = Bl[w], ne = NEl[w], m = 0;
  for (int i = 0; i < 32 && w * 32 + i < nbits; ++i)
    if (bm_get(Bp, (uint64_t)(w * 32 + i) >> D)) m |= 1u << i;
  El[w] = e | (ne & m);
}
__global__ void k_popc(const uint32_t* __restrict__ bm, int64_t nw, int32_t* cnt) {
  const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (w < nw) cnt[w] = __popc(bm[w]);
}
// codes of the set bits of one level (sorted), at exclusive-scan positions
__global__ void k_bm_fill(const uint32_t* __restrict__ bm, const int32_t* __restrict__ pos, int64_t nw,
                          uint64_t* out) {
  const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (w >= nw) return;
  uint32_t x = bm[w];
  int32_t p = pos[w] - pos[0];
  while (x) {
    const int b = __ffs(x) - 1;
    out[p++] = (uint64_t)(w * 32 + b);
    x &= x - 1;
  }
}
// all-coarse trees: the box arrays (code, level) straight from the E bitmaps, every
// level in one launch (box index = level offset + rank within the level)
struct CoarseFill {   // by value
  int64_t woff[12], loff[12];
  int nl;
};
__global__ void k_coarse_boxes(const uint32_t* __restrict__ bmE, const int32_t* __restrict__ posE, CoarseFill cf,
                               uint64_t* code, int32_t* level) {
  const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (w >= cf.woff[cf.nl]) return;
  int l = 0;
  while (w >= cf.woff[l + 1]) ++l;
  uint32_t x = bmE[w];
  int64_t p = cf.loff[l] + (posE[w] - posE[cf.woff[l]]);
  const uint64_t base = (uint64_t)(w - cf.woff[l]) * 32;
  while (x) {
    const int b = __ffs(x) - 1;
    code[p] = base + b;
    level[p] = l;
    ++p;
    x &= x - 1;
  }
}

// per-level totals of a scanned bitmap: tot[l] = pos[woff[l+1]] - pos[woff[l]] (pos has
// one extra trailing entry)
template <int D>
__global__ void k_bm_totals(const int32_t* __restrict__ pos, Coarse<D> cs, int64_t base, int64_t* tot) {
  const int l = threadIdx.x;
  if (l <= Coarse<D>::LBC) tot[l] = pos[base + cs.woff[l + 1]] - pos[base + cs.woff[l]];
}


struct ReadIdx {   // by value
  int64_t v[LMAX + 3];
  int m;
};
// out[i] = fscan[v[i]], out[m + i] = escan[v[i]] (i < m), out[2m] = dlist_off[nbox],
// out[2m + 1] = poff[nbox]: every host-side size of the plan in one read-back
__global__ void k_read_totals(const int32_t* __restrict__ fscan, const int32_t* __restrict__ escan, ReadIdx ri,
                              const int32_t* __restrict__ doff, const int32_t* __restrict__ poff,
                              const int32_t* __restrict__ poff_o, const unsigned long long* __restrict__ nleaf,
                              const int64_t* __restrict__ part_off, const unsigned long long* __restrict__ same_tot,
                              int64_t nbox, int64_t* out) {
  const int i = threadIdx.x;
  if (i < ri.m) {
    out[i] = fscan[ri.v[i]];
    out[ri.m + i] = escan[ri.v[i]];
  }
  if (i == 0) {
    out[2 * ri.m] = doff[nbox];
    out[2 * ri.m + 1] = poff[nbox];
    out[2 * ri.m + 2] = poff_o ? poff_o[nbox] : 0;
    out[2 * ri.m + 3] = nleaf ? (int64_t)*nleaf : 0;
    out[2 * ri.m + 4] = part_off ? part_off[nbox] : 0;
    out[2 * ri.m + 5] = same_tot ? (int64_t)*same_tot : 0;
  }
}


__global__ void k_fill_level(int32_t* lev, int64_t a, int64_t b, int l) {
  int64_t i = a + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < b) lev[i] = l;
}

struct BoxCtx {   // passed by value (no host-to-device copies)
  const uint64_t* code;
  const int32_t* level;
  int64_t loff[LMAX + 2];   // level offsets [nlevels+1]
  const uint64_t* B;        // concatenated non-leaf sets
  int64_t boff[LMAX + 2];   // offsets of B per level [nlevels+1]
  int nlevels;
  const uint64_t* keys;
  int64_t n;
  // coarse levels (<= lbc): B and E bitmaps and the exclusive scan of the E words, so a
  // box's index is a rank (one word and one popcount) instead of a binary search
  int lbc;
  int64_t woff[12];         // word offsets per coarse level
  const uint32_t* bmB;
  const uint32_t* bmE;
  const int32_t* posE;
};
__device__ __forceinline__ int64_t bm_rank(const BoxCtx& c, int l, uint64_t code) {
  const int64_t w0 = c.woff[l], w = w0 + (int64_t)(code >> 5);
  return (int64_t)(c.posE[w] - c.posE[w0]) + __popc(c.bmE[w] & ((1u << (code & 31)) - 1u));
}

template <int D>
__global__ void k_box_attrs(BoxCtx c, int64_t nbox, int32_t* start, int32_t* end, int32_t* parent,
                            int32_t* coll, uint8_t* flags) {
  constexpr int NCOL = Dim<D>::NCOL;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nbox) return;
  int l = c.level[i];
  uint64_t code = c.code[i];
  int sh = D * (NBITS - l);
  uint64_t lo = (sh >= 64) ? 0 : (code << sh);
  uint64_t hiv = (sh >= 64) ? ~0ULL : ((code + 1) << sh);
  int64_t s = lower_bound_u64(c.keys, c.n, lo);
  int64_t e = (l == 0) ? c.n : lower_bound_u64(c.keys, c.n, hiv);
  start[i] = (int32_t)s;
  end[i] = (int32_t)e;
  if (l <= c.lbc) {
    flags[i] = bm_get(c.bmB + c.woff[l], code) ? 0 : 1;
    parent[i] = l > 0 ? (int32_t)(c.loff[l - 1] + bm_rank(c, l - 1, code >> D)) : -1;
    int x[3];
    decode<D>(code, x);
    const int n1 = 1 << l;
    for (int k = 0; k < NCOL; ++k) {
      int cc[3], rem = k;
      bool ok = true;
      for (int d = D - 1; d >= 0; --d) {
        cc[d] = x[d] + (rem % 3) - 1;
        rem /= 3;
        ok = ok && cc[d] >= 0 && cc[d] < n1;
      }
      int32_t r = -1;
      if (ok) {
        const uint64_t nb = encode<D>(cc);
        if (bm_get(c.bmE + c.woff[l], nb)) r = (int32_t)(c.loff[l] + bm_rank(c, l, nb));
      }
      coll[NCOL * i + k] = r;
    }
    return;
  }
  bool leaf = bsearch_u64(c.B + c.boff[l], c.boff[l + 1] - c.boff[l], code) < 0;
  flags[i] = leaf ? 1 : 0;
  if (l > 0) {
    int64_t j = bsearch_u64(c.code + c.loff[l - 1], c.loff[l] - c.loff[l - 1], code >> D);
    parent[i] = (int32_t)(j < 0 ? -1 : c.loff[l - 1] + j);
  } else {
    parent[i] = -1;
  }
  int x[3];
  decode<D>(code, x);
  int n1 = 1 << l;
  const uint64_t* lv = c.code + c.loff[l];
  int64_t nl = c.loff[l + 1] - c.loff[l];
  // slot k enumerates offsets in {-1,0,1}^D, last axis fastest
  for (int k = 0; k < NCOL; ++k) {
    int cc[3], rem = k;
    bool ok = true;
    for (int d = D - 1; d >= 0; --d) {
      cc[d] = x[d] + (rem % 3) - 1;
      rem /= 3;
      ok = ok && cc[d] >= 0 && cc[d] < n1;
    }
    int32_t r = -1;
    if (ok) {
      int64_t j = bsearch_u64(lv, nl, encode<D>(cc));
      if (j >= 0) r = (int32_t)(c.loff[l] + j);
    }
    coll[NCOL * i + k] = r;
  }
}

template <int D>
__global__ void k_children(const uint64_t* code, const int32_t* parent, int64_t nbox, int32_t* child) {
  constexpr int NCH = Dim<D>::NCH;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nbox) return;
  int32_t p = parent[i];
  if (p >= 0) child[NCH * (int64_t)p + (code[i] & (NCH - 1))] = (int32_t)i;
}

// flags: bit0 leaf, bit1 F_out, bit2 F_in, bit3 has local expansion
__global__ void k_flags_out(const int32_t* start, const int32_t* end, const int32_t* level, int min_level,
                            int64_t nbox, uint8_t* flags, uint8_t* fout) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nbox) return;
  bool leaf = flags[i] & 1;
  // forced coarse boxes (level < min_level) carry outgoing expansions even when locally
  // empty: their moments are injected from the other ranks (dmk_level_moments)
  bool f = !leaf && (end[i] > start[i] || level[i] < min_level);
  flags[i] = (uint8_t)((leaf ? 1 : 0) | (f ? 2 : 0));
  fout[i] = f ? 1 : 0;
}
template <int D>
__global__ void k_flags_in(const int32_t* start, const int32_t* end, const int32_t* coll, int64_t nbox,
                           uint8_t* flags, uint8_t* exp) {
  constexpr int NCOL = Dim<D>::NCOL;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nbox) return;
  uint8_t f = flags[i];
  bool nonempty = end[i] > start[i];
  bool fin = false;
  if (nonempty)
    for (int k = 0; k < NCOL; ++k) {
      int32_t s = coll[NCOL * i + k];
      if (s >= 0 && (flags[s] & 2)) fin = true;
    }
  // a local expansion only where there are targets (bit 4, k_flag_targets)
  bool e = nonempty && (f & 16) && (!(f & 1) || fin);
  // other threads only read bit 1 (F_out), which this write leaves unchanged
  flags[i] = (uint8_t)(f | (fin ? 4 : 0) | (e ? 8 : 0));
  exp[i] = e ? 1 : 0;
}

// bit 4 (F_TGT): the box holds at least one target point (all points, unless the plan
// was given n_targets < n: then the first n_targets caller points)
__global__ void k_target_flag_pts(const int32_t* __restrict__ perm, int64_t n, int64_t n_targets, int32_t* tf) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) tf[i] = perm[i] < n_targets ? 1 : 0;
}
__global__ void k_flag_targets(const int32_t* start, const int32_t* end, const int32_t* tscan, int64_t nbox,
                               uint8_t* flags) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nbox) return;
  const bool tgt = tscan ? tscan[end[i]] > tscan[start[i]] : end[i] > start[i];
  if (tgt) flags[i] |= 16;
}

// ranks in the compact F_out / local-expansion arrays and the compact box lists
// themselves (scatter by rank), both kinds in one pass
__global__ void k_ranks_lists(const int32_t* __restrict__ fscan, const uint8_t* __restrict__ fsel,
                              const int32_t* __restrict__ escan, const uint8_t* __restrict__ esel, int64_t nbox,
                              int32_t* frank, int32_t* erank, int32_t* flist, int32_t* elist) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nbox) return;
  const bool f = fsel[i], e = esel[i];
  frank[i] = f ? fscan[i] : -1;
  erank[i] = e ? escan[i] : -1;
  if (f) flist[fscan[i]] = (int32_t)i;
  if (e) elist[escan[i]] = (int32_t)i;
}

// direct lists: pass 0 counts, pass 1 fills; one warp per box, lanes over the colleague
// slots (and over the 3^D x 2^D fine-neighbour candidates), ballots for the positions
// box centre and side in fp32 (exact: dyadic, level <= 20): (c_x, c_y, c_z, 2^-l)
__device__ __forceinline__ float4 box_c4f(uint64_t c, int l) {
  const float sd = ldexpf(1.0f, -l);
  return make_float4(((float)compact3d(c >> 2) + 0.5f) * sd, ((float)compact3d(c >> 1) + 0.5f) * sd,
                     ((float)compact3d(c) + 0.5f) * sd, sd);
}
// Outputs of the direct-list passes for the symmetric near field (kernels.cu,
// k_p2p32s): per box the number of same-level entries (the list's prefix) and of
// (entry, target) partial-sum slots they need (count pass, with the total of
// same-level entries); per entry its owner box and per box the first mixed-level entry
// (fill pass).  Null pointers: not wanted.
struct NearAux {
  int32_t* same = nullptr;
  int64_t* slots = nullptr;
  unsigned long long* same_tot = nullptr;
  uint32_t* cmask = nullptr;        // per box: bit k = colleague k is a non-empty leaf (count pass)
  int32_t* owner = nullptr;
  int32_t* mbeg = nullptr;
  SymTask* tasks = nullptr;         // fill pass: the symmetric tasks (S >= B), appended
  int32_t* ntask = nullptr;
  const int64_t* part_off = nullptr;
};
template <int D, bool FILL>
__global__ void k_dlist(const int32_t* start, const int32_t* end, const int32_t* parent, const int32_t* child,
                        const int32_t* coll, const uint8_t* flags, const uint64_t* code, const int32_t* level,
                        int64_t nbox, int32_t* cnt, const int32_t* off, int32_t* items, NearAux aux) {
  constexpr int NCH = Dim<D>::NCH, NCOL = Dim<D>::NCOL;
  const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= nbox) return;
  const bool is_target = (flags[i] & 1) && end[i] > start[i];
  if (!is_target) {
    if (!FILL && lane == 0) {
      cnt[i] = 0;
      if (aux.same) aux.same[i] = 0;
      if (aux.slots) aux.slots[i] = 0;
    }
    return;
  }
  const unsigned below = (1u << lane) - 1;
  int n_ = 0;
  const int64_t base = FILL ? off[i] : 0;
  int64_t a = i;
  while (a >= 0) {   // B and its ancestors: leaf colleagues at that level
    int32_t s = lane < NCOL ? coll[NCOL * a + lane] : -1;
    const bool ok = s >= 0 && (flags[s] & 1) && end[s] > start[s];
    const unsigned m = __ballot_sync(0xffffffffu, ok);
    if (FILL && ok) {
      items[base + n_ + __popc(m & below)] = s;
      if (aux.owner) aux.owner[base + n_ + __popc(m & below)] = (int32_t)i;
    }
    if constexpr (FILL && D == 3) {
      if (a == i && aux.tasks) {
        // symmetric near-field tasks: colleague k = S (a non-empty leaf of B's level)
        // with S >= B; B is S's colleague 26 - k, so its entry in S's list is the number
        // of S's leaf colleagues before that slot
        const bool tk = ok && s >= (int32_t)i;
        const unsigned tm = __ballot_sync(0xffffffffu, tk);
        int pos = 0;
        if (tm) {
          int b0 = 0;
          if (lane == __ffs(tm) - 1) b0 = atomicAdd(aux.ntask, __popc(tm));
          pos = __shfl_sync(0xffffffffu, b0, __ffs(tm) - 1) + __popc(tm & below);
        }
        if (tk) {
          const int eB = __popc(m & below);
          const int eS = s == (int32_t)i ? eB : __popc(aux.cmask[s] & ((1u << (26 - lane)) - 1u));
          const int bB = start[i], nB = end[i] - bB, bS = start[s], nS = end[s] - bS;
          const float4 cB = box_c4f(code[i], level[i]), cS = box_c4f(code[s], level[s]);
          SymTask t;
          t.rng = make_int4(bB, nB, bS, s == (int32_t)i ? -nB : nS);
          t.slot = make_longlong2(aux.part_off[i] + (int64_t)eB * nB, aux.part_off[s] + (int64_t)eS * nS);
          t.geo = make_float4(cB.x - cS.x, cB.y - cS.y, cB.z - cS.z,
                              __int_as_float(0x7F000000 - __float_as_int(cB.w)));
          aux.tasks[pos] = t;
        }
      }
    }
    if (a == i && lane == 0) {
      // the same-level entries (B's own colleague leaves) are the list's prefix: the
      // symmetric near field takes them, the queue form the rest (mixed levels)
      const int ns = __popc(m);
      if (!FILL) {
        if (aux.cmask) aux.cmask[i] = m;
        if (aux.same) aux.same[i] = ns;
        if (aux.slots) aux.slots[i] = (int64_t)ns * (end[i] - start[i]);
        if (aux.same_tot) atomicAdd(aux.same_tot, (unsigned long long)ns);
      } else if (aux.mbeg) {
        aux.mbeg[i] = (int32_t)(base + ns);
      }
    }
    n_ += __popc(m);
    a = parent[a];
  }
  int bc[3];
  decode<D>(code[i], bc);
  for (int c0 = 0; c0 < NCOL * NCH; c0 += 32) {   // fine neighbours: leaves one level down touching B
    const int c = c0 + lane;
    bool ok = false;
    int32_t ch = -1;
    if (c < NCOL * NCH) {
      const int32_t s = coll[NCOL * i + c / NCH];
      if (s >= 0 && !(flags[s] & 1)) {
        ch = child[NCH * (int64_t)s + c % NCH];
        if (ch >= 0 && (flags[ch] & 1) && end[ch] > start[ch]) {
          int cc[3];
          decode<D>(code[ch], cc);
          ok = true;
          for (int d = 0; d < D; ++d) ok = ok && cc[d] >= 2 * bc[d] - 1 && cc[d] <= 2 * bc[d] + 2;
        }
      }
    }
    const unsigned m = __ballot_sync(0xffffffffu, ok);
    if (FILL && ok) {
      items[base + n_ + __popc(m & below)] = ch;
      if (aux.owner) aux.owner[base + n_ + __popc(m & below)] = (int32_t)i;
    }
    n_ += __popc(m);
  }
  if (!FILL && lane == 0) cnt[i] = n_;
}

// P2P work items: (leaf, first target) for every chunk of 32 targets
__global__ void k_p2p_count(const int32_t* start, const int32_t* end, const uint8_t* flags, int64_t nbox,
                            int32_t* cnt) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nbox) return;
  int n_ = end[i] - start[i];
  cnt[i] = ((flags[i] & 1) && (flags[i] & 16) && n_ > 0) ? (n_ + 31) / 32 : 0;
}
// Sec. 3.4, 3D: the octants of every leaf (its points are Morton
// sorted, so octant k is a contiguous range): oct[8 b + k] = first point of octant k.
__global__ void k_leaf_oct(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ code,
                           const int32_t* __restrict__ level, const int32_t* __restrict__ start,
                           const int32_t* __restrict__ end, const uint8_t* __restrict__ flags, int64_t nbox,
                           int32_t* oct) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t b = t >> 3;
  const int k = (int)(t & 7);
  if (b >= nbox) return;
  if (!(flags[b] & 1)) return;
  const int l = level[b];
  int64_t lo = start[b], hi = end[b];
  if (k > 0 && l < NBITS) {
    const int sh = 3 * (NBITS - l - 1);
    const uint64_t v = ((code[b] << 3) | (uint64_t)k) << sh;
    while (lo < hi) {   // first point of the leaf with key >= v
      const int64_t mid = (lo + hi) >> 1;
      if (keys[mid] < v) lo = mid + 1; else hi = mid;
    }
  } else if (k > 0) {
    lo = end[b];        // level-NBITS leaf: one octant
  }
  oct[8 * b + k] = (int32_t)lo;
}
// octant work items of the target leaves: (leaf, octant, t0, t1), <= 32 targets each;
// also counts the target leaves (for the host's choice of the P2P form)
__global__ void k_p2p_count_o(const int32_t* __restrict__ start, const int32_t* __restrict__ end,
                              const uint8_t* __restrict__ flags, const int32_t* __restrict__ oct, int64_t nbox,
                              int32_t* cnt, unsigned long long* nleaf) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nbox) return;
  int c = 0;
  if ((flags[i] & 1) && (flags[i] & 16) && end[i] > start[i]) {
    for (int k = 0; k < 8; ++k) {
      const int a = oct[8 * i + k], e = k < 7 ? oct[8 * i + k + 1] : end[i];
      c += (e - a + 31) / 32;
    }
    atomicAdd(nleaf, 1ull);
  }
  cnt[i] = c;
}
__global__ void k_p2p_fill_o(const int32_t* __restrict__ end, const int32_t* __restrict__ oct,
                             const int32_t* __restrict__ cnt, const int32_t* __restrict__ off, int64_t nbox,
                             int4* items) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nbox || cnt[i] == 0) return;
  int p = off[i];
  for (int k = 0; k < 8; ++k) {
    const int a = oct[8 * i + k], e = k < 7 ? oct[8 * i + k + 1] : end[i];
    for (int t0 = a; t0 < e; t0 += 32) items[p++] = make_int4((int)i, k, t0, min(e, t0 + 32));
  }
}
__global__ void k_p2p_fill(const int32_t* start, const int32_t* cnt, const int32_t* off, int64_t nbox,
                           int32_t* items) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nbox) return;
  for (int k = 0; k < cnt[i]; ++k) {
    items[2 * (off[i] + k)] = (int32_t)i;
    items[2 * (off[i] + k) + 1] = start[i] + 32 * k;
  }
}

// Leaf-local double-single source records for the fp32 P2P tier (reading R16): for the
// leaf B holding point i, d = x_i - c_B (fp64, exact), hi = fl32(d), lo = fl32(d - hi);
// xl4[i] = (hi_x, hi_y, hi_z, rho_i) (the charge slot is filled per evaluation) and
// xl4lo[i] = (lo_x, lo_y, lo_z, 0).
__global__ void k_leaf_local4(const uint64_t* code, const int32_t* level, const int32_t* start, const int32_t* end,
                              const uint8_t* flags, int64_t nbox, const double* xs, const double* ys,
                              const double* zs, float4* xl4, float4* xl4lo) {
  const int64_t b = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (b >= nbox || !(flags[b] & 1)) return;
  double c[3], ih;
  box_geom(code[b], level[b], c, ih);
  for (int i = start[b] + lane; i < end[b]; i += 32) {
    const double dx = xs[i] - c[0], dy = ys[i] - c[1], dz = zs[i] - c[2];
    const float hx = (float)dx, hy = (float)dy, hz = (float)dz;
    xl4[i] = make_float4(hx, hy, hz, 0.0f);
    xl4lo[i] = make_float4((float)(dx - hx), (float)(dy - hy), (float)(dz - hz), 0.0f);
  }
}

// box centres and sizes in fp32 (exact: dyadic, level <= 20): (c_x, c_y, c_z, 2^-l)
__global__ void k_box_c4(const uint64_t* code, const int32_t* level, int64_t nbox, float4* c4) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= nbox) return;
  const uint64_t c = code[b];
  const float s = ldexpf(1.0f, -level[b]);
  c4[b] = make_float4(((float)compact3d(c >> 2) + 0.5f) * s, ((float)compact3d(c >> 1) + 0.5f) * s,
                      ((float)compact3d(c) + 0.5f) * s, s);
}

// ---------------------------------------------------------------- host helpers
int64_t select_flagged(cudaStream_t s, const uint64_t* in, const uint8_t* flags, int64_t n,
                       DevBuf<uint64_t>& out) {
  DevBuf<uint64_t> tmp;
  tmp.alloc(n ? n : 1, s);
  DevBuf<int64_t> cnt;
  cnt.alloc(1, s);
  cub_run(s, [&](void* t, size_t& b) {
    return cub::DeviceSelect::Flagged(t, b, in, flags, tmp.p, cnt.p, n, s);
  });
  int64_t h = 0;
  DMK_CUDA(cudaMemcpyAsync(&h, cnt.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  DMK_CUDA(cudaStreamSynchronize(s));
  out.alloc(h ? h : 1, s);
  if (h) DMK_CUDA(cudaMemcpyAsync(out.p, tmp.p, h * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
  return h;
}

// sort + unique of n codes with `bits` significant bits
int64_t sort_unique(cudaStream_t s, const uint64_t* in, int64_t n, int bits, DevBuf<uint64_t>& out) {
  if (n == 0) {
    out.alloc(1, s);
    return 0;
  }
  DevBuf<uint64_t> sorted;
  sorted.alloc(n, s);
  cub_run(s, [&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortKeys(t, b, in, sorted.p, (int64_t)n, 0, bits > 0 ? bits : 1, s);
  });
  DevBuf<uint64_t> tmp;
  tmp.alloc(n, s);
  DevBuf<int64_t> cnt;
  cnt.alloc(1, s);
  cub_run(s, [&](void* t, size_t& b) {
    return cub::DeviceSelect::Unique(t, b, sorted.p, tmp.p, cnt.p, (int64_t)n, s);
  });
  int64_t h = 0;
  DMK_CUDA(cudaMemcpyAsync(&h, cnt.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  DMK_CUDA(cudaStreamSynchronize(s));
  out.alloc(h, s);
  DMK_CUDA(cudaMemcpyAsync(out.p, tmp.p, h * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
  return h;
}

__global__ void k_is_sentinel(const uint64_t* a, const int64_t* cnt, uint64_t sentinel, int64_t* out) {
  const int64_t c = *cnt;
  out[0] = c;
  out[1] = (c > 0 && a[c - 1] == sentinel) ? 1 : 0;
}

// sort + unique of n codes < 2^bits plus possibly the sentinel 2^bits (dropped): one
// round trip for the count
int64_t sort_unique_drop(cudaStream_t s, const uint64_t* in, int64_t n, int bits, DevBuf<uint64_t>& out) {
  const uint64_t sentinel = (uint64_t)1 << bits;
  DevBuf<uint64_t> sorted, tmp;
  sorted.alloc(n, s);
  tmp.alloc(n, s);
  cub_run(s, [&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortKeys(t, b, in, sorted.p, (int64_t)n, 0, bits + 1, s);
  });
  DevBuf<int64_t> cnt, res;
  cnt.alloc(1, s);
  res.alloc(2, s);
  cub_run(s, [&](void* t, size_t& b) {
    return cub::DeviceSelect::Unique(t, b, sorted.p, tmp.p, cnt.p, (int64_t)n, s);
  });
  k_is_sentinel<<<1, 1, 0, s>>>(tmp.p, cnt.p, sentinel, res.p);
  int64_t h[2];
  DMK_CUDA(cudaMemcpyAsync(h, res.p, sizeof(h), cudaMemcpyDeviceToHost, s));
  DMK_CUDA(cudaStreamSynchronize(s));
  const int64_t m = h[0] - h[1];
  out.alloc(m ? m : 1, s);
  if (m) DMK_CUDA(cudaMemcpyAsync(out.p, tmp.p, m * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
  return m;
}

void exclusive_scan(cudaStream_t s, const int32_t* in, int32_t* out, int64_t n) {
  cub_run(s, [&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, in, out, n, s); });
}
void exclusive_scan_u8(cudaStream_t s, const uint8_t* in, int32_t* out, int64_t n) {
  cub::TransformInputIterator<int32_t, cub::CastOp<int32_t>, const uint8_t*> it(in, cub::CastOp<int32_t>());
  cub_run(s, [&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, it, out, n, s); });
}

template <class T>
T d2h_at(cudaStream_t s, const T* p) {
  T h;
  DMK_CUDA(cudaMemcpyAsync(&h, p, sizeof(T), cudaMemcpyDeviceToHost, s));
  DMK_CUDA(cudaStreamSynchronize(s));
  return h;
}

}  // namespace

// Build the tree of plan P from n points (device pointer, row-major n x D).
template <int D>
static void build_tree_d(dmk_plan_s* P, const double* dpts) {
  constexpr int NCH = Dim<D>::NCH, NCOL = Dim<D>::NCOL;
  cudaStream_t s = P->stream;
  const int64_t n = P->n;
  const int ns = P->ns;
  // phase timing (DMK_PROFILE=1): synchronising wall-clock marks, plan time only
  auto t_last = std::chrono::steady_clock::now();
  auto mark = [&](const char* name) {
    if (!P->profile_tree) return;
    cudaStreamSynchronize(s);
    auto now = std::chrono::steady_clock::now();
    P->tree_timings.push_back({name, std::chrono::duration<double, std::milli>(now - t_last).count()});
    t_last = now;
  };

  // ---- root cube (reading R5), or the caller's (distributed plans share one root):
  // computed on the device; the host copy (pinned) is read after the next round trip
  static thread_local Geo* hgeo = nullptr;
  if (!hgeo) DMK_CUDA(cudaHostAlloc((void**)&hgeo, sizeof(Geo), cudaHostAllocDefault));
  DevBuf<Geo> dgeo;
  dgeo.alloc(1, s);
  if (P->root_fixed) {
    if (!(P->side > 0) || !std::isfinite(P->side)) fail(DMK_ERR_ARG, "fixed root side must be > 0");
    Geo g{};
    for (int d = 0; d < 3; ++d) g.lo[d] = d < D ? P->lo[d] : 0.0;
    g.side = P->side;
    g.scale = (double)(1 << NBITS) / P->side;
    *hgeo = g;
    DMK_CUDA(cudaMemcpyAsync(dgeo.p, hgeo, sizeof(Geo), cudaMemcpyHostToDevice, s));
  } else {
    int nb = std::min(nblk(n), 1024);
    DevBuf<double> part;
    part.alloc(6 * nb, s);
    k_bbox_partial<D><<<nb, TPB, 0, s>>>(dpts, n, part.p);
    k_bbox_final<D><<<1, TPB, 0, s>>>(part.p, nb, dgeo.p);
    DMK_LAUNCH_CHECK();
    DMK_CUDA(cudaMemcpyAsync(hgeo, dgeo.p, sizeof(Geo), cudaMemcpyDeviceToHost, s));
  }
  mark("bbox");

  // ---- Morton keys, stable sort, sorted normalised coordinates
  {
    DevBuf<uint64_t> k0;
    DevBuf<int32_t> i0;
    k0.alloc(n, s);
    i0.alloc(n, s);
    k_keys<D><<<nblk(n), TPB, 0, s>>>(dpts, n, dgeo.p, k0.p, i0.p);
    DMK_LAUNCH_CHECK();
    P->keys.alloc(n, s);
    P->perm.alloc(n, s);
    // 3D: first the top 24 bits (3 radix passes instead of 8): levels <= 8 are sorted,
    // which is all the tree needs unless a level-7 box must be refined (checked with the
    // level counts below; then the rest of the key is sorted too, stably, which composes
    // to the full stable sort of reading R5)
    const int b0 = (D == 3 && P->fast_sort) ? D * NBITS - 24 : 0;
    P->sorted_from_bit = b0;
    cub_run(s, [&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, k0.p, P->keys.p, i0.p, P->perm.p, (int64_t)n, b0, D * NBITS, s);
    });
    P->xs.alloc(n, s);
    P->ys.alloc(n, s);
    if (D == 3) P->zs.alloc(n, s);
    k_gather_pts<D><<<nblk(n), TPB, 0, s>>>(dpts, P->perm.p, n, dgeo.p, P->xs.p, P->ys.p, P->zs.p);
    DMK_LAUNCH_CHECK();
  }

  mark("sort");
  // ---- unbalanced refinement: U[l] = level-l boxes with > ns points.  Coarse levels
  // (<= LBC) are dense bitmaps filled in one pass over the keys; finer levels are
  // selected as sorted lists.
  using CS = Coarse<D>;
  constexpr int LBC = CS::LBC;
  CS cs;
  cs.woff[0] = 0;
  for (int l = 0; l <= LBC; ++l) cs.woff[l + 1] = cs.woff[l] + std::max<int64_t>(1, ((int64_t)1 << (D * l)) / 32);
  const int64_t W = cs.woff[LBC + 1];
  auto nbits = [](int l) { return (int64_t)1 << (D * l); };
  DevBuf<uint32_t> bmbuf;   // [U | NE | B | E], W words each
  bmbuf.alloc(4 * W, s);
  uint32_t *bmU = bmbuf.p, *bmNE = bmU + W, *bmB = bmNE + W, *bmE = bmB + W;
  DMK_CUDA(cudaMemsetAsync(bmbuf.p, 0, 4 * W * sizeof(uint32_t), s));
  std::vector<DevBuf<uint64_t>> U(LMAX);
  std::vector<int64_t> nU(LMAX, 0);
  int ltop = -1;
  {
    // the counts of every level in one pass and one round trip, then the selections
    DevBuf<unsigned long long> dcnt;
    dcnt.alloc(LMAX, s);
    DMK_CUDA(cudaMemsetAsync(dcnt.p, 0, LMAX * sizeof(unsigned long long), s));
    k_count_big<D><<<std::min(nblk(n), 4 * 148), TPB, 0, s>>>(P->keys.p, n, ns, P->min_level, dcnt.p);
    DMK_LAUNCH_CHECK();
    k_mark_coarse<D><<<nblk(n), TPB, 0, s>>>(P->keys.p, n, ns, P->min_level, cs, bmU, bmNE);
    DMK_LAUNCH_CHECK();
    for (int l = 0; l < P->min_level && l <= LBC; ++l) {
      k_bm_all<<<nblk(nbits(l) / 32 + 1), TPB, 0, s>>>(bmU + cs.woff[l], nbits(l));
      DMK_LAUNCH_CHECK();
    }
    unsigned long long hc[LMAX];
    DMK_CUDA(cudaMemcpyAsync(hc, dcnt.p, sizeof(hc), cudaMemcpyDeviceToHost, s));
    DMK_CUDA(cudaStreamSynchronize(s));
    if (P->sorted_from_bit > 0 && hc[7] > 0) {
      // a level-7 box holds > n_s points: the tree may go below level 8, where the top
      // 24 bits do not order the keys -- finish the stable sort and recount
      DevBuf<uint64_t> k1;
      DevBuf<int32_t> i1;
      k1.alloc(n, s);
      i1.alloc(n, s);
      cub_run(s, [&](void* t, size_t& b) {
        return cub::DeviceRadixSort::SortPairs(t, b, P->keys.p, k1.p, P->perm.p, i1.p, (int64_t)n, 0, D * NBITS, s);
      });
      std::swap(P->keys.p, k1.p);
      std::swap(P->perm.p, i1.p);
      P->sorted_from_bit = 0;
      k_gather_pts<D><<<nblk(n), TPB, 0, s>>>(dpts, P->perm.p, n, dgeo.p, P->xs.p, P->ys.p, P->zs.p);
      DMK_LAUNCH_CHECK();
      DMK_CUDA(cudaMemsetAsync(bmbuf.p, 0, 4 * W * sizeof(uint32_t), s));
      DMK_CUDA(cudaMemsetAsync(dcnt.p, 0, LMAX * sizeof(unsigned long long), s));
      k_count_big<D><<<std::min(nblk(n), 4 * 148), TPB, 0, s>>>(P->keys.p, n, ns, P->min_level, dcnt.p);
      DMK_LAUNCH_CHECK();
      k_mark_coarse<D><<<nblk(n), TPB, 0, s>>>(P->keys.p, n, ns, P->min_level, cs, bmU, bmNE);
      DMK_LAUNCH_CHECK();
      for (int l = 0; l < P->min_level && l <= LBC; ++l) {
        k_bm_all<<<nblk(nbits(l) / 32 + 1), TPB, 0, s>>>(bmU + cs.woff[l], nbits(l));
        DMK_LAUNCH_CHECK();
      }
      DMK_CUDA(cudaMemcpyAsync(hc, dcnt.p, sizeof(hc), cudaMemcpyDeviceToHost, s));
      DMK_CUDA(cudaStreamSynchronize(s));
    }
    if (!P->root_fixed) {   // the root cube computed on the device
      if (hgeo->bad) fail(DMK_ERR_ARG, "points contain non-finite coordinates");
      for (int d = 0; d < D; ++d) P->lo[d] = hgeo->lo[d];
      P->side = hgeo->side;
    }
    DevBuf<uint64_t> codes;
    DevBuf<uint8_t> flags;
    DevBuf<int64_t> nsel;
    for (int l = 0; l < LMAX; ++l) {
      if (l < P->min_level) {
        // forced refinement (distributed plans): every box of the levels above min_level
        // exists and is refined, empty or not, so that all ranks share the coarse tree
        nU[l] = (int64_t)1 << (D * l);
        if (l > LBC) fail(DMK_ERR_ARG, "min_level beyond the coarse levels");
        ltop = l;
        continue;
      }
      nU[l] = (int64_t)hc[l];
      if (nU[l] == 0) break;
      ltop = l;
      if (l <= LBC) continue;   // bitmap
      if (!codes.p) {
        codes.alloc(n, s);
        flags.alloc(n, s);
        nsel.alloc(1, s);
      }
      k_big<D><<<nblk(n), TPB, 0, s>>>(P->keys.p, n, l, ns, codes.p, flags.p);
      DMK_LAUNCH_CHECK();
      U[l].alloc(nU[l], s);
      cub_run(s, [&](void* t, size_t& b) {
        return cub::DeviceSelect::Flagged(t, b, codes.p, flags.p, U[l].p, nsel.p, n, s);
      });
    }
  }

  mark("refine");
  // ---- 2:1 balance, bottom-up: B[l] = U[l] + level-l boxes touching B[l+1]
  std::vector<DevBuf<uint64_t>> B(ltop + 1);
  std::vector<int64_t> nB(ltop + 1, 0);
  DMK_CUDA(cudaMemcpyAsync(bmB, bmU, W * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));   // B >= U
  if (ltop > LBC) {
    B[ltop].alloc(nU[ltop], s);
    DMK_CUDA(cudaMemcpyAsync(B[ltop].p, U[ltop].p, nU[ltop] * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
    nB[ltop] = nU[ltop];
  }
  for (int l = ltop - 1; l >= 0; --l) {
    if (l > LBC) {
      int64_t nc = nU[l] + NCH * nB[l + 1];
      DevBuf<uint64_t> cand;
      cand.alloc(nc, s);
      if (nU[l]) DMK_CUDA(cudaMemcpyAsync(cand.p, U[l].p, nU[l] * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
      // out-of-domain touches become the sentinel 2^{D l}, dropped after the sort
      k_touch<D><<<nblk(NCH * nB[l + 1]), TPB, 0, s>>>(B[l + 1].p, nB[l + 1], l, cand.p + nU[l], nullptr,
                                                       (uint64_t)1 << (D * l));
      DMK_LAUNCH_CHECK();
      nB[l] = sort_unique_drop(s, cand.p, nc, D * l, B[l]);
    } else if (l + 1 > LBC) {
      if (nB[l + 1]) {
        k_touch_list_bm<D><<<nblk(nB[l + 1]), TPB, 0, s>>>(B[l + 1].p, nB[l + 1], l, bmB + cs.woff[l]);
        DMK_LAUNCH_CHECK();
      }
    } else {
      k_touch_bm<D><<<nblk(nbits(l + 1)), TPB, 0, s>>>(bmB + cs.woff[l + 1], nbits(l + 1), l, bmB + cs.woff[l]);
      DMK_LAUNCH_CHECK();
    }
  }
  const int nlevels = ltop + 2;
  mark("balance");
  P->th.nlevels = nlevels;

  // ---- box sets per level: E_l = B_l + non-empty children of B_{l-1}
  std::vector<DevBuf<uint64_t>> E(nlevels);
  std::vector<int64_t> nE(nlevels, 0);
  const bool all_coarse = nlevels - 1 <= LBC;
  DevBuf<int32_t> bm_cnt, bm_pos;   // popcounts and exclusive scan of [B | E] bitmap words
  {
    // coarse levels: E bitmaps, then all coarse B and E lists from one scan and one
    // round trip for their sizes
    DMK_CUDA(cudaMemsetAsync(bmE, 1, 1, s));   // E_0 = {root}: first word = 1 (little endian)
    const int lc = std::min(LBC, nlevels - 1);
    for (int l = 1; l <= lc; ++l) {
      k_E_bm<D><<<nblk(nbits(l) / 32 + 1), TPB, 0, s>>>(bmB + cs.woff[l], bmNE + cs.woff[l], bmB + cs.woff[l - 1],
                                                       nbits(l), bmE + cs.woff[l]);
      DMK_LAUNCH_CHECK();
    }
    DevBuf<int32_t>& cnt = bm_cnt;
    DevBuf<int32_t>& pos = bm_pos;
    DevBuf<int64_t> tot;
    cnt.alloc(2 * W + 1, s);
    pos.alloc(2 * W + 1, s);
    tot.alloc(2 * (LBC + 1), s);
    DMK_CUDA(cudaMemsetAsync(cnt.p + 2 * W, 0, sizeof(int32_t), s));
    k_popc<<<nblk(2 * W), TPB, 0, s>>>(bmB, 2 * W, cnt.p);   // B and E are adjacent
    DMK_LAUNCH_CHECK();
    exclusive_scan(s, cnt.p, pos.p, 2 * W + 1);
    k_bm_totals<D><<<1, 32, 0, s>>>(pos.p, cs, 0, tot.p);
    k_bm_totals<D><<<1, 32, 0, s>>>(pos.p, cs, W, tot.p + LBC + 1);
    DMK_LAUNCH_CHECK();
    int64_t ht[2 * (LBC + 1)];
    DMK_CUDA(cudaMemcpyAsync(ht, tot.p, sizeof(ht), cudaMemcpyDeviceToHost, s));
    DMK_CUDA(cudaStreamSynchronize(s));
    for (int l = 0; l <= std::min(LBC, ltop); ++l) nB[l] = ht[l];
    for (int l = 0; l <= lc; ++l) nE[l] = ht[LBC + 1 + l];
    // all levels coarse: the box arrays come straight from the bitmaps (no lists)
    for (int l = 0; l <= std::min(LBC, ltop) && !all_coarse; ++l) {
      B[l].alloc(nB[l] ? nB[l] : 1, s);
      const int64_t nw = cs.woff[l + 1] - cs.woff[l];
      k_bm_fill<<<nblk(nw), TPB, 0, s>>>(bmB + cs.woff[l], pos.p + cs.woff[l], nw, B[l].p);
      DMK_LAUNCH_CHECK();
    }
    for (int l = 0; l <= lc && !all_coarse; ++l) {
      E[l].alloc(nE[l] ? nE[l] : 1, s);
      const int64_t nw = cs.woff[l + 1] - cs.woff[l];
      k_bm_fill<<<nblk(nw), TPB, 0, s>>>(bmE + cs.woff[l], pos.p + W + cs.woff[l], nw, E[l].p);
      DMK_LAUNCH_CHECK();
    }
  }
  for (int l = LBC + 1; l < nlevels; ++l) {
    const int64_t nc = (int64_t)NCH * nB[l - 1];
    const int64_t nb_l = (l <= ltop) ? nB[l] : 0;
    DevBuf<uint64_t> codes;
    DevBuf<uint8_t> flags;
    codes.alloc(nc, s);
    flags.alloc(nc, s);
    k_child_cand<D><<<nblk(nc), TPB, 0, s>>>(B[l - 1].p, nB[l - 1], nb_l ? B[l].p : nullptr, nb_l, P->keys.p, n, l,
                                             codes.p, flags.p);
    DMK_LAUNCH_CHECK();
    nE[l] = select_flagged(s, codes.p, flags.p, nc, E[l]);
  }

  mark("boxsets");
  // ---- global box arrays
  auto& th = P->th;
  th.level_off.assign(nlevels + 1, 0);
  for (int l = 0; l < nlevels; ++l) th.level_off[l + 1] = th.level_off[l] + nE[l];
  const int64_t nbox = P->nbox = th.level_off[nlevels];
  P->box_code.alloc(nbox, s);
  P->box_level.alloc(nbox, s);
  std::vector<int64_t> boff(nlevels + 1, 0);
  DevBuf<uint64_t> Bcat;
  if (all_coarse) {
    CoarseFill cf{};
    for (int l = 0; l <= nlevels; ++l) {
      cf.woff[l] = cs.woff[l];
      cf.loff[l] = th.level_off[l];
    }
    cf.nl = nlevels;
    k_coarse_boxes<<<nblk(cs.woff[nlevels]), TPB, 0, s>>>(bmE, bm_pos.p + W, cf, P->box_code.p, P->box_level.p);
    DMK_LAUNCH_CHECK();
    Bcat.alloc(1, s);   // unused: every level answers from the bitmaps
  } else {
    for (int l = 0; l < nlevels; ++l) {
      DMK_CUDA(cudaMemcpyAsync(P->box_code.p + th.level_off[l], E[l].p, nE[l] * sizeof(uint64_t),
                               cudaMemcpyDeviceToDevice, s));
      k_fill_level<<<nblk(nE[l]), TPB, 0, s>>>(P->box_level.p, th.level_off[l], th.level_off[l + 1], l);
      DMK_LAUNCH_CHECK();
    }
    for (int l = 0; l < nlevels; ++l) boff[l + 1] = boff[l] + ((l <= ltop) ? nB[l] : 0);
    Bcat.alloc(boff[nlevels] ? boff[nlevels] : 1, s);
    for (int l = 0; l <= ltop; ++l)
      if (nB[l])
        DMK_CUDA(cudaMemcpyAsync(Bcat.p + boff[l], B[l].p, nB[l] * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
  }

  P->box_start.alloc(nbox, s);
  P->box_end.alloc(nbox, s);
  P->box_parent.alloc(nbox, s);
  P->box_coll.alloc(NCOL * nbox, s);
  P->box_child.alloc(NCH * nbox, s);
  P->box_flags.alloc(nbox, s);
  static_assert(LBC + 2 <= 12, "BoxCtx::woff");
  BoxCtx ctx{};
  ctx.code = P->box_code.p;
  ctx.level = P->box_level.p;
  ctx.B = Bcat.p;
  ctx.nlevels = nlevels;
  ctx.keys = P->keys.p;
  ctx.n = n;
  ctx.lbc = LBC;
  ctx.bmB = bmB;
  ctx.bmE = bmE;
  ctx.posE = bm_pos.p + W;
  for (int l = 0; l <= nlevels; ++l) {
    ctx.loff[l] = th.level_off[l];
    ctx.boff[l] = boff[l];
  }
  for (int l = 0; l <= LBC + 1; ++l) ctx.woff[l] = cs.woff[l];
  k_box_attrs<D><<<nblk(nbox), TPB, 0, s>>>(ctx, nbox, P->box_start.p, P->box_end.p, P->box_parent.p,
                                         P->box_coll.p, P->box_flags.p);
  DMK_LAUNCH_CHECK();
  DMK_CUDA(cudaMemsetAsync(P->box_child.p, 0xff, NCH * nbox * sizeof(int32_t), s));
  k_children<D><<<nblk(nbox), TPB, 0, s>>>(P->box_code.p, P->box_parent.p, nbox, P->box_child.p);
  DMK_LAUNCH_CHECK();

  mark("boxattrs");
  // ---- flags, ranks, compact lists
  DevBuf<uint8_t> fsel, esel;
  fsel.alloc(nbox + 1, s);
  esel.alloc(nbox + 1, s);
  DMK_CUDA(cudaMemsetAsync(fsel.p + nbox, 0, 1, s));
  DMK_CUDA(cudaMemsetAsync(esel.p + nbox, 0, 1, s));
  k_flags_out<<<nblk(nbox), TPB, 0, s>>>(P->box_start.p, P->box_end.p, P->box_level.p, P->min_level, nbox,
                                         P->box_flags.p, fsel.p);
  DMK_LAUNCH_CHECK();
  {
    DevBuf<int32_t> tf, tscan;
    if (P->n_targets < n) {
      tf.alloc(n + 1, s);
      tscan.alloc(n + 1, s);
      DMK_CUDA(cudaMemsetAsync(tf.p + n, 0, sizeof(int32_t), s));
      k_target_flag_pts<<<nblk(n), TPB, 0, s>>>(P->perm.p, n, P->n_targets, tf.p);
      DMK_LAUNCH_CHECK();
      exclusive_scan(s, tf.p, tscan.p, n + 1);
    }
    k_flag_targets<<<nblk(nbox), TPB, 0, s>>>(P->box_start.p, P->box_end.p, P->n_targets < n ? tscan.p : nullptr,
                                              nbox, P->box_flags.p);
    DMK_LAUNCH_CHECK();
  }
  k_flags_in<D><<<nblk(nbox), TPB, 0, s>>>(P->box_start.p, P->box_end.p, P->box_coll.p, nbox, P->box_flags.p,
                                        esel.p);
  DMK_LAUNCH_CHECK();
  DevBuf<int32_t> fscan, escan;
  fscan.alloc(nbox + 1, s);
  escan.alloc(nbox + 1, s);
  exclusive_scan_u8(s, fsel.p, fscan.p, nbox + 1);
  exclusive_scan_u8(s, esel.p, escan.p, nbox + 1);
  P->fout_rank.alloc(nbox, s);
  P->exp_rank.alloc(nbox, s);
  P->fout_list.alloc(nbox, s);   // capacity nbox: filled before the sizes are known on the host
  P->exp_list.alloc(nbox, s);
  k_ranks_lists<<<nblk(nbox), TPB, 0, s>>>(fscan.p, fsel.p, escan.p, esel.p, nbox, P->fout_rank.p, P->exp_rank.p,
                                           P->fout_list.p, P->exp_list.p);
  DMK_LAUNCH_CHECK();
  // direct lists (CSR over boxes) and P2P work items: counts and scans, then the flag
  // totals, per-level rank offsets and list sizes in ONE round trip, then the fills
  DevBuf<int32_t> dcnt, pcnt, poff;
  dcnt.alloc(nbox + 1, s);
  pcnt.alloc(nbox + 1, s);
  poff.alloc(nbox + 1, s);
  DMK_CUDA(cudaMemsetAsync(dcnt.p, 0, (nbox + 1) * sizeof(int32_t), s));
  DMK_CUDA(cudaMemsetAsync(pcnt.p, 0, (nbox + 1) * sizeof(int32_t), s));
  // symmetric near field (3D): same-level counts and partial-sum slots per box
  DevBuf<int64_t> slots;
  DevBuf<unsigned long long> same_tot;
  NearAux aux{};
  if (D == 3) {
    P->dlist_same.alloc(nbox, s);
    P->dlist_cmask.alloc(nbox, s);
    slots.alloc(nbox + 1, s);
    same_tot.alloc(1, s);
    DMK_CUDA(cudaMemsetAsync(slots.p + nbox, 0, sizeof(int64_t), s));
    DMK_CUDA(cudaMemsetAsync(same_tot.p, 0, sizeof(unsigned long long), s));
    aux.same = P->dlist_same.p;
    aux.cmask = P->dlist_cmask.p;
    aux.slots = slots.p;
    aux.same_tot = same_tot.p;
  }
  k_dlist<D, false><<<nblk(32 * nbox), TPB, 0, s>>>(P->box_start.p, P->box_end.p, P->box_parent.p, P->box_child.p,
                                                    P->box_coll.p, P->box_flags.p, P->box_code.p, P->box_level.p,
                                                    nbox, dcnt.p, nullptr, nullptr, aux);
  DMK_LAUNCH_CHECK();
  if (D == 3) {
    P->part_off.alloc(nbox + 1, s);
    cub_run(s, [&](void* t, size_t& b) {
      return cub::DeviceScan::ExclusiveSum(t, b, slots.p, P->part_off.p, (int64_t)(nbox + 1), s);
    });
  }
  k_p2p_count<<<nblk(nbox), TPB, 0, s>>>(P->box_start.p, P->box_end.p, P->box_flags.p, nbox, pcnt.p);
  DMK_LAUNCH_CHECK();
  P->dlist_off.alloc(nbox + 1, s);
  exclusive_scan(s, dcnt.p, P->dlist_off.p, nbox + 1);
  exclusive_scan(s, pcnt.p, poff.p, nbox + 1);
  // octant items (Sec. 3.4 P2P form, 3D), chosen at evaluation for big leaves
  DevBuf<int32_t> ocnt, ooff;
  DevBuf<unsigned long long> nleaf;
  const char* pform = std::getenv("DMK_P2P_FORM");
  const bool build_oct = D == 3 && pform && std::strcmp(pform, "octant") == 0;   // opt-in form
  if (build_oct) {
    P->leaf_oct.alloc(8 * nbox, s);
    k_leaf_oct<<<nblk(8 * nbox), TPB, 0, s>>>(P->keys.p, P->box_code.p, P->box_level.p, P->box_start.p,
                                              P->box_end.p, P->box_flags.p, nbox, P->leaf_oct.p);
    DMK_LAUNCH_CHECK();
    ocnt.alloc(nbox + 1, s);
    ooff.alloc(nbox + 1, s);
    nleaf.alloc(1, s);
    DMK_CUDA(cudaMemsetAsync(ocnt.p + nbox, 0, sizeof(int32_t), s));
    DMK_CUDA(cudaMemsetAsync(nleaf.p, 0, sizeof(unsigned long long), s));
    k_p2p_count_o<<<nblk(nbox), TPB, 0, s>>>(P->box_start.p, P->box_end.p, P->box_flags.p, P->leaf_oct.p, nbox,
                                             ocnt.p, nleaf.p);
    DMK_LAUNCH_CHECK();
    exclusive_scan(s, ocnt.p, ooff.p, nbox + 1);
  }
  {
    ReadIdx ri{};
    const int m = nlevels + 1;
    for (int l = 0; l < nlevels; ++l) ri.v[l] = th.level_off[l];
    ri.v[nlevels] = nbox;
    ri.m = m;
    DevBuf<int64_t> dout;
    dout.alloc(2 * m + 6, s);
    k_read_totals<<<1, 64, 0, s>>>(fscan.p, escan.p, ri, P->dlist_off.p, poff.p, build_oct ? ooff.p : nullptr,
                                   build_oct ? nleaf.p : nullptr, D == 3 ? P->part_off.p : nullptr,
                                   D == 3 ? same_tot.p : nullptr, nbox, dout.p);
    DMK_LAUNCH_CHECK();
    std::vector<int64_t> h(2 * m + 6);
    DMK_CUDA(cudaMemcpyAsync(h.data(), dout.p, h.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    DMK_CUDA(cudaStreamSynchronize(s));
    P->nfout = h[nlevels];
    P->nexp = h[m + nlevels];
    th.fout_off.assign(nlevels + 1, 0);
    th.exp_off.assign(nlevels + 1, 0);
    for (int l = 0; l <= nlevels; ++l) {
      th.fout_off[l] = h[l];
      th.exp_off[l] = h[m + l];
    }
    P->ndlist = h[2 * m];
    P->np2p = h[2 * m + 1];
    P->np2p_o = h[2 * m + 2];
    P->nleaf_t = h[2 * m + 3];
    P->npart = h[2 * m + 4];
    P->nmixed = P->ndlist - h[2 * m + 5];
  }
  mark("flags");
  P->dlist.alloc(P->ndlist ? P->ndlist : 1, s);
  NearAux faux{};
  if (D == 3) {
    P->dlist_mbeg.alloc(nbox, s);
    faux.mbeg = P->dlist_mbeg.p;
    P->sym_cap = P->ndlist - P->nmixed;   // the same-level entries (tasks: about half)
    P->sym_tasks.alloc(P->sym_cap ? P->sym_cap : 1, s);
    P->sym_ntask.alloc(1, s);
    DMK_CUDA(cudaMemsetAsync(P->sym_ntask.p, 0, sizeof(int32_t), s));
    faux.cmask = P->dlist_cmask.p;
    faux.tasks = P->sym_tasks.p;
    faux.ntask = P->sym_ntask.p;
    faux.part_off = P->part_off.p;
  }
  k_dlist<D, true><<<nblk(32 * nbox), TPB, 0, s>>>(P->box_start.p, P->box_end.p, P->box_parent.p, P->box_child.p,
                                                   P->box_coll.p, P->box_flags.p, P->box_code.p, P->box_level.p,
                                                   nbox, nullptr, P->dlist_off.p, P->dlist.p, faux);
  DMK_LAUNCH_CHECK();
  mark("dlists");
  P->p2p_items.alloc(2 * (P->np2p ? P->np2p : 1), s);
  k_p2p_fill<<<nblk(nbox), TPB, 0, s>>>(P->box_start.p, pcnt.p, poff.p, nbox, P->p2p_items.p);
  DMK_LAUNCH_CHECK();
  if (build_oct) {
    P->p2p_items_o.alloc(P->np2p_o ? P->np2p_o : 1, s);
    k_p2p_fill_o<<<nblk(nbox), TPB, 0, s>>>(P->box_end.p, P->leaf_oct.p, ocnt.p, ooff.p, nbox, P->p2p_items_o.p);
    DMK_LAUNCH_CHECK();
  }
  if (D == 3) {
    P->box_c4.alloc(nbox, s);
    k_box_c4<<<nblk(nbox), TPB, 0, s>>>(P->box_code.p, P->box_level.p, nbox, P->box_c4.p);
    DMK_LAUNCH_CHECK();

    P->xl4.alloc(n ? n : 1, s);
    P->xl4lo.alloc(n ? n : 1, s);
    k_leaf_local4<<<nblk(32 * nbox), TPB, 0, s>>>(P->box_code.p, P->box_level.p, P->box_start.p, P->box_end.p,
                                                   P->box_flags.p, nbox, P->xs.p, P->ys.p, P->zs.p, P->xl4.p,
                                                   P->xl4lo.p);
    DMK_LAUNCH_CHECK();
  }
  // no final synchronisation: everything the host needs was read back above, the rest is
  // stream-ordered before the evaluation (mark() synchronises when profiling)
  mark("p2pitems");
}


void build_tree(dmk_plan_s* P, const double* dpts) {
  if (P->dim == 2) build_tree_d<2>(P, dpts);
  else build_tree_d<3>(P, dpts);
}

}  // namespace dmk
