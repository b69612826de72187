// kernels.cu -- the DMK hot path on the device (Sec. 3.5 Steps 2-5).
//
// Representation: the upward pass carries Chebyshev *moments*
// mu_n(B) = sum_j rho_j T_n(xi_j) instead of the proxy charges rho~ = V^{-T} mu of
// Def. 2.1 -- a fixed linear bijection, folded into the plane-wave matrix
// Q = E V^{-T} (so Phi_l(B) of Eq. 3.42 is bit-for-bit the same quantity), and
// c2p (Lemma 2.2) becomes the exact re-expansion mu^P = (A (x) A (x) A) mu^C.
// The downward pass carries Chebyshev coefficients Lambda (Eq. 3.43) and splits
// them with T_p2c = A^T (Lemma 2.3).  Plane-wave expansions are stored for m3 >= 0
// only (Hermitian symmetry of real sources).
//
// Kernels (one CTA per box unless noted):
//   k_gather_q     charges into Morton order (+ the charge slot of the fp32 P2P records)
//   k_anterp_mma<P>   moments of each F_out box from the points of its leaf children
//                  (fp64 tensor-core GEMMs, DMMA)
//   k_c2p_grp<P>   child -> parent moments by parent groups (8 children, 3 DMMA
//                  contractions over K = 2p), one tree level per launch
//   k_prox2pw<P,H>    outgoing plane waves F(B) from mu(B) (T_prox2pw, DMMA)
//   k_pwshift<H>   fp32 tier: colleague translation (Eq. 3.39) + weights for the 8
//                  children of a parent from the 4x4x4 window of outgoing expansions
//   k_pwlocal<P,H>    translation (p = 28) or its k_pwshift result, then T_pw2poly
//                  Lambda_own(B) = (Gr (x) Gr (x) Gr) Psi_l(B)
//   k_p2c_grp<P>   Lambda(children) += (A^T)^{(x)3} Lambda(parent) by parent groups
//   k_eval32<P> / k_eval_mma<P>   far field at targets from Lambda (fp32 tier / DMMA)
//   k_p2p<K> / k_p2p32<K>   residual kernel R_{L_S} over the direct lists (warp per
//                  item of <= 32 targets, fp64 or the fp32 tier), self terms
//   k_combine      (u_far + u_near)/side, scattered to the caller's order
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "device.cuh"
#include "umma.cuh"

namespace dmk {

// ---------------------------------------------------------------- gather
// q[i] = charges[perm[i]] (Morton order, fp64); with the fp32 P2P tier also the charge
// slot of the leaf-local source record.
__global__ void k_gather_q(const double* __restrict__ charges, const int32_t* __restrict__ perm, int64_t n,
                           double* q, float4* __restrict__ xl4) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double v = charges[perm[i]];
  q[i] = v;
  if (xl4) xl4[i].w = (float)v;
}

// ---- fp32 tier (reading R16, p <= 18): anterpolation and evaluation on the FP32 pipes
// (2x the fp64 rate).  Chebyshev values are computed in fp64 and rounded once; partial
// sums run in fp32 over at most 32 points (anterpolation) or one Chebyshev index pair
// (evaluation, 2 x p terms), then are added in fp64, so the relative error of a moment
// or a potential stays at a few fp32 roundings (~2e-7), below the fp32 rounding of the
// stored plane waves that R16 already accepts.
//
// k_anterp32: mu[n1][n2][n3] = sum_j (rho_j Tx_j[n1] Ty_j[n2]) Tz_j[n3]; thread (n1, m)
// owns the two rows n2 = 2m, 2m+1 over n3 (one pass over the Tz vector feeds both, as
// packed FFMA2), fp32 partial sums over 32 points folded into the fp64 moment cube
// kept in shared memory, which is written out coalesced at the end.
template <int P>
struct Ant32 {
  static constexpr int H2 = (P + 1) / 2, NW = P * H2, NT = (NW + 31) / 32 * 32, CH = 128, PZ = (P + 3) & ~3;
  static constexpr int PY = 2 * H2;   // Ty rows padded to an even length (float2 loads)
  static constexpr int P3A = (P * P * P + 1) & ~1;   // 16-byte aligned float tables after the cube
  static constexpr size_t smem = sizeof(double) * (size_t)P3A + sizeof(float) * (size_t)CH * (P + PY + PZ);
};
template <int P>
__global__ void __launch_bounds__(Ant32<P>::NT) k_anterp32(DevTree t, const int32_t* __restrict__ boxes,
                                                           const double* __restrict__ q, double* __restrict__ mom) {
  using A_ = Ant32<P>;
  constexpr int P2 = P * P, P3 = P2 * P, NT = A_::NT, CH = A_::CH, PZ = A_::PZ, PY = A_::PY, H2 = A_::H2;
  extern __shared__ double smd[];
  double* cube = smd;                                    // [P][P][P] fp64 moments
  float* sx = reinterpret_cast<float*>(cube + A_::P3A);  // [CH][P]   rho T_n1(x)
  float* sy = sx + CH * P;                               // [CH][PY]  T_n2(y)
  float* sz = sy + CH * PY;                              // [CH][PZ]  T_n3(z), 16-byte aligned
  __shared__ int2 rg[8];
  __shared__ int nr_s, tot_s;
  const int b = boxes[blockIdx.x], tid = threadIdx.x;
  if (tid < 32) box_ranges_w<false>(t, b, rg, nr_s, tot_s);
  for (int i = tid; i < P3; i += NT) cube[i] = 0.0;
  __syncthreads();
  const int nr = nr_s, tot = tot_s;
  if (tot == 0) return;   // moments were zeroed by the caller
  double cen[3], ih;
  box_geom(t.code[b], t.level[b], cen, ih);
  const int n1 = tid / H2, m = tid % H2;
  const bool own = tid < A_::NW;
  const bool second = 2 * m + 1 < P;   // odd p: the last m owns one row
  for (int c0 = 0; c0 < tot; c0 += CH) {
    const int nc = min(CH, tot - c0);
    for (int w = tid; w < CH * 3; w += NT) {
      // Chebyshev values by the recurrence in fp64, rounded once (no register array)
      const int j = w / 3, d = w % 3;
      float* dst = d == 0 ? sx + j * P : (d == 1 ? sy + j * PY : sz + j * PZ);
      const int len = d == 0 ? P : (d == 1 ? PY : PZ);
      if (j < nc) {
        const int pi = range_point(rg, nr, c0 + j);
        const double xx = ((d == 0 ? t.xs[pi] : d == 1 ? t.ys[pi] : t.zs[pi]) - cen[d]) * ih;
        const double sc = d == 0 ? q[pi] : 1.0;
        double ta = 1.0, tb = xx;
        dst[0] = (float)sc;
        if (P > 1) dst[1] = (float)(sc * xx);
#pragma unroll 4
        for (int n = 2; n < P; ++n) {
          const double tn = 2.0 * xx * tb - ta;
          dst[n] = (float)(sc * tn);
          ta = tb;
          tb = tn;
        }
        for (int n = P; n < len; ++n) dst[n] = 0.0f;
      } else {
        for (int n = 0; n < len; ++n) dst[n] = 0.0f;
      }
    }
    __syncthreads();
    if (own) {
      for (int j0 = 0; j0 < nc; j0 += 32) {   // fp32 partial sums over <= 32 points
        float2 aa[PZ / 2], ab[PZ / 2];
#pragma unroll
        for (int v = 0; v < PZ / 2; ++v) aa[v] = ab[v] = make_float2(0.0f, 0.0f);
        const int j1 = min(nc, j0 + 32);
#pragma unroll 2
        for (int j = j0; j < j1; ++j) {
          const float2 wy = *reinterpret_cast<const float2*>(sy + j * PY + 2 * m);
          const float wx = sx[j * P + n1];
          const float2 wa = make_float2(wx * wy.x, wx * wy.x), wb = make_float2(wx * wy.y, wx * wy.y);
          const float4* zr = reinterpret_cast<const float4*>(sz + j * PZ);
#pragma unroll
          for (int v = 0; v < PZ / 4; ++v) {
            const float4 z = zr[v];
            const float2 z0 = make_float2(z.x, z.y), z1 = make_float2(z.z, z.w);
            aa[2 * v] = __ffma2_rn(wa, z0, aa[2 * v]);
            aa[2 * v + 1] = __ffma2_rn(wa, z1, aa[2 * v + 1]);
            ab[2 * v] = __ffma2_rn(wb, z0, ab[2 * v]);
            ab[2 * v + 1] = __ffma2_rn(wb, z1, ab[2 * v + 1]);
          }
        }
        double* ra = cube + ((size_t)n1 * P + 2 * m) * P;
#pragma unroll
        for (int v = 0; v < PZ / 2; ++v) {
          if (2 * v < P) ra[2 * v] += (double)aa[v].x;
          if (2 * v + 1 < P) ra[2 * v + 1] += (double)aa[v].y;
          if (second) {
            if (2 * v < P) ra[P + 2 * v] += (double)ab[v].x;
            if (2 * v + 1 < P) ra[P + 2 * v + 1] += (double)ab[v].y;
          }
        }
      }
    }
    __syncthreads();
  }
  double* out = mom + (size_t)t.fout_rank[b] * P3;
  for (int i = tid; i < P3; i += NT) out[i] = cube[i];
}

// ---- fp32 tier on the 5th-generation tensor cores (tcgen05, kind::tf32 with the 3xTF32
// split): the same contraction as a GEMM per F_out box with the points as K,
//   mu[(n1 n2)][n3] = sum_j W[(n1 n2)][j] Tz[n3][j],   W[(n1 n2)][j] = rho_j Tx_j[n1] Ty_j[n2],
// M = p^2 rows in MT tiles of 128 (TMEM lanes), N = p padded to NP (a multiple of 16),
// K = the points.  Warp-specialised pipeline: 4 MT producer warps (one thread per row m)
// compute the Chebyshev values of a super-chunk of SC points in fp64 (rounded once into
// shared tables), then write W and Tz of each chunk of KC points, split as
// hi = tf32(v), lo = tf32(v - hi), into one of two operand buffers (K-major, no swizzle,
// umma.cuh) and arrive on its "full" mbarrier; one MMA warp waits for it, issues
// A_hi B_hi + A_lo B_hi + A_hi B_lo (MT tiles x 3 MMAs) into the super-chunk's TMEM
// accumulator and commits the buffer's "free" mbarrier (the tensor core releases it when
// its MMAs complete).  Each super-chunk accumulates in one of two TMEM accumulators; the
// producers read it (tcgen05.ld) into fp64 registers one super-chunk later, so the fp32
// sums run over at most SC points (as k_anterp32's 32) and fp64 across super-chunks.
#ifndef ANT_TC_KC
#define ANT_TC_KC 8      // points per operand chunk (one K = 8 MMA step)
#endif
#ifndef ANT_TC_MINB
#define ANT_TC_MINB 2    // two CTAs per SM (shared memory and TMEM allow two)
#endif
template <int P>
struct AntTC {
  static constexpr int P2 = P * P, MT = (P2 + 127) / 128, NP = (P + 15) / 16 * 16;
  static constexpr int KC = ANT_TC_KC, SC = 64, NCH = SC / KC;
  static constexpr int NPROD = 128 * MT;                  // producer threads: one per row
  static constexpr int NT = NPROD + 32;                   // + the MMA warp
  static constexpr int ACOLS = MT * NP;                   // TMEM columns per accumulator
  static constexpr int TCOLS = 2 * ACOLS <= 32 ? 32 : (2 * ACOLS <= 64 ? 64 : (2 * ACOLS <= 128 ? 128 : 256));
  static constexpr size_t A_WORDS = (size_t)MT * 128 * KC, B_WORDS = (size_t)NP * KC;
  static constexpr size_t BUF_WORDS = 2 * A_WORDS + 2 * B_WORDS;   // hi + lo
  static constexpr size_t smem = sizeof(float) * (2 * BUF_WORDS + (size_t)2 * 3 * SC * P) + 128;
};
__device__ __forceinline__ int umma_koff(int row, int k, int kc) {   // K-major, no swizzle (umma.cuh)
  return (row >> 3) * (kc / 4) * 32 + (k >> 2) * 32 + (row & 7) * 4 + (k & 3);
}
template <int P>
__global__ void __launch_bounds__(AntTC<P>::NT, ANT_TC_MINB) k_anterp_tc(DevTree t, const int32_t* __restrict__ boxes,
                                                               const double* __restrict__ q,
                                                               double* __restrict__ mom) {
  using C = AntTC<P>;
  constexpr int P2 = C::P2, MT = C::MT, NP = C::NP, KC = C::KC, SC = C::SC, NCH = C::NCH;
  constexpr int NPROD = C::NPROD, ACOLS = C::ACOLS;
  extern __shared__ __align__(128) float smf[];
  float* buf[2] = {smf, smf + C::BUF_WORDS};   // [Ah | Al | Bh | Bl] per operand buffer
  float* tab[2] = {smf + 2 * C::BUF_WORDS, smf + 2 * C::BUF_WORDS + 3 * SC * P};   // [sx|sy|sz][SC][P]
  __shared__ __align__(8) uint64_t full[2], freeb[2], dfull[2], dfree[2];
  __shared__ uint32_t tbase;
  __shared__ int2 rg[8];
  __shared__ int nr_s, tot_s;
  const int b = boxes[blockIdx.x], tid = threadIdx.x, warp = tid >> 5;
  if (tid < 32) box_ranges_w<false>(t, b, rg, nr_s, tot_s);
  __syncthreads();
  const int nr = nr_s, tot = tot_s;
  if (tot == 0) return;   // moments were zeroed by the caller
  // zero the padding once (never rewritten): A rows >= p^2, B rows >= p, both buffers
  for (int i = tid; i < (MT * 128 - P2) * KC; i += C::NT) {
    const int r = P2 + i / KC, k = i % KC;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      buf[u][umma_koff(r, k, KC)] = 0.0f;
      buf[u][C::A_WORDS + umma_koff(r, k, KC)] = 0.0f;
    }
  }
  for (int i = tid; i < (NP - P) * KC; i += C::NT) {
    const int r = P + i / KC, k = i % KC;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      buf[u][2 * C::A_WORDS + umma_koff(r, k, KC)] = 0.0f;
      buf[u][2 * C::A_WORDS + C::B_WORDS + umma_koff(r, k, KC)] = 0.0f;
    }
  }
  if (warp == 0) umma::tmem_alloc<C::TCOLS>(&tbase);
  if (tid == 0) {
    for (int u = 0; u < 2; ++u) {
      umma::mbar_init(&full[u], NPROD / 32);   // one arrival per producer warp
      umma::mbar_init(&freeb[u], 1);           // tcgen05.commit
      umma::mbar_init(&dfull[u], 1);           // tcgen05.commit
      umma::mbar_init(&dfree[u], NPROD / 32);
    }
  }
  umma::fence_smem_to_async();
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tmem = tbase;
  const int nsc = (tot + SC - 1) / SC;   // super-chunks
  if (warp == NPROD / 32) {
    // ================= MMA warp
    if ((tid & 31) == 0) {
      const uint32_t idesc = umma::idesc_tf32(128, NP);
      int g = 0;   // global chunk index
      for (int sc = 0; sc < nsc; ++sc) {
        const int d = sc & 1;
        if (sc >= 2) umma::mbar_wait(&dfree[d], (uint32_t)(((sc - 2) >> 1) & 1));   // producers read it
        const int nch = min(NCH, (tot - sc * SC + KC - 1) / KC);
        for (int c = 0; c < nch; ++c, ++g) {
          const int u = g & 1;
          umma::mbar_wait(&full[u], (uint32_t)((g >> 1) & 1));
          umma::fence_after_sync();
          const float* B0 = buf[u];
          const uint64_t dAh = umma::sdesc_kmajor(B0, 128, 32 * KC);
          const uint64_t dAl = umma::sdesc_kmajor(B0 + C::A_WORDS, 128, 32 * KC);
          const uint64_t dBh = umma::sdesc_kmajor(B0 + 2 * C::A_WORDS, 128, 32 * KC);
          const uint64_t dBl = umma::sdesc_kmajor(B0 + 2 * C::A_WORDS + C::B_WORDS, 128, 32 * KC);
          const uint32_t dbase = tmem + (uint32_t)(d * ACOLS);
#pragma unroll
          for (int pr = 0; pr < 3; ++pr) {   // hi.hi, lo.hi, hi.lo
            const uint64_t da = pr == 1 ? dAl : dAh, db = pr == 2 ? dBl : dBh;
#pragma unroll
            for (int s8 = 0; s8 < KC / 8; ++s8)
#pragma unroll
              for (int tm = 0; tm < MT; ++tm)
                umma::mma_tf32(dbase + tm * NP, da + (uint64_t)(tm * 32 * KC + s8 * 16), db + (uint64_t)(s8 * 16),
                               idesc, pr > 0 || c > 0 || s8 > 0);
          }
          umma::commit(&freeb[u]);   // the buffer is free once these MMAs complete
        }
        umma::commit(&dfull[d]);     // the super-chunk's accumulator is complete
      }
    }
    __syncwarp();
  } else {
    // ================= producer warps: thread m owns accumulator row m = (n1, n2)
    const int m = tid;
    const int n1 = m / P, n2 = m - n1 * P;
    const bool real = m < P2;
    double cen[3], ih;
    box_geom(t.code[b], t.level[b], cen, ih);
    double acc[P];
#pragma unroll
    for (int n = 0; n < P; ++n) acc[n] = 0.0;
    // Chebyshev work items: point j = w / 3 of the super-chunk, axis d = w % 3
    auto cheb = [&](int sc) {
      for (int w = tid; w < 3 * SC; w += NPROD) {
        const int jw = w / 3, dw = w % 3;
        const double* coord = dw == 0 ? t.xs : (dw == 1 ? t.ys : t.zs);
        float* dst = tab[sc & 1] + dw * SC * P + jw * P;
        const int j = sc * SC + jw;
        if (j < tot) {
          const int pi = range_point(rg, nr, j);
          const double xx = (coord[pi] - cen[dw]) * ih, sc0 = dw == 0 ? q[pi] : 1.0;
          double ta = 1.0, tb = xx;
          dst[0] = (float)sc0;
          if (P > 1) dst[1] = (float)(sc0 * xx);
#pragma unroll 6
          for (int n = 2; n < P; ++n) {
            const double tn = 2.0 * xx * tb - ta;
            dst[n] = (float)(sc0 * tn);
            ta = tb;
            tb = tn;
          }
        } else {
#pragma unroll
          for (int n = 0; n < P; ++n) dst[n] = 0.0f;
        }
      }
    };
    auto flush = [&](int sc) {   // the accumulator of super-chunk sc -> fp64 registers
      const int d = sc & 1;
      umma::mbar_wait(&dfull[d], (uint32_t)((sc >> 1) & 1));
      umma::fence_after_sync();
      float v[32];
      const uint32_t col = (uint32_t)(d * ACOLS + (m >> 7) * NP);
      if constexpr (NP >= 32) umma::ld32x32b_x32(tmem + ((uint32_t)(32 * (warp & 3)) << 16) + col, v);
      else umma::ld32x32b_x16(tmem + ((uint32_t)(32 * (warp & 3)) << 16) + col, v);
#pragma unroll
      for (int n = 0; n < P; ++n) acc[n] += (double)v[n];
      umma::fence_before_sync();
      __syncwarp();
      if ((tid & 31) == 0) umma::mbar_arrive(&dfree[d]);
    };
    int g = 0;
    cheb(0);
    for (int sc = 0; sc < nsc; ++sc) {
      umma::bar_sync(1, NPROD);   // the super-chunk's tables are written
      const float* sx = tab[sc & 1];
      const float* sy = sx + SC * P;
      const float* sz = sy + SC * P;
      const int nch = min(NCH, (tot - sc * SC + KC - 1) / KC);
      for (int c = 0; c < nch; ++c, ++g) {
        const int u = g & 1;
        if (g >= 2) umma::mbar_wait(&freeb[u], (uint32_t)(((g - 2) >> 1) & 1));
        float* Ah = buf[u];
        float* Al = Ah + C::A_WORDS;
        float* Bh = Al + C::A_WORDS;
        float* Bl = Bh + C::B_WORDS;
        if (real) {
#pragma unroll
          for (int k4 = 0; k4 < KC; k4 += 4) {
            float4 h, l;
            float* hv = &h.x;
            float* lv = &l.x;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int j = c * KC + k4 + e;
              const float w = sx[j * P + n1] * sy[j * P + n2];
              hv[e] = umma::tf32_rna(w);
              lv[e] = umma::tf32_rna(w - hv[e]);
            }
            const int o = umma_koff(m, k4, KC);
            *reinterpret_cast<float4*>(Ah + o) = h;
            *reinterpret_cast<float4*>(Al + o) = l;
          }
        }
        if (m < P * (KC / 4)) {
          const int n3 = m / (KC / 4), k4 = 4 * (m % (KC / 4));
          float4 h, l;
          float* hv = &h.x;
          float* lv = &l.x;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float z = sz[(c * KC + k4 + e) * P + n3];
            hv[e] = umma::tf32_rna(z);
            lv[e] = umma::tf32_rna(z - hv[e]);
          }
          const int o = umma_koff(n3, k4, KC);
          *reinterpret_cast<float4*>(Bh + o) = h;
          *reinterpret_cast<float4*>(Bl + o) = l;
        }
        umma::fence_smem_to_async();
        __syncwarp();
        if ((tid & 31) == 0) umma::mbar_arrive(&full[u]);
      }
      // next super-chunk's tables (the other table buffer: its last readers finished
      // before this super-chunk's bar_sync), then the previous accumulator
      if (sc + 1 < nsc) cheb(sc + 1);
      if (sc >= 1) flush(sc - 1);
    }
    flush(nsc - 1);
    if (real) {
      double* out = mom + (size_t)t.fout_rank[b] * P * P2 + (size_t)m * P;
#pragma unroll
      for (int n = 0; n < P; ++n) out[n] = acc[n];
    }
  }
  umma::fence_before_sync();
  __syncthreads();
  if (warp == 0) umma::tmem_free<C::TCOLS>(tmem);
}

// ---- fp32 tier far-field evaluation on the tensor cores (tcgen05 kind::tf32, 3xTF32):
//   G[j][(n1 n2)] = sum_n3 Tz_j[n3] Lambda[(n1 n2)][n3]          (UMMA: M = 128 targets,
//   u_j = sum_n1 Tx_j[n1] sum_n2 Ty_j[n2] G[j][(n1 n2)]           N = p^2 in chunks, K = p)
// One CTA per local-expansion box, one thread per target of a 128-target tile (its
// Chebyshev values in fp64, rounded once; Tz split hi/lo into its A row).  Lambda (own +
// inherited part) is split into hi/lo B rows once per box.  The p^2 columns run in NCH
// chunks of NCW through two TMEM accumulators: chunk c + 2 is issued as soon as the
// threads have read chunk c, so the tensor core works while the threads contract.
template <int P>
struct EvTC {
  static constexpr int P2 = P * P, KP = (P + 7) / 8 * 8, NB = (P2 + 15) / 16 * 16;
  static constexpr int NCH = NB <= 128 ? 1 : (NB + 111) / 112, NCW = NB <= 128 ? NB : 112;
  static constexpr int NT = 128;
  static constexpr int TCOLS = (NCH > 1 ? 2 : 1) * NCW <= 128 ? 128 : 256;
  static constexpr size_t A_WORDS = (size_t)128 * KP, B_WORDS = (size_t)NCH * NCW * KP;
  static constexpr size_t smem = sizeof(float) * (2 * A_WORDS + 2 * B_WORDS) + 128;
};
template <int P>
__global__ void __launch_bounds__(EvTC<P>::NT, 2) k_eval_tc(DevTree t, const int32_t* __restrict__ boxes,
                                                            const double* __restrict__ lam,
                                                            double* __restrict__ ufar) {
  using C = EvTC<P>;
  constexpr int P2 = C::P2, KP = C::KP, NCH = C::NCH, NCW = C::NCW, NT = C::NT;
  extern __shared__ __align__(128) float smf[];
  float* Ah = smf;                  // [128][KP]  Tz of the tile's targets
  float* Al = Ah + C::A_WORDS;
  float* Bh = Al + C::A_WORDS;      // [NCH*NCW][KP]  Lambda rows (n1 n2)
  float* Bl = Bh + C::B_WORDS;
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ uint32_t tbase;
  __shared__ int2 rg[8];
  __shared__ int nr_s, tot_s;
  const int b = boxes[blockIdx.x], tid = threadIdx.x, warp = tid >> 5;
  if (tid < 32) box_ranges_w<true>(t, b, rg, nr_s, tot_s);
  __syncthreads();
  const int nr = nr_s, tot = tot_s;
  if (tot == 0) return;
  // ---- B: the box's local expansion (own + inherited, k_p2c_grp) as hi/lo tf32 rows
  {
    const double* src = lam + (size_t)t.exp_rank[b] * P * P2;
    // one row (n1 n2) of p values per thread and pass: all its loads in flight together
    for (int r = tid; r < NCH * NCW; r += NT) {
      double v[KP];
#pragma unroll
      for (int k = 0; k < KP; ++k) v[k] = 0.0;
      if (r < P2) {
#pragma unroll
        for (int k = 0; k < P; ++k) v[k] = __ldg(src + (size_t)r * P + k);
      }
#pragma unroll
      for (int k4 = 0; k4 < KP; k4 += 4) {
        float4 h, l;
        float* hv = &h.x;
        float* lv = &l.x;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float f = (float)v[k4 + e];
          hv[e] = umma::tf32_rna(f);
          lv[e] = umma::tf32_rna(f - hv[e]);
        }
        const int o = umma_koff(r, k4, KP);
        *reinterpret_cast<float4*>(Bh + o) = h;
        *reinterpret_cast<float4*>(Bl + o) = l;
      }
    }
  }
  if (warp == 0) umma::tmem_alloc<C::TCOLS>(&tbase);
  if (tid == 0) {
    umma::mbar_init(&mbar[0], 1);
    umma::mbar_init(&mbar[1], 1);
  }
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tmem = tbase;
  double cen[3], ih;
  box_geom(t.code[b], t.level[b], cen, ih);
  const uint32_t idesc = umma::idesc_tf32(128, NCW);
  const uint64_t dAh = umma::sdesc_kmajor(Ah, 128, 32 * KP), dAl = umma::sdesc_kmajor(Al, 128, 32 * KP);
  const uint64_t dBh = umma::sdesc_kmajor(Bh, 128, 32 * KP), dBl = umma::sdesc_kmajor(Bl, 128, 32 * KP);
  uint32_t ph0 = 0, ph1 = 0;   // completed phases of the two accumulators' mbarriers
  auto issue = [&](int c) {    // chunk c of the p^2 columns into accumulator c % 2
    umma::fence_after_sync();
    const uint32_t d = tmem + (uint32_t)((c & 1) * NCW);
    const uint64_t boff = (uint64_t)(c * NCW / 8) * (32 * KP / 16);   // rows c NCW.. (16-byte units)
#pragma unroll
    for (int pr = 0; pr < 3; ++pr) {   // hi.hi, lo.hi, hi.lo
      const uint64_t da = pr == 1 ? dAl : dAh, db = (pr == 2 ? dBl : dBh) + boff;
#pragma unroll
      for (int s = 0; s < KP / 8; ++s) umma::mma_tf32(d, da + (uint64_t)(s * 16), db + (uint64_t)(s * 16), idesc, pr > 0 || s > 0);
    }
    umma::commit(&mbar[c & 1]);
  };
  for (int t0 = 0; t0 < tot; t0 += 128) {
    const int j = t0 + tid;
    const bool real = j < tot;
    const int pi = real ? range_point(rg, nr, j) : 0;
    float tx[P], ty[P];
    {
      double tz[P];
      cheb_vec(real ? (t.xs[pi] - cen[0]) * ih : 0.0, tz, P, 1.0);
#pragma unroll
      for (int n = 0; n < P; ++n) tx[n] = (float)tz[n];
      cheb_vec(real ? (t.ys[pi] - cen[1]) * ih : 0.0, tz, P, 1.0);
#pragma unroll
      for (int n = 0; n < P; ++n) ty[n] = (float)tz[n];
      cheb_vec(real ? (t.zs[pi] - cen[2]) * ih : 0.0, tz, P, real ? 1.0 : 0.0);
#pragma unroll
      for (int k4 = 0; k4 < KP; k4 += 4) {
        float4 h, l;
        float* hv = &h.x;
        float* lv = &l.x;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float z = k4 + e < P ? (float)tz[k4 + e] : 0.0f;
          hv[e] = umma::tf32_rna(z);
          lv[e] = umma::tf32_rna(z - hv[e]);
        }
        const int o = umma_koff(tid, k4, KP);
        *reinterpret_cast<float4*>(Ah + o) = h;
        *reinterpret_cast<float4*>(Al + o) = l;
      }
    }
    umma::fence_smem_to_async();
    umma::fence_before_sync();
    __syncthreads();
    if (tid == 0) {
      issue(0);
      if (NCH > 1) issue(1);
    }
    float s[P];
#pragma unroll
    for (int n = 0; n < P; ++n) s[n] = 0.0f;
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      umma::mbar_wait(&mbar[c & 1], (c & 1) ? ph1 : ph0);
      if (c & 1) ph1 ^= 1;
      else ph0 ^= 1;
      umma::fence_after_sync();
      const uint32_t base = tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)((c & 1) * NCW);
#pragma unroll
      for (int c32 = 0; c32 < NCW; c32 += 32) {
        float g[32];
        if (c32 + 32 <= NCW) umma::ld32x32b_x32(base + c32, g);
        else umma::ld32x32b_x16(base + c32, g);
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const int r = c * NCW + c32 + e;   // row (n1 n2), compile-time after unrolling
          if (c32 + e < NCW && r < P2) s[r / P] = fmaf(ty[r % P], g[e], s[r / P]);
        }
      }
      umma::fence_before_sync();
      __syncthreads();   // accumulator c % 2 read by every thread
      if (tid == 0 && c + 2 < NCH) issue(c + 2);
    }
    double u = 0.0;
#pragma unroll
    for (int n = 0; n < P; ++n) u = fma((double)tx[n], (double)s[n], u);
    if (real) ufar[pi] = u;
  }
  umma::fence_before_sync();
  __syncthreads();
  if (warp == 0) umma::tmem_free<C::TCOLS>(tmem);
}

// k_eval32: u_i = sum_n1 T_n1(x_i) sum_n2 T_n2(y_i) sum_n3 Lambda[n1 n2 n3] T_n3(z_i), two
// targets per thread (each Lambda row read from shared memory serves both), the n3 sums
// as packed FFMA2 (even/odd n3 halves), T_n1 by the recurrence in fp64, the n1 sum in fp64.
template <int P>
struct Ev32 {
  static constexpr int NT = 128, PZ = (P + 3) & ~3;
  static constexpr size_t smem = sizeof(float) * (size_t)P * P * PZ;
};
template <int P>
__global__ void __launch_bounds__(Ev32<P>::NT) k_eval32(DevTree t, const int32_t* __restrict__ boxes,
                                                        const double* __restrict__ lam,
                                                        double* __restrict__ ufar) {
  using E = Ev32<P>;
  constexpr int NT = E::NT, PZ = E::PZ, P2 = P * P;
  extern __shared__ float4 sl4[];   // [P2][PZ/4]
  float* sl = reinterpret_cast<float*>(sl4);
  __shared__ int2 rg[8];
  __shared__ int nr_s, tot_s;
  const int b = boxes[blockIdx.x], tid = threadIdx.x;
  if (tid < 32) box_ranges_w<true>(t, b, rg, nr_s, tot_s);
  __syncthreads();
  const int nr = nr_s, tot = tot_s;
  if (tot == 0) return;
  // the box's local expansion (own + inherited, k_p2c_grp)
  const double* src = lam + (size_t)t.exp_rank[b] * P * P2;
  for (int i = tid; i < P2 * PZ; i += NT) {
    const int r = i / PZ, c = i - r * PZ;
    sl[i] = c < P ? (float)src[r * P + c] : 0.0f;
  }
  double cen[3], ih;
  box_geom(t.code[b], t.level[b], cen, ih);
  __syncthreads();
  for (int k0 = 2 * tid; k0 < tot; k0 += 2 * NT) {
    const bool two = k0 + 1 < tot;
    const int pa = range_point(rg, nr, k0), pb = two ? range_point(rg, nr, k0 + 1) : pa;
    const double xa = (t.xs[pa] - cen[0]) * ih, xb = (t.xs[pb] - cen[0]) * ih;
    float2 fy[P], fza[PZ / 2], fzb[PZ / 2];
    {
      double ta[P], tb[P];
      cheb_vec((t.ys[pa] - cen[1]) * ih, ta, P, 1.0);
      cheb_vec((t.ys[pb] - cen[1]) * ih, tb, P, 1.0);
#pragma unroll
      for (int n = 0; n < P; ++n) fy[n] = make_float2((float)ta[n], (float)tb[n]);
      cheb_vec((t.zs[pa] - cen[2]) * ih, ta, P, 1.0);
      cheb_vec((t.zs[pb] - cen[2]) * ih, tb, P, 1.0);
#pragma unroll
      for (int v = 0; v < PZ / 2; ++v) {
        fza[v] = make_float2(2 * v < P ? (float)ta[2 * v] : 0.0f, 2 * v + 1 < P ? (float)ta[2 * v + 1] : 0.0f);
        fzb[v] = make_float2(2 * v < P ? (float)tb[2 * v] : 0.0f, 2 * v + 1 < P ? (float)tb[2 * v + 1] : 0.0f);
      }
    }
    double ua = 0.0, ub = 0.0, aa = 1.0, ab = xa, ba = 1.0, bb = xb;   // T_n1, T_{n1+1}
#pragma unroll 1
    for (int n1 = 0; n1 < P; ++n1) {
      const float4* row = sl4 + (size_t)n1 * P * (PZ / 4);
      float2 s1 = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int n2 = 0; n2 < P; ++n2) {
        float2 sa = make_float2(0.0f, 0.0f), sb = make_float2(0.0f, 0.0f);
#pragma unroll
        for (int v = 0; v < PZ / 4; ++v) {
          const float4 l4 = row[n2 * (PZ / 4) + v];
          const float2 l0 = make_float2(l4.x, l4.y), l1 = make_float2(l4.z, l4.w);
          sa = __ffma2_rn(l0, fza[2 * v], sa);
          sa = __ffma2_rn(l1, fza[2 * v + 1], sa);
          sb = __ffma2_rn(l0, fzb[2 * v], sb);
          sb = __ffma2_rn(l1, fzb[2 * v + 1], sb);
        }
        s1 = __ffma2_rn(make_float2(sa.x + sa.y, sb.x + sb.y), fy[n2], s1);
      }
      ua = fma((double)s1.x, aa, ua);
      ub = fma((double)s1.y, ba, ub);
      const double na = 2.0 * xa * ab - aa, nb = 2.0 * xb * bb - ba;
      aa = ab;
      ab = na;
      ba = bb;
      bb = nb;
    }
    ufar[pa] = ua;
    if (two) ufar[pb] = ub;
  }
}

// ---------------------------------------------------------------- c2p / p2c
// ---- c2p / p2c by parent groups on fp64 tensor cores (Lemmas 2.2-2.3).
// The 8 children of a parent share the axis factors: with octant o = (o1 o2 o3),
//   c2p: mu_P = sum_o (A_o1 (x) A_o2 (x) A_o3) mu_o
//           = sum_o3 [sum_o2 [sum_o1 A_o1 mu_(o1 o2 o3)]_axis1 ...]
// so the axis-1 contraction runs over K = 2p (both o1) for each (o2, o3), the axis-2
// one over K = 2p for each o3, and the axis-3 one over K = 2p once: 14 p^4 instead of
// 48 p^4 flops per parent.  p2c is the transpose (axis 1 first, expanding 1 -> 2 -> 4
// -> 8).  A CTA owns a tile of MT rows of the first-contracted axis (c2p: output rows
// m1 of the parent; p2c: output rows k1 of the children), intermediates in shared
// memory, each contraction a DMMA GEMM (c2p: grp_tiles, per-lane precomputed operand
// offsets, A fragments kept across n-tiles, two tiles of global B loads in flight:
// 0.276 -> 0.235 ms at config 1, 1.49 -> 1.17 ms at eps = 1e-9; p2c: mma_tiles, where
// the same rewrite measured slower, 0.29 -> 0.33 ms).
constexpr int cmin(int a, int b) { return a < b ? a : b; }
template <int P, int MT>
struct GrpCfg {
  // p = 28: one CTA per SM fits (shared memory), so 16 warps instead of 8 keep more
  // tiles' operand loads in flight
  static constexpr int NT = P > 18 ? 512 : 256;
  static constexpr int P2 = P * P, NTILE = (P + MT - 1) / MT;
  static constexpr int KS2 = (2 * P + 3) / 4, KS1 = (P + 3) / 4;
  static constexpr size_t smem_c2p = sizeof(double) * ((size_t)2 * P2 + 6 * (size_t)MT * P2);
  static constexpr size_t smem_p2c = sizeof(double) * ((size_t)2 * P2 + 6 * (size_t)MT * P2);
  // resident CTAs per SM the shared memory allows (registers held to match)
  static constexpr int MINB_C2P = P > 18 ? 1 : cmin((int)((227 * 1024) / (smem_c2p + 1024)), 4);
};
// Warp-level fp64 GEMM on 8x8 output tiles (mma.sync m8n8k4, DMMA) for the group
// kernels, with the operand addressing precomputed per lane by the caller:
//   fa(mt, ks) = A[8 mt + g][4 ks + q],  fb(nt, ks) = B[4 ks + q][8 nt + g],
//   fc(mt, nt, c0, c1) consumes C[8 mt + g][8 nt + 2q + {0, 1}]   (g = lane/4, q = lane%4).
// Tiles are dealt to the warps round-robin in mt-major order; a warp keeps its A
// fragments while the m-tile does not change (axis contractions whose M is one or two
// tiles reuse them over all n-tiles), and loads the next tile's B fragments during the
// current tile's DMMA chain (NB tiles per step: more loads in flight, for global B).
// FPRE (accumulating epilogues): fpre(mt, nt, p0, p1) loads the current output values
// before the chain.
template <int KS, int NB = 1, class FA, class FB, class FC, class FP>
__device__ __forceinline__ void grp_tiles(int mtiles, int ntiles, FA fa, FB fb, FC fc, FP fpre) {
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int ntot = mtiles * ntiles;
  int t = warp;
  if (t >= ntot) return;
  int cur = -1;
  double av[KS], bv[NB][KS];
  // a step takes NB tiles t, t + nw, ..., whose B loads are all in flight together (the
  // next step's are issued before this step's DMMA chains)
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    const int tj = t + j * nw;
    const int nt = (tj < ntot ? tj : t) % ntiles;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) bv[j][ks] = fb(nt, ks);
  }
  for (; t < ntot; t += NB * nw) {
    double bn[NB][KS];
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const int tn = t + (NB + j) * nw;
      if (tn < ntot) {
        const int ntn = tn % ntiles;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) bn[j][ks] = fb(ntn, ks);
      }
    }
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const int tj = t + j * nw;
      if (tj < ntot) {
        const int mt = tj / ntiles, nt = tj - mt * ntiles;
        if (mt != cur) {
          cur = mt;
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) av[ks] = fa(mt, ks);
        }
        double p0 = 0.0, p1 = 0.0;
        fpre(mt, nt, p0, p1);
        double c0 = 0.0, c1 = 0.0;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) dmma(c0, c1, av[ks], bv[j][ks]);
        fc(mt, nt, c0 + p0, c1 + p1);
      }
    }
#pragma unroll
    for (int j = 0; j < NB; ++j)
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) bv[j][ks] = bn[j][ks];
  }
}
struct NoPre {
  __device__ __forceinline__ void operator()(int, int, double&, double&) const {}
};
// K index k = 4 ks + q of a contraction over both halves o (K = 2p): o = k >= p,
// k' = k - o p; k >= 2p is padding
template <int P>
__device__ __forceinline__ void split_k2(int k, int& o, int& kk, bool& ok) {
  ok = k < 2 * P;
  o = k >= P;
  kk = k - o * P;
}
template <int P, int MT>
__global__ void __launch_bounds__(GrpCfg<P, MT>::NT, GrpCfg<P, MT>::MINB_C2P) k_c2p_grp(DevTree t, const int32_t* __restrict__ parents,
                                                 const double* __restrict__ A, double* __restrict__ mom) {
  using C = GrpCfg<P, MT>;
  constexpr int P2 = C::P2, P3 = P2 * P, KS2 = C::KS2;
  constexpr int NT1 = (P2 + 7) / 8;            // axis-1 n tiles per group
  constexpr int NT2 = (MT * P + 7) / 8;        // axis-2 n tiles per o3
  extern __shared__ double sm[];
  double* sA = sm;                  // [2][P][P]: A_s[n][k]
  double* xi = sA + 2 * P2;         // [(o2 o3)][MT][P2]
  double* eta = xi + 4 * MT * P2;   // [o3][MT][P2]
  __shared__ const double* ch[8];
  // 1D grid, the tiles of a parent adjacent (they read the same children: L2 reuse)
  const int b = parents[blockIdx.x / C::NTILE], tid = threadIdx.x, m0 = (blockIdx.x % C::NTILE) * MT;
  const int lane = tid & 31, g = lane >> 2, q = lane & 3;
  if (tid < 8) {
    const int c = t.child[8 * (int64_t)b + tid];
    ch[tid] = (c >= 0 && (t.flags[c] & F_OUT)) ? mom + (size_t)t.fout_rank[c] * P3 : nullptr;
  }
  for (int i = tid; i < 2 * P2; i += C::NT) sA[i] = A[i];
  __syncthreads();
  bool any = false;
#pragma unroll
  for (int o = 0; o < 8; ++o) any |= ch[o] != nullptr;
  if (!any) return;
  // ---- axis 1: xi[gg][i][n2n3] = sum_{o1,k1} A_o1[m0+i][k1] mu_(o1 gg)[k1][n2n3]
  // M = MT rows (one tile for MT <= 8), K = 2p, N = 4 groups x p^2 columns
  {
    int koff[KS2];   // per k step: k1 p^2, or -1 (padding)
    bool kh[KS2];    // o1 of the k step
#pragma unroll
    for (int ks = 0; ks < KS2; ++ks) {
      int o, kk;
      bool ok;
      split_k2<P>(4 * ks + q, o, kk, ok);
      koff[ks] = ok ? kk * P2 : -1;
      kh[ks] = o;
    }
    grp_tiles<KS2, (P <= 18 ? 2 : 1)>(
        (MT + 7) / 8, 4 * NT1,
        [&](int mt, int ks) {
          int o, kk;
          bool ok;
          split_k2<P>(4 * ks + q, o, kk, ok);
          const int i = mt * 8 + g;
          return (ok && i < MT && m0 + i < P) ? sA[(o * P + m0 + i) * P + kk] : 0.0;
        },
        [&](int nt, int ks) {
          const int gg = nt / NT1, n = min((nt - gg * NT1) * 8 + g, P2 - 1);
          const double* c = ch[(kh[ks] ? 4 : 0) + gg];
          return (c && koff[ks] >= 0) ? __ldg(c + koff[ks] + n) : 0.0;
        },
        [&](int mt, int nt, double v0, double v1) {
          const int gg = nt / NT1, n = (nt - gg * NT1) * 8 + 2 * q, i = mt * 8 + g;
          if (i < MT) {
            double* row = xi + (gg * MT + i) * P2;
            if (n < P2) row[n] = v0;
            if (n + 1 < P2) row[n + 1] = v1;
          }
        },
        NoPre{});
  }
  __syncthreads();
  // ---- axis 2: eta[o3][i][m2 n3] = sum_{o2,k2} A_o2[m2][k2] xi[(o2 o3)][i][k2 n3]
  // M = p rows m2, K = 2p, N = 2 (o3) x MT p columns (i, n3)
  {
    int koff[KS2];   // per k step: o2 2 MT p^2 + k2 p, or -1
#pragma unroll
    for (int ks = 0; ks < KS2; ++ks) {
      int o, kk;
      bool ok;
      split_k2<P>(4 * ks + q, o, kk, ok);
      koff[ks] = ok ? o * 2 * MT * P2 + kk * P : -1;
    }
    grp_tiles<KS2>(
        (P + 7) / 8, 2 * NT2,
        [&](int mt, int ks) {
          int o, kk;
          bool ok;
          split_k2<P>(4 * ks + q, o, kk, ok);
          const int m2 = mt * 8 + g;
          return (ok && m2 < P) ? sA[(o * P + m2) * P + kk] : 0.0;
        },
        [&](int nt, int ks) {
          const int o3 = nt >= NT2, n = (nt - o3 * NT2) * 8 + g, i = n / P, n3 = n - i * P;
          return (koff[ks] >= 0 && i < MT) ? xi[koff[ks] + (o3 * MT + i) * P2 + n3] : 0.0;
        },
        [&](int mt, int nt, double v0, double v1) {
          const int m2 = mt * 8 + g;
          if (m2 >= P) return;
          const int o3 = nt >= NT2;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int n = (nt - o3 * NT2) * 8 + 2 * q + e, i = n / P, n3 = n - i * P;
            if (i < MT) eta[(o3 * MT + i) * P2 + m2 * P + n3] = e ? v1 : v0;
          }
        },
        NoPre{});
  }
  __syncthreads();
  // ---- axis 3: mu_P[m0+i][m2][m3] += sum_{o3,k3} eta[o3][i][m2][k3] A_o3[m3][k3]
  // M = MT p rows (i, m2), K = 2p, N = p columns m3
  {
    int koff[KS2];   // per k step: o3 MT p^2 + k3, or -1
#pragma unroll
    for (int ks = 0; ks < KS2; ++ks) {
      int o, kk;
      bool ok;
      split_k2<P>(4 * ks + q, o, kk, ok);
      koff[ks] = ok ? o * MT * P2 + kk : -1;
    }
    double* dst = mom + (size_t)t.fout_rank[b] * P3;
    grp_tiles<KS2>(
        (MT * P + 7) / 8, (P + 7) / 8,
        [&](int mt, int ks) {
          const int m = mt * 8 + g, i = m / P, m2 = m - i * P;
          return (koff[ks] >= 0 && i < MT) ? eta[koff[ks] + i * P2 + m2 * P] : 0.0;
        },
        [&](int nt, int ks) {
          int o, kk;
          bool ok;
          split_k2<P>(4 * ks + q, o, kk, ok);
          const int m3 = nt * 8 + g;
          return (ok && m3 < P) ? sA[(o * P + m3) * P + kk] : 0.0;
        },
        [&](int mt, int nt, double v0, double v1) {
          const int m = mt * 8 + g, i = m / P, m2 = m - i * P, n = nt * 8 + 2 * q;
          if (i >= MT || m0 + i >= P) return;
          // one writer per element: fire-and-forget reductions (RED), no read latency
          double* row = dst + (size_t)(m0 + i) * P2 + m2 * P;
          if (n < P) atomicAdd(row + n, v0);
          if (n + 1 < P) atomicAdd(row + n + 1, v1);
        },
        NoPre{});
  }
}

template <int P, int MT>
__global__ void __launch_bounds__(GrpCfg<P, MT>::NT) k_p2c_grp(DevTree t, const int32_t* __restrict__ parents,
                                                 const double* __restrict__ A, double* __restrict__ lam) {
  using C = GrpCfg<P, MT>;
  constexpr int P2 = C::P2, P3 = P2 * P, KS1 = C::KS1, KS2 = C::KS2;
  extern __shared__ double sm[];
  double* sA = sm;                   // [2][P][P]: A_s[n][k]
  double* zeta = sA + 2 * P2;        // [o1][MT][P2]        (k1 m2 m3)
  double* zeta2 = zeta + 2 * MT * P2;   // [o1][o2][MT][P2]  (k1 k2 m3)
  __shared__ double* ch[8];
  // 1D grid, the tiles of a parent adjacent (they read the same parent: L2 reuse)
  const int b = parents[blockIdx.x / C::NTILE], tid = threadIdx.x, k0 = (blockIdx.x % C::NTILE) * MT;
  if (tid < 8) {
    const int c = t.child[8 * (int64_t)b + tid];
    ch[tid] = (c >= 0 && (t.flags[c] & F_EXP)) ? lam + (size_t)t.exp_rank[c] * P3 : nullptr;
  }
  for (int i = tid; i < 2 * P2; i += C::NT) sA[i] = A[i];
  __syncthreads();
  bool any = false;
#pragma unroll
  for (int o = 0; o < 8; ++o) any |= ch[o] != nullptr;
  if (!any) return;
  // the parent's full local expansion (its own part plus what it inherited: the level above
  // was completed by the previous launch)
  const double* src = lam + (size_t)t.exp_rank[b] * P3;
  // axis 1: zeta[o1][i][m2m3] = sum_m1 A_o1[m1][k0+i] Lambda_P[m1][m2m3]
  mma_tiles<KS1>(
      (2 * MT + 7) / 8, (P2 + 7) / 8,
      [&](int m, int k) {
        const int o1 = m >= MT, i = m - o1 * MT;
        return (m < 2 * MT && k0 + i < P && k < P) ? sA[(o1 * P + k) * P + k0 + i] : 0.0;
      },
      [&](int k, int n) {
        return (k < P && n < P2) ? src[(size_t)k * P2 + n] : 0.0;
      },
      [&](int m, int n, double v0, double v1) {
        if (m < 2 * MT) {
          if (n < P2) zeta[m * P2 + n] = v0;
          if (n + 1 < P2) zeta[m * P2 + n + 1] = v1;
        }
      });
  __syncthreads();
  // axis 2: zeta2[o1][o2][i][k2 m3] = sum_m2 A_o2[m2][k2] zeta[o1][i][m2 m3]
  mma_tiles<KS1>(
      (2 * P + 7) / 8, (2 * MT * P + 7) / 8,
      [&](int m, int k) {
        const int o2 = m >= P, k2 = m - o2 * P;
        return (m < 2 * P && k < P) ? sA[(o2 * P + k) * P + k2] : 0.0;
      },
      [&](int k, int n) {
        const int r = n / P, m3 = n - r * P;   // r = o1 * MT + i
        return (k < P && r < 2 * MT) ? zeta[r * P2 + k * P + m3] : 0.0;
      },
      [&](int m, int n, double v0, double v1) {
        if (m >= 2 * P) return;
        const int o2 = m >= P, k2 = m - o2 * P;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int nn = n + e, r = nn / P, m3 = nn - r * P;
          if (r < 2 * MT) {
            const int o1 = r >= MT, i = r - o1 * MT;
            zeta2[((o1 * 2 + o2) * MT + i) * P2 + k2 * P + m3] = e ? v1 : v0;
          }
        }
      });
  __syncthreads();
  // axis 3: Lambda_(o1 o2 o3)[k0+i][k2][k3] += sum_m3 zeta2[o1][o2][i][k2][m3] A_o3[m3][k3]
  // (added to the child's own part written by the back transforms: the current values are
  // loaded before each tile's DMMA chain)
  auto out_ptr = [&](int m, int nn) -> double* {
    const int r = m / P, k2 = m - r * P;   // r = (o1 o2) * MT + i
    if (r >= 4 * MT || nn >= 2 * P) return nullptr;
    const int g = r / MT, i = r - g * MT;
    if (k0 + i >= P) return nullptr;
    const int o3 = nn >= P, k3 = nn - o3 * P;
    double* c = ch[g * 2 + o3];
    return c ? c + (size_t)(k0 + i) * P2 + k2 * P + k3 : nullptr;
  };
  mma_tiles_acc<KS1>(
      (4 * MT * P + 7) / 8, (2 * P + 7) / 8,
      [&](int m, int k) { return (m < 4 * MT * P && k < P) ? zeta2[(size_t)(m / P) * P2 + (m % P) * P + k] : 0.0; },
      [&](int k, int n) {
        const int o3 = n >= P, k3 = n - o3 * P;
        return (k < P && n < 2 * P) ? sA[(o3 * P + k) * P + k3] : 0.0;
      },
      [&](int m, int n, double& p0, double& p1) {
        const double* a = out_ptr(m, n);
        const double* b = out_ptr(m, n + 1);
        p0 = a ? *a : 0.0;
        p1 = b ? *b : 0.0;
      },
      [&](int m, int n, double v0, double v1) {
        double* a = out_ptr(m, n);
        double* b = out_ptr(m, n + 1);
        if (a) *a = v0;   // one writer per element
        if (b) *b = v1;
      });
}

// ---------------------------------------------------------------- plane waves
// Real parity-split representation of the plane-wave expansions.  With Qr (tables.cu:
// Q[m][n] = Qr[|m|][n] i^{n mod 2} sgn(m)^{n mod 2}) the outgoing expansion of Eq. 3.42,
//   Phi(m1,m2,m3) = sum_n Q[m1][n1] Q[m2][n2] Q[m3][n3] mu[n1 n2 n3],
// splits by the index parities pi_d = n_d mod 2 into eight REAL arrays on the octant
// a, b, c in [0, nf]:
//   F_pi[a][b][c] = sum_{n_d = pi_d (mod 2)} Qr[a][n1] Qr[b][n2] Qr[c][n3] mu[n1 n2 n3],
//   Phi(m) = sum_pi i^{|pi|} sgn(m1)^pi1 sgn(m2)^pi2 sgn(m3)^pi3 F_pi[|m1|][|m2|][|m3|].
// The colleague shift exp(i h_l m_d delta_d r_l) of Eq. 3.39 (h_l r_l = 2 pi/3) acts on
// each parity pair (F_{pi_d=0}, F_{pi_d=1}) of axis d as a rotation by 2 pi |m_d| delta_d/3;
// the weights w_l(|m|) act diagonally; and T_pw2poly (Eqs. 3.43-3.44: sum over all m,
// real part) collapses to
//   Lambda[n1 n2 n3] = sum_{abc} Gr[n1][a] Gr[n2][b] Gr[n3][c] Psi_{(n1,n2,n3) mod 2}[a][b][c]
// with Gr[n][a] = c_a Qr[a][n], c_0 = 1, c_a = 2.  Everything is real and each 1D factor
// has half of p columns: 4x fewer flops than the complex form.
// Per-box layout F[a][pi][b][c], pi = 4 pi1 + 2 pi2 + pi3: one slab a is contiguous.
// Storage precision of the outgoing plane waves F (precision tier, DESIGN.md reading
// R16): fp32 for eps >= 1e-6 (p <= 18) -- F is re-read 27 times per level from L2 and
// its rounding adds < 2% of the 1e-6 error budget -- fp64 for eps = 1e-9.  All
// arithmetic is fp64; only the stored values are rounded.
template <int P>
using FStore = typename std::conditional<(P <= 18), float, double>::type;

template <int P, int H>
struct PwGeom {
  static constexpr int PP = (P + 1) & ~1, HH = (H + 1) & ~1, P2 = P * P, HSQ = H * H;
  static constexpr int SLAB = 8 * H * H;            // doubles per slab a
  static constexpr size_t BOX = (size_t)H * SLAB;   // doubles per box
};

// 1D transform of P values held in registers by the p-row of an smem matrix (row
// length even, double2 loads), restricted to one parity class of n.
template <int P, int PAR>
__device__ __forceinline__ double dot_par(const double* __restrict__ row, const double* v) {
  double s = 0.0;
#pragma unroll
  for (int n = 0; n < P; n += 2) {
    const double2 q = *(const double2*)(row + n);
    if (PAR == 0) s = fma(q.x, v[n], s);
    else if (n + 1 < P) s = fma(q.y, v[n + 1], s);
  }
  return s;
}

// Outgoing expansion F(B) of an F_out box from its moments (T_prox2pw, Eq. 3.42):
// three axis transforms as fp64 tensor-core GEMMs (DMMA m8n8k4, K = ceil(p/2) padded
// to 4), per parity of the axis being contracted:
//   S1 (n3 -> c):  X1[n1 n2][c]  = sum_j mu[n1 n2][2j+pi3] Qr[c][2j+pi3]
//   S2 (n2 -> b):  X2[b][n1][c]  = sum_j Qr[b][2j+pi2] X1[n1 (2j+pi2)][c]
//   S3 (n1 -> a):  F[a][pi][b c] = sum_j Qr[a][2j+pi1] X2[b][2j+pi1][c]   -> global
// over column chunks of CH values of c (all of them when they fit).
template <int P, int H, int CH>
struct Prox2pw {
  using G = PwGeom<P, H>;
  // p = 28: one CTA per SM (shared memory), 16 warps to keep more DMMA tiles in flight
  static constexpr int NT = P > 18 ? 512 : 256, KS = ((P + 1) / 2 + 3) / 4, HP = (H + 7) / 8 * 8;
  static constexpr size_t smem = sizeof(double) * ((size_t)2 * HP * KS * 4 + (size_t)P * P * CH + (size_t)H * P * CH);
};
// RB: the register-blocked sweeps (device.cuh mma_sweep_m / mma_sweep_n: the 1D transform
// matrix's fragments stay in registers, one load of the large operand per 8-column tile
// and HP/8 (or CH/8) DMMA chains on it) instead of independent 8x8 tiles.
template <int P, int H, int CH, bool RB>
__global__ void __launch_bounds__(Prox2pw<P, H, CH>::NT) k_prox2pw(DevTree t, const int32_t* __restrict__ boxes,
                                                 const double* __restrict__ Qr, const double* __restrict__ mom,
                                                 FStore<P>* __restrict__ F, size_t base, size_t stride) {
  using G = PwGeom<P, H>;
  using C = Prox2pw<P, H, CH>;
  using TF = FStore<P>;
  constexpr int NT = C::NT, P2 = G::P2, PP = G::PP, KS = C::KS, K4 = KS * 4, HP = C::HP, HSQ = G::HSQ;
  // H and CH even (the non-root boxes at p = 28): a lane's two outputs (n, n + 1) stay in
  // one row of c and are stored as one 16-byte word (smem intermediates and F)
  constexpr bool EV = RB && H % 2 == 0 && CH % 2 == 0;
  extern __shared__ __align__(16) double sm_px[];
  double* sQ = sm_px;                  // [2][HP][K4]: sQ[pi][a][j] = Qr[a][2j+pi], zero padded
  double* X1 = sQ + 2 * HP * K4;     // [P2][CH]
  double* X2 = X1 + P2 * CH;         // [H][P][CH]
  const int b = boxes[blockIdx.x], tid = threadIdx.x;
  const int r = t.fout_rank[b];
  const double* mu = mom + (size_t)r * P * P2;
  TF* out = F + base + (size_t)(r == 0 ? 0 : r - 1) * stride;
  for (int i = tid; i < 2 * HP * K4; i += NT) {
    const int j = i % K4, a = (i / K4) % HP, pi = i / (K4 * HP), n = 2 * j + pi;
    sQ[i] = (a < H && n < P) ? Qr[a * PP + n] : 0.0;
  }
  __syncthreads();
  for (int c0 = 0; c0 < H; c0 += CH) {
    const int nc = min(CH, H - c0);
    for (int pi3 = 0; pi3 < 2; ++pi3) {
      const double* q3 = sQ + pi3 * HP * K4;
      // S1: M = P2 rows (n1 n2), N = nc, K = j
      {
        auto fa = [&](int m, int k) { return (m < P2 && 2 * k + pi3 < P) ? __ldg(mu + m * P + 2 * k + pi3) : 0.0; };
        auto fb = [&](int k, int n) { return (n < nc && c0 + n < H) ? q3[(c0 + n) * K4 + k] : 0.0; };
        auto fc = [&](int m, int n, double v0, double v1) {
          if (m < P2) {
            if constexpr (EV) {   // n, nc even: one 16-byte store
              if (n < nc) *reinterpret_cast<double2*>(X1 + m * CH + n) = make_double2(v0, v1);
            } else {
              if (n < nc) X1[m * CH + n] = v0;
              if (n + 1 < nc) X1[m * CH + n + 1] = v1;
            }
          }
        };
        if constexpr (RB) mma_sweep_m<KS, (CH + 7) / 8>((P2 + 7) / 8, fa, fb, fc);
        else mma_tiles<KS>((P2 + 7) / 8, (nc + 7) / 8, fa, fb, fc);
      }
      __syncthreads();
      for (int pi2 = 0; pi2 < 2; ++pi2) {
        const double* q2 = sQ + pi2 * HP * K4;
        // S2: M = H rows b, N = (n1, c) = P CH (c >= nc padded), K = j
        {
          auto fa = [&](int m, int k) { return q2[m * K4 + k]; };
          auto fb = [&](int k, int n) {
            const int n1 = n / CH, c = n - n1 * CH;
            return (n1 < P && c < nc && 2 * k + pi2 < P) ? X1[(n1 * P + 2 * k + pi2) * CH + c] : 0.0;
          };
          auto fc = [&](int m, int n, double v0, double v1) {
            if (m < H) {
              if constexpr (EV) {
                if (n < P * CH) *reinterpret_cast<double2*>(X2 + m * P * CH + n) = make_double2(v0, v1);
              } else {
                if (n < P * CH) X2[m * P * CH + n] = v0;
                if (n + 1 < P * CH) X2[m * P * CH + n + 1] = v1;
              }
            }
          };
          if constexpr (RB) mma_sweep_n<KS, HP / 8>((P * CH + 7) / 8, fa, fb, fc);
          else mma_tiles<KS>(HP / 8, (P * CH + 7) / 8, fa, fb, fc);
        }
        __syncthreads();
        for (int pi1 = 0; pi1 < 2; ++pi1) {
          const double* q1 = sQ + pi1 * HP * K4;
          TF* o = out + (size_t)(4 * pi1 + 2 * pi2 + pi3) * HSQ + c0;
          // S3: M = H rows a, N = (b, c) = H CH (c >= nc skipped), K = j
          auto fa = [&](int m, int k) { return q1[m * K4 + k]; };
          auto fb = [&](int k, int n) {
            const int bb = n / CH, c = n - bb * CH;
            return (bb < H && 2 * k + pi1 < P) ? X2[(bb * P + 2 * k + pi1) * CH + c] : 0.0;
          };
          auto fc = [&](int m, int n, double v0, double v1) {
            if (m < H) {
              const int bb = n / CH, c = n - bb * CH;   // n even, CH may be odd
              if constexpr (EV && sizeof(TF) == 8) {   // (c, c + 1) in one row, 16-byte aligned
                if (bb < H && c < nc)
                  __stcs(reinterpret_cast<double2*>(o + (size_t)m * G::SLAB + bb * H + c), make_double2(v0, v1));
                return;
              }
              if (bb < H && c < nc) o[(size_t)m * G::SLAB + bb * H + c] = (TF)v0;
              const int b1 = (n + 1) / CH, c1 = n + 1 - b1 * CH;
              if (b1 < H && c1 < nc) o[(size_t)m * G::SLAB + b1 * H + c1] = (TF)v1;
            }
          };
          if constexpr (RB) mma_sweep_n<KS, HP / 8>((H * CH + 7) / 8, fa, fb, fc);
          else mma_tiles<KS>(HP / 8, (H * CH + 7) / 8, fa, fb, fc);
        }
        __syncthreads();   // X2 is rewritten by the next pi2
      }
    }
  }
}

// fp32 tier: T_prox2pw (Eq. 3.42) of every F_out box as three whole-box axis
// contractions with packed FFMA2: an axis contraction over n of one parity class is a
// sum over the input pairs (2j, 2j+1), and (Qr[m][2j], Qr[m][2j+1]) x (v[2j], v[2j+1])
// accumulates the parity-0 and parity-1 outputs in the two halves of one register:
//   axis 3: X1[n1][n2][c]  = (sum_{n3 even}, sum_{n3 odd}) Qr[c][n3] mu[n1][n2][n3]
//   axis 2: X2[n1][pi3][b][c] = (pi2 = 0, 1) halves over n2
//   axis 1: F[a][pi][b][c] (fp32, global) over n1.
template <int P, int H>
struct Px32 {
  static constexpr int NT = 256, PH = (P + 1) / 2, PP = 2 * PH;
  static constexpr size_t smem =
      sizeof(float2) * ((size_t)H * PH + (size_t)P * P * H + (size_t)P * 2 * H * H);
};
template <int P, int H>
__global__ void __launch_bounds__(Px32<P, H>::NT) k_prox2pw32(DevTree t, const int32_t* __restrict__ boxes,
                                                              const double* __restrict__ Qr,
                                                              const double* __restrict__ mom, float* __restrict__ F,
                                                              size_t base, size_t stride) {
  using C = Px32<P, H>;
  constexpr int NT = C::NT, PH = C::PH, PP = C::PP, HSQ = H * H, P2 = P * P;
  extern __shared__ float2 smx[];
  float2* QP = smx;              // [m][j] = (Qr[m][2j], Qr[m][2j+1])
  float2* X1 = QP + H * PH;      // [n1][n2][c]      (pi3 halves)
  float2* X2 = X1 + P2 * H;      // [n1][pi3][b][c]  (pi2 halves)
  const int b = boxes[blockIdx.x], tid = threadIdx.x;
  const int r = t.fout_rank[b];
  const double* mu = mom + (size_t)r * P * P2;
  float* out = F + base + (size_t)(r == 0 ? 0 : r - 1) * stride;
  for (int i = tid; i < H * PH; i += NT) {
    const int m = i / PH, j = i - m * PH;
    QP[i] = make_float2((float)Qr[m * PP + 2 * j], (float)Qr[m * PP + 2 * j + 1]);   // Qr rows are zero-padded
  }
  __syncthreads();
  // axis 3: one (n1, n2) row of mu per unit
  for (int u = tid; u < P2; u += NT) {
    float2 v[PH];
#pragma unroll
    for (int j = 0; j < PH; ++j)
      v[j] = make_float2((float)mu[(size_t)u * P + 2 * j], 2 * j + 1 < P ? (float)mu[(size_t)u * P + 2 * j + 1] : 0.0f);
#pragma unroll 1
    for (int c = 0; c < H; ++c) {
      float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int j = 0; j < PH; ++j) acc = __ffma2_rn(QP[c * PH + j], v[j], acc);
      X1[u * H + c] = acc;
    }
  }
  __syncthreads();
  // axis 2: unit (n1, pi3, c): inputs X1[n1][n2][c].pi3 over n2
  for (int u = tid; u < P * 2 * H; u += NT) {
    const int n1 = u / (2 * H), p3 = (u / H) % 2, c = u % H;
    float2 v[PH];
#pragma unroll
    for (int j = 0; j < PH; ++j) {
      const float2 e0 = X1[(n1 * P + 2 * j) * H + c];
      const float2 e1 = 2 * j + 1 < P ? X1[(n1 * P + 2 * j + 1) * H + c] : make_float2(0.0f, 0.0f);
      v[j] = p3 ? make_float2(e0.y, e1.y) : make_float2(e0.x, e1.x);
    }
#pragma unroll 1
    for (int bb = 0; bb < H; ++bb) {
      float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int j = 0; j < PH; ++j) acc = __ffma2_rn(QP[bb * PH + j], v[j], acc);
      X2[((n1 * 2 + p3) * H + bb) * H + c] = acc;
    }
  }
  __syncthreads();
  // axis 1: unit (pi2, pi3, b, c): inputs X2[n1][pi3][b][c].pi2 over n1 -> F[a][pi][b][c]
  for (int u = tid; u < 4 * HSQ; u += NT) {
    const int g = u / HSQ, bc = u - g * HSQ, p2 = g >> 1, p3 = g & 1;
    float2 v[PH];
#pragma unroll
    for (int j = 0; j < PH; ++j) {
      const float2 e0 = X2[((2 * j) * 2 + p3) * HSQ + bc];
      const float2 e1 = 2 * j + 1 < P ? X2[((2 * j + 1) * 2 + p3) * HSQ + bc] : make_float2(0.0f, 0.0f);
      v[j] = p2 ? make_float2(e0.y, e1.y) : make_float2(e0.x, e1.x);
    }
#pragma unroll 1
    for (int a = 0; a < H; ++a) {
      float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int j = 0; j < PH; ++j) acc = __ffma2_rn(QP[a * PH + j], v[j], acc);
      float* o = out + (size_t)a * 8 * HSQ + bc;
      o[(2 * p2 + p3) * HSQ] = acc.x;         // pi1 = 0
      o[(4 + 2 * p2 + p3) * HSQ] = acc.y;     // pi1 = 1
    }
  }
}

// Rotation-accumulate along one axis (bit ST of the parity index): acc += R(delta phi) g.
template <int ST, int DELTA>
__device__ __forceinline__ void rot_acc(double* acc, const double* g, double C, double S) {
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    if (p & ST) continue;
    const double g0 = g[p], g1 = g[p + ST];
    if (DELTA == 0) {
      acc[p] += g0;
      acc[p + ST] += g1;
    } else if (DELTA > 0) {
      acc[p] = fma(C, g0, fma(-S, g1, acc[p]));
      acc[p + ST] = fma(S, g0, fma(C, g1, acc[p + ST]));
    } else {
      acc[p] = fma(C, g0, fma(S, g1, acc[p]));
      acc[p + ST] = fma(-S, g0, fma(C, g1, acc[p + ST]));
    }
  }
}
__device__ __forceinline__ void rot_cs(int m, double& C, double& S) {
  const int e = m % 3;   // angle 2 pi m / 3
  C = e == 0 ? 1.0 : -0.5;
  S = e == 0 ? 0.0 : (e == 1 ? 0.86602540378443864676 : -0.86602540378443864676);
}

// ---- fp32 tier (reading R16, p <= 18): translation by parent groups.
// The 8 children of a parent B have their 27 colleagues inside the 4x4x4 window of
// level-l boxes around them (the children of B's colleagues), so one pass over the
// window's 64 outgoing expansions serves all 8 (64 instead of 8 x 27 = 216 reads of F,
// which is re-read from L2 and bounds the per-box form).  For one mode (a, b, c) a
// thread keeps the window sums in registers as three separable passes (Eq. 3.39 with
// e^{i h m . delta r_l} = product of per-axis rotations by 2 pi m_d delta_d / 3 of the
// parity pairs): Z over w3, Y over w2, X over w1, for child offsets o in {0,1}^3 with
// delta = o + 1 - w.  Sums in fp32 (the F values are fp32-rounded already); the level's
// difference-kernel weights are applied and the weighted incoming expansion of each
// local-expansion child is written to T[exp_rank] for k_pwlocal<..., FROMT>.
template <int ST, int DELTA>
__device__ __forceinline__ void rot_accf(float* acc, const float* g, float C, float S) {
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    if (p & ST) continue;
    const float g0 = g[p], g1 = g[p + ST];
    if (DELTA == 0) {
      acc[p] += g0;
      acc[p + ST] += g1;
    } else if (DELTA > 0) {
      acc[p] = fmaf(C, g0, fmaf(-S, g1, acc[p]));
      acc[p + ST] = fmaf(S, g0, fmaf(C, g1, acc[p + ST]));
    } else {
      acc[p] = fmaf(C, g0, fmaf(S, g1, acc[p]));
      acc[p + ST] = fmaf(-S, g0, fmaf(C, g1, acc[p + ST]));
    }
  }
}
template <int ST>
__device__ __forceinline__ void rot_accf_d(int delta, float* acc, const float* g, float C, float S) {
  if (delta > 0) rot_accf<ST, 1>(acc, g, C, S);
  else if (delta < 0) rot_accf<ST, -1>(acc, g, C, S);
  else rot_accf<ST, 0>(acc, g, C, S);
}
__device__ __forceinline__ void rot_csf(int m, float& C, float& S) {
  const int e = m % 3;   // angle 2 pi m / 3
  C = e == 0 ? 1.0f : -0.5f;
  S = e == 0 ? 0.0f : (e == 1 ? 0.866025403784438647f : -0.866025403784438647f);
}
constexpr int PWS_NT = 128, PWS_GY = 2;
template <int H>
__global__ void __launch_bounds__(PWS_NT, 3)
    k_pwshift(DevTree t, const int32_t* __restrict__ parents, const float* __restrict__ F, size_t base,
              size_t stride, const double* __restrict__ W, size_t wstride, float* __restrict__ Tout) {
  constexpr int HSQ = H * H, NM = H * HSQ, SLAB = 8 * HSQ;
  __shared__ const float* win[64];   // window box (w1 w2 w3), null: absent or not F_out
  __shared__ int rank[8];            // exp rank of child o = (o1 o2 o3), -1: none
  __shared__ int lvl;
  // 1D grid, the PWS_GY mode slices of a parent adjacent (same window: L2 reuse)
  const int pb = parents[blockIdx.x / PWS_GY], slice = blockIdx.x % PWS_GY, tid = threadIdx.x;
  if (tid < 64) {
    const int w1 = tid >> 4, w2 = (tid >> 2) & 3, w3 = tid & 3;
    // window index w = 2 D + c + 1 for the child c of the parent colleague B + D
    const int D1 = w1 == 0 ? -1 : (w1 == 3 ? 1 : 0), D2 = w2 == 0 ? -1 : (w2 == 3 ? 1 : 0),
              D3 = w3 == 0 ? -1 : (w3 == 3 ? 1 : 0);
    const int c1 = w1 - 2 * D1 - 1, c2 = w2 - 2 * D2 - 1, c3 = w3 - 2 * D3 - 1;
    const int S = t.coll[27 * (int64_t)pb + (D1 + 1) * 9 + (D2 + 1) * 3 + (D3 + 1)];
    const float* ptr = nullptr;
    if (S >= 0) {
      const int ch = t.child[8 * (int64_t)S + (c1 << 2) + (c2 << 1) + c3];
      if (ch >= 0 && (t.flags[ch] & F_OUT)) ptr = F + base + (size_t)(t.fout_rank[ch] - 1) * stride;
    }
    win[tid] = ptr;
  } else if (tid < 72) {
    const int ch = t.child[8 * (int64_t)pb + (tid - 64)];
    rank[tid - 64] = (ch >= 0 && (t.flags[ch] & F_EXP)) ? t.exp_rank[ch] : -1;
    if (tid == 64) lvl = t.level[pb] + 1;
  }
  __syncthreads();
  bool any = false;
#pragma unroll
  for (int o = 0; o < 8; ++o) any |= rank[o] >= 0;
  if (!any) return;
  const double* Wl = W + (size_t)lvl * wstride;
  for (int m = slice * PWS_NT + tid; m < NM; m += PWS_GY * PWS_NT) {
    const int a = m / HSQ, bc = m - a * HSQ;
    float Ca, Sa, Cb, Sb, Cc, Sc;
    rot_csf(a, Ca, Sa);
    rot_csf(bc / H, Cb, Sb);
    rot_csf(bc % H, Cc, Sc);
    const size_t off = (size_t)a * SLAB + bc;
    float X[8][8];
#pragma unroll
    for (int o = 0; o < 8; ++o)
#pragma unroll
      for (int p = 0; p < 8; ++p) X[o][p] = 0.0f;
#pragma unroll
    for (int w1 = 0; w1 < 4; ++w1) {
      float Y[2][2][8];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int p = 0; p < 8; ++p) Y[i][j][p] = 0.0f;
#pragma unroll
      for (int w2 = 0; w2 < 4; ++w2) {
        float g[4][8];
#pragma unroll
        for (int w3 = 0; w3 < 4; ++w3) {
          const float* sp = win[w1 * 16 + w2 * 4 + w3];
#pragma unroll
          for (int p = 0; p < 8; ++p) g[w3][p] = sp ? __ldg(sp + off + p * HSQ) : 0.0f;
        }
        float Z[2][8];
#pragma unroll
        for (int o3 = 0; o3 < 2; ++o3) {
#pragma unroll
          for (int p = 0; p < 8; ++p) Z[o3][p] = 0.0f;
#pragma unroll
          for (int w3 = o3; w3 < o3 + 3; ++w3) rot_accf_d<1>(o3 + 1 - w3, Z[o3], g[w3], Cc, Sc);
        }
#pragma unroll
        for (int o2 = 0; o2 < 2; ++o2) {
          if (w2 < o2 || w2 > o2 + 2) continue;
#pragma unroll
          for (int o3 = 0; o3 < 2; ++o3) rot_accf_d<2>(o2 + 1 - w2, Y[o2][o3], Z[o3], Cb, Sb);
        }
      }
#pragma unroll
      for (int o1 = 0; o1 < 2; ++o1) {
        if (w1 < o1 || w1 > o1 + 2) continue;
#pragma unroll
        for (int o2 = 0; o2 < 2; ++o2)
#pragma unroll
          for (int o3 = 0; o3 < 2; ++o3) rot_accf_d<4>(o1 + 1 - w1, X[o1 * 4 + o2 * 2 + o3], Y[o2][o3], Ca, Sa);
      }
    }
    const float wt = (float)__ldg(Wl + m);
#pragma unroll
    for (int o = 0; o < 8; ++o) {
      const int r = rank[o];
      if (r < 0) continue;
      float* dst = Tout + (size_t)r * H * SLAB + off;
#pragma unroll
      for (int p = 0; p < 8; ++p) dst[p * HSQ] = wt * X[o][p];
    }
  }
}

// ---- eps = 1e-9 tier (p = 28, fp64): the same parent-group translation in double
// precision.  The 8 x 8 fp64 window sums of one mode do not fit one thread's registers,
// so a thread owns one mode and one half of the children (o1), and walks the 3 x 4 x 4
// part of the window that half needs (48 instead of 64 reads of F per mode and half;
// per child 24 instead of the 27 x 8 = 216 reads of the per-box form).  The weighted
// incoming expansions go to T (fp64) for the back transforms (k_pwlocal<..., FROMT>).
constexpr int PWS64_NT = 128;
template <int H>
__global__ void __launch_bounds__(PWS64_NT, 2)
    k_pwshift64(DevTree t, const int32_t* __restrict__ parents, const double* __restrict__ F, size_t base,
                size_t stride, const double* __restrict__ W, size_t wstride, double* __restrict__ Tout) {
  constexpr int HSQ = H * H, NM = H * HSQ, SLAB = 8 * HSQ;
  __shared__ const double* win[64];   // window box (w1 w2 w3), null: absent or not F_out
  __shared__ int rank[8];             // exp rank of child o = (o1 o2 o3), -1: none
  __shared__ int lvl;
  const int pb = parents[blockIdx.x], tid = threadIdx.x;   // grid: (parent, mode block, o1)
  if (tid < 64) {
    const int w1 = tid >> 4, w2 = (tid >> 2) & 3, w3 = tid & 3;
    const int D1 = w1 == 0 ? -1 : (w1 == 3 ? 1 : 0), D2 = w2 == 0 ? -1 : (w2 == 3 ? 1 : 0),
              D3 = w3 == 0 ? -1 : (w3 == 3 ? 1 : 0);
    const int c1 = w1 - 2 * D1 - 1, c2 = w2 - 2 * D2 - 1, c3 = w3 - 2 * D3 - 1;
    const int S = t.coll[27 * (int64_t)pb + (D1 + 1) * 9 + (D2 + 1) * 3 + (D3 + 1)];
    const double* ptr = nullptr;
    if (S >= 0) {
      const int ch = t.child[8 * (int64_t)S + (c1 << 2) + (c2 << 1) + c3];
      if (ch >= 0 && (t.flags[ch] & F_OUT)) ptr = F + base + (size_t)(t.fout_rank[ch] - 1) * stride;
    }
    win[tid] = ptr;
  } else if (tid < 72) {
    const int ch = t.child[8 * (int64_t)pb + (tid - 64)];
    rank[tid - 64] = (ch >= 0 && (t.flags[ch] & F_EXP)) ? t.exp_rank[ch] : -1;
    if (tid == 64) lvl = t.level[pb] + 1;
  }
  __syncthreads();
  const int o1 = blockIdx.z;
  bool any = false;
#pragma unroll
  for (int o = 0; o < 4; ++o) any |= rank[o1 * 4 + o] >= 0;
  if (!any) return;
  const double* Wl = W + (size_t)lvl * wstride;
  const int m = blockIdx.y * PWS64_NT + tid;
  if (m >= NM) return;
  const int a = m / HSQ, bc = m - a * HSQ;
  double Ca, Sa, Cb, Sb, Cc, Sc;
  rot_cs(a, Ca, Sa);
  rot_cs(bc / H, Cb, Sb);
  rot_cs(bc % H, Cc, Sc);
  const size_t off = (size_t)a * SLAB + bc;
  double X[2][2][8];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int p = 0; p < 8; ++p) X[i][j][p] = 0.0;
#pragma unroll 1
  for (int w1 = o1; w1 < o1 + 3; ++w1) {
    double Y[2][2][8];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int p = 0; p < 8; ++p) Y[i][j][p] = 0.0;
#pragma unroll
    for (int w2 = 0; w2 < 4; ++w2) {
      double Z[2][8];
#pragma unroll
      for (int p = 0; p < 8; ++p) Z[0][p] = Z[1][p] = 0.0;
#pragma unroll
      for (int w3 = 0; w3 < 4; ++w3) {
        const double* sp = win[w1 * 16 + w2 * 4 + w3];
        if (sp == nullptr) continue;
        double g[8];
#pragma unroll
        for (int p = 0; p < 8; ++p) g[p] = __ldg(sp + off + p * HSQ);
        // child o3 takes window w3 in o3..o3+2 with delta = o3 + 1 - w3
        if (w3 <= 2) {
          if (w3 == 0) rot_acc<1, 1>(Z[0], g, Cc, Sc);
          else if (w3 == 1) rot_acc<1, 0>(Z[0], g, Cc, Sc);
          else rot_acc<1, -1>(Z[0], g, Cc, Sc);
        }
        if (w3 >= 1) {
          if (w3 == 1) rot_acc<1, 1>(Z[1], g, Cc, Sc);
          else if (w3 == 2) rot_acc<1, 0>(Z[1], g, Cc, Sc);
          else rot_acc<1, -1>(Z[1], g, Cc, Sc);
        }
      }
#pragma unroll
      for (int o2 = 0; o2 < 2; ++o2) {
        if (w2 < o2 || w2 > o2 + 2) continue;
        const int d = o2 + 1 - w2;
#pragma unroll
        for (int o3 = 0; o3 < 2; ++o3) {
          if (d > 0) rot_acc<2, 1>(Y[o2][o3], Z[o3], Cb, Sb);
          else if (d < 0) rot_acc<2, -1>(Y[o2][o3], Z[o3], Cb, Sb);
          else rot_acc<2, 0>(Y[o2][o3], Z[o3], Cb, Sb);
        }
      }
    }
    const int d = o1 + 1 - w1;
#pragma unroll
    for (int o2 = 0; o2 < 2; ++o2)
#pragma unroll
      for (int o3 = 0; o3 < 2; ++o3) {
        if (d > 0) rot_acc<4, 1>(X[o2][o3], Y[o2][o3], Ca, Sa);
        else if (d < 0) rot_acc<4, -1>(X[o2][o3], Y[o2][o3], Ca, Sa);
        else rot_acc<4, 0>(X[o2][o3], Y[o2][o3], Ca, Sa);
      }
  }
  const double wt = __ldg(Wl + m);
#pragma unroll
  for (int o2 = 0; o2 < 2; ++o2)
#pragma unroll
    for (int o3 = 0; o3 < 2; ++o3) {
      const int r = rank[o1 * 4 + o2 * 2 + o3];
      if (r < 0) continue;
      double* dst = Tout + (size_t)r * H * SLAB + off;
#pragma unroll
      for (int p = 0; p < 8; ++p) dst[p * HSQ] = wt * X[o2][o3][p];
    }
}

// ---- Parent-group translation staged through shared memory (both tiers; TT = the
// plane-wave storage type, float for p <= 18, double for p = 28).  The same window sums
// as k_pwshift / k_pwshift64 (Eq. 3.39, separable per-axis rotations by 2 pi m_d delta_d
// / 3), over chunks of MC modes of one slab a, in two passes:
//   ZY: a thread owns (w1, pi1, mode i) and walks w2 = 0..3: it loads the 16 values
//       F[w1 w2 w3][pi1 pi2 pi3][m] (w3, pi2, pi3), sums the Z taps over w3 for both
//       children o3 in registers and accumulates the Y taps into Y[o2][o3][pi2 pi3];
//       the 16 results go to YS[w1 o2 o3][pi][MC] (shared, double buffered by chunk);
//   X:  a thread owns (child o, pi2 pi3, i): the three w1 taps from YS, the weights,
//       T (global).
// One barrier per chunk.  The three taps of an axis combine as  R(+1) g_l + g_m + R(-1) g_r
// for a child with window rows (l, m, r) = (o, o + 1, o + 2)  (delta = o + 1 - w).
template <class TT>
__device__ __forceinline__ void rot3(TT l0, TT l1, TT m0, TT m1, TT r0, TT r1, TT C, TT S, TT& o0, TT& o1) {
  const TT s0 = l0 + r0, s1 = l1 + r1, d0 = l0 - r0, d1 = l1 - r1;
  o0 = C * s0 + (m0 - S * d1);
  o1 = C * s1 + (m1 + S * d0);
}
template <int DELTA, class TT>
__device__ __forceinline__ void racc(TT& a0, TT& a1, TT g0, TT g1, TT C, TT S) {
  if (DELTA == 0) {
    a0 += g0;
    a1 += g1;
  } else if (DELTA > 0) {
    a0 += C * g0 - S * g1;
    a1 += S * g0 + C * g1;
  } else {
    a0 += C * g0 + S * g1;
    a1 += C * g1 - S * g0;
  }
}
template <class TT>
__device__ __forceinline__ void rcs(int m, TT& C, TT& S) {
  const int e = m % 3;   // angle 2 pi m / 3
  C = e == 0 ? TT(1) : TT(-0.5);
  S = e == 0 ? TT(0) : (e == 1 ? TT(0.86602540378443864676) : TT(-0.86602540378443864676));
}
template <int H, class TT>
struct PwsS {
  static constexpr int NT = 256, HSQ = H * H, MC = 32, NCH = (HSQ + MC - 1) / MC;
  static constexpr int YSZ = 16 * 8 * MC;   // one YS buffer
  static constexpr size_t smem = sizeof(TT) * (size_t)2 * YSZ;
  static constexpr int MINB = 2;
  static_assert(8 * MC == NT, "one ZY item per thread");
};
template <int H, class TT>
__global__ void __launch_bounds__(PwsS<H, TT>::NT, PwsS<H, TT>::MINB)
    k_pwshift_s(DevTree t, const int32_t* __restrict__ parents, const TT* __restrict__ F, size_t base, size_t stride,
                const double* __restrict__ W, size_t wstride, TT* __restrict__ Tout) {
  using C = PwsS<H, TT>;
  constexpr int NT = C::NT, HSQ = H * H, SLAB = 8 * HSQ, MC = C::MC, NCH = C::NCH, YSZ = C::YSZ;
  extern __shared__ __align__(16) unsigned char pws_raw[];
  TT* YSb = reinterpret_cast<TT*>(pws_raw);   // [2][(w1 o2) o3][pi][MC]
  __shared__ const TT* win[64];               // window box (w1 w2 w3), null: absent or not F_out
  __shared__ int rank[8];                     // exp rank of child o = (o1 o2 o3), -1: none
  __shared__ int lvl;
  const int pb = parents[blockIdx.x], tid = threadIdx.x;
  if (tid < 64) {
    const int w1 = tid >> 4, w2 = (tid >> 2) & 3, w3 = tid & 3;
    const int D1 = w1 == 0 ? -1 : (w1 == 3 ? 1 : 0), D2 = w2 == 0 ? -1 : (w2 == 3 ? 1 : 0),
              D3 = w3 == 0 ? -1 : (w3 == 3 ? 1 : 0);
    const int c1 = w1 - 2 * D1 - 1, c2 = w2 - 2 * D2 - 1, c3 = w3 - 2 * D3 - 1;
    const int S = t.coll[27 * (int64_t)pb + (D1 + 1) * 9 + (D2 + 1) * 3 + (D3 + 1)];
    const TT* ptr = nullptr;
    if (S >= 0) {
      const int ch = t.child[8 * (int64_t)S + (c1 << 2) + (c2 << 1) + c3];
      if (ch >= 0 && (t.flags[ch] & F_OUT)) ptr = F + base + (size_t)(t.fout_rank[ch] - 1) * stride;
    }
    win[tid] = ptr;
  } else if (tid < 72) {
    const int ch = t.child[8 * (int64_t)pb + (tid - 64)];
    rank[tid - 64] = (ch >= 0 && (t.flags[ch] & F_EXP)) ? t.exp_rank[ch] : -1;
    if (tid == 64) lvl = t.level[pb] + 1;
  }
  __syncthreads();
  bool any = false;
#pragma unroll
  for (int o = 0; o < 8; ++o) any |= rank[o] >= 0;
  if (!any) return;
  const double* Wl = W + (size_t)lvl * wstride;
  // ZY item of this thread: (w1, pi1) warp-uniform, i = lane
  const int zi = tid % MC, zg = tid / MC, pi1 = zg & 1, w1 = zg >> 1;
  int nb = 0;
  for (int ch = blockIdx.y; ch < H * NCH; ch += gridDim.y, ++nb) {
    const int a = ch / NCH, m0 = (ch - a * NCH) * MC;
    const size_t aoff = (size_t)a * SLAB;
    TT* YS = YSb + (nb & 1) * YSZ;
    {
      const int m = m0 + zi;
      const bool ok = m < HSQ;
      TT Cc, Sc, Cb, Sb;
      rcs(m % H, Cc, Sc);
      rcs(m / H, Cb, Sb);
      TT Y[2][2][4];   // [o2][o3][pi2 pi3]
#pragma unroll
      for (int o2 = 0; o2 < 2; ++o2)
#pragma unroll
        for (int o3 = 0; o3 < 2; ++o3)
#pragma unroll
          for (int p = 0; p < 4; ++p) Y[o2][o3][p] = TT(0);
#pragma unroll
      for (int w2 = 0; w2 < 4; ++w2) {
        TT g[4][4];   // [w3][pi2 pi3]
#pragma unroll
        for (int w3 = 0; w3 < 4; ++w3) {
          const TT* sp = ok ? win[w1 * 16 + w2 * 4 + w3] : nullptr;
#pragma unroll
          for (int p = 0; p < 4; ++p) g[w3][p] = sp ? __ldg(sp + aoff + (pi1 * 4 + p) * HSQ + m) : TT(0);
        }
        // Z taps: pairs (pi3 = 0, 1) for pi2 = 0, 1; child o3 from w3 = o3 .. o3 + 2
        TT Z[2][4];
#pragma unroll
        for (int o3 = 0; o3 < 2; ++o3)
#pragma unroll
          for (int p2 = 0; p2 < 2; ++p2)
            rot3(g[o3][2 * p2], g[o3][2 * p2 + 1], g[o3 + 1][2 * p2], g[o3 + 1][2 * p2 + 1], g[o3 + 2][2 * p2],
                 g[o3 + 2][2 * p2 + 1], Cc, Sc, Z[o3][2 * p2], Z[o3][2 * p2 + 1]);
        // Y taps: pairs (pi2 = 0, 1) for pi3 = 0, 1; child o2 takes w2 in o2 .. o2 + 2
#pragma unroll
        for (int o2 = 0; o2 < 2; ++o2) {
          if (w2 < o2 || w2 > o2 + 2) continue;
          constexpr int dummy = 0;
          (void)dummy;
#pragma unroll
          for (int o3 = 0; o3 < 2; ++o3)
#pragma unroll
            for (int p3 = 0; p3 < 2; ++p3) {
              TT& y0 = Y[o2][o3][p3];
              TT& y1 = Y[o2][o3][2 + p3];
              const int d = o2 + 1 - w2;
              if (d > 0) racc<1>(y0, y1, Z[o3][p3], Z[o3][2 + p3], Cb, Sb);
              else if (d < 0) racc<-1>(y0, y1, Z[o3][p3], Z[o3][2 + p3], Cb, Sb);
              else racc<0>(y0, y1, Z[o3][p3], Z[o3][2 + p3], Cb, Sb);
            }
        }
      }
#pragma unroll
      for (int o2 = 0; o2 < 2; ++o2)
#pragma unroll
        for (int o3 = 0; o3 < 2; ++o3)
#pragma unroll
          for (int p = 0; p < 4; ++p) YS[(((w1 * 2 + o2) * 2 + o3) * 8 + pi1 * 4 + p) * MC + zi] = Y[o2][o3][p];
    }
    __syncthreads();
    // ---- X: child o1 from w1 = o1 .. o1 + 2 (axis 1, mode a), weights, T; pairs (p, p + 4)
    TT Ca, Sa;
    rcs(a, Ca, Sa);
#pragma unroll
    for (int u = 0; u < 32 * MC / NT; ++u) {
      const int it = tid + u * NT, i = it % MC, g = it / MC, p = g & 3, o = g >> 2, m = m0 + i;
      const int r = rank[o];
      if (m >= HSQ || r < 0) continue;
      const TT* yl = YS + ((((o >> 2) * 2 + ((o >> 1) & 1)) * 2 + (o & 1)) * 8 + p) * MC + i;
      TT x0, x1;
      rot3(yl[0], yl[4 * MC], yl[32 * MC], yl[36 * MC], yl[64 * MC], yl[68 * MC], Ca, Sa, x0, x1);
      const TT wt = (TT)__ldg(Wl + (size_t)a * HSQ + m);
      TT* dst = Tout + (size_t)r * H * SLAB + aoff + m;
      dst[p * HSQ] = wt * x0;
      dst[(p + 4) * HSQ] = wt * x1;
    }
    // YS is double buffered: the next chunk writes the other buffer, and this buffer
    // again only after the next chunk's barrier (every thread is past this X pass)
  }
}

// eps = 1e-9 tier: T_pw2poly (Eqs. 3.43-3.44) of every non-root local box from the fp64
// weighted incoming expansion T[a][pi][b][c], all three axis contractions on DMMA
// (m8n8k4 f64).  The slabs a stream through shared memory AC = 2 at a time (cp.async
// double buffer): axis 3 (over c, output parity n3 % 2 picks pi3) into U[a][pi12][b][n3],
// axis 2 (over b) into V[a][pi1][n2 n3] for 4 slabs, then the axis-1 contraction over
// those 4 slabs as one DMMA k-step into Lambda accumulators that stay in registers for
// the whole box (each warp owns a fixed set of (n2 n3) column tiles).
template <int P, int H>
struct Pw2p64 {
  static constexpr int NT = 384, NW = NT / 32, AC = 2, HH = (H + 1) & ~1, P2 = P * P;
  static constexpr int PH = (P + 1) / 2, MT = (PH + 7) / 8;   // tiles of one parity class
  static constexpr int NT1 = (P2 + 7) / 8, TPW = (NT1 + NW - 1) / NW;
  static constexpr int TSZ = AC * 8 * H * H;
  static constexpr size_t smem =
      sizeof(double) * ((size_t)P * HH + 2 * (size_t)TSZ + (size_t)AC * 4 * H * P + 4 * 2 * (size_t)P2);
};
template <int P, int H>
__global__ void __launch_bounds__(Pw2p64<P, H>::NT, 1)
    k_pw2poly64(DevTree t, const int32_t* __restrict__ boxes, const double* __restrict__ Gr,
                const double* __restrict__ Tin, double* __restrict__ lam) {
  using C = Pw2p64<P, H>;
  constexpr int NT = C::NT, NW = C::NW, AC = C::AC, HH = C::HH, P2 = C::P2, MT = C::MT, NT1 = C::NT1,
                TPW = C::TPW, TSZ = C::TSZ, HSQ = H * H, SLAB = 8 * HSQ, NCHUNK = H / AC;
  constexpr int R3 = AC * 4 * H, MT3 = R3 / 8, KS = (H + 3) / 4, NT3 = (P + 7) / 8;
  static_assert(H % 4 == 0 && R3 % 8 == 0, "slab chunking");
  extern __shared__ __align__(16) double sm[];
  double* sG = sm;                   // [P][HH]
  double* Tc = sG + P * HH;          // [2][AC][8][H][H]
  double* U = Tc + 2 * TSZ;          // [AC][4][H][P]
  double* V = U + AC * 4 * H * P;    // [4][2][P2]
  const int b = boxes[blockIdx.x], tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2,
            q = lane & 3;
  const double* tb = Tin + (size_t)t.exp_rank[b] * H * SLAB;
  auto load = [&](int k) {
    const double* src = tb + (size_t)k * TSZ;
    double* dst = Tc + (k & 1) * TSZ;
    for (int i = tid; i < TSZ / 2; i += NT) cp_async16(dst + 2 * i, src + 2 * i);
    cp_async_commit();
  };
  load(0);
  for (int i = tid; i < P * HH; i += NT) sG[i] = Gr[i];
  double acc[TPW][2][MT][2];
#pragma unroll
  for (int s = 0; s < TPW; ++s)
#pragma unroll
    for (int par = 0; par < 2; ++par)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) acc[s][par][mt][0] = acc[s][par][mt][1] = 0.0;
#pragma unroll 1
  for (int k = 0; k < NCHUNK; ++k) {
    if (k + 1 < NCHUNK) {
      load(k + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    // ---- axis 3: U[r = (ac pi12 b)][n3] = sum_c Gr[n3][c] T[ac][2 pi12 + n3 % 2][b][c];
    // a warp takes one row tile and both column tiles of a parity (two DMMA chains)
    const double* Tk = Tc + (k & 1) * TSZ;
    static_assert(MT == 2, "two column tiles per parity");
    for (int u = warp; u < 2 * MT3; u += NW) {
      const int par = u / MT3, mt = u - par * MT3;
      const int r = mt * 8 + g, ac = r / (4 * H), pi12 = (r / H) & 3, bb = r % H;
      const double* arow = Tk + ((ac * 8 + 2 * pi12 + par) * H + bb) * H;
      const int n3a = 2 * g + par, n3b = 2 * (8 + g) + par;
      const double* brow0 = sG + n3a * HH;
      const double* brow1 = sG + (n3b < P ? n3b : 0) * HH;
      double av[KS], b0[KS], b1[KS];
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const int kk = ks * 4 + q;
        av[ks] = kk < H ? arow[kk] : 0.0;
        b0[ks] = kk < H ? brow0[kk] : 0.0;
        b1[ks] = (n3b < P && kk < H) ? brow1[kk] : 0.0;
      }
      double c0 = 0.0, c1 = 0.0, d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        dmma(c0, c1, av[ks], b0[ks]);
        dmma(d0, d1, av[ks], b1[ks]);
      }
      double* urow = U + r * P;
      const int na = 4 * q + par, nb = 2 * (8 + 2 * q) + par;
      urow[na] = c0;          // 4q + par + 2 < 16 <= P
      urow[na + 2] = c1;
      if (nb < P) urow[nb] = d0;
      if (nb + 2 < P) urow[nb + 2] = d1;
    }
    __syncthreads();
    // ---- axis 2: V[slot ac][pi1][n2][n3] = sum_b Gr[n2][b] U[ac][2 pi1 + n2 % 2][b][n3];
    // a warp takes one column tile of a group and both row tiles (two DMMA chains)
    for (int u = warp; u < AC * 4 * NT3; u += NW) {
      const int grp = u / NT3, nt = u - grp * NT3;
      const int ac = grp >> 2, pi1 = (grp >> 1) & 1, par2 = grp & 1;
      const int n2a = 2 * g + par2, n2b = 2 * (8 + g) + par2, n3 = nt * 8 + g;
      const double* arow0 = sG + n2a * HH;
      const double* arow1 = sG + (n2b < P ? n2b : 0) * HH;
      const double* ucol = U + ((ac * 4 + 2 * pi1 + par2) * H) * P + (n3 < P ? n3 : 0);
      double a0v[KS], a1v[KS], bv[KS];
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const int kk = ks * 4 + q;
        a0v[ks] = kk < H ? arow0[kk] : 0.0;
        a1v[ks] = (n2b < P && kk < H) ? arow1[kk] : 0.0;
        bv[ks] = (n3 < P && kk < H) ? ucol[kk * P] : 0.0;
      }
      double c0 = 0.0, c1 = 0.0, d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        dmma(c0, c1, a0v[ks], bv[ks]);
        dmma(d0, d1, a1v[ks], bv[ks]);
      }
      const int c3 = nt * 8 + 2 * q;
      double* vb = V + ((size_t)(((k & 1) * AC + ac) * 2 + pi1)) * P2;
      double* vr0 = vb + n2a * P;
      if (c3 < P) vr0[c3] = c0;
      if (c3 + 1 < P) vr0[c3 + 1] = c1;
      if (n2b < P) {
        double* vr1 = vb + n2b * P;
        if (c3 < P) vr1[c3] = d0;
        if (c3 + 1 < P) vr1[c3 + 1] = d1;
      }
    }
    if (k & 1) {
      __syncthreads();
      // ---- axis 1 over the 4 slabs a0 .. a0 + 3 in V: one k-step per (parity, tile)
      const int a0 = (k >> 1) * 4;
      double af[2][MT];
#pragma unroll
      for (int par = 0; par < 2; ++par)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const int n1 = 2 * (mt * 8 + g) + par;
          af[par][mt] = n1 < P ? sG[n1 * HH + a0 + q] : 0.0;
        }
#pragma unroll
      for (int s = 0; s < TPW; ++s) {
        const int nt = warp + s * NW;
        if (nt < NT1) {
          const int n = nt * 8 + g;
#pragma unroll
          for (int par = 0; par < 2; ++par) {
            const double bv = n < P2 ? V[(q * 2 + par) * P2 + n] : 0.0;
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) dmma(acc[s][par][mt][0], acc[s][par][mt][1], af[par][mt], bv);
          }
        }
      }
    }
  }
  double* dst = lam + (size_t)t.exp_rank[b] * P * P2;
#pragma unroll
  for (int s = 0; s < TPW; ++s) {
    const int nt = warp + s * NW;
    if (nt >= NT1) continue;
    const int n = nt * 8 + 2 * q;
#pragma unroll
    for (int par = 0; par < 2; ++par)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int n1 = 2 * (mt * 8 + g) + par;
        if (n1 >= P) continue;
        if (n < P2) dst[(size_t)n1 * P2 + n] = acc[s][par][mt][0];
        if (n + 1 < P2) dst[(size_t)n1 * P2 + n + 1] = acc[s][par][mt][1];
      }
  }
}

// fp32 tier: T_pw2poly (Eqs. 3.43-3.44) of every non-root local box from the weighted
// incoming expansion T[a][pi][b][c] written by k_pwshift, as three axis contractions
// over the whole box (no slab chunking, two barriers): axis 3 rows (a, pi12, b) from
// global memory into U[a][pi12][b][n3], axis 2 columns into V[a][pi1][n2][n3], axis 1
// into Lambda[n1][n2][n3] (fp64, global).  The output index n of each axis picks the
// input parity n mod 2, so output pairs (2k, 2k+1) take (Gr[2k][.], Gr[2k+1][.]) times
// (parity-0, parity-1) inputs: one packed FFMA2 per input index.
template <int P, int H>
struct Pw2p {
  static constexpr int NT = 256, PH = (P + 1) / 2, PE = 2 * PH, HH = (H + 1) & ~1;
  static constexpr int NU = H * 4 * H * PE, NV = H * 2 * PE * P;
  static constexpr size_t smem = sizeof(float2) * (size_t)H * PH + sizeof(float) * (size_t)(NU + NV);
};
template <int P, int H>
__global__ void __launch_bounds__(Pw2p<P, H>::NT, 2)
    k_pw2poly32(DevTree t, const int32_t* __restrict__ boxes, const double* __restrict__ Gr,
                const float* __restrict__ Tin, double* __restrict__ lam) {
  using C = Pw2p<P, H>;
  constexpr int NT = C::NT, PH = C::PH, PE = C::PE, HH = C::HH, HSQ = H * H, SLAB = 8 * HSQ, P2 = P * P;
  extern __shared__ float2 smp[];
  float2* GP = smp;                                        // [c][k] = (Gr[2k][c], Gr[2k+1][c])
  float* U = reinterpret_cast<float*>(GP + H * PH);        // [a][pi12][b][PE]
  float* V = U + C::NU;                                    // [a][pi1][PE][P]
  const int b = boxes[blockIdx.x], tid = threadIdx.x;
  for (int i = tid; i < H * PH; i += NT) {
    const int c = i / PH, k = i - c * PH;
    GP[i] = make_float2((float)Gr[(2 * k) * HH + c], 2 * k + 1 < P ? (float)Gr[(2 * k + 1) * HH + c] : 0.0f);
  }
  __syncthreads();
  const float* tb = Tin + (size_t)t.exp_rank[b] * H * SLAB;
  // axis 3: U[a][g][bb][n3] = sum_c Gr[n3][c] T[a][2 g + n3%2][bb][c]
  for (int u = tid; u < H * 4 * H; u += NT) {
    const int a = u / (4 * H), g = (u / H) % 4, bb = u % H;
    const float* r0 = tb + (size_t)a * SLAB + (2 * g) * HSQ + bb * H;
    float2 tv[H];
#pragma unroll
    for (int c = 0; c < H; ++c) tv[c] = make_float2(__ldg(r0 + c), __ldg(r0 + HSQ + c));
    float2* dst = reinterpret_cast<float2*>(U + (size_t)u * PE);
#pragma unroll 1
    for (int k = 0; k < PH; ++k) {
      float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int c = 0; c < H; ++c) acc = __ffma2_rn(GP[c * PH + k], tv[c], acc);
      dst[k] = acc;
    }
  }
  __syncthreads();
  // axis 2: V[a][p1][n2][n3] = sum_bb Gr[n2][bb] U[a][2 p1 + n2%2][bb][n3]
  for (int u = tid; u < H * 2 * P; u += NT) {
    const int a = u / (2 * P), p1 = (u / P) % 2, n3 = u % P;
    const float* c0 = U + ((size_t)(a * 4 + 2 * p1) * H) * PE + n3;
    float2 uv[H];
#pragma unroll
    for (int bb = 0; bb < H; ++bb) uv[bb] = make_float2(c0[bb * PE], c0[(H + bb) * PE]);
    float* dst = V + ((size_t)(a * 2 + p1) * PE) * P + n3;
#pragma unroll 1
    for (int k = 0; k < PH; ++k) {
      float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int bb = 0; bb < H; ++bb) acc = __ffma2_rn(GP[bb * PH + k], uv[bb], acc);
      dst[(2 * k) * P] = acc.x;
      dst[(2 * k + 1) * P] = acc.y;
    }
  }
  __syncthreads();
  // axis 1: Lambda[n1][n2][n3] = sum_a Gr[n1][a] V[a][n1%2][n2][n3]
  double* out = lam + (size_t)t.exp_rank[b] * P * P2;
  for (int u = tid; u < P2; u += NT) {
    float2 vv[H];
#pragma unroll
    for (int a = 0; a < H; ++a) vv[a] = make_float2(V[(size_t)(a * 2) * PE * P + u], V[(size_t)(a * 2 + 1) * PE * P + u]);
#pragma unroll 1
    for (int k = 0; k < PH; ++k) {
      float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int a = 0; a < H; ++a) acc = __ffma2_rn(GP[a * PH + k], vv[a], acc);
      out[(size_t)(2 * k) * P2 + u] = (double)acc.x;
      if (2 * k + 1 < P) out[(size_t)(2 * k + 1) * P2 + u] = (double)acc.y;
    }
  }
}

// Incoming expansion + conversion to Chebyshev coefficients of one local-expansion box
// (Eq. 3.39 fused with Eqs. 3.43-3.44): per chunk of AC slabs a, the 27-colleague
// translation (separable rotations: three nested 3-point sums), the weights, then the
// axis-3 and axis-2 back transforms in shared memory.  The axis-1 contraction over a
// either runs at the end as one DMMA GEMM over all slabs kept in shared memory
// (VSMEM, p <= 18), or as rank-AC updates of register accumulators (p = 28, whose
// slabs do not fit).  ROOT: the root box with the window weights (its only colleague
// is itself, delta = 0).
template <int P, int H, int AC>
struct PwLocal {
  using G = PwGeom<P, H>;
  static constexpr bool VSMEM = P <= 18;
  static constexpr int NT = ((VSMEM || P * P <= AC * H * H ? AC * H * H : P * P) + 31) / 32 * 32;
  static constexpr int KSA = (H + 3) / 4;   // axis-1 DMMA k steps (slabs, zero padded)
  static constexpr size_t smem =
      sizeof(double) * ((size_t)P * G::HH + (size_t)AC * G::SLAB + (size_t)AC * 4 * H * P +
                        (VSMEM ? (size_t)H * 2 * G::P2 : (size_t)AC * 2 * G::P2));
  static constexpr int MINB = (VSMEM && NT <= 352) ? 2 : 1;
};
template <int P, int H, int AC, bool ROOT, bool FROMT = false, class TT = float>
__global__ void __launch_bounds__(PwLocal<P, H, AC>::NT, PwLocal<P, H, AC>::MINB)
    k_pwlocal(DevTree t, const int32_t* __restrict__ boxes, const double* __restrict__ Gr,
              const double* __restrict__ W, size_t wstride, const FStore<P>* __restrict__ F, size_t base,
              size_t stride, double* __restrict__ lam, const TT* __restrict__ Tin = nullptr) {
  using G = PwGeom<P, H>;
  using C = PwLocal<P, H, AC>;
  using TF = FStore<P>;
  constexpr bool VSMEM = C::VSMEM;
  constexpr int NT = C::NT, P2 = G::P2, HH = G::HH, HSQ = G::HSQ, SLAB = G::SLAB, KSA = C::KSA;
  constexpr int NACC = VSMEM ? 1 : P;
  extern __shared__ double sm[];
  double* sG = sm;                  // [P][HH]
  double* T = sG + P * HH;          // [AC][8][H][H]  translated + weighted slabs
  double* U = T + AC * SLAB;        // [AC][4][H][P]  axis 3 done
  double* V = U + AC * 4 * H * P;   // [a][2][P2]     axes 3, 2 done (VSMEM: all slabs)
  __shared__ const TF* src[27];   // by delta slot (d1+1)*9 + (d2+1)*3 + (d3+1)
  const int b = boxes[blockIdx.x], tid = threadIdx.x;
  if (!(t.flags[b] & F_IN)) return;   // (never: every local box has F_in, tree.cu)
  const int l = t.level[b];
  const double* Wl = W + (ROOT ? 0 : (size_t)l * wstride);
  for (int i = tid; i < P * HH; i += NT) sG[i] = Gr[i];
  if (!FROMT && tid < 27) {
    // colleague slot k = (dx+1)*9 + (dy+1)*3 + (dz+1) holds B + (dx,dy,dz); its
    // delta = c_B - c_S = -(dx,dy,dz) has slot 26 - k
    const TF* p = nullptr;
    if (ROOT) {
      if (tid == 13) p = F;
    } else {
      const int s = t.coll[27 * (int64_t)b + tid];
      if (s >= 0 && (t.flags[s] & F_OUT)) p = F + base + (size_t)(t.fout_rank[s] - 1) * stride;
    }
    src[26 - tid] = p;
  }
  __syncthreads();
  double acc[NACC];
#pragma unroll
  for (int n = 0; n < NACC; ++n) acc[n] = 0.0;
  for (int a0 = 0; a0 < H; a0 += AC) {
    const int nac = min(AC, H - a0);
    // ---- translation (Eq. 3.39) and weights
    for (int w = tid; w < nac * HSQ; w += NT) {
      const int ac = w / HSQ, bc = w % HSQ, a = a0 + ac;
      const size_t off = (size_t)a * SLAB + bc;
      double o[8];
      if (FROMT) {   // translated and weighted by k_pwshift
        const TT* tb = Tin + (size_t)t.exp_rank[b] * H * SLAB + off;
#pragma unroll
        for (int p = 0; p < 8; ++p) o[p] = (double)__ldg(tb + p * HSQ);
      } else if (ROOT) {
#pragma unroll
        for (int p = 0; p < 8; ++p) o[p] = (double)__ldg(src[13] + off + p * HSQ);
      } else {
        double Ca, Sa, Cb, Sb, Cc, Sc;
        rot_cs(a, Ca, Sa);
        rot_cs(bc / H, Cb, Sb);
        rot_cs(bc % H, Cc, Sc);
#pragma unroll
        for (int p = 0; p < 8; ++p) o[p] = 0.0;
#pragma unroll
        for (int d1 = 0; d1 < 3; ++d1) {
          double x[8];
#pragma unroll
          for (int p = 0; p < 8; ++p) x[p] = 0.0;
#pragma unroll
          for (int d2 = 0; d2 < 3; ++d2) {
            double y[8];
#pragma unroll
            for (int p = 0; p < 8; ++p) y[p] = 0.0;
#pragma unroll
            for (int d3 = 0; d3 < 3; ++d3) {
              const TF* s = src[d1 * 9 + d2 * 3 + d3];
              if (s == nullptr) continue;
              double g[8];
#pragma unroll
              for (int p = 0; p < 8; ++p) g[p] = (double)__ldg(s + off + p * HSQ);
              if (d3 == 0) rot_acc<1, -1>(y, g, Cc, Sc);
              else if (d3 == 1) rot_acc<1, 0>(y, g, Cc, Sc);
              else rot_acc<1, 1>(y, g, Cc, Sc);
            }
            if (d2 == 0) rot_acc<2, -1>(x, y, Cb, Sb);
            else if (d2 == 1) rot_acc<2, 0>(x, y, Cb, Sb);
            else rot_acc<2, 1>(x, y, Cb, Sb);
          }
          if (d1 == 0) rot_acc<4, -1>(o, x, Ca, Sa);
          else if (d1 == 1) rot_acc<4, 0>(o, x, Ca, Sa);
          else rot_acc<4, 1>(o, x, Ca, Sa);
        }
      }
      const double wt = FROMT ? 1.0 : __ldg(Wl + (size_t)a * HSQ + bc);
#pragma unroll
      for (int p = 0; p < 8; ++p) T[(ac * 8 + p) * HSQ + bc] = wt * o[p];
    }
    __syncthreads();
    // ---- axis 3: U[ac][pi12][b][n3] = sum_c Gr[n3][c] T[ac][pi12*2 + n3%2][b][c]
    for (int w = tid; w < nac * 4 * H * 2; w += NT) {
      const int par = w & 1, row = w >> 1;   // row = (ac*4 + pi12)*H + b
      const int bb = row % H, g = row / H;
      double z[HH];
#pragma unroll
      for (int c = 0; c < HH; ++c) z[c] = c < H ? T[((g * 2 + par) * H + bb) * H + c] : 0.0;
#pragma unroll
      for (int n = par; n < P; n += 2) {
        const double* gr = sG + n * HH;
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < HH; c += 2) {
          const double2 q = *(const double2*)(gr + c);
          s = fma(q.x, z[c], fma(q.y, z[c + 1], s));
        }
        U[row * P + n] = s;
      }
    }
    __syncthreads();
    // ---- axis 2: V[a][pi1][n2][n3] = sum_b Gr[n2][b] U[ac][pi1*2 + n2%2][b][n3]
    double* Va = VSMEM ? V + (size_t)a0 * 2 * P2 : V;
    for (int w = tid; w < nac * 2 * P * 2; w += NT) {
      const int par = w & 1, n3 = (w >> 1) % P, g = (w >> 1) / P;   // g = ac*2 + pi1
      double z[HH];
#pragma unroll
      for (int bb = 0; bb < HH; ++bb) z[bb] = bb < H ? U[((g * 2 + par) * H + bb) * P + n3] : 0.0;
#pragma unroll
      for (int n = par; n < P; n += 2) {
        const double* gr = sG + n * HH;
        double s = 0.0;
#pragma unroll
        for (int bb = 0; bb < HH; bb += 2) {
          const double2 q = *(const double2*)(gr + bb);
          s = fma(q.x, z[bb], fma(q.y, z[bb + 1], s));
        }
        Va[(g * P + n) * P + n3] = s;
      }
    }
    __syncthreads();
    if (!VSMEM && tid < P2) {
      // ---- axis 1 (registers): Lambda[n1][n2 n3] += sum_ac Gr[n1][a0+ac] V[ac][n1%2][n2 n3]
      for (int ac = 0; ac < nac; ++ac) {
        const double v0 = V[(ac * 2 + 0) * P2 + tid], v1 = V[(ac * 2 + 1) * P2 + tid];
#pragma unroll
        for (int n = 0; n < NACC; ++n) acc[n] = fma(sG[n * HH + a0 + ac], (n & 1) ? v1 : v0, acc[n]);
      }
    }
    // next chunk: T's last readers (axis 3) finished before the barrier above; U and V
    // are rewritten only after the next chunk's barriers
  }
  double* dst = lam + (size_t)t.exp_rank[b] * P * P2;
  if (VSMEM) {
    // ---- axis 1 (DMMA): Lambda[2i+pi1][n2n3] = sum_a Gr[2i+pi1][a] V[a][pi1][n2n3]
    constexpr int PH = (P + 1) / 2;
#pragma unroll 1
    for (int pi1 = 0; pi1 < 2; ++pi1)
      mma_tiles<KSA>(
          (PH + 7) / 8, (P2 + 7) / 8,
          [&](int m, int k) { return (2 * m + pi1 < P && k < H) ? sG[(2 * m + pi1) * HH + k] : 0.0; },
          [&](int k, int n) { return (n < P2 && k < H) ? V[(k * 2 + pi1) * P2 + n] : 0.0; },
          [&](int m, int n, double v0, double v1) {
            const int n1 = 2 * m + pi1;
            if (n1 < P) {
              if (n < P2) dst[(size_t)n1 * P2 + n] = v0;
              if (n + 1 < P2) dst[(size_t)n1 * P2 + n + 1] = v1;
            }
          });
  } else if (tid < P2) {
#pragma unroll
    for (int n = 0; n < NACC; ++n) dst[(size_t)n * P2 + tid] = acc[n];
  }
}

// ---------------------------------------------------------------- evaluation (p = 28)
// Far-field evaluation: u_j = sum_a (Tx_j[n1] Ty_j[n2]) G[j][a],  G = V Lambda^T,
// V[j][b] = Tz_j[b]  (a = n1 P + n2, b = n3).  One CTA per local-expansion box,
// Lambda in smem in DMMA-fragment order, each warp evaluates tiles of 8 targets.
template <int P>
struct EvalMma {
  static constexpr int P2 = P * P, KS = (P + 3) / 4, NT8 = (P2 + 7) / 8, NW = 8;
  static constexpr size_t smem = sizeof(double) * ((size_t)NT8 * KS * 32 + (size_t)NW * 8 * 3 * P);
};
template <int P>
__global__ void __launch_bounds__(256) k_eval_mma(DevTree t, const int32_t* __restrict__ boxes,
                                                  const double* __restrict__ lam,
                                                  double* __restrict__ ufar) {
  using E = EvalMma<P>;
  constexpr int P2 = E::P2, KS = E::KS, NT8 = E::NT8, NW = E::NW;
  extern __shared__ double sm[];
  double* lamF = sm;                        // [NT8][KS][32]
  double* Tv = lamF + NT8 * KS * 32;        // [NW][8 targets][3 dims][P]
  __shared__ int2 rg[8];
  __shared__ int nr_s, tot_s;
  const int b = boxes[blockIdx.x], tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < 32) box_ranges_w<true>(t, b, rg, nr_s, tot_s);
  const double* src = lam + (size_t)t.exp_rank[b] * P * P2;   // own + inherited (p2c) expansion
  for (int i = tid; i < NT8 * KS * 32; i += NW * 32) {
    int ln = i & 31, ks = (i >> 5) % KS, nt = (i >> 5) / KS;
    int a = nt * 8 + (ln >> 2), bb = ks * 4 + (ln & 3);
    lamF[i] = (a < P2 && bb < P) ? src[a * P + bb] : 0.0;
  }
  __syncthreads();
  const int nr = nr_s, tot = tot_s;
  if (tot == 0) return;
  double cen[3], ih;
  box_geom(t.code[b], t.level[b], cen, ih);
  double* T = Tv + warp * 8 * 3 * P;
  const int g = lane >> 2, q4 = lane & 3;
  for (int tt = warp * 8; tt < tot; tt += NW * 8) {
    const int nv = min(8, tot - tt);
    if (lane < 24) {
      const int j = lane / 3, d = lane % 3;
      double Tl[P];
      if (j < nv) {
        int pi = range_point(rg, nr, tt + j);
        double x = (d == 0 ? t.xs[pi] : d == 1 ? t.ys[pi] : t.zs[pi]);
        cheb_vec((x - cen[d]) * ih, Tl, P, 1.0);
      } else {
#pragma unroll
        for (int n = 0; n < P; ++n) Tl[n] = 0.0;
      }
#pragma unroll
      for (int n = 0; n < P; ++n) T[(j * 3 + d) * P + n] = Tl[n];
    }
    __syncwarp();
    double af[KS];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      int bb = ks * 4 + q4;
      af[ks] = bb < P ? T[(g * 3 + 2) * P + bb] : 0.0;
    }
    const double* Tx = T + (g * 3 + 0) * P;
    const double* Ty = T + (g * 3 + 1) * P;
    double part = 0.0;
#pragma unroll 1
    for (int nt = 0; nt < NT8; nt += 2) {
      double c0 = 0.0, c1 = 0.0, d0 = 0.0, d1 = 0.0;
      const bool two = nt + 1 < NT8;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        dmma(c0, c1, af[ks], lamF[(nt * KS + ks) * 32 + lane]);
        if (two) dmma(d0, d1, af[ks], lamF[((nt + 1) * KS + ks) * 32 + lane]);
      }
      int a = nt * 8 + 2 * q4;
      if (a < P2) part = fma(c0, Tx[a / P] * Ty[a % P], part);
      if (a + 1 < P2) part = fma(c1, Tx[(a + 1) / P] * Ty[(a + 1) % P], part);
      a += 8;
      if (two && a < P2) part = fma(d0, Tx[a / P] * Ty[a % P], part);
      if (two && a + 1 < P2) part = fma(d1, Tx[(a + 1) / P] * Ty[(a + 1) % P], part);
    }
    part += __shfl_xor_sync(0xffffffffu, part, 1);
    part += __shfl_xor_sync(0xffffffffu, part, 2);
    if (q4 == 0 && g < nv) ufar[range_point(rg, nr, tt + g)] = part;
    __syncwarp();
  }
}

// Anterpolation: mu[a][b] = sum_j (rho_j Tx_j[n1] Ty_j[n2]) Tz_j[b] as C = U^T V with
// the points as the DMMA k dimension; each warp keeps its m-tiles x all n-tiles of mu
// in registers.  One CTA per F_out box.
template <int P>
struct AntMma {
  static constexpr int P2 = P * P, MT = (P2 + 7) / 8, NTB = (P + 7) / 8, NW = (P >= 18) ? 16 : 8;
  static constexpr int MPW = (MT + NW - 1) / NW, CH = 128;
  static constexpr size_t smem = sizeof(double) * 3 * CH * P;
};
template <int P>
__global__ void __launch_bounds__(AntMma<P>::NW * 32)
    k_anterp_mma(DevTree t, const int32_t* __restrict__ boxes, const double* __restrict__ q,
                 double* __restrict__ mom) {
  using A_ = AntMma<P>;
  constexpr int P2 = A_::P2, MT = A_::MT, NTB = A_::NTB, NW = A_::NW, MPW = A_::MPW, CH = A_::CH;
  constexpr int NT = NW * 32;
  extern __shared__ double sm[];
  double* Tx = sm;             // [CH][P] (times rho)
  double* Ty = Tx + CH * P;    // [CH][P]
  double* Tz = Ty + CH * P;    // [CH][P]
  __shared__ int2 rg[8];
  __shared__ int nr_s, tot_s;
  const int b = boxes[blockIdx.x], tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < 32) box_ranges_w<false>(t, b, rg, nr_s, tot_s);
  __syncthreads();
  const int nr = nr_s, tot = tot_s;
  if (tot == 0) return;   // moments were zeroed by the caller
  double cen[3], ih;
  box_geom(t.code[b], t.level[b], cen, ih);
  const int g = lane >> 2, q4 = lane & 3;
  double acc[MPW][NTB][2];
#pragma unroll
  for (int i = 0; i < MPW; ++i)
#pragma unroll
    for (int nb = 0; nb < NTB; ++nb) acc[i][nb][0] = acc[i][nb][1] = 0.0;
  for (int c0 = 0; c0 < tot; c0 += CH) {
    const int nc = min(CH, tot - c0);
    for (int w = tid; w < CH * 3; w += NT) {
      int j = w / 3, d = w % 3;
      double Tl[P];
      if (j < nc) {
        int pi = range_point(rg, nr, c0 + j);
        double x = (d == 0 ? t.xs[pi] : d == 1 ? t.ys[pi] : t.zs[pi]);
        cheb_vec((x - cen[d]) * ih, Tl, P, d == 0 ? q[pi] : 1.0);
      } else {
#pragma unroll
        for (int n = 0; n < P; ++n) Tl[n] = 0.0;
      }
      double* dst = (d == 0 ? Tx : d == 1 ? Ty : Tz) + j * P;
#pragma unroll
      for (int n = 0; n < P; ++n) dst[n] = Tl[n];
    }
    __syncthreads();
    const int nks = (nc + 3) / 4;
    for (int ks = 0; ks < nks; ++ks) {
      const int j = ks * 4 + q4;
      double bf[NTB];
#pragma unroll
      for (int nb = 0; nb < NTB; ++nb) {
        int bb = nb * 8 + g;
        bf[nb] = bb < P ? Tz[j * P + bb] : 0.0;
      }
#pragma unroll
      for (int i = 0; i < MPW; ++i) {
        const int mt = warp + i * NW;
        if (mt < MT) {
          const int a = mt * 8 + g;
          const double af = a < P2 ? Tx[j * P + a / P] * Ty[j * P + a % P] : 0.0;
#pragma unroll
          for (int nb = 0; nb < NTB; ++nb) dmma(acc[i][nb][0], acc[i][nb][1], af, bf[nb]);
        }
      }
    }
    __syncthreads();
  }
  double* out = mom + (size_t)t.fout_rank[b] * P * P2;
#pragma unroll
  for (int i = 0; i < MPW; ++i) {
    const int mt = warp + i * NW;
    const int a = mt * 8 + g;
    if (mt >= MT || a >= P2) continue;
#pragma unroll
    for (int nb = 0; nb < NTB; ++nb) {
      const int bb = nb * 8 + 2 * q4;
      if (bb < P) out[a * P + bb] = acc[i][nb][0];
      if (bb + 1 < P) out[a * P + bb + 1] = acc[i][nb][1];
    }
  }
}

// ---------------------------------------------------------------- P2P
struct ResPoly {
  double a[25];   // monomial coefficients in s = 2 r^2/r_L^2 - 1
};
constexpr int KER_LAPLACE = 0, KER_YUKAWA = 1;

// FULL: root is a leaf -> the kernel itself (no far field).  Otherwise the residual of
// the SOURCE level L, R_L(r) = K(r) - m_L(r/r_L)/r_L for r < r_L
// with K = 1/r (Eq. 3.66) or exp(-lam r)/r (Eq. 4.18), and the r = 0 (self / coincident)
// term is -m_L(0)/r_L = -M_L(0) (Step 5 folded in).  1/r uses one polynomial for all
// levels (rp, by value); Yukawa reads the level's coefficients from lvpoly.
// one warp (work item) per CTA: items differ in length, and single-warp CTAs keep the
// SMs evenly loaded (measured 1.24 -> 1.16 ms for k_p2p32 at config 1 against 4 warps)
constexpr int P2P32_NW = 1;
template <int K, int KER, bool FULL>
__global__ void __launch_bounds__(P2P32_NW * 32) k_p2p(DevTree t, const int32_t* __restrict__ items, int64_t nitems,
                                             const int32_t* __restrict__ doff, const int32_t* __restrict__ dlist,
                                             const double* __restrict__ q, const double* __restrict__ ufar,
                                             const int32_t* __restrict__ perm, double inv_side, ResPoly rp,
                                             const double* __restrict__ lvpoly, double lam,
                                             double* __restrict__ unear, double* __restrict__ out) {
  __shared__ double4 ssrc[P2P32_NW][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t it = (int64_t)blockIdx.x * P2P32_NW + warp;
  if (it >= nitems) return;
  const int B = items[2 * it], t0 = items[2 * it + 1];
  const int nt = min(32, t.end[B] - t0);
  const int ti = t0 + min(lane, nt - 1);
  const double xt = t.xs[ti], yt = t.ys[ti], zt = t.zs[ti];
  double acc = 0.0;
  for (int e = doff[B]; e < doff[B + 1]; ++e) {
    const int S = dlist[e];
    const int L = t.level[S];
    const double irl = ldexp(1.0, L), two_irl2 = ldexp(2.0, 2 * L), rl2 = ldexp(1.0, -2 * L);
    double a[K + 1];
#pragma unroll
    for (int j = 0; j <= K; ++j) a[j] = (KER == KER_YUKAWA) ? __ldg(lvpoly + L * (K + 1) + j) : rp.a[j];
    for (int s0 = t.start[S]; s0 < t.end[S]; s0 += 32) {
      const int ns = min(32, t.end[S] - s0);
      if (lane < ns) {
        int j = s0 + lane;
        ssrc[warp][lane] = make_double4(t.xs[j], t.ys[j], t.zs[j], q[j]);
      }
      __syncwarp();
      for (int k = 0; k < ns; ++k) {
        const double4 sp = ssrc[warp][k];
        const double dx = xt - sp.x, dy = yt - sp.y, dz = zt - sp.z;
        const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
        if (FULL) {
          if (r2 > 0.0) {
            const double rinv = rsqrt(r2);
            acc += (KER == KER_YUKAWA) ? sp.w * exp(-lam * r2 * rinv) * rinv : sp.w * rinv;
          }
        } else if (r2 < rl2) {
          const double s = fma(r2, two_irl2, -1.0);
          double pv = a[K];
#pragma unroll
          for (int j = K - 1; j >= 0; --j) pv = fma(pv, s, a[j]);
          double kv = 0.0;
          if (r2 > 0.0) {
            const double rinv = rsqrt(r2);
            kv = (KER == KER_YUKAWA) ? exp(-lam * r2 * rinv) * rinv : rinv;
          }
          acc = fma(sp.w, fma(-pv, irl, kv), acc);
        }
      }
      __syncwarp();
    }
  }
  if (lane < nt) unear[t0 + lane] = acc;
}

// fp32 tier (reading R16, p <= 18, eps >= 1e-6).  The same sum as k_p2p, every pair
// evaluated in single precision on leaf-local double-single coordinates: a source
// record holds x - c_S split as hi + lo (k_leaf_local4), the target's record is shifted
// once per list entry by c_T - c_S (exact in fp32: dyadic centres, level <= 20) with an
// error-free TwoSum, and a pair difference is (x_hi - y_hi) + (x_lo - y_lo), so |dx|
// carries a relative error of ~2^-23 whatever its size against r_L (plain fp32
// coordinates would carry 2^-25 r_L absolute: 4x the eps = 1e-6 error budget on
// surface distributions).  The terms of one list entry are summed in fp32 and added to
// an fp64 accumulator.  R_L(r) = K(r) - m_L(s)/r_L as in k_p2p (Horner in fp32: the
// monomial coefficients of m are O(1), |s| <= 1).
__device__ __forceinline__ float rsqrt_approx(float x) {   // MUFU.RSQ, flush-to-zero
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void sts_f32(uint32_t addr, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void two_sum(float a, float b, float& s, float& e) {
  s = __fadd_rn(a, b);
  const float bb = __fsub_rn(s, a);
  e = __fadd_rn(__fsub_rn(a, __fsub_rn(s, bb)), __fsub_rn(b, bb));
}
// Two sources per lane and instruction: the pair arithmetic runs on packed fp32x2
// (FFMA2/FADD2/FMUL2, sm_100), which halves the issue slots of the distance test and of
// the Horner polynomial (the kernel is issue-bound).  A source tile is staged as pairs
// (2k, 2k+1) in structure-of-pairs form with negated coordinates (x_t + (-y) rounds
// exactly like x_t - y); an odd tail is padded with a far-away, chargeless source.
template <int K, int KER>
__global__ void __launch_bounds__(P2P32_NW * 32) k_p2p32(DevTree t, const int32_t* __restrict__ items, int64_t nitems,
                                               const int32_t* __restrict__ doff, const int32_t* __restrict__ dlist,
                                               const float4* __restrict__ boxc, const float4* __restrict__ src,
                                               const float4* __restrict__ srclo, ResPoly rp,
                                               const double* __restrict__ lvpoly, float lam,
                                               double* __restrict__ unear) {
  __shared__ float4 sA[P2P32_NW][16], sB[P2P32_NW][16], sC[P2P32_NW][16];   // (-x, -y) hi, (-z hi, rho), (-x, -y) lo
  __shared__ float2 sD[P2P32_NW][16];                         // -z lo
  __shared__ double red[P2P32_NW][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t it = (int64_t)blockIdx.x * P2P32_NW + warp;
  if (it >= nitems) return;
  const int B = items[2 * it], t0 = items[2 * it + 1];
  const int nt = min(32, t.end[B] - t0);
  // an item of nt < 16 targets (the tail of a leaf) splits each source tile over
  // f = 32/nt lane groups: lane = target + nt * phase, phase strides the source pairs
  const int f = 32 / nt, tj = lane % nt, ph = lane / nt;
  const float4 tp = src[t0 + tj], tl = srclo[t0 + tj];
  const float4 cB = boxc[B];
  float2 a2[K + 1];
  if (KER == KER_LAPLACE) {
#pragma unroll
    for (int j = 0; j <= K; ++j) a2[j] = make_float2((float)rp.a[j], (float)rp.a[j]);
  }
  float* fA = reinterpret_cast<float*>(sA[warp]);
  float* fB = reinterpret_cast<float*>(sB[warp]);
  float* fC = reinterpret_cast<float*>(sC[warp]);
  float* fD = reinterpret_cast<float*>(sD[warp]);
  const float2 m1 = make_float2(-1.0f, -1.0f);
  double acc = 0.0;
  for (int e = doff[B]; e < doff[B + 1]; ++e) {
    const int S = dlist[e];
    const float4 cS = boxc[S];   // centre and side 2^-L (fp32, exact)
    // c_T - c_S, exact: both are dyadic with <= 22 significant bits
    float xt, yt, zt, xe, ye, ze;
    two_sum(tp.x, cB.x - cS.x, xt, xe);
    two_sum(tp.y, cB.y - cS.y, yt, ye);
    two_sum(tp.z, cB.z - cS.z, zt, ze);
    xe += tl.x;
    ye += tl.y;
    ze += tl.z;
    const float2 xt2 = make_float2(xt, xt), yt2 = make_float2(yt, yt), zt2 = make_float2(zt, zt);
    const float2 xe2 = make_float2(xe, xe), ye2 = make_float2(ye, ye), ze2 = make_float2(ze, ze);
    const float irl = __int_as_float(0x7F000000 - __float_as_int(cS.w));   // 2^L
    const float rl2 = cS.w * cS.w;
    const float2 tw2 = make_float2(2.0f * irl * irl, 2.0f * irl * irl), nirl2 = make_float2(-irl, -irl);
    if (KER == KER_YUKAWA) {
      const int L = t.level[S];
#pragma unroll
      for (int j = 0; j <= K; ++j) {
        const float c = (float)__ldg(lvpoly + L * (K + 1) + j);
        a2[j] = make_float2(c, c);
      }
    }
    float2 part = make_float2(0.0f, 0.0f);
    for (int s0 = t.start[S]; s0 < t.end[S]; s0 += 32) {
      const int ns = min(32, t.end[S] - s0), npair = (ns + 1) >> 1;
      const int j = lane >> 1, h = lane & 1;
      if (lane < ns) {
        const float4 hi = src[s0 + lane], lo = srclo[s0 + lane];
        fA[4 * j + h] = -hi.x;
        fA[4 * j + 2 + h] = -hi.y;
        fB[4 * j + h] = -hi.z;
        fB[4 * j + 2 + h] = hi.w;
        fC[4 * j + h] = -lo.x;
        fC[4 * j + 2 + h] = -lo.y;
        fD[2 * j + h] = -lo.z;
      } else if (lane == ns && h == 1) {
        // odd tail: a chargeless source at (4, 4, 4) r_L, outside the ball of every
        // target (|x_t| <= 2.5 r_L per axis) yet close enough that the polynomial of
        // its packed partner lane stays finite (s < 260)
        const float pad = -4.0f * cS.w;
        fA[4 * j + 1] = pad;
        fA[4 * j + 3] = pad;
        fB[4 * j + 1] = pad;
        fB[4 * j + 3] = 0.0f;
        fC[4 * j + 1] = 0.0f;
        fC[4 * j + 3] = 0.0f;
        fD[2 * j + 1] = 0.0f;
      }
      __syncwarp();
#pragma unroll 4
      for (int jp = ph; jp < npair; jp += f) {
        const float4 A = sA[warp][jp], Bv = sB[warp][jp], C = sC[warp][jp];
        const float2 Dv = sD[warp][jp];
        const float2 dx = __fadd2_rn(__fadd2_rn(xt2, make_float2(A.x, A.y)), __fadd2_rn(xe2, make_float2(C.x, C.y)));
        const float2 dy = __fadd2_rn(__fadd2_rn(yt2, make_float2(A.z, A.w)), __fadd2_rn(ye2, make_float2(C.z, C.w)));
        const float2 dz = __fadd2_rn(__fadd2_rn(zt2, make_float2(Bv.x, Bv.y)), __fadd2_rn(ze2, Dv));
        const float2 r2 = __ffma2_rn(dx, dx, __ffma2_rn(dy, dy, __fmul2_rn(dz, dz)));
        const bool i0 = r2.x < rl2, i1 = r2.y < rl2;
        if (i0 || i1) {
          const float2 s2 = __ffma2_rn(r2, tw2, m1);
          float2 pv = a2[K];
#pragma unroll
          for (int q = K - 1; q >= 0; --q) pv = __ffma2_rn(pv, s2, a2[q]);
          // r^2 below FLT_MIN (|x_t - x_s| < 1e-19 r_L) counts as coincident
          const float ri0 = rsqrt_approx(r2.x), ri1 = rsqrt_approx(r2.y);
          float k0 = (KER == KER_YUKAWA) ? expf(-lam * r2.x * ri0) * ri0 : ri0;
          float k1 = (KER == KER_YUKAWA) ? expf(-lam * r2.y * ri1) * ri1 : ri1;
          const float2 kv = make_float2(r2.x >= 1.17549435e-38f ? k0 : 0.0f, r2.y >= 1.17549435e-38f ? k1 : 0.0f);
          const float2 w = make_float2(i0 ? Bv.z : 0.0f, i1 ? Bv.w : 0.0f);
          part = __ffma2_rn(w, __ffma2_rn(pv, nirl2, kv), part);
        }
      }
      __syncwarp();
    }
    acc += (double)part.x + (double)part.y;
  }
  red[warp][lane] = ph < f ? acc : 0.0;
  __syncwarp();
  if (lane < nt) {
    double u = 0.0;
    for (int k = 0; k < f; ++k) u += red[warp][lane + k * nt];
    unear[t0 + lane] = u;
  }
}

// ---- fp32 tier, queue form (the default).  k_p2p32 is issue-bound on divergence: the
// residual polynomial runs whenever ANY lane of the warp holds an in-ball pair, which is
// almost every iteration although only ~16% of the list pairs of a uniform tree lie
// inside r_L (ball 4 pi/3 out of 27 boxes).  Here the pass over
// the list (phase A) only measures the pairs -- coordinates in units of the source leaf's
// r_L (an exact power-of-two scaling) -- and appends each in-ball pair to a lane-private
// queue in shared memory as two floats: u = r^2 / r_L^2 and w = rho_j / r_L.  When a
// lane's queue is nearly full, and at the end of the item, the warp drains the queues
// (phase B): with s = 2u - 1,
//   R_L(r) rho_j = (rho_j / r_L) (u^{-1/2} - m_L(s))               (Laplace, Eq. 3.66)
//   R_L(r) rho_j = (rho_j / r_L) (e^{-lam r} u^{-1/2} - m_L(s))    (Yukawa, Eq. 4.18)
// two queue entries per packed FFMA2, every lane busy except for the tail of the
// longest queue.  u = 0 (coincident pair, self term) gives -w m_L(-1) = -M_L(0) rho_j
// (Step 5).  Yukawa's polynomial and kernel depend on the source
// level: its queue holds one level at a time (drained when the level changes).
// Phase A measures with the high parts of the double-single coordinates only (error
// <= ~2^-24 * 2.5 r_L per coordinate, i.e. <= ~1.5e-7 r_L / r relative on r): a pair
// closer than sqrt(tc) r_L -- rare, a warp-uniform branch over CHK iterations --
// is re-measured with the full double-single difference (hi + lo) like k_p2p32.
// The list's entries are read 32 at a time into registers (lane k holds entry k's
// range and box) and broadcast by shuffles; the source tile k+1 is loaded into
// registers while tile k is measured.
template <int K, int KER, int QC>
struct P2PQ {
  // resident one-warp CTAs per SM that the shared memory allows (queue + staging + the
  // 1 KB per-CTA reservation); the register allocation is held to the same count
  static constexpr int MINB = (228 * 1024) / (256 * QC + 1400 + 1024);
  static constexpr int CHK = 4;   // pair iterations between queue-capacity votes
  static_assert(QC >= 4 * CHK + 2, "queue too small");   // drained at QC - 2 CHK
};
struct ResPoly32 {
  float a[25];   // the residual polynomial's coefficients in fp32 (kernel parameter space)
};
// u = r^2 / r_L^2 (queued), w = rho_j / r_L; s = 2u - 1; coefficients c[q] (Laplace: the
// kernel parameter, constant bank; Yukawa: the queued level's, registers)
template <int K, int KER, class CF>
__device__ __forceinline__ float2 p2pq_term(float2 u, float2 w, const CF& c, float lam_rl, bool v0, bool v1) {
  const float2 s = __ffma2_rn(u, make_float2(2.0f, 2.0f), make_float2(-1.0f, -1.0f));
  float2 pv = make_float2(c[K], c[K]);
#pragma unroll
  for (int q = K - 1; q >= 0; --q) pv = __ffma2_rn(pv, s, make_float2(c[q], c[q]));
  // r_L / r; u below FLT_MIN (|x_t - x_s| < 1e-19 r_L) counts as coincident
  float k0 = rsqrt_approx(u.x), k1 = rsqrt_approx(u.y);
  if (KER == KER_YUKAWA) {   // e^{-lam r}, r = r_L sqrt(u) = r_L u (r_L/r)
    k0 *= __expf(-lam_rl * u.x * k0);
    k1 *= __expf(-lam_rl * u.y * k1);
  }
  const float2 kv = make_float2(u.x >= 1.17549435e-38f ? k0 : 0.0f, u.y >= 1.17549435e-38f ? k1 : 0.0f);
  const float2 r = __fmul2_rn(w, __fadd2_rn(kv, make_float2(-pv.x, -pv.y)));
  return make_float2(v0 ? r.x : 0.0f, v1 ? r.y : 0.0f);
}
template <int K, int KER, int QC>
__global__ void __launch_bounds__(32, P2PQ<K, KER, QC>::MINB) k_p2p32q(DevTree t, const int32_t* __restrict__ items, int64_t nitems,
                                               const int32_t* __restrict__ doff, const int32_t* __restrict__ dlist,
                                               const float4* __restrict__ boxc, const float4* __restrict__ src,
                                               const float4* __restrict__ srclo, ResPoly32 rp,
                                               const double* __restrict__ lvpoly, float lam, float tc,
                                               double* __restrict__ unear, const int32_t* __restrict__ dbeg) {
  constexpr int CHK = P2PQ<K, KER, QC>::CHK;
  // staged tile as 16 source pairs + slot 16, a permanent pad; slots past the tile's pairs
  // are pads too (a chargeless source at (4, 4, 4) r_L, outside every target's ball)
  __shared__ float4 sA[17], sB[17], sC[17];   // (-x, -y) hi, (-z hi, rho/r_L), (-x, -y) lo
  __shared__ float2 sD[17];                   // -z lo
  __shared__ float qT[2 * QC * 32];           // lane-private queues: t at [slot][lane], w QC slots later
  __shared__ double red[32];
  const int lane = threadIdx.x;
  const int64_t it = blockIdx.x;
  if (it >= nitems) return;
  const int B = items[2 * it], t0 = items[2 * it + 1];
  const int nt = min(32, t.end[B] - t0);
  // an item of nt < 16 targets (the tail of a leaf) splits each source tile over
  // f = 32/nt lane groups: lane = target + nt * phase, phase strides the source pairs
  const int f = 32 / nt, tj = lane % nt, ph = lane / nt;
  const bool act = ph < f;
  const float4 tp = src[t0 + tj], tl = srclo[t0 + tj];
  const float4 cB = boxc[B];
  float cy[KER == KER_YUKAWA ? K + 1 : 1];   // Yukawa: the queued level's coefficients
  float* fA = reinterpret_cast<float*>(sA);
  float* fB = reinterpret_cast<float*>(sB);
  float* fC = reinterpret_cast<float*>(sC);
  float* fD = reinterpret_cast<float*>(sD);
  if (lane == 0) {
    sA[16] = make_float4(-1e30f, -1e30f, -1e30f, -1e30f);
    sB[16] = make_float4(-1e30f, -1e30f, 0.0f, 0.0f);
    sC[16] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    sD[16] = make_float2(0.0f, 0.0f);
  }
  // next free slot of this lane's queue as a shared-memory byte address (t; w at +128 QC)
  const uint32_t qa0 = (uint32_t)__cvta_generic_to_shared(qT + lane);
  uint32_t qa = qa0;
  const uint32_t qlim = qa0 + 128 * (QC - 2 * CHK);
  int qlev = -1;
  float qlam = 0.0f;   // Yukawa: lam * r_L of the queued level
  double acc = 0.0;
  auto drain = [&]() {
    const int cnt = (int)(qa - qa0) >> 7;
    const int mx = __reduce_max_sync(0xffffffffu, cnt);
    float2 ap = make_float2(0.0f, 0.0f);
    for (int i = 0; i < mx; i += 2) {
      const float2 tt = make_float2(qT[32 * i + lane], qT[32 * (i + 1) + lane]);
      const float2 ww = make_float2(qT[32 * (QC + i) + lane], qT[32 * (QC + i + 1) + lane]);
      if constexpr (KER == KER_YUKAWA)
        ap = __fadd2_rn(ap, p2pq_term<K, KER>(tt, ww, cy, qlam, i < cnt, i + 1 < cnt));
      else
        ap = __fadd2_rn(ap, p2pq_term<K, KER>(tt, ww, rp.a, qlam, i < cnt, i + 1 < cnt));
    }
    acc += (double)ap.x + (double)ap.y;
    qa = qa0;
  };
  // ---- the list in batches of 32 entries: lane k holds entry e0 + k (dbeg: the
  // list's suffix from dbeg[B], the mixed-level entries beside the symmetric form)
  const int e_beg = dbeg ? dbeg[B] : doff[B], e_end = doff[B + 1];
  int eb = e_beg;   // first entry of the batch in registers
  int m_start = 0, m_end = 0, m_lev = 0;
  float4 m_c = cB;
  auto load_batch = [&](int e0) {
    eb = e0;
    if (e0 + lane < e_end) {
      const int S = dlist[e0 + lane];
      m_start = t.start[S];
      m_end = t.end[S];
      m_c = boxc[S];
      if (KER == KER_YUKAWA) m_lev = t.level[S];
    }
  };
  load_batch(e_beg);
  int e = e_beg;
  int s0 = __shfl_sync(0xffffffffu, m_start, 0), sE = __shfl_sync(0xffffffffu, m_end, 0);
  float4 rh = make_float4(0.0f, 0.0f, 0.0f, 0.0f), rl = rh;
  if (s0 + lane < sE) {
    rh = src[s0 + lane];
    rl = srclo[s0 + lane];
  }
  while (true) {
    const int k = e - eb;
    const float4 cS = make_float4(__shfl_sync(0xffffffffu, m_c.x, k), __shfl_sync(0xffffffffu, m_c.y, k),
                                  __shfl_sync(0xffffffffu, m_c.z, k), __shfl_sync(0xffffffffu, m_c.w, k));
    const int L = KER == KER_YUKAWA ? __shfl_sync(0xffffffffu, m_lev, k) : 0;
    const int ns = min(32, sE - s0), npair = (ns + 1) >> 1;
    const float irl = __int_as_float(0x7F000000 - __float_as_int(cS.w));   // 2^L
    // ---- stage the current tile (all lanes finished reading the previous one)
    __syncwarp();
    {
      const bool real = lane < ns;
      const int j = lane >> 1, h = lane & 1;
      const float pad = -4.0f * cS.w;
      const float nirl = -irl;   // coordinates in units of r_L, negated
      fA[4 * j + h] = real ? rh.x * nirl : pad;
      fA[4 * j + 2 + h] = real ? rh.y * nirl : pad;
      fB[4 * j + h] = real ? rh.z * nirl : pad;
      fB[4 * j + 2 + h] = real ? rh.w * irl : 0.0f;
      fC[4 * j + h] = real ? rl.x * nirl : 0.0f;
      fC[4 * j + 2 + h] = real ? rl.y * nirl : 0.0f;
      fD[2 * j + h] = real ? rl.z * nirl : 0.0f;
    }
    __syncwarp();
    // ---- advance the cursor and prefetch the next tile into registers
    int ns0 = s0 + 32, nsE = sE;
    bool more = true;
    if (ns0 >= sE) {
      ++e;
      if (e < e_end) {
        if (e - eb == 32) load_batch(e);
        ns0 = __shfl_sync(0xffffffffu, m_start, e - eb);
        nsE = __shfl_sync(0xffffffffu, m_end, e - eb);
      } else {
        more = false;
      }
    }
    if (more && ns0 + lane < nsE) {
      rh = src[ns0 + lane];
      rl = srclo[ns0 + lane];
    }
    // ---- level constants (Yukawa: the queue holds one level)
    if (KER == KER_YUKAWA) {
      if (L != qlev) {
        if (__any_sync(0xffffffffu, qa != qa0)) drain();
        qlev = L;
        qlam = lam * cS.w;
#pragma unroll
        for (int j = 0; j <= K; ++j) cy[KER == KER_YUKAWA ? j : 0] = (float)__ldg(lvpoly + L * (K + 1) + j);
      }
    }
    // ---- the target in the source leaf's frame (exact centre difference + TwoSum), in
    // units of r_L (exact power-of-two scaling, as the staged sources)
    float xt, yt, zt, xe, ye, ze;
    two_sum(tp.x, cB.x - cS.x, xt, xe);
    two_sum(tp.y, cB.y - cS.y, yt, ye);
    two_sum(tp.z, cB.z - cS.z, zt, ze);
    xe = (xe + tl.x) * irl;
    ye = (ye + tl.y) * irl;
    ze = (ze + tl.z) * irl;
    xt *= irl;
    yt *= irl;
    zt *= irl;
    // ---- phase A: measure, queue the in-ball pairs.  f == 1 (warp-uniform): every lane
    // walks the same pair slots, padded to a multiple of CHK (pads never enter the ball)
    const float lim = act ? 1.0f : -1.0f;   // in-ball test u < 1; idle lanes queue nothing
    auto phase_a = [&](auto uni_) {
      constexpr bool UNI = decltype(uni_)::value;
      const int kmax = UNI ? npair : (npair + f - 1) / f;   // warp-uniform trip count
      for (int k0 = 0; k0 < kmax; k0 += CHK) {
        if (__any_sync(0xffffffffu, qa > qlim)) drain();
        float2 tt[CHK], ww[CHK];
        int jj[CHK];
        bool close = false;
#pragma unroll
        for (int kk = 0; kk < CHK; ++kk) {
          const int jp = UNI ? k0 + kk : ph + (k0 + kk) * f;
          jj[kk] = UNI ? jp : (act && jp < npair ? jp : 16);
          const float4 A = sA[jj[kk]], Bv = sB[jj[kk]];
          const float2 dx = __fadd2_rn(make_float2(xt, xt), make_float2(A.x, A.y));
          const float2 dy = __fadd2_rn(make_float2(yt, yt), make_float2(A.z, A.w));
          const float2 dz = __fadd2_rn(make_float2(zt, zt), make_float2(Bv.x, Bv.y));
          tt[kk] = __ffma2_rn(dx, dx, __ffma2_rn(dy, dy, __fmul2_rn(dz, dz)));
          ww[kk] = make_float2(Bv.z, Bv.w);
          close |= fminf(tt[kk].x, tt[kk].y) < tc;
        }
        if (__any_sync(0xffffffffu, close)) {   // rare: close pairs need the low parts
#pragma unroll
          for (int kk = 0; kk < CHK; ++kk) {
            const float4 A = sA[jj[kk]], Bv = sB[jj[kk]], C = sC[jj[kk]];
            const float2 Dv = sD[jj[kk]];
            const float2 dx = __fadd2_rn(__fadd2_rn(make_float2(xt, xt), make_float2(A.x, A.y)),
                                         __fadd2_rn(make_float2(xe, xe), make_float2(C.x, C.y)));
            const float2 dy = __fadd2_rn(__fadd2_rn(make_float2(yt, yt), make_float2(A.z, A.w)),
                                         __fadd2_rn(make_float2(ye, ye), make_float2(C.z, C.w)));
            const float2 dz = __fadd2_rn(__fadd2_rn(make_float2(zt, zt), make_float2(Bv.x, Bv.y)),
                                         __fadd2_rn(make_float2(ze, ze), Dv));
            tt[kk] = __ffma2_rn(dx, dx, __ffma2_rn(dy, dy, __fmul2_rn(dz, dz)));
          }
        }
#pragma unroll
        for (int kk = 0; kk < CHK; ++kk) {
          if (tt[kk].x < lim) {
            sts_f32(qa, tt[kk].x);
            sts_f32(qa + 128 * QC, ww[kk].x);
            qa += 128;
          }
          if (tt[kk].y < lim) {
            sts_f32(qa, tt[kk].y);
            sts_f32(qa + 128 * QC, ww[kk].y);
            qa += 128;
          }
        }
      }
    };
    if (f == 1) phase_a(std::true_type{});
    else phase_a(std::false_type{});
    if (!more) break;
    s0 = ns0;
    sE = nsE;
  }
  drain();
  red[lane] = act ? acc : 0.0;
  __syncwarp();
  if (lane < nt) {
    double u = 0.0;
    for (int k = 0; k < f; ++k) u += red[lane + k * nt];
    unear[t0 + lane] = u;
  }
}

// ---- fp32 tier, symmetric form (the default).  R_L depends only on the source leaf's
// level, so for two leaves B, S of the SAME level the pair (x, y)
// contributes R_L(|x - y|) rho_y to u(x) and R_L(|x - y|) rho_x to u(y): one evaluation
// serves both.  The same-level entries of a leaf's direct list are its colleague leaves
// (the list's prefix, tree.cu); a warp takes one entry (B, S) with S > B (S < B: S's
// warp does it) and evaluates every pair of B's and S's points once, densely -- the lanes
// hold up to 32 points of one leaf, the other leaf's points are broadcast from shared
// memory two at a time (packed fp32x2), the pairs outside the ball r < r_L weighted 0
// (~16% of the pairs are inside; culling first costs more on a SIMT
// machine, profiles/r02_p2p_nbr_experiments.md).  The lanes' side sums stay in registers;
// the broadcast side's per-point sums are collected in 32 registers per lane and
// reduced across the warp by a butterfly transpose (31 shuffles).  S == B (the leaf
// itself) runs one-sided, with the r = 0 pair giving the Step 5 self term
// -w m_L(-1).  Each (target, same-level entry) sum is an fp32
// partial in its own slot (part), summed per target in list order by k_p2p_psum (fp64),
// so the result does not depend on scheduling (bitwise deterministic).  Mixed-level
// entries (adaptive trees) stay with the queue form k_p2p32q on the list's suffix.
// Coordinates: the lane leaf's frame in units of r_L (exact scaling), the broadcast
// points shifted in with TwoSum (double-single); as in the queue form (reading R16) u
// comes from the high parts and a group of pairs where some pair is closer than
// sqrt(tc) r_L is re-evaluated on the full double-single difference.
constexpr int P2PS_NW = 4;
// compile-time experiments (both measured slower, profiles/r02_p2p_tail_ab.jsonl, off):
// records past a chunk's tail skip the kernel evaluation (warp-uniform); records with
// no pair inside any lane's ball skip it (one vote per record)
#ifndef DMK_P2PS_TAIL
#define DMK_P2PS_TAIL 0
#endif
#ifndef DMK_P2PS_RSKIP
#define DMK_P2PS_RSKIP 0
#endif
constexpr bool P2PS_TAIL = DMK_P2PS_TAIL, P2PS_RSKIP = DMK_P2PS_RSKIP;
constexpr int P2PS_PER_DEFAULT = 64;
// (blocks of consecutive tasks per warp visit instead of the round-robin deal measured
// slower: profiles/r02_p2ps_bl.jsonl, commit 'task-block assignment experiment')
// -DDMK_P2PS_MINB=5|6 caps the registers at 96|80 (spills; profiles/r02_p2ps_minb.jsonl)
#ifdef DMK_P2PS_MINB
#define DMK_P2PS_BOUNDS __launch_bounds__(P2PS_NW * 32, DMK_P2PS_MINB)
#else
#define DMK_P2PS_BOUNDS __launch_bounds__(P2PS_NW * 32)
#endif
template <int K, int KER>
__global__ void DMK_P2PS_BOUNDS k_p2p32s(const SymTask* __restrict__ tasks,
                                                        const int32_t* __restrict__ ntask_p,
                                                        const float4* __restrict__ src,
                                                        const float4* __restrict__ srclo, ResPoly32 rp,
                                                        const double* __restrict__ lvpoly, float lam, float tc,
                                                        float* __restrict__ part) {
  // per warp: 16 broadcast pair records (P0 = (x0, x1, y0, y1), P1 = (z0, z1, w0, w1)
  // high parts, P2 = (x0, x1, y0, y1), P3 = (z0, z1, -, -) low parts; negated)
  __shared__ float4 sbuf[P2PS_NW][4][16];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntask = *ntask_p;
  const int gw = blockIdx.x * P2PS_NW + warp, nwarps = gridDim.x * P2PS_NW;
  float4* P0 = sbuf[warp][0];
  float4* P1 = sbuf[warp][1];
  float4* P2 = sbuf[warp][2];
  float4* P3 = sbuf[warp][3];
  float* f0 = reinterpret_cast<float*>(P0);
  float* f1 = reinterpret_cast<float*>(P1);
  float* f2 = reinterpret_cast<float*>(P2);
  float* f3 = reinterpret_cast<float*>(P3);
  float cf[K + 1];
  int lev = -1;
  if constexpr (KER != KER_YUKAWA) {
#pragma unroll
    for (int q = 0; q <= K; ++q) cf[q] = rp.a[q];
  }
  // persistent: the next task's record is loaded while this one runs
  SymTask nx{};
  if (gw < ntask) nx = tasks[gw];
  for (int ti = gw; ti < ntask; ti += nwarps) {
    const SymTask tk = nx;
    if (ti + nwarps < ntask) nx = tasks[ti + nwarps];
    const bool self_task = tk.rng.w < 0;
    const int bB = tk.rng.x, nB = tk.rng.y, bS = tk.rng.z, nS = self_task ? nB : tk.rng.w;
    const float irl = tk.geo.w;
    if constexpr (KER == KER_YUKAWA) {   // the pair's level (both leaves): its residual polynomial
      const int L = (__float_as_int(irl) >> 23) - 127;
      if (L != lev) {
        lev = L;
#pragma unroll
        for (int q = 0; q <= K; ++q) cf[q] = (float)__ldg(lvpoly + L * (K + 1) + q);
      }
    }
    const float lamr = lam * __int_as_float(0x7F000000 - __float_as_int(irl));   // Yukawa: lambda r_L
    const int64_t slotB = tk.slot.x, slotS = tk.slot.y;
    const int ncB = (nB + 31) >> 5, ncS = (nS + 31) >> 5;
    // one chunk pair (B chunk cb, S chunk cs); SELF: the leaf with itself, one-sided
    auto chunk_pair = [&](auto self_, int cb, int cs, float& accS1) {
      constexpr bool self = decltype(self_)::value;
      {
        const int nb = min(32, nB - 32 * cb), ns = min(32, nS - 32 * cs);
        // lanes take the larger chunk (one-sided: always B's targets)
        const bool swap = !self && ns > nb;
        const int nxp = swap ? ns : nb, ny = swap ? nb : ns;
        const int gx = (swap ? bS + 32 * cs : bB + 32 * cb), gy = (swap ? bB + 32 * cb : bS + 32 * cs);
        // c_X - c_Y
        const float sgn = swap ? -1.0f : 1.0f;
        const float dcx = sgn * tk.geo.x, dcy = sgn * tk.geo.y, dcz = sgn * tk.geo.z;
        // the lane's point (target side), in units of r_L
        const bool lv = lane < nxp;
        const float4 th = src[gx + (lv ? lane : 0)], tl = srclo[gx + (lv ? lane : 0)];
        const float2 xt = make_float2(th.x * irl, th.x * irl), yt = make_float2(th.y * irl, th.y * irl),
                     zt = make_float2(th.z * irl, th.z * irl);
        const float2 xtl = make_float2(tl.x * irl, tl.x * irl), ytl = make_float2(tl.y * irl, tl.y * irl),
                     ztl = make_float2(tl.z * irl, tl.z * irl);
        const float wi = lv ? th.w * irl : 0.0f;
        // stage the broadcast chunk: -(y + c_Y - c_X) = (-y) + (c_X - c_Y), TwoSum'd
        __syncwarp();
        {
          const int j = lane, h = j & 1, r = j >> 1;
          // pads: far away (u > 1e10, never 0) and chargeless
          float sx = 1e5f, sy = 1e5f, sz = 1e5f, lx = 0.0f, ly = 0.0f, lz = 0.0f, w = 0.0f;
          if (j < ny) {
            const float4 hi = src[gy + j], lo = srclo[gy + j];
            float ex, ey, ez;
            two_sum(-hi.x, dcx, sx, ex);
            two_sum(-hi.y, dcy, sy, ey);
            two_sum(-hi.z, dcz, sz, ez);
            sx *= irl;
            sy *= irl;
            sz *= irl;
            lx = (ex - lo.x) * irl;
            ly = (ey - lo.y) * irl;
            lz = (ez - lo.z) * irl;
            w = hi.w * irl;
          }
          f0[4 * r + h] = sx;
          f0[4 * r + 2 + h] = sy;
          f1[4 * r + h] = sz;
          f1[4 * r + 2 + h] = w;
          f2[4 * r + h] = lx;
          f2[4 * r + 2 + h] = ly;
          f3[4 * r + h] = lz;
          f3[4 * r + 2 + h] = 0.0f;
        }
        __syncwarp();
        const int npy = (ny + 1) >> 1;
        float2 accX = make_float2(0.0f, 0.0f);
        // the broadcast points' terms; columns of pads and of records past the chunk are
        // never read back (a column's butterfly sum lands in its own lane only)
        float v[32];
#pragma unroll
        for (int g = 0; g < 4; ++g) {   // groups of 4 pair records (8 points)
          if (4 * g >= npy) break;
          float2 u[4];
          float4 Q[4];
          bool close = false;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int r = 4 * g + k;
            const float4 A = P0[r];
            Q[k] = P1[r];
            const float2 dx = __fadd2_rn(xt, make_float2(A.x, A.y));
            const float2 dy = __fadd2_rn(yt, make_float2(A.z, A.w));
            const float2 dz = __fadd2_rn(zt, make_float2(Q[k].x, Q[k].y));
            u[k] = __ffma2_rn(dx, dx, __ffma2_rn(dy, dy, __fmul2_rn(dz, dz)));
            close |= fminf(u[k].x, u[k].y) < tc;
          }
          {   // no pair of the group inside any lane's ball (corner colleagues, mostly): next
            const float um = fminf(fminf(fminf(u[0].x, u[0].y), fminf(u[1].x, u[1].y)),
                                   fminf(fminf(u[2].x, u[2].y), fminf(u[3].x, u[3].y)));
            if (!__any_sync(0xffffffffu, lv && um < 1.0f)) {
              if (!self) {
#pragma unroll
                for (int c = 0; c < 8; ++c) v[8 * g + c] = 0.0f;
              }
              continue;
            }
          }
          if (__any_sync(0xffffffffu, close)) {   // rare (always on the self chunk's diagonal)
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int r = 4 * g + k;
              const float4 A = P0[r], L = P2[r], Z = P3[r];
              const float2 dx = __fadd2_rn(__fadd2_rn(xt, make_float2(A.x, A.y)), __fadd2_rn(xtl, make_float2(L.x, L.y)));
              const float2 dy = __fadd2_rn(__fadd2_rn(yt, make_float2(A.z, A.w)), __fadd2_rn(ytl, make_float2(L.z, L.w)));
              const float2 dz = __fadd2_rn(__fadd2_rn(zt, make_float2(Q[k].x, Q[k].y)), __fadd2_rn(ztl, make_float2(Z.x, Z.y)));
              u[k] = __ffma2_rn(dx, dx, __ffma2_rn(dy, dy, __fmul2_rn(dz, dz)));
            }
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int r = 4 * g + k;
            if (P2PS_TAIL && r >= npy) {   // records past the chunk's tail (warp-uniform): no pairs
              if (!self) v[2 * r] = v[2 * r + 1] = 0.0f;
              continue;
            }
            if (P2PS_RSKIP && !__any_sync(0xffffffffu, lv && fminf(u[k].x, u[k].y) < 1.0f)) {
              if (!self) v[2 * r] = v[2 * r + 1] = 0.0f;
              continue;
            }
            // R_L outside the ball is 0 (the mask folded into R); the lane's side gets
            // w_y R, the broadcast side w_x R (pads and idle lanes have w = 0; an idle
            // lane's own sum is not written)
            const bool in0 = u[k].x < 1.0f, in1 = u[k].y < 1.0f;
            const float2 uu = (K > 12) ? make_float2(fminf(u[k].x, 1.0f), fminf(u[k].y, 1.0f)) : u[k];
            const float2 s2 = __ffma2_rn(uu, make_float2(2.0f, 2.0f), make_float2(-1.0f, -1.0f));
            float2 pv = make_float2(cf[K], cf[K]);
#pragma unroll
            for (int q = K - 1; q >= 0; --q) pv = __ffma2_rn(pv, s2, make_float2(cf[q], cf[q]));
            float k0v = rsqrt_approx(uu.x), k1v = rsqrt_approx(uu.y);
            if constexpr (KER == KER_YUKAWA) {
              k0v *= __expf(-lamr * uu.x * k0v);
              k1v *= __expf(-lamr * uu.y * k1v);
            }
            float2 kv = make_float2(k0v, k1v);
            // the leaf with itself: u below FLT_MIN (|x - y| < 1e-19 r_L, the r = 0 self
            // pair) counts as coincident (two different leaves have no coincident pair)
            if (self) kv = make_float2(uu.x >= 1.17549435e-38f ? k0v : 0.0f, uu.y >= 1.17549435e-38f ? k1v : 0.0f);
            float2 R = __fadd2_rn(kv, make_float2(-pv.x, -pv.y));
            R = make_float2(in0 ? R.x : 0.0f, in1 ? R.y : 0.0f);
            accX = __ffma2_rn(make_float2(Q[k].z, Q[k].w), R, accX);
            if (!self) {
              const float2 vb = __fmul2_rn(make_float2(wi, wi), R);
              v[2 * r] = vb.x;
              v[2 * r + 1] = vb.y;
            }
          }
        }
        const float ax = accX.x + accX.y;
        if (self) {
          accS1 += ax;
          return;
        }
        // the broadcast side's sums: butterfly transpose-reduce, lane j gets point j's
#pragma unroll
        for (int sft = 16; sft >= 1; sft >>= 1) {
          const bool up = lane & sft;
#pragma unroll
          for (int k = 0; k < sft; ++k) {
            const float send = up ? v[k] : v[k + sft];
            const float keep = up ? v[k + sft] : v[k];
            v[k] = keep + __shfl_xor_sync(0xffffffffu, send, sft);
          }
        }
        // slots: B-chunk cb's targets first written at cs = 0, S-chunk cs's at cb = 0
        // (later chunk pairs add, in this fixed order)
        const int64_t sx_ = swap ? slotS + 32 * cs : slotB + 32 * cb;
        const int64_t sy_ = swap ? slotB + 32 * cb : slotS + 32 * cs;
        const bool firstX = swap ? cb == 0 : cs == 0, firstY = swap ? cs == 0 : cb == 0;
        if (lane < nxp) part[sx_ + lane] = firstX ? ax : part[sx_ + lane] + ax;
        if (lane < ny) part[sy_ + lane] = firstY ? v[0] : part[sy_ + lane] + v[0];
      }
    };
    for (int cb = 0; cb < ncB; ++cb) {
      float accS1 = 0.0f;   // one-sided (self): the lane's sum over all of B's chunks
      if (self_task) {
        for (int cs = 0; cs < ncS; ++cs) chunk_pair(std::true_type{}, cb, cs, accS1);
        if (lane < min(32, nB - 32 * cb)) part[slotB + 32 * cb + lane] = accS1;
      } else {
        for (int cs = 0; cs < ncS; ++cs) chunk_pair(std::false_type{}, cb, cs, accS1);
      }
    }
  }
}

// near-field sums per target: the same-level entries' partials in list order (fp64),
// plus the queue form's mixed-level sum (already in unear) when there are mixed entries
__global__ void k_p2p_psum(DevTree t, const int32_t* __restrict__ items, int64_t nitems,
                           const int32_t* __restrict__ nsame, const int64_t* __restrict__ part_off,
                           const float* __restrict__ part, bool mixed, double* __restrict__ unear) {
  const int64_t it = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (it >= nitems) return;
  const int B = items[2 * it], t0 = items[2 * it + 1];
  const int b0 = t.start[B], nB = t.end[B] - b0, i = t0 - b0 + lane;
  if (i >= nB || lane >= 32) return;
  const int ns = nsame[B];
  const float* pp = part + part_off[B] + i;
  double u = 0.0;
  int e = 0;
  for (; e + 8 <= ns; e += 8) {   // 8 loads in flight, summed in list order
    float v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldg(pp + (int64_t)(e + k) * nB);
#pragma unroll
    for (int k = 0; k < 8; ++k) u += (double)v[k];
  }
  for (; e < ns; ++e) u += (double)__ldg(pp + (int64_t)e * nB);
  if (mixed) u += unear[b0 + i];
  unear[b0 + i] = u;
}

template <int K, int KER>
__global__ void __launch_bounds__(128) k_p2p32o(DevTree t, const int4* __restrict__ items, int64_t nitems,
                                                const int32_t* __restrict__ oct,
                                               const int32_t* __restrict__ doff, const int32_t* __restrict__ dlist,
                                               const float4* __restrict__ boxc, const float4* __restrict__ src,
                                               const float4* __restrict__ srclo, ResPoly rp,
                                               const double* __restrict__ lvpoly, float lam,
                                               double* __restrict__ unear) {
  __shared__ float4 sA[4][16], sB[4][16], sC[4][16];   // (-x, -y) hi, (-z hi, rho), (-x, -y) lo
  __shared__ float2 sD[4][16];                         // -z lo
  __shared__ double red[4][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t it = (int64_t)blockIdx.x * 4 + warp;
  if (it >= nitems) return;
  const int4 itm = items[it];
  const int B = itm.x, o = itm.y, t0 = itm.z;
  const int nt = itm.w - itm.z;
  // an item of nt < 16 targets (the tail of a leaf) splits each source tile over
  // f = 32/nt lane groups: lane = target + nt * phase, phase strides the source pairs
  const int f = 32 / nt, tj = lane % nt, ph = lane / nt;
  const float4 tp = src[t0 + tj], tl = srclo[t0 + tj];
  const float4 cB = boxc[B];
  // the target octant's box (Sec. 3.4: one more level of refinement for the culling)
  const float hT = 0.25f * cB.w;
  const float ox = cB.x + ((o >> 2) & 1 ? hT : -hT), oy = cB.y + ((o >> 1) & 1 ? hT : -hT),
              oz = cB.z + (o & 1 ? hT : -hT);
  __shared__ int sOa[4][8], sOx[4][8];   // selected source octants: first point, exclusive prefix
  float2 a2[K + 1];
  if (KER == KER_LAPLACE) {
#pragma unroll
    for (int j = 0; j <= K; ++j) a2[j] = make_float2((float)rp.a[j], (float)rp.a[j]);
  }
  float* fA = reinterpret_cast<float*>(sA[warp]);
  float* fB = reinterpret_cast<float*>(sB[warp]);
  float* fC = reinterpret_cast<float*>(sC[warp]);
  float* fD = reinterpret_cast<float*>(sD[warp]);
  const float2 m1 = make_float2(-1.0f, -1.0f);
  double acc = 0.0;
  for (int e = doff[B]; e < doff[B + 1]; ++e) {
    const int S = dlist[e];
    const float4 cS = boxc[S];   // centre and side 2^-L (fp32, exact)
    // c_T - c_S, exact: both are dyadic with <= 22 significant bits
    float xt, yt, zt, xe, ye, ze;
    two_sum(tp.x, cB.x - cS.x, xt, xe);
    two_sum(tp.y, cB.y - cS.y, yt, ye);
    two_sum(tp.z, cB.z - cS.z, zt, ze);
    xe += tl.x;
    ye += tl.y;
    ze += tl.z;
    const float2 xt2 = make_float2(xt, xt), yt2 = make_float2(yt, yt), zt2 = make_float2(zt, zt);
    const float2 xe2 = make_float2(xe, xe), ye2 = make_float2(ye, ye), ze2 = make_float2(ze, ze);
    const float irl = __int_as_float(0x7F000000 - __float_as_int(cS.w));   // 2^L
    const float rl2 = cS.w * cS.w;
    const float2 tw2 = make_float2(2.0f * irl * irl, 2.0f * irl * irl), nirl2 = make_float2(-irl, -irl);
    if (KER == KER_YUKAWA) {
      const int L = t.level[S];
#pragma unroll
      for (int j = 0; j <= K; ++j) {
        const float c = (float)__ldg(lvpoly + L * (K + 1) + j);
        a2[j] = make_float2(c, c);
      }
    }
    // source octants of S within r_L of the target octant (closed boxes: every pair of a
    // culled octant has r >= r_L, where R_L = 0): lanes 0-7 test one octant each
    bool sel = false;
    int oa = 0, oc = 0;
    if (lane < 8) {
      oa = oct[8 * (int64_t)S + lane];
      oc = (lane < 7 ? oct[8 * (int64_t)S + lane + 1] : t.end[S]) - oa;
      if (oc > 0) {
        const float hS = 0.25f * cS.w;
        const float gx = fmaxf(0.0f, fabsf(ox - (cS.x + ((lane >> 2) & 1 ? hS : -hS))) - hT - hS);
        const float gy = fmaxf(0.0f, fabsf(oy - (cS.y + ((lane >> 1) & 1 ? hS : -hS))) - hT - hS);
        const float gz = fmaxf(0.0f, fabsf(oz - (cS.z + (lane & 1 ? hS : -hS))) - hT - hS);
        sel = fmaf(gx, gx, fmaf(gy, gy, gz * gz)) < rl2 * 1.000001f;
      }
    }
    if (!__any_sync(0xffffffffu, sel)) continue;
    int c = sel ? oc : 0, incl = c;
#pragma unroll
    for (int d = 1; d < 8; d <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += v;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 7);
    if (lane < 8) {
      sOa[warp][lane] = oa;
      sOx[warp][lane] = sel ? incl - c : 0x7fffffff;   // unselected: never matched
    }
    __syncwarp();
    float2 part = make_float2(0.0f, 0.0f);
    for (int s0 = 0; s0 < total; s0 += 32) {
      const int ns = min(32, total - s0), npair = (ns + 1) >> 1;
      const int j = lane >> 1, h = lane & 1;
      if (lane < ns) {
        const int g = s0 + lane;
        int kk = 0, best = -1;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int x0 = sOx[warp][k];
          if (x0 <= g && x0 >= best) {
            best = x0;
            kk = k;
          }
        }
        const int si = sOa[warp][kk] + (g - best);
        const float4 hi = src[si], lo = srclo[si];
        fA[4 * j + h] = -hi.x;
        fA[4 * j + 2 + h] = -hi.y;
        fB[4 * j + h] = -hi.z;
        fB[4 * j + 2 + h] = hi.w;
        fC[4 * j + h] = -lo.x;
        fC[4 * j + 2 + h] = -lo.y;
        fD[2 * j + h] = -lo.z;
      } else if (lane == ns && h == 1) {
        // odd tail: a chargeless source at (4, 4, 4) r_L, outside the ball of every
        // target (|x_t| <= 2.5 r_L per axis) yet close enough that the polynomial of
        // its packed partner lane stays finite (s < 260)
        const float pad = -4.0f * cS.w;
        fA[4 * j + 1] = pad;
        fA[4 * j + 3] = pad;
        fB[4 * j + 1] = pad;
        fB[4 * j + 3] = 0.0f;
        fC[4 * j + 1] = 0.0f;
        fC[4 * j + 3] = 0.0f;
        fD[2 * j + 1] = 0.0f;
      }
      __syncwarp();
#pragma unroll 4
      for (int jp = ph; jp < npair; jp += f) {
        const float4 A = sA[warp][jp], Bv = sB[warp][jp], C = sC[warp][jp];
        const float2 Dv = sD[warp][jp];
        const float2 dx = __fadd2_rn(__fadd2_rn(xt2, make_float2(A.x, A.y)), __fadd2_rn(xe2, make_float2(C.x, C.y)));
        const float2 dy = __fadd2_rn(__fadd2_rn(yt2, make_float2(A.z, A.w)), __fadd2_rn(ye2, make_float2(C.z, C.w)));
        const float2 dz = __fadd2_rn(__fadd2_rn(zt2, make_float2(Bv.x, Bv.y)), __fadd2_rn(ze2, Dv));
        const float2 r2 = __ffma2_rn(dx, dx, __ffma2_rn(dy, dy, __fmul2_rn(dz, dz)));
        const bool i0 = r2.x < rl2, i1 = r2.y < rl2;
        if (i0 || i1) {
          const float2 s2 = __ffma2_rn(r2, tw2, m1);
          float2 pv = a2[K];
#pragma unroll
          for (int q = K - 1; q >= 0; --q) pv = __ffma2_rn(pv, s2, a2[q]);
          // r^2 below FLT_MIN (|x_t - x_s| < 1e-19 r_L) counts as coincident
          const float ri0 = rsqrt_approx(r2.x), ri1 = rsqrt_approx(r2.y);
          float k0 = (KER == KER_YUKAWA) ? expf(-lam * r2.x * ri0) * ri0 : ri0;
          float k1 = (KER == KER_YUKAWA) ? expf(-lam * r2.y * ri1) * ri1 : ri1;
          const float2 kv = make_float2(r2.x >= 1.17549435e-38f ? k0 : 0.0f, r2.y >= 1.17549435e-38f ? k1 : 0.0f);
          const float2 w = make_float2(i0 ? Bv.z : 0.0f, i1 ? Bv.w : 0.0f);
          part = __ffma2_rn(w, __ffma2_rn(pv, nirl2, kv), part);
        }
      }
      __syncwarp();
    }
    acc += (double)part.x + (double)part.y;
  }
  red[warp][lane] = ph < f ? acc : 0.0;
  __syncwarp();
  if (lane < nt) {
    double u = 0.0;
    for (int k = 0; k < f; ++k) u += red[warp][lane + k * nt];
    unear[t0 + lane] = u;
  }
}

// u = (u_far + u_near)/side, scattered to the caller's order (after both branches)
__global__ void k_combine(const double* __restrict__ ufar, const double* __restrict__ unear,
                          const int32_t* __restrict__ perm, int64_t n, double inv_side, double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[perm[i]] = (ufar[i] + unear[i]) * inv_side;
}

// ---------------------------------------------------------------- host launchers
void resolve_timings(dmk_plan_s* P) {
  if (P->ev_marks.empty()) return;
  // marks live on several streams (the near field on the side stream): wait for every
  // one, and commit the sums only when all of them resolved
  for (auto& m : P->ev_marks) DMK_CUDA(cudaEventSynchronize(m.e1));
  std::vector<std::pair<const char*, double>> acc(P->timings);
  for (auto& m : P->ev_marks) {
    float ms = 0;
    DMK_CUDA(cudaEventElapsedTime(&ms, m.e0, m.e1));
    bool found = false;
    for (auto& pr : acc)
      if (std::strcmp(pr.first, m.name) == 0) { pr.second += ms; found = true; }
    if (!found) acc.push_back({m.name, (double)ms});
  }
  P->timings.swap(acc);
  P->ev_marks.clear();
}

// prox2pw: columns c per chunk, all of them when the intermediates fit 200 KB, else
// balanced chunks.  pwlocal: 2 slabs per chunk unless the translation items of two
// slabs exceed 1024 threads.
constexpr int px_ch(int P, int H) {
  int best = 1;
  for (int ch = 1; ch <= H; ++ch) {
    size_t sm = sizeof(double) * ((size_t)2 * ((H + 7) / 8 * 8) * ((((P + 1) / 2) + 3) / 4 * 4) + (size_t)P * P * ch +
                                  (size_t)H * P * ch);
    if (sm <= 200 * 1024) best = ch;
  }
  const int nchunk = (H + best - 1) / best;
  return (H + nchunk - 1) / nchunk;
}
constexpr int pw_ac(int H) { return 2 * H * H <= 1024 ? 2 : 1; }

static bool anterp_tc() {   // validation in progress: opt-in (DMK_ANTERP=tc)
  const char* e = std::getenv("DMK_ANTERP");
  return e && std::strcmp(e, "tc") == 0;
}

static bool eval_tc() {   // default: tensor cores; DMK_EVAL=ffma selects k_eval32
  const char* e = std::getenv("DMK_EVAL");
  return !(e && std::strcmp(e, "ffma") == 0);
}

// eps = 1e-9 translation + back transforms, chosen at plan time (the T buffer is sized
// then): parent groups staged through shared memory (k_pwshift_s<H, double>) into an
// fp64 T, back transforms on DMMA (k_pw2poly64) -- the default, 1.97 + 1.53 ms at
// config 1 (profiles/r02_pw64_forms_v3.jsonl); DMK_PW64=box: the 27-colleague per-box
// form k_pwlocal (8.4 ms); DMK_PW64=group: register window sums k_pwshift64 + k_pwlocal
// from T (7.0 + 3.6 ms: 204 registers, 8 warps per SM, latency-bound)
constexpr int PW64_BOX = 0, PW64_GROUP = 1, PW64_STAGED = 2;
static int pw64_form() {
  const char* e = std::getenv("DMK_PW64");
  if (e && std::strcmp(e, "group") == 0) return PW64_GROUP;
  if (e && std::strcmp(e, "box") == 0) return PW64_BOX;
  return PW64_STAGED;
}
bool pw64_group_env() { return pw64_form() != PW64_BOX; }
#define pw64_group() (PL->pwt64.n > 0)
// fp32-tier translation: k_pwshift (register window sums) or k_pwshift_s (DMK_PWS=staged)
static bool pws_staged() {
  const char* e = std::getenv("DMK_PWS");
  return e && std::strcmp(e, "staged") == 0;
}
constexpr unsigned PWS_S_GY = 4;   // CTAs per parent (each walks every 4th mode chunk)

// Phases of run_eval: UP = anterpolation + c2p (Step 2), DOWN = Step 3; C2P_ONLY =
// c2p for the levels above `top` only (after dmk_level_moments injected level `top`).
constexpr int PH_ANTERP = 1, PH_DOWN = 2, PH_C2P_ONLY = 4, PH_C2P = 8, PH_UP = PH_ANTERP | PH_C2P;

// c2p into the level-l parents (k_c2p_grp: parent groups, MT parent rows per CTA)
template <int P>
constexpr int grp_mt() { return P <= 9 ? 9 : (P <= 18 ? 6 : 4); }
// p2c tiles: smaller for p = 18 (6 tiles per parent; measured 0.30 -> 0.28 ms at config 1)
template <int P>
constexpr int grp_mt_p2c() { return P <= 9 ? 9 : (P <= 18 ? 3 : 4); }
template <int P>
static void run_c2p_level(dmk_plan_s* PL, const DevTree& dt, int l) {
  cudaStream_t s = PL->stream;
  const auto& th = PL->th;
  const int64_t a = th.fout_off[l], b = th.fout_off[l + 1];
  const int64_t ca = th.fout_off[l + 1], cb = th.fout_off[l + 2];
  if (b <= a || cb <= ca) return;
  auto go = [&](auto mt_) {
    constexpr int MT = decltype(mt_)::value;
    using G = GrpCfg<P, MT>;
    set_smem(k_c2p_grp<P, MT>, G::smem_c2p);
    const unsigned grid = (unsigned)((b - a) * G::NTILE);
    k_c2p_grp<P, MT><<<grid, G::NT, G::smem_c2p, s>>>(dt, PL->fout_list.p + a, PL->tab->dA, PL->mom.p);
    DMK_LAUNCH_CHECK();
  };
  go(std::integral_constant<int, grp_mt<P>()>());
}

template <int P, int NF, int NF0>
static void run_eval(dmk_plan_s* PL, int phase = PH_UP | PH_DOWN, int top = 0) {
  cudaStream_t s = PL->stream;
  const Tables& T = *PL->tab;
  DevTree dt = dev_tree(PL);
  const auto& th = PL->th;
  const int nl = th.nlevels;
  constexpr int P3 = P * P * P;
  Timer tm(PL);
  const int64_t n = PL->n;
  if (nl > 1 && (phase & PH_C2P_ONLY)) {
    for (int l = top - 1; l >= 0; --l) run_c2p_level<P>(PL, dt, l);
    return;
  }
  if (nl > 1 && (phase & PH_ANTERP)) {
    // ---- Step 2: upward pass
    tm.begin("anterp");
    DMK_CUDA(cudaMemsetAsync(PL->mom.p, 0, PL->mom.bytes(), s));
    if (PL->nfout) {
      if constexpr (P <= 18) {   // fp32 tier (R16): tensor cores (tcgen05), or FFMA2 (DMK_ANTERP=ffma)
        if (anterp_tc()) {
          set_smem(k_anterp_tc<P>, AntTC<P>::smem);
          k_anterp_tc<P><<<(int)PL->nfout, AntTC<P>::NT, AntTC<P>::smem, s>>>(dt, PL->fout_list.p, PL->q.p,
                                                                              PL->mom.p);
        } else {
          set_smem(k_anterp32<P>, Ant32<P>::smem);
          k_anterp32<P><<<(int)PL->nfout, Ant32<P>::NT, Ant32<P>::smem, s>>>(dt, PL->fout_list.p, PL->q.p,
                                                                            PL->mom.p);
        }
      } else {
        size_t sm = AntMma<P>::smem;
        set_smem(k_anterp_mma<P>, sm);
        k_anterp_mma<P><<<(int)PL->nfout, AntMma<P>::NW * 32, sm, s>>>(dt, PL->fout_list.p, PL->q.p, PL->mom.p);
      }
      DMK_LAUNCH_CHECK();
    }
    tm.end();
  }
  if (nl > 1 && (phase & PH_C2P)) {
    tm.begin("c2p");
    for (int l = nl - 2; l >= 0; --l) run_c2p_level<P>(PL, dt, l);
    tm.end();
  }
  if (nl > 1 && (phase & PH_DOWN)) {
    // ---- Step 3: downward pass
    // the root box's chain (prox2pw, pwlocal: one CTA each, H0 > H) runs on its own
    // stream beside the other boxes' launches; joined before p2c
    cudaStream_t sr = PL->serial ? s : PL->root_stream;
    if (!PL->serial) {
      DMK_CUDA(cudaEventRecord(PL->ev_fork, s));
      DMK_CUDA(cudaStreamWaitEvent(sr, PL->ev_fork, 0));
    }
    tm.begin("prox2pw");
    {
      constexpr int H = NF + 1, H0 = NF0 + 1, AC = px_ch(P, H), AC0 = px_ch(P, H0);
      using K1 = Prox2pw<P, H, AC>;
      using K0 = Prox2pw<P, H0, AC0>;
      // DMK_PROX2PW=tiles: the independent-tile form (before the register-blocked sweeps)
      const char* pxe = std::getenv("DMK_PROX2PW");
      const bool px_rb = !(pxe && std::strcmp(pxe, "tiles") == 0);
      if constexpr (P > 18) {
        set_smem(k_prox2pw<P, H0, AC0, true>, K0::smem);
        set_smem(k_prox2pw<P, H, AC, true>, K1::smem);
        set_smem(k_prox2pw<P, H, AC, false>, K1::smem);
      }
      FStore<P>* Fp = reinterpret_cast<FStore<P>*>(PL->phi.p);
      if constexpr (P <= 18) {   // fp32 tier (R16)
        using X0 = Px32<P, H0>;
        using X1 = Px32<P, H>;
        set_smem(k_prox2pw32<P, H0>, X0::smem);
        set_smem(k_prox2pw32<P, H>, X1::smem);
        k_prox2pw32<P, H0><<<1, X0::NT, X0::smem, sr>>>(dt, PL->fout_list.p, T.dQr0, PL->mom.p, Fp, 0, 0);
        DMK_LAUNCH_CHECK();
        if (PL->nfout > 1) {
          k_prox2pw32<P, H><<<(int)(PL->nfout - 1), X1::NT, X1::smem, s>>>(dt, PL->fout_list.p + 1, T.dQr1, PL->mom.p,
                                                                          Fp, PL->phi_size0, PL->phi_size1);
          DMK_LAUNCH_CHECK();
        }
      } else {
        k_prox2pw<P, H0, AC0, true><<<1, K0::NT, K0::smem, sr>>>(dt, PL->fout_list.p, T.dQr0, PL->mom.p, Fp, 0, 0);
        DMK_LAUNCH_CHECK();
        if (PL->nfout > 1) {
          if (px_rb)
            k_prox2pw<P, H, AC, true><<<(int)(PL->nfout - 1), K1::NT, K1::smem, s>>>(
                dt, PL->fout_list.p + 1, T.dQr1, PL->mom.p, Fp, PL->phi_size0, PL->phi_size1);
          else
            k_prox2pw<P, H, AC, false><<<(int)(PL->nfout - 1), K1::NT, K1::smem, s>>>(
                dt, PL->fout_list.p + 1, T.dQr1, PL->mom.p, Fp, PL->phi_size0, PL->phi_size1);
          DMK_LAUNCH_CHECK();
        }
      }
    }
    tm.end();
    tm.begin("pwlocal");
    {
      constexpr int H = NF + 1, H0 = NF0 + 1, AC = pw_ac(H), AC0 = pw_ac(H0);
      using K1 = PwLocal<P, H, AC>;
      using K0 = PwLocal<P, H0, AC0>;
      set_smem(k_pwlocal<P, H0, AC0, true>, K0::smem);
      set_smem(k_pwlocal<P, H, AC, false>, K1::smem);
      // root: exp rank 0, F_out rank 0
      const FStore<P>* Fp = reinterpret_cast<const FStore<P>*>(PL->phi.p);
      k_pwlocal<P, H0, AC0, true><<<1, K0::NT, K0::smem, sr>>>(dt, PL->exp_list.p, T.dGr0, T.dW0, 0, Fp, 0, 0,
                                                               PL->lam.p);
      DMK_LAUNCH_CHECK();
      if (!PL->serial) DMK_CUDA(cudaEventRecord(PL->ev_root, sr));
      if (PL->nexp > 1) {
        if constexpr (P <= 18) {
          // parent-group translation (k_pwshift) into T, then the back transforms
          tm.end();
          tm.begin("pwshift");
          if (PL->nfout > 0) {
            if (pws_staged()) {
              using KS = PwsS<H, float>;
              set_smem(k_pwshift_s<H, float>, KS::smem);
              const dim3 grid((unsigned)PL->nfout, PWS_S_GY);
              k_pwshift_s<H, float><<<grid, KS::NT, KS::smem, s>>>(dt, PL->fout_list.p,
                                                                  reinterpret_cast<const float*>(Fp), PL->phi_size0,
                                                                  PL->phi_size1, T.dW, T.wstride, PL->pwt.p);
            } else {
              const unsigned grid = (unsigned)(PL->nfout * PWS_GY);
              k_pwshift<H><<<grid, PWS_NT, 0, s>>>(dt, PL->fout_list.p, reinterpret_cast<const float*>(Fp),
                                                    PL->phi_size0, PL->phi_size1, T.dW, T.wstride, PL->pwt.p);
            }
            DMK_LAUNCH_CHECK();
          }
          tm.end();
          tm.begin("pw2poly");
          using K2 = Pw2p<P, H>;
          set_smem(k_pw2poly32<P, H>, K2::smem);
          k_pw2poly32<P, H><<<(int)(PL->nexp - 1), K2::NT, K2::smem, s>>>(dt, PL->exp_list.p + 1, T.dGr1, PL->pwt.p,
                                                                         PL->lam.p);
        } else if (pw64_group()) {
          // eps = 1e-9: fp64 parent-group translation into T, then the back transforms
          tm.end();
          tm.begin("pwshift");
          const bool staged = pw64_form() == PW64_STAGED;
          if (PL->nfout > 0) {
            if (staged) {
              using KS = PwsS<H, double>;
              set_smem(k_pwshift_s<H, double>, KS::smem);
              const dim3 grid((unsigned)PL->nfout, PWS_S_GY);
              k_pwshift_s<H, double><<<grid, KS::NT, KS::smem, s>>>(dt, PL->fout_list.p,
                                                                   reinterpret_cast<const double*>(Fp), PL->phi_size0,
                                                                   PL->phi_size1, T.dW, T.wstride, PL->pwt64.p);
            } else {
              const dim3 grid((unsigned)PL->nfout, (unsigned)((H * H * H + PWS64_NT - 1) / PWS64_NT), 2);
              k_pwshift64<H><<<grid, PWS64_NT, 0, s>>>(dt, PL->fout_list.p, reinterpret_cast<const double*>(Fp),
                                                       PL->phi_size0, PL->phi_size1, T.dW, T.wstride, PL->pwt64.p);
            }
            DMK_LAUNCH_CHECK();
          }
          tm.end();
          tm.begin("pw2poly");
          if (staged) {
            using K2 = Pw2p64<P, H>;
            set_smem(k_pw2poly64<P, H>, K2::smem);
            k_pw2poly64<P, H><<<(int)(PL->nexp - 1), K2::NT, K2::smem, s>>>(dt, PL->exp_list.p + 1, T.dGr1,
                                                                             PL->pwt64.p, PL->lam.p);
          } else {
            set_smem(k_pwlocal<P, H, AC, false, true, double>, K1::smem);
            k_pwlocal<P, H, AC, false, true, double><<<(int)(PL->nexp - 1), K1::NT, K1::smem, s>>>(
                dt, PL->exp_list.p + 1, T.dGr1, T.dW, T.wstride, Fp, PL->phi_size0, PL->phi_size1, PL->lam.p,
                PL->pwt64.p);
          }
        } else {
          k_pwlocal<P, H, AC, false><<<(int)(PL->nexp - 1), K1::NT, K1::smem, s>>>(
              dt, PL->exp_list.p + 1, T.dGr1, T.dW, T.wstride, Fp, PL->phi_size0, PL->phi_size1, PL->lam.p);
        }
        DMK_LAUNCH_CHECK();
      }
    }
    tm.end();
    if (!PL->serial) DMK_CUDA(cudaStreamWaitEvent(s, PL->ev_root, 0));
    // inherited local expansions: k_p2c_grp adds each parent's full expansion, split to
    // its children (Lemma 2.3), into the children's own parts written by the back transforms
    tm.begin("p2c");
    {
      // parents at level l-1 push their local expansions into their level-l children
      auto go = [&](auto mt_, int64_t a, int64_t b) {
        constexpr int MT = decltype(mt_)::value;
        using G = GrpCfg<P, MT>;
        set_smem(k_p2c_grp<P, MT>, G::smem_p2c);
        const unsigned grid = (unsigned)((b - a) * G::NTILE);
        k_p2c_grp<P, MT><<<grid, G::NT, G::smem_p2c, s>>>(dt, PL->exp_list.p + a, T.dA, PL->lam.p);
        DMK_LAUNCH_CHECK();
      };
      for (int l = 1; l < nl; ++l) {
        const int64_t a = th.exp_off[l - 1], b = th.exp_off[l];
        if (b <= a || th.exp_off[l + 1] <= th.exp_off[l]) continue;
        go(std::integral_constant<int, grp_mt_p2c<P>()>(), a, b);
      }
    }
    tm.end();
    tm.begin("eval");
    {
      if (PL->nexp) {
        if constexpr (P <= 18) {   // fp32 tier (R16): tensor cores, or FFMA2 (DMK_EVAL=ffma)
          if (eval_tc()) {
            set_smem(k_eval_tc<P>, EvTC<P>::smem);
            k_eval_tc<P><<<(int)PL->nexp, EvTC<P>::NT, EvTC<P>::smem, s>>>(dt, PL->exp_list.p, PL->lam.p,
                                                                              PL->ufar.p);
          } else {
            set_smem(k_eval32<P>, Ev32<P>::smem);
            k_eval32<P><<<(int)PL->nexp, Ev32<P>::NT, Ev32<P>::smem, s>>>(dt, PL->exp_list.p, PL->lam.p,
                                                                            PL->ufar.p);
          }
        } else {
          size_t sm = EvalMma<P>::smem;
          set_smem(k_eval_mma<P>, sm);
          k_eval_mma<P><<<(int)PL->nexp, 256, sm, s>>>(dt, PL->exp_list.p, PL->lam.p, PL->ufar.p);
        }
        DMK_LAUNCH_CHECK();
      }
    }
    tm.end();
  } else if (nl == 1 && (phase & PH_DOWN)) {
    DMK_CUDA(cudaMemsetAsync(PL->ufar.p, 0, n * sizeof(double), s));
  }
}

// P2P dispatch on the kernel and the residual-polynomial degree
template <int KER, bool FULL>
static void run_p2p_deg(dmk_plan_s* PL, double* out, const ResPoly& rp, int K, cudaStream_t st) {
  DevTree dt = dev_tree(PL);
  int nb = (int)((PL->np2p + P2P32_NW - 1) / P2P32_NW);
  if (nb == 0) return;
  const Tables& T = *PL->tab;
#define DMK_P2P_CASE(KK)                                                                                          \
  case KK:                                                                                                        \
    k_p2p<KK, KER, FULL><<<nb, P2P32_NW * 32, 0, st>>>(dt, PL->p2p_items.p, PL->np2p, PL->dlist_off.p, PL->dlist.p,         \
                                                      PL->q.p, PL->ufar.p, PL->perm.p, 1.0 / PL->side, rp,        \
                                                      T.dRespoly, T.lam, PL->unear.p, out);                       \
    break;
  switch (K) {
    DMK_P2P_CASE(4) DMK_P2P_CASE(6) DMK_P2P_CASE(8) DMK_P2P_CASE(10) DMK_P2P_CASE(12) DMK_P2P_CASE(14)
    DMK_P2P_CASE(16) DMK_P2P_CASE(18) DMK_P2P_CASE(20) DMK_P2P_CASE(22) DMK_P2P_CASE(24)
    default: fail(DMK_ERR_UNSUPPORTED, "residual polynomial degree out of range");
  }
#undef DMK_P2P_CASE
  DMK_LAUNCH_CHECK();
}

template <int KER>
static void run_p2p32_deg(dmk_plan_s* PL, const ResPoly& rp, int K, cudaStream_t st) {
  DevTree dt = dev_tree(PL);
  int nb = (int)((PL->np2p + P2P32_NW - 1) / P2P32_NW);
  if (nb == 0) return;
  const Tables& T = *PL->tab;
#define DMK_P2P_CASE(KK)                                                                                   \
  case KK:                                                                                                 \
    k_p2p32<KK, KER><<<nb, P2P32_NW * 32, 0, st>>>(dt, PL->p2p_items.p, PL->np2p, PL->dlist_off.p, PL->dlist.p,      \
                                         PL->box_c4.p, PL->xl4.p, PL->xl4lo.p, rp, T.dRespoly, (float)T.lam, PL->unear.p);            \
    break;
  switch (K) {
    DMK_P2P_CASE(4) DMK_P2P_CASE(6) DMK_P2P_CASE(8) DMK_P2P_CASE(10) DMK_P2P_CASE(12) DMK_P2P_CASE(14)
    DMK_P2P_CASE(16) DMK_P2P_CASE(18) DMK_P2P_CASE(20) DMK_P2P_CASE(22) DMK_P2P_CASE(24)
    default: fail(DMK_ERR_UNSUPPORTED, "residual polynomial degree out of range");
  }
#undef DMK_P2P_CASE
  DMK_LAUNCH_CHECK();
}

// queue form (default): DMK_P2P_QC selects the queue capacity, DMK_P2P_TC the u = r^2/r_L^2
// below which a pair is re-measured with the double-single low parts (tuning)
static float p2p_tc() {
  const char* e = std::getenv("DMK_P2P_TC");
  return e ? (float)std::atof(e) : 0.0025f;   // r < 0.05 r_L
}
template <int KER, int QC>
static void run_p2p32q_deg(dmk_plan_s* PL, const ResPoly& rp64, int K, cudaStream_t st,
                           const int32_t* dbeg = nullptr) {
  DevTree dt = dev_tree(PL);
  ResPoly32 rp{};
  for (int k = 0; k < 25; ++k) rp.a[k] = (float)rp64.a[k];
  const int64_t nb = PL->np2p;
  if (nb == 0) return;
  const Tables& T = *PL->tab;
#define DMK_P2P_CASE(KK)                                                                                   \
  case KK:                                                                                                 \
    k_p2p32q<KK, KER, QC><<<(unsigned)nb, 32, 0, st>>>(dt, PL->p2p_items.p, PL->np2p, PL->dlist_off.p,      \
                                                      PL->dlist.p, PL->box_c4.p, PL->xl4.p, PL->xl4lo.p, rp, \
                                                      T.dRespoly, (float)T.lam, p2p_tc(), PL->unear.p, dbeg); \
    break;
  switch (K) {
    DMK_P2P_CASE(4) DMK_P2P_CASE(6) DMK_P2P_CASE(8) DMK_P2P_CASE(10) DMK_P2P_CASE(12) DMK_P2P_CASE(14)
    DMK_P2P_CASE(16) DMK_P2P_CASE(18) DMK_P2P_CASE(20) DMK_P2P_CASE(22) DMK_P2P_CASE(24)
    default: fail(DMK_ERR_UNSUPPORTED, "residual polynomial degree out of range");
  }
#undef DMK_P2P_CASE
  DMK_LAUNCH_CHECK();
}
template <int KER>
static void run_p2p32q(dmk_plan_s* PL, const ResPoly& rp, int K, cudaStream_t st, const int32_t* dbeg = nullptr) {
  const char* e = std::getenv("DMK_P2P_QC");
  const int qc = e ? std::atoi(e) : 32;
  if (qc == 48) run_p2p32q_deg<KER, 48>(PL, rp, K, st, dbeg);
  else if (qc == 24) run_p2p32q_deg<KER, 24>(PL, rp, K, st, dbeg);
  else run_p2p32q_deg<KER, 32>(PL, rp, K, st, dbeg);
}
// symmetric form (default): same-level pairs once (k_p2p32s, one warp per direct-list
// entry), the mixed-level suffixes by the queue form into unear, then the per-target
// sums of the partials (k_p2p_psum)
template <int KER>
static void run_p2p32s(dmk_plan_s* PL, const ResPoly& rp64, int K, cudaStream_t st) {
  DevTree dt = dev_tree(PL);
  ResPoly32 rp{};
  for (int k = 0; k < 25; ++k) rp.a[k] = (float)rp64.a[k];
  if (PL->np2p == 0) return;
  const Tables& T = *PL->tab;
  if (PL->nmixed > 0) run_p2p32q<KER>(PL, rp64, K, st, PL->dlist_mbeg.p);
  if (PL->sym_cap > 0) {
    // persistent: enough warps to fill the SMs (the task count stays on the device);
    // the SM count and occupancy are queried once per process and kernel
    static thread_local int nsm = 0;
    if (!nsm) {
      int dev = 0;
      DMK_CUDA(cudaGetDevice(&dev));
      DMK_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    }
    // resident CTAs per SM: all that fit by default; DMK_P2PS_PER = k caps them (leaves
    // registers for the far-field kernels of the other stream), 0 = one task per warp
    const char* pe = std::getenv("DMK_P2PS_PER");
    const int per_env = pe ? std::atoi(pe) : P2PS_PER_DEFAULT;
#define DMK_P2P_CASE(KK)                                                                                      \
  case KK: {                                                                                                  \
    static thread_local int per = 0;                                                                          \
    if (!per) DMK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_p2p32s<KK, KER>, P2PS_NW * 32, 0)); \
    k_p2p32s<KK, KER><<<(unsigned)std::min<int64_t>(per_env == 0 ? INT64_MAX : (int64_t)nsm * std::max(std::min(per, per_env), 1), \
                                                    (PL->sym_cap + P2PS_NW - 1) / P2PS_NW),                   \
                        P2PS_NW * 32, 0, st>>>(PL->sym_tasks.p, PL->sym_ntask.p, PL->xl4.p, PL->xl4lo.p, rp,   \
                                               T.dRespoly, (float)T.lam, p2p_tc(), PL->part.p);               \
    break;                                                                                                    \
  }
    switch (K) {
      DMK_P2P_CASE(4) DMK_P2P_CASE(6) DMK_P2P_CASE(8) DMK_P2P_CASE(10) DMK_P2P_CASE(12) DMK_P2P_CASE(14)
      DMK_P2P_CASE(16) DMK_P2P_CASE(18) DMK_P2P_CASE(20) DMK_P2P_CASE(22) DMK_P2P_CASE(24)
      default: fail(DMK_ERR_UNSUPPORTED, "residual polynomial degree out of range");
    }
#undef DMK_P2P_CASE
    DMK_LAUNCH_CHECK();
  }
  k_p2p_psum<<<(unsigned)((PL->np2p + 3) / 4), 128, 0, st>>>(dt, PL->p2p_items.p, PL->np2p, PL->dlist_same.p,
                                                            PL->part_off.p, PL->part.p, PL->nmixed > 0,
                                                            PL->unear.p);
  DMK_LAUNCH_CHECK();
}
// 0 symmetric (default), 1 leaf (k_p2p32), 2 octant (k_p2p32o), 3 queue (k_p2p32q)
static int p2p_form(const dmk_plan_s* PL) {
  const char* e = std::getenv("DMK_P2P_FORM");
  if (!e) return 0;
  if (std::strcmp(e, "leaf") == 0) return 1;
  if (std::strcmp(e, "octant") == 0 && PL->np2p_o > 0) return 2;
  if (std::strcmp(e, "queue") == 0) return 3;
  return 0;
}

// Sec. 3.4 form: octant items and per-octant source culling (58% of the pairs of a
// uniform tree).  Opt-in (DMK_P2P_FORM=octant): measured slower than k_p2p32 on both
// config 1 (3.36 vs 1.23 ms, ~30-point leaves) and config 2 (43 vs 26 ms, mean 52
// points per leaf): octants of ~4-8 targets leave a warp's lanes with one or two source
// pairs per list entry, so the per-entry culling and gather cost more than the pairs
// saved.  Kept as a tested alternative for much bigger leaves.
template <int KER>
static void run_p2p32o_deg(dmk_plan_s* PL, const ResPoly& rp, int K, cudaStream_t st) {
  DevTree dt = dev_tree(PL);
  int nb = (int)((PL->np2p_o + 3) / 4);
  if (nb == 0) return;
  const Tables& T = *PL->tab;
#define DMK_P2P_CASE(KK)                                                                                    \
  case KK:                                                                                                  \
    k_p2p32o<KK, KER><<<nb, 128, 0, st>>>(dt, PL->p2p_items_o.p, PL->np2p_o, PL->leaf_oct.p, PL->dlist_off.p, \
                                          PL->dlist.p, PL->box_c4.p, PL->xl4.p, PL->xl4lo.p, rp, T.dRespoly,  \
                                          (float)T.lam, PL->unear.p);                                       \
    break;
  switch (K) {
    DMK_P2P_CASE(4) DMK_P2P_CASE(6) DMK_P2P_CASE(8) DMK_P2P_CASE(10) DMK_P2P_CASE(12) DMK_P2P_CASE(14)
    DMK_P2P_CASE(16) DMK_P2P_CASE(18) DMK_P2P_CASE(20) DMK_P2P_CASE(22) DMK_P2P_CASE(24)
    default: fail(DMK_ERR_UNSUPPORTED, "residual polynomial degree out of range");
  }
#undef DMK_P2P_CASE
  DMK_LAUNCH_CHECK();
}

template <class F>
static void dispatch_p(dmk_plan_s* PL, F f) {
  switch (PL->tab->p) {
    case 9: f(std::integral_constant<int, 9>(), std::integral_constant<int, 6>(), std::integral_constant<int, 10>()); break;
    case 18: f(std::integral_constant<int, 18>(), std::integral_constant<int, 12>(), std::integral_constant<int, 19>()); break;
    case 28: f(std::integral_constant<int, 28>(), std::integral_constant<int, 19>(), std::integral_constant<int, 28>()); break;
    default: fail(DMK_ERR_UNSUPPORTED, "unsupported Chebyshev order");
  }
}

// Step 2 (charges -> moments), 3D: gather the charges into Morton order, anterpolate,
// c2p.  The moments stay in the plan for eval_downward().
// Stream structure of one evaluation (3D).  The near field (Steps 4-5, P2P) needs only
// the gathered charges; it runs on a LOW-priority side stream while the far field
// (Steps 2-3) runs on a HIGH-priority stream, so the far field's level-by-level
// launches keep their SMs and the P2P blocks fill whatever they leave idle.  Both
// branches fork from and join back into the caller's plan stream.
struct StreamSwap {   // run_eval launches on PL->stream: point it at a branch stream
  dmk_plan_s* P;
  cudaStream_t keep;
  StreamSwap(dmk_plan_s* p, cudaStream_t st) : P(p), keep(p->stream) { p->stream = st; }
  ~StreamSwap() { P->stream = keep; }
};
static void fork_to(dmk_plan_s* PL, cudaStream_t from, cudaStream_t to) {
  DMK_CUDA(cudaEventRecord(PL->ev_fork, from));
  DMK_CUDA(cudaStreamWaitEvent(to, PL->ev_fork, 0));
}

void eval_upward(dmk_plan_s* PL, const double* dcharges) {
  cudaStream_t s = PL->stream, slo = PL->side_stream, shi = PL->hi_stream;
  PL->timings.clear();
  PL->ev_marks.clear();
  PL->ev_used = 0;
  Timer tm(PL);
  // a near-field branch of an earlier call may still read q: join it first
  if (PL->p2p_pending) DMK_CUDA(cudaStreamWaitEvent(s, PL->ev_join, 0));
  tm.begin("gather");
  const bool p2p32 = PL->dim == 3 && PL->tab->p <= 18 && PL->th.nlevels > 1;   // reading R16
  k_gather_q<<<(int)((PL->n + 255) / 256), 256, 0, s>>>(dcharges, PL->perm.p, PL->n, PL->q.p,
                                                        p2p32 ? PL->xl4.p : nullptr);
  DMK_LAUNCH_CHECK();
  tm.end();
  if (PL->dim == 2) return;   // the 2D path runs as one piece (eval_plan_2d)
  if (PL->serial) slo = s;    // DMK_SERIAL=1: no overlap (per-stage timing / profiling)
  fork_to(PL, s, slo);
  ResPoly rp{};
  const auto& poly = PL->tab->respoly;
  int K = (int)poly.size() - 1;
  for (int k = 0; k <= K && k < 25; ++k) rp.a[k] = poly[k];
  tm.begin("p2p", slo);
  const bool full = PL->th.nlevels == 1;
  const int form = p2p32 ? p2p_form(PL) : -1;
  if (PL->tab->kernel == DMK_KERNEL_YUKAWA) {
    K = PL->tab->respoly_deg;
    if (form == 2) run_p2p32o_deg<KER_YUKAWA>(PL, rp, K, slo);
    else if (form == 1) run_p2p32_deg<KER_YUKAWA>(PL, rp, K, slo);
    else if (form == 3) run_p2p32q<KER_YUKAWA>(PL, rp, K, slo);
    else if (form == 0) run_p2p32s<KER_YUKAWA>(PL, rp, K, slo);
    else if (full) run_p2p_deg<KER_YUKAWA, true>(PL, nullptr, rp, K, slo);
    else run_p2p_deg<KER_YUKAWA, false>(PL, nullptr, rp, K, slo);
  } else {
    if (form == 2) run_p2p32o_deg<KER_LAPLACE>(PL, rp, K, slo);
    else if (form == 1) run_p2p32_deg<KER_LAPLACE>(PL, rp, K, slo);
    else if (form == 3) run_p2p32q<KER_LAPLACE>(PL, rp, K, slo);
    else if (form == 0) run_p2p32s<KER_LAPLACE>(PL, rp, K, slo);
    else if (full) run_p2p_deg<KER_LAPLACE, true>(PL, nullptr, rp, K, slo);
    else run_p2p_deg<KER_LAPLACE, false>(PL, nullptr, rp, K, slo);
  }
  tm.end(slo);
  DMK_CUDA(cudaEventRecord(PL->ev_join, slo));
  PL->p2p_pending = true;
  // far field, upward part, on the high-priority stream; joined back into s
  fork_to(PL, s, shi);
  {
    StreamSwap sw(PL, shi);
    dispatch_p(PL, [&](auto P_, auto NF_, auto NF0_) { run_eval<P_(), NF_(), NF0_()>(PL, PH_UP); });
  }
  fork_to(PL, shi, s);
}

// Step 3 on the high-priority stream, then the join with the near-field branch and the
// combine on the plan stream.
void eval_downward(dmk_plan_s* PL, double* dout) {
  if (PL->dim == 2) {
    eval_plan_2d(PL, dout);
    return;
  }
  cudaStream_t s = PL->stream, shi = PL->hi_stream;
  fork_to(PL, s, shi);
  {
    StreamSwap sw(PL, shi);
    dispatch_p(PL, [&](auto P_, auto NF_, auto NF0_) { run_eval<P_(), NF_(), NF0_()>(PL, PH_DOWN); });
  }
  fork_to(PL, shi, s);
  DMK_CUDA(cudaStreamWaitEvent(s, PL->ev_join, 0));
  PL->p2p_pending = false;
  k_combine<<<(int)((PL->n + 255) / 256), 256, 0, s>>>(PL->ufar.p, PL->unear.p, PL->perm.p, PL->n, 1.0 / PL->side,
                                                       dout);
  DMK_LAUNCH_CHECK();
}

void eval_plan(dmk_plan_s* PL, const double* dcharges, double* dout) {
  eval_upward(PL, dcharges);
  eval_downward(PL, dout);
}

// ---- level moments (distributed evaluation): dense [2^{3l}][p^3] by Morton code
__global__ void k_level_get(const uint64_t* __restrict__ code, const int32_t* __restrict__ fout_rank, int64_t b0,
                            int p3, const double* __restrict__ mom, double* __restrict__ dense) {
  const int64_t i = b0 + blockIdx.x;
  const int r = fout_rank[i];
  if (r < 0) return;
  const double* src = mom + (size_t)r * p3;
  double* dst = dense + (size_t)code[i] * p3;
  for (int k = threadIdx.x; k < p3; k += blockDim.x) dst[k] = src[k];
}
__global__ void k_level_set(const uint64_t* __restrict__ code, const int32_t* __restrict__ fout_rank, int64_t b0,
                            int p3, const double* __restrict__ dense, double* __restrict__ mom) {
  const int64_t i = b0 + blockIdx.x;
  const int r = fout_rank[i];
  if (r < 0) return;
  const double* src = dense + (size_t)code[i] * p3;
  double* dst = mom + (size_t)r * p3;
  for (int k = threadIdx.x; k < p3; k += blockDim.x) dst[k] = src[k];
}

// sparse form (locally essential tree exchange): the boxes of a forced level are all
// present in Morton order, so the box of code c is level_off[level] + c
__global__ void k_box_moments(const int32_t* __restrict__ fout_rank, int64_t b0, int64_t nmax,
                              const int64_t* __restrict__ codes, int p3, double* __restrict__ mom,
                              double* __restrict__ vals, int set) {
  const int64_t k = blockIdx.x;
  const int64_t c = codes[k];
  if (c < 0 || c >= nmax) return;
  const int r = fout_rank[b0 + c];
  if (r < 0) return;
  double* m = mom + (size_t)r * p3;
  double* v = vals + (size_t)k * p3;
  for (int i = threadIdx.x; i < p3; i += blockDim.x) {
    if (set) m[i] = v[i];
    else v[i] = m[i];
  }
}

void box_moments(dmk_plan_s* PL, int level, const int64_t* dcodes, int64_t nb, double* dvals, bool set) {
  if (PL->dim != 3) fail(DMK_ERR_UNSUPPORTED, "box moments are implemented for dim = 3");
  if (level < 0 || level >= PL->min_level) fail(DMK_ERR_ARG, "level must be in [0, min_level)");
  if (level >= PL->th.nlevels - 1) fail(DMK_ERR_STATE, "the tree has no non-leaf boxes at that level");
  if (nb == 0) return;
  const int p3 = PL->tab->p * PL->tab->p * PL->tab->p;
  k_box_moments<<<(unsigned)nb, 256, 0, PL->stream>>>(PL->fout_rank.p, PL->th.level_off[level],
                                                       (int64_t)1 << (3 * level), dcodes, p3, PL->mom.p, dvals,
                                                       set ? 1 : 0);
  DMK_LAUNCH_CHECK();
}

void level_moments(dmk_plan_s* PL, int level, double* ddense, bool set) {
  if (PL->dim != 3) fail(DMK_ERR_UNSUPPORTED, "level moments are implemented for dim = 3");
  if (level < 0 || level >= PL->min_level) fail(DMK_ERR_ARG, "level must be in [0, min_level)");
  if (level >= PL->th.nlevels - 1) fail(DMK_ERR_STATE, "the tree has no non-leaf boxes at that level");
  cudaStream_t s = PL->stream;
  const int p3 = PL->tab->p * PL->tab->p * PL->tab->p;
  const int64_t a = PL->th.level_off[level], b = PL->th.level_off[level + 1];
  if (!set) {
    DMK_CUDA(cudaMemsetAsync(ddense, 0, ((size_t)1 << (3 * level)) * p3 * sizeof(double), s));
    k_level_get<<<(int)(b - a), 256, 0, s>>>(PL->box_code.p, PL->fout_rank.p, a, p3, PL->mom.p, ddense);
    DMK_LAUNCH_CHECK();
    return;
  }
  // levels above `level` are pure c2p sums (all their children are forced non-leaf), so
  // zero them, inject `level`, and rebuild them
  const int64_t r0 = PL->th.fout_off[0], r1 = PL->th.fout_off[level];
  if (r1 > r0) DMK_CUDA(cudaMemsetAsync(PL->mom.p + (size_t)r0 * p3, 0, (size_t)(r1 - r0) * p3 * sizeof(double), s));
  k_level_set<<<(int)(b - a), 256, 0, s>>>(PL->box_code.p, PL->fout_rank.p, a, p3, ddense, PL->mom.p);
  DMK_LAUNCH_CHECK();
  dispatch_p(PL, [&](auto P_, auto NF_, auto NF0_) { run_eval<P_(), NF_(), NF0_()>(PL, PH_C2P_ONLY, level); });
}

}  // namespace dmk
