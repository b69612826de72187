// kernels2d.cu -- the DMK hot path in 2D for K(r) = -log r (BASELINE config 3), Sec. 3.5
// Steps 2-5 on a quadtree, with the Fourier-space PSWF split of
// Sec. 4.6 at lam = 0 (tables.cu build_log2d_tables).
//
// Same representation as the 3D path (kernels.cu): Chebyshev moments in the upward
// pass, the real parity-split plane-wave form F[a][pi][b] (pi = 2 pi1 + pi2, a, b =
// |m1|, |m2| in [0, nf]) with the colleague shift as per-axis rotations, Chebyshev
// coefficients Lambda in the downward pass.  Everything per box is p^2 or (nf+1)^2, so
// these are plain fp64 kernels: one CTA per box, operands in shared memory.
//
//   k_anterp2   moments mu[n1][n2] = sum_j rho_j T_n1(xi_j) T_n2(eta_j)  (Def. 2.1)
//   k_c2p2      child -> parent moments (Lemma 2.2), one level per launch
//   k_prox2pw2  F = (Qr (x) Qr) mu per parity class (Eq. 3.42)
//   k_pwlocal2  9-colleague translation (Eq. 3.39) + weights + (Gr (x) Gr) (Eqs. 3.43-3.44)
//   k_p2c2      Lambda(B) += (A^T (x) A^T) Lambda(parent) (Lemma 2.3)
//   k_eval2     far field at the targets
//   k_p2p2      residual of the source level over the direct lists, Step 5, the
//               -log(side) rescaling, scatter to caller order
#include "device.cuh"

namespace dmk {
namespace {

constexpr int NCH2 = 4, NCOL2 = 9;

__device__ __forceinline__ uint32_t compact2d(uint64_t x) {
  x &= 0x5555555555555555ULL;
  x = (x ^ (x >> 1)) & 0x3333333333333333ULL;
  x = (x ^ (x >> 2)) & 0x0f0f0f0f0f0f0f0fULL;
  x = (x ^ (x >> 4)) & 0x00ff00ff00ff00ffULL;
  x = (x ^ (x >> 8)) & 0x0000ffff0000ffffULL;
  x = (x ^ (x >> 16)) & 0x00000000ffffffffULL;
  return (uint32_t)x;
}
__device__ __forceinline__ void box_geom2(uint64_t code, int l, double c[2], double& inv_half) {
  double s = ldexp(1.0, -l);
  c[0] = ((double)compact2d(code >> 1) + 0.5) * s;
  c[1] = ((double)compact2d(code) + 0.5) * s;
  inv_half = ldexp(1.0, l + 1);
}

// ---------------------------------------------------------------- anterpolation
template <int P>
__global__ void __launch_bounds__(256) k_anterp2(DevTree t, const int32_t* __restrict__ boxes,
                                                 const double* __restrict__ q, double* __restrict__ mom) {
  constexpr int NT = 256, CH = 64, P2 = P * P, NO = (P2 + NT - 1) / NT;
  __shared__ double Tx[CH][P], Ty[CH][P];
  __shared__ int2 rg[NCH2];
  __shared__ int nr_s, tot_s;
  const int b = boxes[blockIdx.x], tid = threadIdx.x;
  if (tid < 32) box_ranges_w<false, NCH2>(t, b, rg, nr_s, tot_s);
  __syncthreads();
  const int nr = nr_s, tot = tot_s;
  double* out = mom + (size_t)t.fout_rank[b] * P2;
  if (tot == 0) return;   // zeroed by the caller
  double cen[2], ih;
  box_geom2(t.code[b], t.level[b], cen, ih);
  double acc[NO];
#pragma unroll
  for (int i = 0; i < NO; ++i) acc[i] = 0.0;
  for (int c0 = 0; c0 < tot; c0 += CH) {
    const int nc = min(CH, tot - c0);
    for (int w = tid; w < 2 * CH; w += NT) {
      const int j = w >> 1, d = w & 1;
      double T[P];
      if (j < nc) {
        const int pi = range_point(rg, nr, c0 + j);
        cheb_vec(((d ? t.ys[pi] : t.xs[pi]) - cen[d]) * ih, T, P, d ? 1.0 : q[pi]);
      } else {
#pragma unroll
        for (int n = 0; n < P; ++n) T[n] = 0.0;
      }
      double* dst = d ? Ty[j] : Tx[j];
#pragma unroll
      for (int n = 0; n < P; ++n) dst[n] = T[n];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < NO; ++i) {
      const int o = tid + i * NT;
      if (o < P2) {
        const int n1 = o / P, n2 = o % P;
        double s = acc[i];
        for (int j = 0; j < nc; ++j) s = fma(Tx[j][n1], Ty[j][n2], s);
        acc[i] = s;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < NO; ++i)
    if (tid + i * NT < P2) out[tid + i * NT] = acc[i];
}

// ---------------------------------------------------------------- c2p / p2c
// Y[n1][m] = sum_k X[n1][k] M2(m,k) then Z[m][n2] = sum_k M1(m,k) Y[k][n2], with
// M(m,k) = A_s[m][k] (c2p) or A_s[k][m] (p2c); child bits: bit1 = x (n1), bit0 = y (n2).
template <int P, bool TRANS>
__device__ __forceinline__ void sq_transform(double* X, double* Y, const double* M1, const double* M2, int tid,
                                             int nt) {
  constexpr int P2 = P * P;
  for (int o = tid; o < P2; o += nt) {
    const int r = o / P, m = o % P;
    double s = 0.0;
    for (int k = 0; k < P; ++k) s = fma(X[r * P + k], TRANS ? M2[k * P + m] : M2[m * P + k], s);
    Y[o] = s;
  }
  __syncthreads();
  for (int o = tid; o < P2; o += nt) {
    const int m = o / P, c = o % P;
    double s = 0.0;
    for (int k = 0; k < P; ++k) s = fma(TRANS ? M1[k * P + m] : M1[m * P + k], Y[k * P + c], s);
    X[o] = s;
  }
  __syncthreads();
}

template <int P>
__global__ void __launch_bounds__(256) k_c2p2(DevTree t, const int32_t* __restrict__ boxes,
                                              const double* __restrict__ A, double* __restrict__ mom) {
  constexpr int NT = 256, P2 = P * P;
  __shared__ double X[P2], Y[P2], sA[2 * P2];
  const int b = boxes[blockIdx.x], tid = threadIdx.x;
  for (int i = tid; i < 2 * P2; i += NT) sA[i] = A[i];
  double* dst = mom + (size_t)t.fout_rank[b] * P2;
  for (int o = 0; o < NCH2; ++o) {
    const int ch = t.child[NCH2 * (int64_t)b + o];
    if (ch < 0 || !(t.flags[ch] & F_OUT)) continue;
    const double* src = mom + (size_t)t.fout_rank[ch] * P2;
    __syncthreads();
    for (int i = tid; i < P2; i += NT) X[i] = src[i];
    __syncthreads();
    sq_transform<P, false>(X, Y, sA + ((o >> 1) & 1) * P2, sA + (o & 1) * P2, tid, NT);
    for (int i = tid; i < P2; i += NT) dst[i] += X[i];   // this CTA owns mu(parent)
  }
}

template <int P>
__global__ void __launch_bounds__(256) k_p2c2(DevTree t, const int32_t* __restrict__ boxes,
                                              const double* __restrict__ A, double* __restrict__ lam) {
  constexpr int NT = 256, P2 = P * P;
  __shared__ double X[P2], Y[P2], sA[2 * P2];
  const int b = boxes[blockIdx.x], tid = threadIdx.x;
  const int par = t.parent[b], o = (int)(t.code[b] & 3);
  for (int i = tid; i < 2 * P2; i += NT) sA[i] = A[i];
  const double* src = lam + (size_t)t.exp_rank[par] * P2;
  for (int i = tid; i < P2; i += NT) X[i] = src[i];
  __syncthreads();
  sq_transform<P, true>(X, Y, sA + ((o >> 1) & 1) * P2, sA + (o & 1) * P2, tid, NT);
  double* dst = lam + (size_t)t.exp_rank[b] * P2;
  for (int i = tid; i < P2; i += NT) dst[i] += X[i];
}

// ---------------------------------------------------------------- plane waves
// F[a][pi1 pi2][b] = sum_{n_d = pi_d (2)} Qr[a][n1] Qr[b][n2] mu[n1][n2]
template <int P, int H>
__global__ void __launch_bounds__(256) k_prox2pw2(DevTree t, const int32_t* __restrict__ boxes,
                                                  const double* __restrict__ Qr, const double* __restrict__ mom,
                                                  double* __restrict__ F, size_t base, size_t stride) {
  constexpr int NT = 256, P2 = P * P, PP = (P + 1) & ~1;
  __shared__ double sQ[H * PP], mu[P2], X[P * 2 * H];
  const int b = boxes[blockIdx.x], tid = threadIdx.x;
  const int r = t.fout_rank[b];
  double* out = F + base + (size_t)(r == 0 ? 0 : r - 1) * stride;
  for (int i = tid; i < H * PP; i += NT) sQ[i] = Qr[i];
  for (int i = tid; i < P2; i += NT) mu[i] = mom[(size_t)r * P2 + i];
  __syncthreads();
  for (int o = tid; o < P * 2 * H; o += NT) {   // X[n1][pi2][b]
    const int n1 = o / (2 * H), pi2 = (o / H) & 1, bb = o % H;
    double s = 0.0;
    for (int n2 = pi2; n2 < P; n2 += 2) s = fma(sQ[bb * PP + n2], mu[n1 * P + n2], s);
    X[o] = s;
  }
  __syncthreads();
  for (int o = tid; o < 4 * H * H; o += NT) {   // F[a][pi][b]
    const int a = o / (4 * H), pi = (o / H) & 3, bb = o % H, pi1 = pi >> 1, pi2 = pi & 1;
    double s = 0.0;
    for (int n1 = pi1; n1 < P; n1 += 2) s = fma(sQ[a * PP + n1], X[(n1 * 2 + pi2) * H + bb], s);
    out[o] = s;
  }
}

// rotation-accumulate on a 4-vector along the axis of parity bit ST (2: axis 1, 1: axis 2)
template <int ST, int DELTA>
__device__ __forceinline__ void rot_acc4(double* acc, const double* g, double C, double S) {
#pragma unroll
  for (int p = 0; p < 4; ++p) {
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
__device__ __forceinline__ void rot_cs2(int m, double& C, double& S) {
  const int e = m % 3;
  C = e == 0 ? 1.0 : -0.5;
  S = e == 0 ? 0.0 : (e == 1 ? 0.86602540378443864676 : -0.86602540378443864676);
}

// Psi = w (.) sum over the 9 colleagues of the rotated F; Lambda = (Gr (x) Gr) Psi per parity
template <int P, int H, bool ROOT>
__global__ void __launch_bounds__(256) k_pwlocal2(DevTree t, const int32_t* __restrict__ boxes,
                                                  const double* __restrict__ Gr, const double* __restrict__ W,
                                                  size_t wstride, const double* __restrict__ F, size_t base,
                                                  size_t stride, double* __restrict__ lam) {
  constexpr int NT = 256, P2 = P * P, HH = (H + 1) & ~1;
  __shared__ double sG[P * HH], Tm[4 * H * H], Y[2 * H * P];
  __shared__ const double* src[NCOL2];
  const int b = boxes[blockIdx.x], tid = threadIdx.x;
  if (!(t.flags[b] & F_IN)) return;
  const double* Wl = W + (ROOT ? 0 : (size_t)t.level[b] * wstride);
  for (int i = tid; i < P * HH; i += NT) sG[i] = Gr[i];
  if (tid < NCOL2) {
    // slot k = (dx+1)*3 + (dy+1) holds B + (dx,dy); delta = -(dx,dy) has slot 8 - k
    const double* p = nullptr;
    if (ROOT) {
      if (tid == 4) p = F;
    } else {
      const int s = t.coll[NCOL2 * (int64_t)b + tid];
      if (s >= 0 && (t.flags[s] & F_OUT)) p = F + base + (size_t)(t.fout_rank[s] - 1) * stride;
    }
    src[8 - tid] = p;
  }
  __syncthreads();
  for (int o = tid; o < H * H; o += NT) {   // translation at mode (a, b)
    const int a = o / H, bb = o % H;
    double out4[4] = {0.0, 0.0, 0.0, 0.0};
    if (ROOT) {
#pragma unroll
      for (int p = 0; p < 4; ++p) out4[p] = src[4][(a * 4 + p) * H + bb];
    } else {
      double Ca, Sa, Cb, Sb;
      rot_cs2(a, Ca, Sa);
      rot_cs2(bb, Cb, Sb);
#pragma unroll
      for (int d1 = 0; d1 < 3; ++d1) {
        double x[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int d2 = 0; d2 < 3; ++d2) {
          const double* s = src[d1 * 3 + d2];
          if (!s) continue;
          double g[4];
#pragma unroll
          for (int p = 0; p < 4; ++p) g[p] = __ldg(s + (a * 4 + p) * H + bb);
          if (d2 == 0) rot_acc4<1, -1>(x, g, Cb, Sb);
          else if (d2 == 1) rot_acc4<1, 0>(x, g, Cb, Sb);
          else rot_acc4<1, 1>(x, g, Cb, Sb);
        }
        if (d1 == 0) rot_acc4<2, -1>(out4, x, Ca, Sa);
        else if (d1 == 1) rot_acc4<2, 0>(out4, x, Ca, Sa);
        else rot_acc4<2, 1>(out4, x, Ca, Sa);
      }
    }
    const double wt = Wl[a * H + bb];
#pragma unroll
    for (int p = 0; p < 4; ++p) Tm[(p * H + a) * H + bb] = wt * out4[p];
  }
  __syncthreads();
  for (int o = tid; o < 2 * H * P; o += NT) {   // Y[pi1][a][n2] = sum_b Gr[n2][b] T[2 pi1 + n2%2][a][b]
    const int pi1 = o / (H * P), a = (o / P) % H, n2 = o % P;
    const double* tr = Tm + ((2 * pi1 + (n2 & 1)) * H + a) * H;
    double s = 0.0;
    for (int bb = 0; bb < H; ++bb) s = fma(sG[n2 * HH + bb], tr[bb], s);
    Y[o] = s;
  }
  __syncthreads();
  double* dst = lam + (size_t)t.exp_rank[b] * P2;
  for (int o = tid; o < P2; o += NT) {   // Lambda[n1][n2] = sum_a Gr[n1][a] Y[n1%2][a][n2]
    const int n1 = o / P, n2 = o % P;
    const double* yr = Y + (n1 & 1) * H * P + n2;
    double s = 0.0;
    for (int a = 0; a < H; ++a) s = fma(sG[n1 * HH + a], yr[a * P], s);
    dst[o] = s;
  }
}

// ---------------------------------------------------------------- evaluation
template <int P>
__global__ void __launch_bounds__(128) k_eval2(DevTree t, const int32_t* __restrict__ boxes,
                                               const double* __restrict__ lam, double* __restrict__ ufar) {
  constexpr int NT = 128, P2 = P * P;
  __shared__ double L[P2];
  __shared__ int2 rg[NCH2];
  __shared__ int nr_s, tot_s;
  const int b = boxes[blockIdx.x], tid = threadIdx.x;
  if (tid < 32) box_ranges_w<true, NCH2>(t, b, rg, nr_s, tot_s);
  const double* src = lam + (size_t)t.exp_rank[b] * P2;
  for (int i = tid; i < P2; i += NT) L[i] = src[i];
  __syncthreads();
  const int nr = nr_s, tot = tot_s;
  double cen[2], ih;
  box_geom2(t.code[b], t.level[b], cen, ih);
  for (int j = tid; j < tot; j += NT) {
    const int pi = range_point(rg, nr, j);
    double Tx[P], Ty[P];
    cheb_vec((t.xs[pi] - cen[0]) * ih, Tx, P, 1.0);
    cheb_vec((t.ys[pi] - cen[1]) * ih, Ty, P, 1.0);
    double u = 0.0;
    for (int n1 = 0; n1 < P; ++n1) {
      double s = 0.0;
#pragma unroll
      for (int n2 = 0; n2 < P; ++n2) s = fma(L[n1 * P + n2], Ty[n2], s);
      u = fma(Tx[n1], s, u);
    }
    ufar[pi] = u;
  }
}

// ---------------------------------------------------------------- P2P
struct ResPoly2 {
  double a[25];
};
// total charge, deterministic: pass 1 gives SUMB fixed-order block partials, pass 2 adds
// them in order (one block of SUMB threads)
constexpr int SUMB = 512;
__global__ void k_sum_part(const double* __restrict__ q, int64_t n, double* part) {
  __shared__ double s[256];
  double v = 0.0;
  for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)SUMB * 256) v += q[i];
  s[threadIdx.x] = v;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = s[0];
}
__global__ void k_sum(const double* __restrict__ part, double* out) {
  __shared__ double s[SUMB];
  s[threadIdx.x] = part[threadIdx.x];
  __syncthreads();
  for (int w = SUMB / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = s[0];
}

// R_L(r) = -log r + log r_L - g(s), s = 2 r^2/r_L^2 - 1, for 0 < r < r_L (source level L);
// r = 0 (self / coincident): -M_L(0) = log r_L - g(-1) (Step 5), and the coincident
// charge is accumulated for the rescaling u = u' - log(side) (Q - q_coinc) back to the
// caller's units.  FULL: the root is a leaf, the kernel itself.
template <int K, bool FULL>
__global__ void __launch_bounds__(128) k_p2p2(DevTree t, const int32_t* __restrict__ items, int64_t nitems,
                                              const int32_t* __restrict__ doff, const int32_t* __restrict__ dlist,
                                              const double* __restrict__ q, const double* __restrict__ ufar,
                                              const int32_t* __restrict__ perm, double log_side,
                                              const double* __restrict__ qtot, ResPoly2 rp,
                                              double* __restrict__ unear, double* __restrict__ out) {
  __shared__ double2 sxy[4][32];
  __shared__ double sq[4][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t it = (int64_t)blockIdx.x * 4 + warp;
  if (it >= nitems) return;
  const int B = items[2 * it], t0 = items[2 * it + 1];
  const int nt = min(32, t.end[B] - t0);
  const int ti = t0 + min(lane, nt - 1);
  const double xt = t.xs[ti], yt = t.ys[ti];
  double acc = 0.0, qc = 0.0;
  for (int e = doff[B]; e < doff[B + 1]; ++e) {
    const int S = dlist[e];
    const int L = t.level[S];
    const double two_irl2 = ldexp(2.0, 2 * L), rl2 = ldexp(1.0, -2 * L);
    const double log_rl = -L * 0.69314718055994530942;
    for (int s0 = t.start[S]; s0 < t.end[S]; s0 += 32) {
      const int ns = min(32, t.end[S] - s0);
      if (lane < ns) {
        const int j = s0 + lane;
        sxy[warp][lane] = make_double2(t.xs[j], t.ys[j]);
        sq[warp][lane] = q[j];
      }
      __syncwarp();
      for (int k = 0; k < ns; ++k) {
        const double2 sp = sxy[warp][k];
        const double w = sq[warp][k];
        const double dx = xt - sp.x, dy = yt - sp.y;
        const double r2 = fma(dx, dx, dy * dy);
        if (r2 == 0.0) qc += w;
        if (FULL) {
          if (r2 > 0.0) acc = fma(w, -0.5 * log(r2), acc);
        } else if (r2 < rl2) {
          const double s = fma(r2, two_irl2, -1.0);
          double pv = rp.a[K];
#pragma unroll
          for (int j = K - 1; j >= 0; --j) pv = fma(pv, s, rp.a[j]);
          const double kv = r2 > 0.0 ? -0.5 * log(r2) : 0.0;
          acc = fma(w, kv + log_rl - pv, acc);
        }
      }
      __syncwarp();
    }
  }
  if (lane < nt) {
    const int i = t0 + lane;
    unear[i] = acc;
    out[perm[i]] = ufar[i] + acc - log_side * (*qtot - qc);
  }
}

}  // namespace

// ---------------------------------------------------------------- host
template <int P, int NF, int NF0>
static void run_eval2(dmk_plan_s* PL) {
  cudaStream_t s = PL->stream;
  const Tables& T = *PL->tab;
  DevTree dt = dev_tree(PL);
  const auto& th = PL->th;
  const int nl = th.nlevels;
  constexpr int P2 = P * P, H = NF + 1, H0 = NF0 + 1;
  Timer tm(PL);
  if (nl > 1) {
    tm.begin("anterp");
    DMK_CUDA(cudaMemsetAsync(PL->mom.p, 0, PL->mom.bytes(), s));
    if (PL->nfout) {
      k_anterp2<P><<<(int)PL->nfout, 256, 0, s>>>(dt, PL->fout_list.p, PL->q.p, PL->mom.p);
      DMK_LAUNCH_CHECK();
    }
    tm.end();
    tm.begin("c2p");
    for (int l = nl - 2; l >= 0; --l) {
      int64_t a = th.fout_off[l], b = th.fout_off[l + 1];
      if (b > a) {
        k_c2p2<P><<<(int)(b - a), 256, 0, s>>>(dt, PL->fout_list.p + a, T.dA, PL->mom.p);
        DMK_LAUNCH_CHECK();
      }
    }
    tm.end();
    tm.begin("prox2pw");
    k_prox2pw2<P, H0><<<1, 256, 0, s>>>(dt, PL->fout_list.p, T.dQr0, PL->mom.p, PL->phi.p, 0, 0);
    DMK_LAUNCH_CHECK();
    if (PL->nfout > 1) {
      k_prox2pw2<P, H><<<(int)(PL->nfout - 1), 256, 0, s>>>(dt, PL->fout_list.p + 1, T.dQr1, PL->mom.p, PL->phi.p,
                                                           PL->phi_size0, PL->phi_size1);
      DMK_LAUNCH_CHECK();
    }
    tm.end();
    tm.begin("pwlocal");
    k_pwlocal2<P, H0, true><<<1, 256, 0, s>>>(dt, PL->exp_list.p, T.dGr0, T.dW0, 0, PL->phi.p, 0, 0, PL->lam.p);
    DMK_LAUNCH_CHECK();
    if (PL->nexp > 1) {
      k_pwlocal2<P, H, false><<<(int)(PL->nexp - 1), 256, 0, s>>>(dt, PL->exp_list.p + 1, T.dGr1, T.dW, T.wstride,
                                                                  PL->phi.p, PL->phi_size0, PL->phi_size1,
                                                                  PL->lam.p);
      DMK_LAUNCH_CHECK();
    }
    tm.end();
    tm.begin("p2c");
    for (int l = 1; l < nl; ++l) {
      int64_t a = th.exp_off[l], b = th.exp_off[l + 1];
      if (b > a) {
        k_p2c2<P><<<(int)(b - a), 256, 0, s>>>(dt, PL->exp_list.p + a, T.dA, PL->lam.p);
        DMK_LAUNCH_CHECK();
      }
    }
    tm.end();
    tm.begin("eval");
    if (PL->nexp) {
      k_eval2<P><<<(int)PL->nexp, 128, 0, s>>>(dt, PL->exp_list.p, PL->lam.p, PL->ufar.p);
      DMK_LAUNCH_CHECK();
    }
    tm.end();
  } else {
    DMK_CUDA(cudaMemsetAsync(PL->ufar.p, 0, PL->n * sizeof(double), s));
  }
  (void)P2;
}

template <bool FULL>
static void run_p2p2(dmk_plan_s* PL, double* out) {
  DevTree dt = dev_tree(PL);
  const int nb = (int)((PL->np2p + 3) / 4);
  if (nb == 0) return;
  const Tables& T = *PL->tab;
  ResPoly2 rp{};
  const int K = T.respoly_deg;
  for (int k = 0; k <= K && k < 25; ++k) rp.a[k] = T.respoly[k];
  {
    DevBuf<double> part;
    part.alloc(SUMB, PL->stream);
    k_sum_part<<<SUMB, 256, 0, PL->stream>>>(PL->q.p, PL->n, part.p);
    DMK_LAUNCH_CHECK();
    k_sum<<<1, SUMB, 0, PL->stream>>>(part.p, PL->scalar.p);
    DMK_LAUNCH_CHECK();
  }
  const double ls = std::log(PL->side);
#define DMK_P2P2_CASE(KK)                                                                                          \
  case KK:                                                                                                         \
    k_p2p2<KK, FULL><<<nb, 128, 0, PL->stream>>>(dt, PL->p2p_items.p, PL->np2p, PL->dlist_off.p, PL->dlist.p,      \
                                                 PL->q.p, PL->ufar.p, PL->perm.p, ls, PL->scalar.p, rp,             \
                                                 PL->unear.p, out);                                                 \
    break;
  switch (K) {
    DMK_P2P2_CASE(4) DMK_P2P2_CASE(6) DMK_P2P2_CASE(8) DMK_P2P2_CASE(10) DMK_P2P2_CASE(12) DMK_P2P2_CASE(14)
    DMK_P2P2_CASE(16) DMK_P2P2_CASE(18) DMK_P2P2_CASE(20) DMK_P2P2_CASE(22) DMK_P2P2_CASE(24)
    default: fail(DMK_ERR_UNSUPPORTED, "residual polynomial degree out of range");
  }
#undef DMK_P2P2_CASE
  DMK_LAUNCH_CHECK();
}

// Steps 2-5 in 2D (charges already gathered into PL->q)
void eval_plan_2d(dmk_plan_s* PL, double* dout) {
  if (PL->tab->nf0 != (PL->tab->p == 9 ? 10 : PL->tab->p == 18 ? 18 : 26))
    fail(DMK_ERR_UNSUPPORTED, "2D root Fourier width does not match the compiled kernels");
  switch (PL->tab->p) {
    case 9: run_eval2<9, 6, 10>(PL); break;
    case 18: run_eval2<18, 12, 18>(PL); break;
    case 28: run_eval2<28, 19, 26>(PL); break;
    default: fail(DMK_ERR_UNSUPPORTED, "unsupported Chebyshev order");
  }
  Timer tm(PL);
  tm.begin("p2p");
  if (PL->th.nlevels == 1) run_p2p2<true>(PL, dout);
  else run_p2p2<false>(PL, dout);
  tm.end();
}

}  // namespace dmk
