// tables.cu -- Step 1 of the DMK algorithm ("Precomputation"):
// the per-precision constants and 1D operator matrices the device kernels use.
// Host code, computed once per precision and cached.  This is an independent
// implementation (it shares nothing with oracle/); the parity tests compare the
// device results against the oracle.
//
//   PSWF psi_0^c (App. A.5, Eq. A.15): lowest eigenvector of the prolate
//     differential operator in the normalised Legendre basis (symmetric
//     tridiagonal), solved with cyclic Jacobi rotations.
//   Difference-kernel weights w_{l,m} = (h_l/2pi)^3 Dhat_l(h_l |m|)  (Eqs. 3.37, 3.68)
//   Root window weights (W_0 + D_0 = M_1 windowed by the truncated kernel, Sec. 4.7)
//   Q = E V^{-T}: Chebyshev moments -> outgoing plane waves (T_prox2pw, Eq. 3.42)
//     and conj(Q)^T = V^{-1} E: incoming plane waves -> Chebyshev coefficients
//     (T_pw2poly, Eqs. 3.43-3.44), kept in the real parity-split form Qr / Gr
//     (kernels.cu explains the representation)
//   A_s: Chebyshev re-expansion T_n(x/2 + s/2) = sum_k A_s[n][k] T_k(x) which gives
//     both T_c2p in moment form (Lemma 2.2) and T_p2c = A_s^T (Lemma 2.3)
//   Residual polynomial: r_L M_L(r) = m(r/r_L), m(t) = Phi(t)/t, fitted as a
//     polynomial in s = 2 t^2 - 1 ("piecewise polynomial approximation ... Estrin",
//     PAPER.md:2002-2008), so R_L(r) = 1/r - m(r/r_L)/r_L for r < r_L (Eq. 3.66).
#include <math.h>

#include <cmath>
#include <functional>
#include <tuple>
#include <map>
#include <mutex>

#include "common.cuh"

namespace dmk {
namespace {

constexpr double PI = 3.14159265358979323846;

// Table 1: eps, c, N_1, p
struct Row {
  double eps, c;
  int N1, p;
};
const Row TABLE1[] = {
    {1e-3, 7.2462000846862793, 13, 9},
    {1e-6, 13.739999771118164, 25, 18},
    {1e-9, 20.736000061035156, 39, 28},
};

// ---------------------------------------------------------------- PSWF
struct Pswf {
  double c = 0;
  std::vector<double> a;  // plain Legendre coefficients, degree 0..nmax
  double psi0 = 0, c0 = 0, c2 = 0;

  static void legendre_all(double x, int nmax, std::vector<double>& P) {
    P.resize(nmax + 2);
    P[0] = 1.0;
    P[1] = x;
    for (int n = 1; n <= nmax; ++n) P[n + 1] = ((2.0 * n + 1.0) * x * P[n] - n * P[n - 1]) / (n + 1.0);
  }
  double eval(double x) const {  // truncated to 0 outside [-1, 1]
    if (std::fabs(x) > 1.0) return 0.0;
    std::vector<double> P;
    legendre_all(x, (int)a.size(), P);
    double s = 0;
    for (size_t n = 0; n < a.size(); n += 2) s += a[n] * P[n];
    return s;
  }
  double integral0(double t) const {  // int_0^t psi, t in [0,1]
    std::vector<double> P;
    legendre_all(t, (int)a.size(), P);
    double s = a[0] * t;
    for (size_t n = 2; n < a.size(); n += 2) s += a[n] * (P[n + 1] - P[n - 1]) / (2.0 * n + 1.0);
    return s;
  }
  double Phi(double t) const { return t >= 1.0 ? 1.0 : integral0(t) / c0; }
};

void jacobi_lowest(int m, std::vector<double>& A, std::vector<double>& vec) {
  // cyclic Jacobi on a dense symmetric m x m matrix; returns the eigenvector of the
  // smallest eigenvalue.
  std::vector<double> V(m * m, 0.0);
  for (int i = 0; i < m; ++i) V[i * m + i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0, tot = 0;
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) {
        tot += A[i * m + j] * A[i * m + j];
        if (i != j) off += A[i * m + j] * A[i * m + j];
      }
    if (off <= 1e-32 * tot) break;
    for (int p = 0; p < m - 1; ++p)
      for (int q = p + 1; q < m; ++q) {
        double apq = A[p * m + q];
        if (std::fabs(apq) < 1e-300) continue;
        double app = A[p * m + p], aqq = A[q * m + q];
        double theta = (aqq - app) / (2.0 * apq);
        double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        double cs = 1.0 / std::sqrt(t * t + 1.0), sn = t * cs;
        for (int k = 0; k < m; ++k) {  // A <- J^T A J
          double akp = A[k * m + p], akq = A[k * m + q];
          A[k * m + p] = cs * akp - sn * akq;
          A[k * m + q] = sn * akp + cs * akq;
        }
        for (int k = 0; k < m; ++k) {
          double apk = A[p * m + k], aqk = A[q * m + k];
          A[p * m + k] = cs * apk - sn * aqk;
          A[q * m + k] = sn * apk + cs * aqk;
        }
        for (int k = 0; k < m; ++k) {
          double vkp = V[k * m + p], vkq = V[k * m + q];
          V[k * m + p] = cs * vkp - sn * vkq;
          V[k * m + q] = sn * vkp + cs * vkq;
        }
      }
  }
  int best = 0;
  for (int i = 1; i < m; ++i)
    if (A[i * m + i] < A[best * m + best]) best = i;
  vec.resize(m);
  for (int k = 0; k < m; ++k) vec[k] = V[k * m + best];
}

void gauss_legendre(int n, std::vector<double>& x, std::vector<double>& w) {
  x.resize(n);
  w.resize(n);
  for (int i = 0; i < n; ++i) {
    double z = std::cos(PI * (i + 0.75) / (n + 0.5)), pp = 0;
    for (int it = 0; it < 100; ++it) {
      double p1 = 1, p2 = 0;
      for (int j = 1; j <= n; ++j) {
        double p3 = p2;
        p2 = p1;
        p1 = ((2.0 * j - 1.0) * z * p2 - (j - 1.0) * p3) / j;
      }
      pp = n * (z * p1 - p2) / (z * z - 1.0);
      double z1 = z;
      z = z1 - p1 / pp;
      if (std::fabs(z - z1) < 1e-16) break;
    }
    x[i] = z;
    w[i] = 2.0 / ((1.0 - z * z) * pp * pp);
  }
}

Pswf make_pswf(double c) {
  Pswf P;
  P.c = c;
  int nmax = 2 * (int)std::ceil(c) + 60;
  if (nmax % 2) ++nmax;
  int m = nmax / 2 + 1;
  std::vector<double> A(m * m, 0.0);
  for (int k = 0; k < m; ++k) {
    double n = 2.0 * k;
    double b = (2 * n * (n + 1) - 1) / ((2 * n + 3) * (2 * n - 1));   // <Pbar_n, x^2 Pbar_n>
    A[k * m + k] = n * (n + 1) + c * c * b;
    if (k + 1 < m) {
      double a = (n + 1) * (n + 2) / ((2 * n + 3) * std::sqrt((2 * n + 1) * (2 * n + 5)));
      A[k * m + k + 1] = A[(k + 1) * m + k] = c * c * a;
    }
  }
  std::vector<double> v;
  jacobi_lowest(m, A, v);
  P.a.assign(nmax + 1, 0.0);
  for (int k = 0; k < m; ++k) P.a[2 * k] = v[k] * std::sqrt(2.0 * k + 0.5);   // Pbar -> P
  if (P.eval(0.0) < 0)
    for (auto& x : P.a) x = -x;
  P.psi0 = P.eval(0.0);
  P.c0 = P.a[0];   // int_0^1 P_n = 0 for even n >= 2
  std::vector<double> gx, gw;
  gauss_legendre(120, gx, gw);
  double s2 = 0;
  for (int i = 0; i < 120; ++i) {
    double x = 0.5 * (gx[i] + 1.0);
    s2 += 0.5 * gw[i] * x * x * P.eval(x);
  }
  P.c2 = s2;
  return P;
}

// ---------------------------------------------------------------- Chebyshev helpers
inline double cheb_node(int i, int p) { return std::cos(PI * (i + 0.5) / p); }
inline double vinv(int n, int i, int p) {   // V^{-1}[n][i] by discrete orthogonality
  return (n == 0 ? 1.0 : 2.0) / p * std::cos(n * PI * (i + 0.5) / p);
}
void cheb_T(double x, int p, std::vector<double>& T) {
  T.resize(p);
  T[0] = 1.0;
  if (p > 1) T[1] = x;
  for (int n = 2; n < p; ++n) T[n] = 2.0 * x * T[n - 1] - T[n - 2];
}

// Q[m][n] = sum_i exp(-i a m x_i) V^{-1}[n][i],  a = h s / 2, m in [0, nf] only.
// The Chebyshev nodes are symmetric (x_{p-1-i} = -x_i) and V^{-1}[n][.] has parity (-1)^n,
// so Q[m][n] is real for even n and purely imaginary for odd n, and Q[-m][n] =
// conj(Q[m][n]).  Qr keeps the one non-zero part: Qr[m][n] = Re Q (n even), Im Q (n odd),
// row length pp (p rounded up to even, zero padded).  Gr[n][m] = c_m Qr[m][n] with c_0 = 1,
// c_m = 2 (m > 0) is the matching back transform (T_pw2poly summed over +-m).
void make_Qr(int p, int nf, double a, int pp, int hh, std::vector<double>& Qr, std::vector<double>& Gr) {
  int nh = nf + 1;
  Qr.assign((size_t)nh * pp, 0.0);
  Gr.assign((size_t)p * hh, 0.0);
  for (int m = 0; m < nh; ++m)
    for (int n = 0; n < p; ++n) {
      double re = 0, im = 0;
      for (int i = 0; i < p; ++i) {
        double x = cheb_node(i, p), v = vinv(n, i, p);
        re += std::cos(a * m * x) * v;
        im -= std::sin(a * m * x) * v;
      }
      double q = (n % 2 == 0) ? re : im;
      Qr[(size_t)m * pp + n] = q;
      Gr[(size_t)n * hh + m] = (m == 0 ? 1.0 : 2.0) * q;
    }
}

template <class F>
void make_weights(int nf, double h, F fhat, double* W) {   // layout [a][b][c], a, b, c in [0, nf]
  int nh = nf + 1;
  double scale = std::pow(h / (2.0 * PI), 3);
  for (int a = 0; a < nh; ++a)
    for (int b = 0; b < nh; ++b)
      for (int c = 0; c < nh; ++c) {
        double k = h * std::sqrt((double)(a * a + b * b + c * c));
        W[((size_t)a * nh + b) * nh + c] = scale * fhat(k);
      }
}

void upload(const std::vector<double>& h, double** d) {
  DMK_CUDA(cudaMalloc((void**)d, h.size() * sizeof(double)));
  DMK_CUDA(cudaMemcpy(*d, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice));
}

// Fit g(u), u in [0, 1], by a degree-K polynomial in s = 2u - 1 (Chebyshev interpolation,
// then monomial form); the smallest even K <= 24 whose max error on a grid is <= tol.
static std::vector<double> fit_poly_s(const std::function<double(double)>& g, double tol, int ncheck) {
  std::vector<double> best;
  std::vector<double> gv(ncheck + 1);
  for (int i = 0; i <= ncheck; ++i) gv[i] = g((double)i / ncheck);
  for (int K = 4; K <= 24; K += 2) {
    std::vector<double> cc(K + 1, 0.0);   // Chebyshev coefficients in s
    std::vector<double> gn(K + 1);
    for (int j = 0; j <= K; ++j) gn[j] = g((std::cos(PI * (j + 0.5) / (K + 1)) + 1.0) / 2.0);
    for (int k = 0; k <= K; ++k) {
      double sum = 0;
      for (int j = 0; j <= K; ++j) sum += gn[j] * std::cos(k * PI * (j + 0.5) / (K + 1));
      cc[k] = (k == 0 ? 1.0 : 2.0) / (K + 1) * sum;
    }
    std::vector<double> mono(K + 1, 0.0), t0(K + 1, 0.0), t1(K + 1, 0.0), t2(K + 1, 0.0);
    t0[0] = 1.0;
    t1[1] = 1.0;
    for (int k = 0; k <= K; ++k) {
      const std::vector<double>& tk = (k == 0) ? t0 : t1;
      for (int j = 0; j <= K; ++j) mono[j] += cc[k] * tk[j];
      if (k >= 1) {   // t2 = 2 s t1 - t0, then shift
        std::fill(t2.begin(), t2.end(), 0.0);
        for (int j = 0; j < K; ++j) t2[j + 1] += 2.0 * t1[j];
        for (int j = 0; j <= K; ++j) t2[j] -= t0[j];
        t0 = t1;
        t1 = t2;
      }
    }
    double err = 0;
    for (int i = 0; i <= ncheck; ++i) {
      double s = 2.0 * i / ncheck - 1.0, v = 0;
      for (int j = K; j >= 0; --j) v = v * s + mono[j];
      err = std::fmax(err, std::fabs(v - gv[i]));
    }
    best = mono;
    if (err <= tol) break;
  }
  return best;
}

Tables* build_log2d_tables(double eps);

Tables* build_tables(int kernel, double eps, double lam) {
  if (kernel == DMK_KERNEL_LOG) return build_log2d_tables(eps);
  if (kernel != DMK_KERNEL_LAPLACE && kernel != DMK_KERNEL_YUKAWA)
    fail(DMK_ERR_UNSUPPORTED, "kernel not implemented in 3D (DMK_KERNEL_LAPLACE, DMK_KERNEL_YUKAWA)");
  const bool yuk = kernel == DMK_KERNEL_YUKAWA;
  const Row* row = nullptr;
  for (const Row& r : TABLE1)   // the loosest row at least as tight as eps (reading R1)
    if (r.eps <= eps * (1 + 1e-9)) {
      row = &r;
      break;
    }
  if (!row) fail(DMK_ERR_UNSUPPORTED, "eps tighter than 1e-9 is not supported");
  Tables* T = new Tables();
  T->kernel = kernel;
  T->lam = yuk ? lam : 0.0;
  T->eps = row->eps;
  T->c = row->c;
  T->p = row->p;
  T->nf = (row->N1 - 1) / 2;
  T->RT = 1.0 + std::sqrt(3.0);
  T->P0 = 1.0 + T->RT + 0.5;
  T->nf0 = (int)std::ceil(2.0 * T->c * T->P0 / (2.0 * PI));
  const int p = T->p, nf = T->nf, nf0 = T->nf0;
  Pswf P = make_pswf(T->c);
  const double c = T->c;

  // plane-wave <-> Chebyshev matrices: h_l r_l = 2 pi / 3 for every l >= 1 (reading R2)
  T->pp = (p + 1) & ~1;
  make_Qr(p, nf, PI / 3.0, T->pp, (nf + 2) & ~1, T->Qr1, T->Gr1);
  make_Qr(p, nf0, PI / T->P0, T->pp, (nf0 + 2) & ~1, T->Qr0, T->Gr0);

  // Chebyshev re-expansion A_s
  T->A.assign(2 * p * p, 0.0);
  std::vector<double> Tn;
  for (int si = 0; si < 2; ++si) {
    double s = si ? 1.0 : -1.0;
    for (int i = 0; i < p; ++i) {
      cheb_T(cheb_node(i, p) / 2.0 + s / 2.0, p, Tn);
      for (int n = 0; n < p; ++n)
        for (int k = 0; k < p; ++k) T->A[(si * p + n) * p + k] += vinv(k, i, p) * Tn[n];
    }
  }

  // Fourier-space split (Eq. 3.68; Yukawa: Eq. 4.18 times 4 pi): Khat Ghat_l with
  // Ghat_l(k) = psi(sqrt(k^2 + lam^2) r_l/c)/psi(0)
  const double lam2 = T->lam * T->lam;
  auto Ghat = [&](double rl, double k) { return P.eval(std::sqrt(k * k + lam2) * rl / c) / P.psi0; };
  if (yuk && 0.5 * T->lam >= c)
    fail(DMK_ERR_UNSUPPORTED, "Yukawa lambda * (root side) must be < 2 c (level-1 mollifier vanishes)");

  // difference-kernel weights per level
  int nh = nf + 1;
  T->wstride = (size_t)nh * nh * nh;
  T->W.assign((LMAX + 1) * T->wstride, 0.0);
  for (int l = 1; l <= LMAX; ++l) {
    double rl = std::ldexp(1.0, -l), rl1 = std::ldexp(1.0, -l - 1);
    double h = 2.0 * PI / (3.0 * rl);
    auto Dhat = [&](double k) {
      if (yuk) return 4.0 * PI / (k * k + lam2) * (Ghat(rl1, k) - Ghat(rl, k));
      if (k == 0.0) return 2.0 * PI * P.c2 / P.c0 * (rl * rl - rl1 * rl1);
      return 4.0 * PI / P.psi0 * (P.eval(k * rl1 / c) - P.eval(k * rl / c)) / (k * k);
    };
    make_weights(nf, h, Dhat, &T->W[l * T->wstride]);
  }
  // root window: Ghat_1(k) That(k), That the transform of K truncated at R_T (Sec. 4.7):
  //   1/r:            8 pi sin^2(k R_T/2)/k^2
  //   e^{-lam r}/r:   4 pi/(k^2+lam^2) [1 - e^{-lam R_T}(cos k R_T + (lam/k) sin k R_T)]
  {
    int nh0 = nf0 + 1;
    T->W0.assign((size_t)nh0 * nh0 * nh0, 0.0);
    double h0 = 2.0 * PI / T->P0, RT = T->RT, lm = T->lam;
    auto What = [&](double k) {
      double G = Ghat(0.5, k);
      if (yuk) {
        double E = std::exp(-lm * RT);
        if (k == 0.0) return G * 4.0 * PI / lam2 * (1.0 - E * (1.0 + lm * RT));
        return G * 4.0 * PI / (k * k + lam2) * (1.0 - E * (std::cos(k * RT) + lm / k * std::sin(k * RT)));
      }
      if (k == 0.0) return 2.0 * PI * RT * RT;
      double sn = std::sin(k * RT / 2.0);
      return G * 8.0 * PI * sn * sn / (k * k);
    };
    make_weights(nf0, h0, What, T->W0.data());
  }

  // residual R_L(r) = K(r) - M_L(r), r < r_L (Eq. 3.66 / Eq. 4.18): the device evaluates
  // K directly and r_L M_L(t r_L) = g_L(u), u = t^2, as a polynomial in s = 2u - 1
  // ("piecewise polynomial approximation ... Estrin").
  //   1/r: g(u) = Phi(t)/t, the same at every level (scale invariance).
  //   Yukawa: g_L from the radial inverse transform of Khat Ghat_L (Gauss-Legendre over
  //   the support sqrt(k^2+lam^2) <= c/r_L), one polynomial per level.
  if (!yuk) {
    T->m0 = P.psi0 / P.c0;
    auto g = [&](double u) {
      if (u <= 0.0) return T->m0;
      double t = std::sqrt(u);
      return P.Phi(t) / t;
    };
    T->respoly = fit_poly_s(g, 1e-2 * T->eps * T->m0, 4000);
    T->respoly_deg = (int)T->respoly.size() - 1;
    T->respoly_lv.assign((size_t)(LMAX + 1) * (T->respoly_deg + 1), 0.0);
    for (int l = 0; l <= LMAX; ++l)
      for (int j = 0; j <= T->respoly_deg; ++j) T->respoly_lv[l * (T->respoly_deg + 1) + j] = T->respoly[j];
  } else {
    std::vector<double> gx, gw;
    const int NQ = 300;
    gauss_legendre(NQ, gx, gw);
    std::vector<std::vector<double>> polys(LMAX + 1);
    int deg = 0;
    for (int l = 0; l <= LMAX; ++l) {
      const double rl = std::ldexp(1.0, -l), kmax2 = (c / rl) * (c / rl) - lam2;
      std::vector<double> kq(NQ), fq(NQ);   // nodes and weights * Khat Ghat_l
      const double kmax = kmax2 > 0 ? std::sqrt(kmax2) : 0.0;
      for (int i = 0; i < NQ; ++i) {
        kq[i] = 0.5 * kmax * (gx[i] + 1.0);
        fq[i] = 0.5 * kmax * gw[i] * 4.0 * PI / (kq[i] * kq[i] + lam2) * Ghat(rl, kq[i]);
      }
      auto Mr = [&](double r) {   // M_l(r)
        double sum = 0;
        for (int i = 0; i < NQ; ++i)
          sum += fq[i] * kq[i] * kq[i] * (r > 0 ? std::sin(kq[i] * r) / (kq[i] * r) : 1.0);
        return sum / (2.0 * PI * PI);
      };
      const double m0l = rl * Mr(0.0);
      auto g = [&](double u) { return rl * Mr(std::sqrt(u) * rl); };
      polys[l] = fit_poly_s(g, 1e-2 * T->eps * std::fmax(m0l, 1e-300), 600);
      deg = std::max(deg, (int)polys[l].size() - 1);
      if (l == 0) T->m0 = m0l;
    }
    T->respoly_deg = deg;
    T->respoly_lv.assign((size_t)(LMAX + 1) * (deg + 1), 0.0);
    for (int l = 0; l <= LMAX; ++l)
      for (size_t j = 0; j < polys[l].size(); ++j) T->respoly_lv[l * (deg + 1) + j] = polys[l][j];
    T->respoly = polys[LMAX];
    T->respoly.resize(deg + 1, 0.0);
  }

  upload(T->Qr1, &T->dQr1);
  upload(T->Qr0, &T->dQr0);
  upload(T->Gr1, &T->dGr1);
  upload(T->Gr0, &T->dGr0);
  upload(T->A, &T->dA);
  upload(T->W, &T->dW);
  upload(T->W0, &T->dW0);
  upload(T->respoly_lv, &T->dRespoly);
  return T;
}

// 2D, K(r) = -log r: the Fourier-space split of Sec. 4.6 at lam = 0 in 2D
// (PAPER.md:2441-2447): Khat = 2 pi/k^2, Dhat_l = Khat (Ghat_{l+1} - Ghat_l),
// Dhat_l(0) = pi (c2/c0)(r_l^2 - r_{l+1}^2); root window Ghat_1 That with
// That(k) = 2 pi (1 - J0(k R_T))/k^2 - 2 pi R_T log(R_T) J1(k R_T)/k, R_T = (1 + sqrt 2) r_0
// (Sec. 4.7); weights (h/2pi)^2 Dhat(h |m|) on [0, nf]^2.  The residual
// R_L(r) = -log(r/r_L) - g(t^2), t = r/r_L, with
// g(u) = kappa + int_0^1 (psi(x)/psi(0)) (J0(c x sqrt u) - 1)/x dx,
// kappa = log(c/2) + gamma + int_0^1 (psi(x)/psi(0) - 1)/x dx (the same at every level).
Tables* build_log2d_tables(double eps) {
  const Row* row = nullptr;
  for (const Row& r : TABLE1)
    if (r.eps <= eps * (1 + 1e-9)) {
      row = &r;
      break;
    }
  if (!row) fail(DMK_ERR_UNSUPPORTED, "eps tighter than 1e-9 is not supported");
  Tables* T = new Tables();
  T->dim = 2;
  T->kernel = DMK_KERNEL_LOG;
  T->eps = row->eps;
  T->c = row->c;
  T->p = row->p;
  T->nf = (row->N1 - 1) / 2;
  T->RT = 1.0 + std::sqrt(2.0);
  T->P0 = 1.0 + T->RT + 0.5;
  T->nf0 = (int)std::ceil(2.0 * T->c * T->P0 / (2.0 * PI));
  const int p = T->p, nf = T->nf, nf0 = T->nf0;
  Pswf P = make_pswf(T->c);
  const double c = T->c;
  T->pp = (p + 1) & ~1;
  make_Qr(p, nf, PI / 3.0, T->pp, (nf + 2) & ~1, T->Qr1, T->Gr1);
  make_Qr(p, nf0, PI / T->P0, T->pp, (nf0 + 2) & ~1, T->Qr0, T->Gr0);
  T->A.assign(2 * p * p, 0.0);
  std::vector<double> Tn;
  for (int si = 0; si < 2; ++si) {
    double s = si ? 1.0 : -1.0;
    for (int i = 0; i < p; ++i) {
      cheb_T(cheb_node(i, p) / 2.0 + s / 2.0, p, Tn);
      for (int n = 0; n < p; ++n)
        for (int k = 0; k < p; ++k) T->A[(si * p + n) * p + k] += vinv(k, i, p) * Tn[n];
    }
  }
  auto weights2 = [](int nfw, double h, const std::function<double(double)>& fhat, double* W) {
    int nh = nfw + 1;
    double scale = (h / (2.0 * PI)) * (h / (2.0 * PI));
    for (int a = 0; a < nh; ++a)
      for (int b = 0; b < nh; ++b) W[(size_t)a * nh + b] = scale * fhat(h * std::sqrt((double)(a * a + b * b)));
  };
  const int nh = nf + 1;
  T->wstride = (size_t)nh * nh;
  T->W.assign((LMAX + 1) * T->wstride, 0.0);
  for (int l = 1; l <= LMAX; ++l) {
    double rl = std::ldexp(1.0, -l), rl1 = std::ldexp(1.0, -l - 1);
    double h = 2.0 * PI / (3.0 * rl);
    weights2(nf, h, [&](double k) {
      if (k == 0.0) return PI * P.c2 / P.c0 * (rl * rl - rl1 * rl1);
      return 2.0 * PI / P.psi0 * (P.eval(k * rl1 / c) - P.eval(k * rl / c)) / (k * k);
    }, &T->W[l * T->wstride]);
  }
  {
    const int nh0 = nf0 + 1;
    T->W0.assign((size_t)nh0 * nh0, 0.0);
    const double h0 = 2.0 * PI / T->P0, R = T->RT;
    weights2(nf0, h0, [&](double k) {
      double G = P.eval(k * 0.5 / c) / P.psi0;
      if (k == 0.0) return PI * R * R / 2.0 - PI * R * R * std::log(R);
      return G * (2.0 * PI * (1.0 - ::j0(k * R)) / (k * k) - 2.0 * PI * R * std::log(R) * ::j1(k * R) / k);
    }, T->W0.data());
  }
  {
    std::vector<double> gx, gw;
    const int NQ = 240;
    gauss_legendre(NQ, gx, gw);
    std::vector<double> xq(NQ), wq(NQ), pq(NQ);
    double kap = std::log(c / 2.0) + 0.57721566490153286061;
    for (int i = 0; i < NQ; ++i) {
      xq[i] = 0.5 * (gx[i] + 1.0);
      wq[i] = 0.5 * gw[i];
      pq[i] = P.eval(xq[i]) / P.psi0;
      kap += wq[i] * (pq[i] - 1.0) / xq[i];
    }
    T->m0 = kap;
    auto g = [&](double u) {
      double t = std::sqrt(std::fmax(u, 0.0)), sum = 0;
      for (int i = 0; i < NQ; ++i) sum += wq[i] * pq[i] * (::j0(c * xq[i] * t) - 1.0) / xq[i];
      return kap + sum;
    };
    T->respoly = fit_poly_s(g, 1e-2 * T->eps, 1000);
    T->respoly_deg = (int)T->respoly.size() - 1;
    T->respoly_lv.assign((size_t)(LMAX + 1) * (T->respoly_deg + 1), 0.0);
    for (int l = 0; l <= LMAX; ++l)
      for (int j = 0; j <= T->respoly_deg; ++j) T->respoly_lv[l * (T->respoly_deg + 1) + j] = T->respoly[j];
  }
  upload(T->Qr1, &T->dQr1);
  upload(T->Qr0, &T->dQr0);
  upload(T->Gr1, &T->dGr1);
  upload(T->Gr0, &T->dGr0);
  upload(T->A, &T->dA);
  upload(T->W, &T->dW);
  upload(T->W0, &T->dW0);
  upload(T->respoly_lv, &T->dRespoly);
  return T;
}

std::mutex g_mu;
// Cache of Step-1 tables, keyed by (device, kernel, Table 1 row, lambda').  Laplace and
// log tables are one per device and row.  The Yukawa tables depend on lambda' =
// lambda * side, i.e. on the data's bounding cube, so almost every point set gets its own:
// at most YUKAWA_CACHE of them stay cached per process (least recently used evicted);
// plans hold a reference, so an evicted table lives until its last plan is destroyed.
constexpr size_t YUKAWA_CACHE = 8;
struct Entry {
  std::shared_ptr<const Tables> t;
  uint64_t last_use;
};
std::map<std::tuple<int, int, double, double>, Entry> g_cache;
uint64_t g_tick = 0;

}  // namespace

Tables::~Tables() {
  int cur = -1;
  if (cudaGetDevice(&cur) != cudaSuccess) return;
  if (dev >= 0 && dev != cur) cudaSetDevice(dev);
  for (double* d : {dQr1, dQr0, dGr1, dGr0, dA, dW, dW0, dRespoly})
    if (d) cudaFree(d);
  if (dev >= 0 && dev != cur) cudaSetDevice(cur);
}

double snap_eps(double eps) {
  for (const Row& r : TABLE1)
    if (r.eps <= eps * (1 + 1e-9)) return r.eps;
  return 0;
}

std::shared_ptr<const Tables> get_tables(int kernel, double eps, double lam) {
  int dev = 0;
  DMK_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_mu);
  const bool yuk = kernel == DMK_KERNEL_YUKAWA;
  auto key = std::make_tuple(dev, kernel, snap_eps(eps), yuk ? lam : 0.0);
  auto it = g_cache.find(key);
  if (it != g_cache.end()) {
    it->second.last_use = ++g_tick;
    return it->second.t;
  }
  std::shared_ptr<Tables> T(build_tables(kernel, eps, lam));
  T->dev = dev;
  if (yuk) {
    size_t ny = 0;
    auto lru = g_cache.end();
    for (auto e = g_cache.begin(); e != g_cache.end(); ++e)
      if (std::get<1>(e->first) == DMK_KERNEL_YUKAWA) {
        ++ny;
        if (lru == g_cache.end() || e->second.last_use < lru->second.last_use) lru = e;
      }
    if (ny >= YUKAWA_CACHE) g_cache.erase(lru);
  }
  g_cache[key] = Entry{T, ++g_tick};
  return T;
}

size_t tables_cached() {
  std::lock_guard<std::mutex> lk(g_mu);
  return g_cache.size();
}

}  // namespace dmk
