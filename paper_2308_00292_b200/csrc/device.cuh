// device.cuh -- device-side helpers shared by the 3D (kernels.cu) and 2D (kernels2d.cu)
// DMK kernels: the tree view, Chebyshev vectors, the fp64 tensor-core (DMMA) tile
// helper, point-range walks, launch helpers and phase timers.  Internal, not ABI.
#pragma once
#include <cstring>

#include "common.cuh"

namespace dmk {

struct DevTree {
  const uint64_t* code;
  const int32_t* level;
  const int32_t* start;
  const int32_t* end;
  const int32_t* parent;
  const int32_t* child;
  const int32_t* coll;
  const uint8_t* flags;
  const int32_t* fout_rank;
  const int32_t* exp_rank;
  const double* xs;
  const double* ys;
  const double* zs;
};
constexpr uint8_t F_LEAF = 1, F_OUT = 2, F_IN = 4, F_EXP = 8, F_TGT = 16;

__device__ __forceinline__ uint32_t compact3d(uint64_t x) {
  x &= 0x1249249249249249ULL;
  x = (x ^ (x >> 2)) & 0x10c30c30c30c30c3ULL;
  x = (x ^ (x >> 4)) & 0x100f00f00f00f00fULL;
  x = (x ^ (x >> 8)) & 0x1f0000ff0000ffULL;
  x = (x ^ (x >> 16)) & 0x1f00000000ffffULL;
  x = (x ^ (x >> 32)) & 0x1fffffULL;
  return (uint32_t)x;
}
// centre of box (code, level) and the scale 2/side
__device__ __forceinline__ void box_geom(uint64_t code, int l, double c[3], double& inv_half) {
  double s = ldexp(1.0, -l);
  c[0] = ((double)compact3d(code >> 2) + 0.5) * s;
  c[1] = ((double)compact3d(code >> 1) + 0.5) * s;
  c[2] = ((double)compact3d(code) + 0.5) * s;
  inv_half = ldexp(1.0, l + 1);
}

__device__ __forceinline__ void cheb_vec(double x, double* T, int P, double scale0) {
  // T[n] = scale0 * T_n(x)
  double t0 = 1.0, t1 = x;
  T[0] = scale0;
  if (P > 1) T[1] = scale0 * x;
  for (int n = 2; n < P; ++n) {
    double t2 = 2.0 * x * t1 - t0;
    T[n] = scale0 * t2;
    t0 = t1;
    t1 = t2;
  }
}

// ---------------------------------------------------------------- asynchronous global -> shared copies
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---------------------------------------------------------------- fp64 tensor-core (DMMA) versions
// mma.sync.m8n8k4 f64: A[row=lane>>2][col=lane&3], B[row=lane&3][col=lane>>2],
// C[row=lane>>2][col=2*(lane&3)+{0,1}].  Measured on this B200: 37.2 TFLOP/s, the
// same as DFMA, but 256 FMA per warp instruction from 2 register operands, which
// takes the shared-memory bandwidth limit off these small per-box GEMMs.
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Warp-cooperative C = A B over 8x8 output tiles with K = 4 KS (zero padded by the
// operand functors): fa(m, k), fb(k, n) return operand values, fc(m, n, c_n, c_{n+1})
// consumes the two accumulators a lane owns.  Tiles are dealt round-robin to the warps.
// LOOKAHEAD: the next tile's operands are loaded during the current tile's DMMA chain
// (c2p, whose B operands come from global memory: 0.33 -> 0.305 ms at config 1; the
// register cost makes it slower for the shared-memory-fed contractions)
template <int KS, bool LOOKAHEAD = false, class FA, class FB, class FC>
__device__ __forceinline__ void mma_tiles(int mtiles, int ntiles, FA fa, FB fb, FC fc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int ntot = mtiles * ntiles;
  if constexpr (!LOOKAHEAD) {
    for (int t = warp; t < ntot; t += nw) {
      const int m0 = (t / ntiles) * 8, n0 = (t % ntiles) * 8;
      // all operands of the tile first (independent loads in flight), then the DMMA chain
      double av[KS], bv[KS];
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        av[ks] = fa(m0 + g, ks * 4 + q);
        bv[ks] = fb(ks * 4 + q, n0 + g);
      }
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) dmma(c0, c1, av[ks], bv[ks]);
      fc(m0 + g, n0 + 2 * q, c0, c1);
    }
    return;
  }
  int t = warp;
  if (t >= ntot) return;
  double av[KS], bv[KS];
  {
    const int m0 = (t / ntiles) * 8, n0 = (t % ntiles) * 8;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      av[ks] = fa(m0 + g, ks * 4 + q);
      bv[ks] = fb(ks * 4 + q, n0 + g);
    }
  }
  for (; t < ntot; t += nw) {
    const int m0 = (t / ntiles) * 8, n0 = (t % ntiles) * 8;
    const int tn = t + nw;
    double an[KS], bn[KS];
    if (tn < ntot) {
      const int m1 = (tn / ntiles) * 8, n1 = (tn % ntiles) * 8;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        an[ks] = fa(m1 + g, ks * 4 + q);
        bn[ks] = fb(ks * 4 + q, n1 + g);
      }
    }
    double c0 = 0.0, c1 = 0.0;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) dmma(c0, c1, av[ks], bv[ks]);
    fc(m0 + g, n0 + 2 * q, c0, c1);
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      av[ks] = an[ks];
      bv[ks] = bn[ks];
    }
  }
}

// The same with an accumulate-into-memory epilogue: fpre(m, n, p0, p1) loads the two
// existing values of the lane's outputs BEFORE the tile's DMMA chain (their latency
// overlaps the MMAs), fc(m, n, c_n + p0, c_{n+1} + p1) stores the sums.
template <int KS, class FA, class FB, class FP, class FC>
__device__ __forceinline__ void mma_tiles_acc(int mtiles, int ntiles, FA fa, FB fb, FP fpre, FC fc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  for (int t = warp; t < mtiles * ntiles; t += nw) {
    const int m0 = (t / ntiles) * 8, n0 = (t % ntiles) * 8;
    double p0 = 0.0, p1 = 0.0;
    fpre(m0 + g, n0 + 2 * q, p0, p1);
    double av[KS], bv[KS];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      av[ks] = fa(m0 + g, ks * 4 + q);
      bv[ks] = fb(ks * 4 + q, n0 + g);
    }
    double c0 = 0.0, c1 = 0.0;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) dmma(c0, c1, av[ks], bv[ks]);
    fc(m0 + g, n0 + 2 * q, c0 + p0, c1 + p1);
  }
}

// Register-blocked forms for a contraction with one SMALL operand (the 1D transform
// matrix): its fragments stay in registers, so a tile costs KS loads of the large
// operand instead of 2 KS (mma_tiles reloads both per 8x8 tile).
//   mma_sweep_n: A = the small operand (MT m-tiles, all kept), B swept over n-tiles;
//   mma_sweep_m: B = the small operand (NTL n-tiles, all kept), A swept over m-tiles,
//                the next tile's A loaded during the DMMA chain (A may come from global).
template <int KS, int MT, class FA, class FB, class FC>
__device__ __forceinline__ void mma_sweep_n(int ntiles, FA fa, FB fb, FC fc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  double av[MT][KS];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) av[mt][ks] = fa(mt * 8 + g, ks * 4 + q);
  for (int t = warp; t < ntiles; t += nw) {
    const int n0 = t * 8;
    double bv[KS];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) bv[ks] = fb(ks * 4 + q, n0 + g);
    double c[MT][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) c[mt][0] = c[mt][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) dmma(c[mt][0], c[mt][1], av[mt][ks], bv[ks]);
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) fc(mt * 8 + g, n0 + 2 * q, c[mt][0], c[mt][1]);
  }
}
template <int KS, int NTL, class FA, class FB, class FC>
__device__ __forceinline__ void mma_sweep_m(int mtiles, FA fa, FB fb, FC fc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  double bv[NTL][KS];
#pragma unroll
  for (int nt = 0; nt < NTL; ++nt)
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) bv[nt][ks] = fb(ks * 4 + q, nt * 8 + g);
  int t = warp;
  if (t >= mtiles) return;
  double av[KS];
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) av[ks] = fa(t * 8 + g, ks * 4 + q);
  for (; t < mtiles; t += nw) {
    double an[KS];
    if (t + nw < mtiles) {
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) an[ks] = fa((t + nw) * 8 + g, ks * 4 + q);
    }
    double c[NTL][2];
#pragma unroll
    for (int nt = 0; nt < NTL; ++nt) c[nt][0] = c[nt][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
      for (int nt = 0; nt < NTL; ++nt) dmma(c[nt][0], c[nt][1], av[ks], bv[nt][ks]);
#pragma unroll
    for (int nt = 0; nt < NTL; ++nt) fc(t * 8 + g, nt * 8 + 2 * q, c[nt][0], c[nt][1]);
    if (t + nw < mtiles) {
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) av[ks] = an[ks];
    }
  }
}

// collect the point ranges a box works on:
//   ANTERP: leaf children with points (F_out box)
//   EVAL:   own points if the box is a leaf, else leaf children without F_in
template <bool EVAL, int NCH = 8>
__device__ int box_ranges(const DevTree& t, int b, int2* rg) {
  int nr = 0;
  uint8_t f = t.flags[b];
  if (EVAL && (f & F_LEAF)) {
    rg[nr++] = make_int2(t.start[b], t.end[b]);
    return nr;
  }
  for (int o = 0; o < NCH; ++o) {
    int ch = t.child[NCH * (int64_t)b + o];
    if (ch < 0) continue;
    uint8_t fc = t.flags[ch];
    if (!(fc & F_LEAF) || t.end[ch] <= t.start[ch]) continue;
    if (EVAL && ((fc & F_IN) || !(fc & F_TGT))) continue;
    rg[nr++] = make_int2(t.start[ch], t.end[ch]);
  }
  return nr;
}
// the same ranges collected by one warp (lanes 0..NCH-1 examine one child each, in
// parallel: one round of dependent loads instead of NCH), in child order; also writes
// the number of ranges and the total point count.  Call with all 32 lanes of a warp.
template <bool EVAL, int NCH = 8>
__device__ __forceinline__ void box_ranges_w(const DevTree& t, int b, int2* rg, int& nr_out, int& tot_out) {
  const int lane = threadIdx.x & 31;
  const uint8_t f = t.flags[b];
  if (EVAL && (f & F_LEAF)) {
    if (lane == 0) {
      rg[0] = make_int2(t.start[b], t.end[b]);
      nr_out = 1;
      tot_out = t.end[b] - t.start[b];
    }
    return;
  }
  bool keep = false;
  int2 r = make_int2(0, 0);
  if (lane < NCH) {
    const int ch = t.child[NCH * (int64_t)b + lane];
    if (ch >= 0) {
      const uint8_t fc = t.flags[ch];
      r = make_int2(t.start[ch], t.end[ch]);
      keep = (fc & F_LEAF) && r.y > r.x;
      if (EVAL && ((fc & F_IN) || !(fc & F_TGT))) keep = false;
    }
  }
  const unsigned m = __ballot_sync(0xffffffffu, keep);
  if (keep) rg[__popc(m & ((1u << lane) - 1))] = r;
  int len = keep ? r.y - r.x : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) len += __shfl_xor_sync(0xffffffffu, len, o);
  if (lane == 0) {
    nr_out = __popc(m);
    tot_out = len;
  }
}
__device__ __forceinline__ int range_point(const int2* rg, int nr, int idx) {
  for (int r = 0; r < nr; ++r) {
    int len = rg[r].y - rg[r].x;
    if (idx < len) return rg[r].x + idx;
    idx -= len;
  }
  return -1;
}

// ---------------------------------------------------------------- host helpers
static inline DevTree dev_tree(const dmk_plan_s* P) {
  return DevTree{P->box_code.p, P->box_level.p, P->box_start.p, P->box_end.p, P->box_parent.p,
                 P->box_child.p, P->box_coll.p, P->box_flags.p, P->fout_rank.p, P->exp_rank.p,
                 P->xs.p,        P->ys.p,      P->zs.p};
}

template <class Kern>
static inline void set_smem(Kern k, size_t bytes) {
  // always set: dynamic + static shared memory above 48 KB needs the opt-in
  DMK_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

// Phase timing (DMK_PROFILE=1): CUDA events recorded on the plan stream around each
// phase, no host synchronisation; resolved when dmk_eval_timings() is called.
struct Timer {
  dmk_plan_s* P;
  Timer(dmk_plan_s* p) : P(p) {}
  cudaEvent_t ev() {
    if (P->ev_used == P->ev_pool.size()) {
      cudaEvent_t e;
      DMK_CUDA(cudaEventCreate(&e));
      P->ev_pool.push_back(e);
    }
    return P->ev_pool[P->ev_used++];
  }
  void begin(const char* nm, cudaStream_t st = nullptr) {
    if (!P->profile) return;
    cudaEvent_t e = ev();
    DMK_CUDA(cudaEventRecord(e, st ? st : P->stream));
    P->ev_marks.push_back({nm, e, nullptr});
  }
  void end(cudaStream_t st = nullptr) {
    if (!P->profile) return;
    cudaEvent_t e = ev();
    DMK_CUDA(cudaEventRecord(e, st ? st : P->stream));
    P->ev_marks.back().e1 = e;
  }
};

}  // namespace dmk
