// QR tile kernels for sm_100a: GEQRT, UNMQR, TSQRT, TSMQR (reference kinds
// kernels.py:34-38, access lists kernels.py:192-211).  Semantics are LAPACK's
// dgeqrt / dgemqrt / dtpqrt(l=0) / dtpmqrt(l=0) with block size ib (dlarfg
// sign convention; T factors ib x nb in the tile's side area, panel p at
// columns [p*ib, p*ib+sb), upper triangular, zeros below the diagonal).
//
//  k_qr_panel -- Householder factorization of one ib-wide panel by an
//                8-CTA CLUSTER holding the panel rows in shared memory (CTA q
//                owns rows [q*nb/8, (q+1)*nb/8)).  Per column: barrier 1
//                publishes the partial squared norms (and alpha), every CTA
//                forms the reflector identically (dlarfg); barrier 2
//                publishes the partial products x^T [V | A] that give both
//                the column update w and the T-factor inner products y.  The
//                T factor is finished by CTA 0 from y and tau.
//  k_qr_apply -- applies panels [p0, p1) to a column strip:
//                  W = V^T C (UNMQR) or W = top + V_B^T bot (TSMQR),
//                  W <- T^T W,  C -= V W  (resp. top -= W, bot -= V_B W),
//                with W resident in shared memory and the masked unit-lower
//                V blocks loaded element-wise on the diagonal slabs.
#include <cooperative_groups.h>
#include <cstdlib>

#include "dgemm_dmma.cuh"
#include "tiles.h"

namespace cg = cooperative_groups;

namespace hg {

constexpr int kQrCl = 8;
constexpr int kQrThreads = 256;
constexpr int kQrMaxSb = 128;

enum { QR_GEQRT = 0, QR_TSQRT = 1 };

struct QrPanelParams {
  double* A;     // GEQRT: A_kk; TSQRT: A_ik (the B part)
  double* R;     // TSQRT: A_kk (R rows); GEQRT: unused
  double* side;  // side area of A: T factors (ib x nb)
  int nb, ib, ii, sb, mode;
};

// T (ib x sb block at T, ld ib, upper triangular) from y = striu(V^T V) stored above
// its diagonal and tau on it, by the compact-WY identity, in ONE CTA (any size).
__device__ void qr_t_from_y(double* T, int ib, int sb, double* s) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nthr = blockDim.x, nwarp = nthr / 32;
  // T from y and tau by the compact-WY identity T^{-1} = diag(1/tau) + striu(V^T V)
  // (y(k, j) = V_k^T v_j is exactly striu(V^T V)), inverted by 16x16 blocks in
  // order of block distance.  Packed smem: U (strict upper, row-major), T
  // stored transposed in the strict lower part, tau on the side.
  const int LS = sb + 1;
  double* S = s;                 // S[r*LS + c]
  double* tv = s + sb * LS;      // tau[sb]
  double* Wb = tv + sb;          // work blocks: up to 7 x 256
  for (int e = tid; e < sb * sb; e += nthr) {
    int jc = e / sb, k = e % sb;  // T area column jc, row k
    double v = __ldcg(T + size_t(jc) * ib + k);
    if (k < jc) S[k * LS + jc] = v;        // U(k, jc) = y
    else if (k == jc) tv[k] = v;           // tau
  }
  __syncthreads();
  auto Uat = [&](int r, int c) { return S[r * LS + c]; };                        // r < c
  auto Tat = [&](int r, int c) { return r == c ? tv[r] : S[c * LS + r]; };       // r <= c
  const int nbk = sb / 16;
  // level 0: diagonal blocks, one warp each, lane i = column i (back substitution)
  for (int blk = warp; blk < nbk; blk += nwarp) {
    if (lane >= 16) continue;
    const int a0 = blk * 16, i = lane;
    double tcol[16];
#pragma unroll
    for (int r = 15; r >= 0; --r) {
      double v = 0.0;
      if (r == i) v = tv[a0 + i];
      else if (r < i) {
        double acc = 0.0;
#pragma unroll
        for (int m = r + 1; m < 16; ++m)
          if (m <= i) acc = fma(Uat(a0 + r, a0 + m), tcol[m], acc);
        v = -tv[a0 + r] * acc;
      }
      tcol[r] = v;
    }
#pragma unroll
    for (int r = 0; r < 16; ++r)
      if (r < i) S[(a0 + i) * LS + a0 + r] = tcol[r];
  }
  __syncthreads();
  for (int d = 1; d < nbk; ++d) {
    const int nblk = nbk - d;
    // W_ab = sum_{c=a+1}^{b} U_ac T_cb
    for (int e = tid; e < nblk * 256; e += nthr) {
      const int a = e / 256, b = a + d, i = (e % 256) / 16, j = e % 16;
      const int r0 = a * 16 + i, c0 = b * 16 + j;
      double acc = 0.0;
      for (int m = (a + 1) * 16; m <= c0; ++m) acc = fma(Uat(r0, m), Tat(m, c0), acc);
      Wb[e] = acc;
    }
    __syncthreads();
    // T_ab = -T_aa W_ab
    for (int e = tid; e < nblk * 256; e += nthr) {
      const int a = e / 256, b = a + d, i = (e % 256) / 16, j = e % 16;
      const int r0 = a * 16 + i, c0 = b * 16 + j;
      double acc = 0.0;
      for (int m = i; m < 16; ++m) acc = fma(Tat(r0, a * 16 + m), Wb[a * 256 + m * 16 + j], acc);
      S[c0 * LS + r0] = -acc;
    }
    __syncthreads();
  }
  for (int e = tid; e < sb * sb; e += nthr) {
    int jc = e / sb, k = e % sb;
    T[size_t(jc) * ib + k] = k <= jc ? Tat(k, jc) : 0.0;
  }
}

__global__ void __cluster_dims__(kQrCl, 1, 1) __launch_bounds__(kQrThreads) k_qr_panel(QrPanelParams p) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int q = (int)cl.block_rank();
  const int nb = p.nb, sb = p.sb, ii = p.ii, ib = p.ib;
  const int R = nb / kQrCl;
  const int row0 = q * R;
  const int LD = R + 1;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool ts = p.mode == QR_TSQRT;
  double* s = sm;                          // s[c*LD + r]
  double* pw = s + sb * LD;                // [2][sb] partial x^T [V | A]
  double* rrow = pw + 2 * kQrMaxSb;        // [2][sb] TSQRT: R row j
  double* wv = rrow + 2 * kQrMaxSb;        // [sb] reduced w / y
  double* slot = wv + kQrMaxSb;            // [2][2]: partial norm^2, alpha (owner of row j)
  double* vv = slot + 4;                   // [R]  reflector entries of my rows for column jj
  double* ph = vv + kQrMaxSb;              // [2][sb] half-row partial sums
  __shared__ double s_red[kQrThreads / 32];
  __shared__ double s_tau, s_beta, s_scal;
  double* T = p.side + size_t(ii) * ib;    // this panel's ib x sb T block (ld = ib)
  double* A = p.A;

  for (int e = tid; e < sb * R; e += kQrThreads) {
    int c = e / R, r = e % R;
    int gr = row0 + r;
    s[c * LD + r] = (ts || gr >= ii) ? A[size_t(ii + c) * nb + gr] : 0.0;
  }
  __syncthreads();

  // partial ||x||^2 of column jj over my rows strictly below the diagonal row
  auto publish_norm = [&](int jj, int par) {
    const int j = ii + jj;
    double acc = 0.0;
    for (int r = tid; r < R; r += kQrThreads) {
      int gr = row0 + r;
      if (ts || gr > j) {
        double v = s[jj * LD + r];
        acc = fma(v, v, acc);
      }
    }
    acc = warp_sum(acc);
    if (lane == 0) s_red[warp] = acc;
    if (ts)
      for (int c = tid; c < sb; c += kQrThreads) rrow[par * kQrMaxSb + c] = c >= jj ? p.R[size_t(ii + c) * nb + j] : 0.0;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < kQrThreads / 32; ++w) t += s_red[w];
      slot[par * 2 + 0] = t;
      slot[par * 2 + 1] = (!ts && j >= row0 && j < row0 + R) ? s[jj * LD + (j - row0)] : 0.0;
    }
  };

  publish_norm(0, 0);
  for (int jj = 0; jj < sb; ++jj) {
    const int j = ii + jj;
    const int par = jj & 1;
    cl.sync();  // barrier 1: norms + alpha of column jj
    if (tid < 32) {
      double xn2 = 0.0, al = 0.0;
      if (tid < kQrCl) {
        const double* sl = cl.map_shared_rank(slot, tid) + par * 2;
        xn2 = sl[0];
        al = sl[1];  // only the owner of row j publishes a non-zero alpha
      }
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) {
        xn2 += __shfl_xor_sync(0xffffffffu, xn2, o);
        al += __shfl_xor_sync(0xffffffffu, al, o);
      }
      if (tid == 0) {
        double alpha = ts ? rrow[par * kQrMaxSb + jj] : al;
        double tau = 0.0, beta = alpha, scal = 1.0;
        if (xn2 != 0.0) {
          const double xnorm = sqrt(xn2);
          beta = -copysign(hypot(alpha, xnorm), alpha);
          tau = (beta - alpha) / beta;
          scal = 1.0 / (alpha - beta);
        }
        s_tau = tau;
        s_beta = beta;
        s_scal = scal;
      }
    }
    __syncthreads();
    const double tau = s_tau, beta = s_beta, scal = s_scal;
    // scale my part of x (the owner of row j stores beta) and stage v for the products
    for (int r = tid; r < R; r += kQrThreads) {
      int gr = row0 + r;
      double v = 0.0;
      if (ts || gr > j) {
        v = s[jj * LD + r] * scal;
        s[jj * LD + r] = v;
      } else if (gr == j) {
        s[jj * LD + r] = beta;
        v = 1.0;
      }
      vv[r] = v;
    }
    __syncthreads();
    // partial products x^T [V | A]: two threads per panel column, each half of my rows.
    // Left columns need no unit/zero mask: v_r != 0 only for rows >= j > ii + c.
    {
      const int c = tid % kQrMaxSb, half = tid / kQrMaxSb;
      if (c < sb) {
        const int rb = half * (R / 2), re = rb + R / 2;
        double acc[4] = {0.0, 0.0, 0.0, 0.0};  // 4 independent chains (FMA latency)
        if (c != jj) {
          const double* sc = s + c * LD;
          for (int r = rb; r < re; r += 4) {
#pragma unroll
            for (int u = 0; u < 4; ++u) acc[u] = fma(vv[r + u], sc[r + u], acc[u]);
          }
        }
        ph[half * kQrMaxSb + c] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
      }
    }
    __syncthreads();
    for (int c = tid; c < sb; c += kQrThreads) pw[par * kQrMaxSb + c] = ph[c] + ph[kQrMaxSb + c];
    cl.sync();  // barrier 2: partial products
    for (int c = tid; c < sb; c += kQrThreads) {
      double t = 0.0;
      if (c != jj) {
        double part[kQrCl];
#pragma unroll
        for (int c2 = 0; c2 < kQrCl; ++c2) part[c2] = cl.map_shared_rank(pw, c2)[par * kQrMaxSb + c];
#pragma unroll
        for (int c2 = 0; c2 < kQrCl; ++c2) t += part[c2];
      }
      if (ts && c > jj) t += rrow[par * kQrMaxSb + c];  // the unit of v_j sits in R row j
      wv[c] = t;
    }
    __syncthreads();
    // T column jj (y above the diagonal, tau on it) and the R row (TSQRT)
    if (q == 0) {
      for (int c = tid; c < ib; c += kQrThreads) T[size_t(jj) * ib + c] = c < jj ? wv[c] : (c == jj ? tau : 0.0);
      if (ts)
        for (int c = jj + tid; c < sb; c += kQrThreads)
          p.R[size_t(ii + c) * nb + j] = (c == jj) ? beta : rrow[par * kQrMaxSb + c] - tau * wv[c];
    }
    // apply H_j to columns (jj, sb) of my rows
    {
      const int ngroup = kQrThreads / R;
      const int r = tid % R, grp = tid / R;
      const int gr = row0 + r;
      if (grp < ngroup && tau != 0.0) {
        double v;
        if (ts || gr > j) v = s[jj * LD + r];
        else if (gr == j) v = 1.0;
        else v = 0.0;
        if (v != 0.0) {
          const double tv = tau * v;
          int c = jj + 1 + grp;
          // 8 independent read-modify-writes in flight (a plain loop serialises each
          // shared-memory store before the next load)
          for (; c + 7 * ngroup < sb; c += 8 * ngroup) {
            double x[8], w8[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              x[u] = s[(c + u * ngroup) * LD + r];
              w8[u] = wv[c + u * ngroup];
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) s[(c + u * ngroup) * LD + r] = fma(-tv, w8[u], x[u]);
          }
          for (; c < sb; c += ngroup) s[c * LD + r] = fma(-tv, wv[c], s[c * LD + r]);
        }
      }
    }
    __syncthreads();
    if (jj + 1 < sb) publish_norm(jj + 1, par ^ 1);
  }
  __syncthreads();
  for (int e = tid; e < sb * R; e += kQrThreads) {
    int c = e / R, r = e % R;
    int gr = row0 + r;
    if (ts || gr >= ii) A[size_t(ii + c) * nb + gr] = s[c * LD + r];
  }
  __threadfence();
  cl.sync();
  if (q != 0) return;
  qr_t_from_y(T, ib, sb, s);
}

// ---------------------------------------------------------------------------
using CfgQ64 = GemmCfg<128, 64, 16, 32, 32, 3>;  // 8 warps; requires sb == 128
using CfgQ32 = GemmCfg<128, 32, 16, 32, 16, 3>;  // 8 warps (32x16 warp tiles)
using CfgQ16 = GemmCfg<128, 16, 16, 32, 16, 3>;  // 4 warps
using CfgQ4w = GemmCfg<128, 32, 8, 32, 32, 4>;    // 4 warps of 32x32: C -= V W stream (3 CTAs / SM)
using CfgQ4w1 = GemmCfg<128, 32, 8, 32, 32, 3, true>;  //   and its W = V^T C / T^T W phases (swizzled K_MAJOR ring)
constexpr int kWld = kQrMaxSb + 4;  // W stored [n][k]

// Unit-lower reflector block V of panel ii, element (tile row tr, panel col pc):
//   tr > ii + pc: stored value, tr == ii + pc: 1, tr < ii + pc: 0.
// L = K_MAJOR: operand rows = pc (r0 + rr), k = tr   (used for V^T)
// L = M_MAJOR: operand rows = tr (r0 + rr), k = pc   (used for V)
template <class Cfg, int L, int ROWS>
struct VLoader {
  static constexpr int layout = L;
  static constexpr int rows = ROWS;
  const double* v;  // tile + ii*nb: V(tr, pc) at v[pc*ld + tr]
  int ld, r0, ii, masked;
  HG_DEVICE double val(int tr, int pc) const {
    if (!masked || tr > ii + pc) return v[size_t(pc) * ld + tr];
    return tr == ii + pc ? 1.0 : 0.0;
  }
  HG_DEVICE void load(double* s, int k0) const {
    constexpr int BK = Cfg::BK, PAD = Cfg::PAD;
    bool diag;
    if (L == K_MAJOR) diag = masked && k0 < ii + ROWS + r0 && k0 + BK > ii + r0;  // tr window vs ii+pc
    else diag = masked && r0 < ii + k0 + BK && r0 + ROWS > ii + k0;
    if (!diag) {
      if (L == K_MAJOR) load_slab<Cfg, K_MAJOR, ROWS>(s, v, ld, r0, k0);  // element (pc, tr) at v[pc*ld + tr]
      else load_slab<Cfg, M_MAJOR, ROWS>(s, v, ld, r0, k0);               // element (tr, pc) at v[pc*ld + tr]
      return;
    }
    for (int e = threadIdx.x; e < ROWS * BK; e += Cfg::THREADS) {
      int rr = e / BK, kk = e % BK;
      if (L == K_MAJOR) s[Cfg::kmaj(rr, kk)] = val(k0 + kk, r0 + rr);
      else s[kk * (ROWS + PAD) + rr] = val(r0 + rr, k0 + kk);
    }
  }
};

struct QrApplyParams {
  const double* V;     // factor tile (GEQRT: A_kk; TSQRT: A_ik)
  const double* side;  // its side area (T factors)
  double* top;         // UNMQR: the tile C (rows [ii, nb)); TSMQR: A_kj (rows [ii, ii+sb))
  double* bot;         // TSMQR: A_ij; UNMQR: unused
  int nb, ib, p0, p1, col0, mode;
};

// Column-strip variant: one CTA per BN-column strip (no cluster, all rows),
// BN in {16, 32, 64}: narrower strips = more SMs per task (latency), wider =
// more reuse of V per SM (throughput inside the DAG).
// RED: C -= V W as L2 reductions (red.global.add.f64 of -acc); the next panel
// reads C only through cp.async.cg (L2), after the fence in the update loop.
// C1: the configuration of the two K_MAJOR x K_MAJOR phases (W = V^T C, W = T^T W);
// a shallower ring there lets the 4-warp variant fit 3 CTAs per SM.
template <class CfgQ, class C1>
__host__ __device__ constexpr int qr_ring_doubles() {
  constexpr int a = GemmSmem<C1, K_MAJOR, K_MAJOR>::DOUBLES;
  constexpr int b = CfgQ::STAGES * CfgQ::slab_mmaj(CfgQ::BM);
  return a > b ? a : b;
}

template <class CfgQ, bool RED = false, class C1 = CfgQ>
__global__ void __launch_bounds__(CfgQ::THREADS, CfgQ::THREADS == 128 ? 3 : 2) k_qr_apply(QrApplyParams p) {
  static_assert(C1::THREADS == CfgQ::THREADS && C1::BN == CfgQ::BN && C1::BM == CfgQ::BM, "phase config");
  constexpr int kQrBN = CfgQ::BN;
  extern __shared__ double sm[];
  double* ring = sm;
  double* W = sm + qr_ring_doubles<CfgQ, C1>();  // [n][k], ld kWld
  const int nb = p.nb, ib = p.ib;
  const int n0 = p.col0 + blockIdx.x * kQrBN;
  const bool ts = p.mode == QR_TSQRT;
  for (int P = p.p0; P < p.p1; ++P) {
    const int ii = P * ib;
    const double* Vp = p.V + size_t(ii) * nb;  // V(tr, pc) at Vp[pc*nb + tr]
    // ---- W = V^T C   (UNMQR, K over tile rows [ii, nb))  |  top + V_B^T bot (TSMQR)
    {
      double acc[C1::FM][C1::FN][2];
      zero_acc<C1>(acc);
      if (ts) {
        VLoader<C1, K_MAJOR, 128> la{Vp, nb, 0, ii, 0};
        TileLoader<C1, K_MAJOR, kQrBN> lb{p.bot, nb, n0};
        gemm_mainloop<C1>(acc, ring, la, lb, 0, nb);
      } else {
        VLoader<C1, K_MAJOR, 128> la{Vp, nb, 0, ii, 1};
        TileLoader<C1, K_MAJOR, kQrBN> lb{p.top, nb, n0};
        gemm_mainloop<C1>(acc, ring, la, lb, ii, nb);
      }
      if (ts) {  // W = top + V_B^T bot: top loads batched, not one L2 round trip per element
        double tv[C1::FM][C1::FN][2];
        load_like_acc<C1>(tv, p.top + ii, nb, 0, n0);
#pragma unroll
        for (int i = 0; i < C1::FM; ++i)
#pragma unroll
          for (int j = 0; j < C1::FN; ++j) {
            acc[i][j][0] += tv[i][j][0];
            acc[i][j][1] += tv[i][j][1];
          }
      }
      for_each_acc<C1>(acc, [&](int r, int c, double v) { W[c * kWld + r] = v; });
    }
    __syncthreads();
    // ---- W <- T^T W  (T^T(r, k) = T(k, r) at side[(ii + r)*ib + k])
    {
      double acc[C1::FM][C1::FN][2];
      zero_acc<C1>(acc);
      TileLoader<C1, K_MAJOR, 128> la{p.side + size_t(ii) * ib, ib, 0};
      gemm_mainloop_bsmem<C1, decltype(la), true>(acc, ring, la, W, kWld, 0, 128);  // T^T lower
      for_each_acc<C1>(acc, [&](int r, int c, double v) { W[c * kWld + r] = v; });
      if (ts) sub_store<C1>(acc, p.top + ii, nb, 0, n0);  // top -= W (all loads first)
    }
    __syncthreads();
    // ---- C -= V W  (UNMQR rows [ii, nb))  |  bot -= V_B W (TSMQR)
    {
      VLoader<CfgQ, M_MAJOR, 128> la{Vp, nb, 0, ii, ts ? 0 : 1};
      gemm_sub_chunks_bsmem<CfgQ, decltype(la), false, 128, RED>(ring, la, W, kWld, 128, ts ? 0 : ii, nb,
                                                                  ts ? p.bot : p.top, nb, n0);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// k_qr_apply_cl -- the same block-reflector application with the tile ROWS
// split over a 4-CTA cluster, so one TSMQR / UNMQR (or a GEQRT / TSQRT
// trailing update) spreads over (N/32) x 4 SMs instead of N/64:
//   CTA q owns rows [q*nb/4, (q+1)*nb/4) of C (UNMQR) / bot (TSMQR) and a
//   32-column strip.  Per panel:
//     1. W_q = V[rows_q]^T C[rows_q]            (DMMA, split-K partial)
//     2. cluster barrier; CTA q reduces W rows [32q, 32q+32) over DSMEM
//        (+ top rows for TSMQR)
//     3. cluster barrier; every CTA gathers W rows 0..32q+31, forms its
//        slice of W' = T^T W (T upper triangular)
//     4. cluster barrier; every CTA gathers W' (TSMQR: CTA q also applies
//        top -= W' to its slice of the top rows)
//     5. C[rows_q] -= V[rows_q] W'             (DMMA, W' resident in smem)
// Partial / slice buffers alternate by panel parity, so a fast CTA writing
// panel P+1's partials never overwrites a slice a slow CTA still gathers.
constexpr int kQcCl = 4;
constexpr int kQcBN = 32;
using CfgQC = GemmCfg<128, kQcBN, 16, 32, 16, 3>;  // 8 warps, 32x16 warp tiles
constexpr int kQcSlice = kQrMaxSb / kQcCl;          // W rows reduced per CTA

__global__ void __cluster_dims__(kQcCl, 1, 1) __launch_bounds__(CfgQC::THREADS) k_qr_apply_cl(QrApplyParams p) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int q = (int)cl.block_rank();
  constexpr int RING = GemmSmem<CfgQC, K_MAJOR, K_MAJOR>::DOUBLES;
  constexpr int WBUF = kQcBN * kWld;
  double* ring = sm;
  double* Wp = sm + RING;             // [2][WBUF]: partials, then W' slices (by panel parity)
  double* Ws = Wp + 2 * WBUF;         // reduced W slice + gathered W, then gathered W'
  const int nb = p.nb, ib = p.ib;
  const int n0 = p.col0 + (blockIdx.x / kQcCl) * kQcBN;
  const int rows = nb / kQcCl;
  const int r_begin = q * rows, r_end = r_begin + rows;
  const bool ts = p.mode == QR_TSQRT;
  const int tid = threadIdx.x;
  for (int P = p.p0; P < p.p1; ++P) {
    const int ii = P * ib;
    const double* Vp = p.V + size_t(ii) * nb;
    double* C = ts ? p.bot : p.top;
    double* wp = Wp + (P & 1) * WBUF;
    // rows of C this CTA touches in this panel (UNMQR: only tile rows >= ii)
    const int k0 = ts ? r_begin : max(r_begin, ii);
    // ---- 1. partial W_q --------------------------------------------------------
    {
      double acc[CfgQC::FM][CfgQC::FN][2];
      zero_acc<CfgQC>(acc);
      if (k0 < r_end) {
        VLoader<CfgQC, K_MAJOR, 128> la{Vp, nb, 0, ii, ts ? 0 : 1};
        TileLoader<CfgQC, K_MAJOR, kQcBN> lb{C, nb, n0};
        gemm_mainloop<CfgQC>(acc, ring, la, lb, k0, r_end);
      }
      for_each_acc<CfgQC>(acc, [&](int r, int c, double v) { wp[c * kWld + r] = v; });
    }
    cl.sync();
    // ---- 2. reduce my slice of W ------------------------------------------------
    const int s0 = q * kQcSlice;
    {
      const double* parts[kQcCl];
#pragma unroll
      for (int c2 = 0; c2 < kQcCl; ++c2) parts[c2] = cl.map_shared_rank(wp, c2);
      for (int e = tid; e < kQcSlice * kQcBN; e += CfgQC::THREADS) {
        const int c = e / kQcSlice, r = s0 + e % kQcSlice;
        double v[kQcCl];
#pragma unroll
        for (int c2 = 0; c2 < kQcCl; ++c2) v[c2] = parts[c2][c * kWld + r];
        double t = ts ? p.top[size_t(n0 + c) * nb + ii + r] : 0.0;
#pragma unroll
        for (int c2 = 0; c2 < kQcCl; ++c2) t += v[c2];
        Ws[c * kWld + r] = t;
      }
    }
    cl.sync();
    // ---- 3. gather W rows [0, s0) and form my slice of W' = T^T W -------------------
    for (int c2 = 0; c2 < q; ++c2) {
      const double* src = cl.map_shared_rank(Ws, c2);
      for (int e = tid; e < kQcSlice * kQcBN; e += CfgQC::THREADS) {
        const int c = e / kQcSlice, r = c2 * kQcSlice + e % kQcSlice;
        Ws[c * kWld + r] = src[c * kWld + r];
      }
    }
    __syncthreads();
    {
      const double* T = p.side + size_t(ii) * ib;  // T(k, r) at T[r*ib + k], upper triangular
      for (int e = tid; e < kQcSlice * kQcBN; e += CfgQC::THREADS) {
        const int c = e / kQcSlice, r = s0 + e % kQcSlice;
        const double* tc = T + size_t(r) * ib;
        const double* wc = Ws + c * kWld;
        double a0 = 0.0, a1 = 0.0;
        int k = 0;
        for (; k + 1 <= r; k += 2) {
          a0 = fma(__ldg(tc + k), wc[k], a0);
          a1 = fma(__ldg(tc + k + 1), wc[k + 1], a1);
        }
        if (k <= r) a0 = fma(__ldg(tc + k), wc[k], a0);
        wp[c * kWld + r] = a0 + a1;
      }
    }
    cl.sync();
    // ---- 4. gather W' ----------------------------------------------------------------
    for (int c2 = 0; c2 < kQcCl; ++c2) {
      const double* src = cl.map_shared_rank(wp, c2);
      for (int e = tid; e < kQcSlice * kQcBN; e += CfgQC::THREADS) {
        const int c = e / kQcSlice, r = c2 * kQcSlice + e % kQcSlice;
        Ws[c * kWld + r] = src[c * kWld + r];
      }
    }
    __syncthreads();
    if (ts)
      for (int e = tid; e < kQcSlice * kQcBN; e += CfgQC::THREADS) {
        const int c = e / kQcSlice, r = s0 + e % kQcSlice;
        p.top[size_t(n0 + c) * nb + ii + r] -= Ws[c * kWld + r];
      }
    // ---- 5. C[rows] -= V[rows] W' ------------------------------------------------------
    for (int m0 = k0; m0 < r_end; m0 += 128) {
      double acc[CfgQC::FM][CfgQC::FN][2];
      zero_acc<CfgQC>(acc);
      VLoader<CfgQC, M_MAJOR, 128> la{Vp, nb, m0, ii, ts ? 0 : 1};
      gemm_mainloop_bsmem<CfgQC>(acc, ring, la, Ws, kWld, 0, 128);
      sub_store<CfgQC>(acc, C, nb, m0, n0);
    }
    __syncthreads();
  }
  cl.sync();  // no CTA leaves while a peer may still read its W' slice
}

static unsigned qr_apply_cl_smem() {
  return unsigned((GemmSmem<CfgQC, K_MAJOR, K_MAJOR>::DOUBLES + 3 * kQcBN * kWld) * sizeof(double));
}

// ---------------------------------------------------------------------------
// k_qr_panel_sp -- the Householder panel (GEQRT / TSQRT semantics of
// k_qr_panel) blocked into W = 16-column sub-panels held in registers, one
// tile row per thread, 8-CTA cluster (CTA q owns rows [q*R, (q+1)*R)):
//   per column: ONE cluster barrier for the column norm (+ alpha), dlarfg in
//   every thread, ONE cluster barrier for w = v^T A over the <= 15 remaining
//   sub-panel columns, rank-1 update in registers;
//   per sub-panel: the block reflector I - V T V^T of its 16 columns is
//   applied to the panel's right-hand columns with DMMA partials
//   (W = V^T A_right, G = V^T V), a reduce-scatter / all-gather of W over
//   DSMEM, T_sub from G and tau, W' = T_sub^T W, A_right -= V W';
//   per panel: T = the compact-WY T factor of all 128 reflectors, from
//   striu(V^T V) (DMMA partial Gram matrices reduced over DSMEM) and tau.
// The per-column critical path touches 16 registers per row instead of the
// whole 128-column panel (k_qr_panel: ~4.7 us per column).
constexpr int kQsW = 16;
constexpr int kQsThreads = 128;
constexpr int kQsSB = 128;

template <int R>
struct QsSmem {
  static constexpr int LDP = R + 4;                    // panel [col][row] (+4: conflict-free DMMA frags)
  static constexpr int PS = kQsSB * LDP;
  static constexpr int WB = kQsW * (kQsSB + kQsW);     // partial W (| G) [v][col], 16 x (16 + 112)
  static constexpr int MISC = 4 + kQsW * kQsW + 2 * kQsW + kQsW * kQsW + kQsSB;  // slots, Rblk, wpart, Ts, taus
  static constexpr int DOUBLES = PS + 3 * WB + MISC;
  static constexpr int TFY = kQsSB * (kQsSB + 1) + kQsSB + 7 * 256;  // qr_t_from_y scratch
  static constexpr size_t BYTES = size_t(DOUBLES > TFY ? DOUBLES : TFY) * 8;
};

template <int R>
__global__ void __cluster_dims__(kQrCl, 1, 1) __launch_bounds__(kQsThreads) k_qr_panel_sp(QrPanelParams p) {
  constexpr int W = kQsW, SB = kQsSB;
  using S = QsSmem<R>;
  constexpr int LDP = S::LDP;
  constexpr int WLD = SB + W;  // row stride of the W buffers
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int q = (int)cl.block_rank();
  const int nb = p.nb, ii = p.ii, ib = p.ib;
  const int row0 = q * R;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool ts = p.mode == QR_TSQRT;
  const bool mine = tid < R;
  const int gr = row0 + tid;
  const bool live = mine && (ts || gr >= ii);
  double* Ps = sm;
  double* Wp = Ps + S::PS;             // partial [v][col]: W (cols 0..nR) | G (cols nR..nR+16)
  double* Wr = Wp + S::WB;             // reduced rows of this CTA / gathered W
  double* Wg = Wr + S::WB;             // gathered W' (after T_sub^T)
  double* slot = Wg + S::WB;           // [2][2] norm^2, alpha
  double* Rblk = slot + 4;             // [W][W] TSQRT: R rows of the sub-panel
  double* wpart = Rblk + W * W;        // [2][W]
  double* Ts = wpart + 2 * W;          // [W][W] T_sub, Ts[r*W + c]
  double* taus = Ts + W * W;           // [SB]
  __shared__ double red_n[kQsThreads / 32], red_a[kQsThreads / 32];
  __shared__ double red_w[kQsThreads / 32][kQsW];
  double* T = p.side + size_t(ii) * ib;  // this panel's T block (ib x sb, ld ib)
  double* A = p.A;

  for (int e = tid; e < SB * R; e += kQsThreads) {
    const int c = e / R, r = e % R;
    Ps[c * LDP + r] = (ts || row0 + r >= ii) ? A[size_t(ii + c) * nb + row0 + r] : 0.0;
  }
  __syncthreads();

  // V(row r of this CTA, panel column c): GEQRT masks the unit lower structure
  auto Vat = [&](int r, int c) -> double {
    const int g2 = row0 + r, jd = ii + c;
    if (ts) return Ps[c * LDP + r];
    return g2 > jd ? Ps[c * LDP + r] : (g2 == jd ? 1.0 : 0.0);
  };

  for (int c0 = 0; c0 < SB; c0 += W) {
    if (ts)
      for (int e = tid; e < W * W; e += kQsThreads) {
        const int u = e / W, v = e % W;
        Rblk[e] = v >= u ? __ldcg(p.R + size_t(ii + c0 + v) * nb + ii + c0 + u) : 0.0;
      }
    double a[W];
#pragma unroll
    for (int v = 0; v < W; ++v) a[v] = mine ? Ps[(c0 + v) * LDP + tid] : 0.0;
    __syncthreads();
#pragma unroll
    for (int u = 0; u < W; ++u) {
      const int jj = c0 + u, j = ii + jj, par = jj & 1;
      const bool below = live && (ts || gr > j);
      const bool isdiag = live && !ts && gr == j;
      // ---- 1: norm^2 below the diagonal and alpha -> cluster --------------------------
      {
        double n2 = below ? a[u] * a[u] : 0.0;
        double al = isdiag ? a[u] : 0.0;
        n2 = warp_sum(n2);
        al = warp_sum(al);
        if (lane == 0) {
          red_n[warp] = n2;
          red_a[warp] = al;
        }
        __syncthreads();
        if (tid == 0) {
          double t1 = 0.0, t2 = 0.0;
#pragma unroll
          for (int w2 = 0; w2 < kQsThreads / 32; ++w2) {
            t1 += red_n[w2];
            t2 += red_a[w2];
          }
          slot[par * 2] = t1;
          slot[par * 2 + 1] = t2;
        }
      }
      cl.sync();
      double xn2, alpha;
      {
        double v1 = 0.0, v2 = 0.0;
        if (lane < kQrCl) {
          const double* sl = cl.map_shared_rank(slot, lane) + par * 2;
          v1 = sl[0];
          v2 = sl[1];
        }
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) {
          v1 += __shfl_xor_sync(0xffffffffu, v1, o);
          v2 += __shfl_xor_sync(0xffffffffu, v2, o);
        }
        xn2 = __shfl_sync(0xffffffffu, v1, 0);
        alpha = ts ? Rblk[u * W + u] : __shfl_sync(0xffffffffu, v2, 0);
      }
      // ---- 2: dlarfg (every thread) ------------------------------------------------------
      double tau = 0.0, beta = alpha, scal = 1.0;
      if (xn2 != 0.0) {
        const double xnorm = sqrt(xn2);
        beta = -copysign(hypot(alpha, xnorm), alpha);
        tau = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      double v = 0.0;
      if (below) {
        v = a[u] * scal;
        a[u] = v;
      } else if (isdiag) {
        v = 1.0;
        a[u] = beta;
      }
      if (tid == 0) taus[jj] = tau;
      // ---- 3: w = v^T A(:, u+1..W) -> cluster -------------------------------------------
#pragma unroll
      for (int v2 = u + 1; v2 < W; ++v2) {
        const double pw = warp_sum(v * a[v2]);
        if (lane == 0) red_w[warp][v2] = pw;
      }
      __syncthreads();
      if (tid < W && tid > u) {
        double t1 = 0.0;
#pragma unroll
        for (int w2 = 0; w2 < kQsThreads / 32; ++w2) t1 += red_w[w2][tid];
        wpart[par * W + tid] = t1;
      }
      cl.sync();
      double wl = 0.0;  // lane l (< W) of every warp: w[l] summed over the cluster
      if (lane < W && lane > u) {
        double pt[kQrCl];
#pragma unroll
        for (int c2 = 0; c2 < kQrCl; ++c2) pt[c2] = cl.map_shared_rank(wpart, c2)[par * W + lane];
#pragma unroll
        for (int c2 = 0; c2 < kQrCl; ++c2) wl += pt[c2];
        if (ts) wl += Rblk[u * W + lane];  // the unit of v_j sits in R row j
      }
      // ---- 4: rank-1 update of the sub-panel; TSQRT: R row j ----------------------------
#pragma unroll
      for (int v2 = u + 1; v2 < W; ++v2) {
        const double w = __shfl_sync(0xffffffffu, wl, v2);
        a[v2] = fma(-tau * v, w, a[v2]);
        if (ts && q == 0 && tid == v2) p.R[size_t(ii + c0 + v2) * nb + j] = Rblk[u * W + v2] - tau * w;
      }
      if (ts && q == 0 && tid == 0) p.R[size_t(ii + jj) * nb + j] = beta;
    }
    if (mine) {
#pragma unroll
      for (int v = 0; v < W; ++v) Ps[(c0 + v) * LDP + tid] = a[v];
    }
    __syncthreads();
    // ---- sub-panel block reflector on the right-hand columns ------------------------------------
    const int cR = c0 + W, nR = SB - cR;
    if (nR == 0) break;
    // partial W = V^T A_right (16 x nR) and G = V^T V (16 x 16), DMMA over my R rows
    {
      const int ntile = 2 * ((nR + W) / 8);
      for (int w = warp; w < ntile; w += kQsThreads / 32) {
        const int ti = w & 1, tj = w >> 1;            // row tile (reflector), column tile
        const int colt = tj * 8;                       // 0..nR+16 (last two tiles: G)
        double d0 = 0.0, d1 = 0.0;
        const int g = lane >> 2, t = lane & 3;
        for (int k0 = 0; k0 < R; k0 += 4) {
          const double av = Vat(k0 + t, c0 + ti * 8 + g);
          const int cc = colt + g;
          const double bv = cc < nR ? Ps[(cR + cc) * LDP + k0 + t] : Vat(k0 + t, c0 + cc - nR);
          dmma_8x8x4(d0, d1, av, bv);
        }
        Wp[(ti * 8 + g) * WLD + colt + 2 * t] = d0;
        Wp[(ti * 8 + g) * WLD + colt + 2 * t + 1] = d1;
      }
    }
    cl.sync();
    // reduce-scatter: CTA q owns rows v in {2q, 2q+1}; TSQRT adds the R rows (top) to W
    {
      const int ncol = nR + W;
      for (int e = tid; e < 2 * ncol; e += kQsThreads) {
        const int v = 2 * q + e / ncol, c = e % ncol;
        double pt[kQrCl];
#pragma unroll
        for (int c2 = 0; c2 < kQrCl; ++c2) pt[c2] = cl.map_shared_rank(Wp, c2)[v * WLD + c];
        double t1 = 0.0;
#pragma unroll
        for (int c2 = 0; c2 < kQrCl; ++c2) t1 += pt[c2];
        if (ts && c < nR) t1 += __ldcg(p.R + size_t(ii + cR + c) * nb + ii + c0 + v);
        Wr[v * WLD + c] = t1;
      }
    }
    cl.sync();
    // all-gather the 16 rows
    {
      const int ncol = nR + W;
      for (int e = tid; e < W * ncol; e += kQsThreads) {
        const int v = e / ncol, c = e % ncol;
        if (v / 2 != q) Wr[v * WLD + c] = cl.map_shared_rank(Wr, v / 2)[v * WLD + c];
      }
    }
    __syncthreads();
    // T_sub from G (Wr[.][nR + .]) and tau: T(k,k) = tau_k, T(0:k, k) = -tau_k T(0:k, 0:k) G(0:k, k)
    if (warp == 0) {
      const int i = lane;
      double trow[W];
#pragma unroll
      for (int k = 0; k < W; ++k) trow[k] = 0.0;
#pragma unroll
      for (int k = 0; k < W; ++k) {
        const double tk = taus[c0 + k];
        double acc = 0.0;
#pragma unroll
        for (int m = 0; m < k; ++m)
          if (m >= i) acc = fma(trow[m], Wr[m * WLD + nR + k], acc);
        if (i < k) trow[k] = -tk * acc;
        else if (i == k) trow[k] = tk;
      }
      if (i < W) {
#pragma unroll
        for (int k = 0; k < W; ++k) Ts[i * W + k] = trow[k];
      }
    }
    __syncthreads();
    // W' = T_sub^T W: W'(i, c) = sum_{m <= i} T(m, i) W(m, c)
    for (int c = tid; c < nR; c += kQsThreads) {
      double wc[W];
#pragma unroll
      for (int m = 0; m < W; ++m) wc[m] = Wr[m * WLD + c];
#pragma unroll
      for (int i = 0; i < W; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int m = 0; m <= i; ++m) acc = fma(Ts[m * W + i], wc[m], acc);
        Wg[i * WLD + c] = acc;
        if (ts && q == 0) {  // R rows of the sub-panel: top -= W'
          double* rp = p.R + size_t(ii + cR + c) * nb + ii + c0 + i;
          *rp = __ldcg(rp) - acc;
        }
      }
    }
    __syncthreads();
    // A_right -= V W'  (my row: V(r, v) from the registers of this sub-panel)
    if (live) {
      double vr[W];
#pragma unroll
      for (int v = 0; v < W; ++v) vr[v] = ts ? a[v] : (gr > ii + c0 + v ? a[v] : (gr == ii + c0 + v ? 1.0 : 0.0));
      for (int c = 0; c < nR; ++c) {
        double t1 = Ps[(cR + c) * LDP + tid];
#pragma unroll
        for (int v = 0; v < W; ++v) t1 = fma(-vr[v], Wg[v * WLD + c], t1);
        Ps[(cR + c) * LDP + tid] = t1;
      }
    }
    cl.sync();  // Wp / Wr of this sub-panel are no longer read by any CTA
  }
  // ---- write the panel back ------------------------------------------------------------------
  for (int e = tid; e < SB * R; e += kQsThreads) {
    const int c = e / R, r = e % R;
    if (ts || row0 + r >= ii) A[size_t(ii + c) * nb + row0 + r] = Ps[c * LDP + r];
  }
  // ---- y = striu(V^T V) of the whole panel into the T area (tau on the diagonal) ---------------
  // partial Gram over my rows by DMMA: the 136 upper 8x8 tiles (ti <= tj) of the 16 x 16 tile
  // grid, 34 per warp held in registers until every warp has read the panel, then stored over
  // the panel buffer as Gp[tile][64] for CTA 0 to reduce over DSMEM
  {
    constexpr int NT = 136 / (kQsThreads / 32);
    double g0[NT], g1[NT];
    const int g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const int w = warp + n * (kQsThreads / 32);
      int ti = 0, rem = w;
      while (rem >= 16 - ti) {
        rem -= 16 - ti;
        ++ti;
      }
      const int tj = ti + rem;
      double d0 = 0.0, d1 = 0.0;
      for (int k0 = 0; k0 < R; k0 += 4) dmma_8x8x4(d0, d1, Vat(k0 + t, ti * 8 + g), Vat(k0 + t, tj * 8 + g));
      g0[n] = d0;
      g1[n] = d1;
    }
    __syncthreads();
    double* Gp = Ps;
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const int w = warp + n * (kQsThreads / 32);
      Gp[w * 64 + g * 8 + 2 * t] = g0[n];
      Gp[w * 64 + g * 8 + 2 * t + 1] = g1[n];
    }
  }
  __syncthreads();
  cl.sync();
  if (q == 0) {
    // T column jc: rows k < jc = sum over CTAs of G(k, jc); k == jc: tau; below: 0
    for (int e = tid; e < SB * SB; e += kQsThreads) {
      const int jc = e / SB, k = e % SB;
      double v = 0.0;
      if (k < jc) {
        const int ti = k / 8, tj = jc / 8;
        const int w = ti * 16 - ti * (ti - 1) / 2 + (tj - ti);
        const int off = w * 64 + (k % 8) * 8 + (jc % 8);
        double pt[kQrCl];
#pragma unroll
        for (int c2 = 0; c2 < kQrCl; ++c2) pt[c2] = cl.map_shared_rank(Ps, c2)[off];
#pragma unroll
        for (int c2 = 0; c2 < kQrCl; ++c2) v += pt[c2];
      } else if (k == jc) {
        v = taus[jc];
      }
      T[size_t(jc) * ib + k] = v;
    }
  }
  __threadfence();
  cl.sync();  // every CTA's partial Gram has been read
  if (q != 0) return;
  qr_t_from_y(T, ib, SB, sm);
}

// ---------------------------------------------------------------------------
static unsigned qr_panel_smem(int nb, int sb) {
  const int R = nb / kQrCl;
  size_t d = size_t(sb) * (R + 1);
  size_t t = size_t(sb) * (sb + 1) + sb + 7 * 256;
  if (t > d) d = t;
  d += 8 * kQrMaxSb + 8;
  return unsigned(d * sizeof(double));
}

template <class CfgQ, class C1 = CfgQ>
static unsigned qr_apply_smem() {
  return unsigned((qr_ring_doubles<CfgQ, C1>() + CfgQ::BN * kWld) * sizeof(double));
}

#define HG_QATTR(fn, attr, val)                                                                  \
  do {                                                                                           \
    cudaError_t e_ = cudaFuncSetAttribute(fn, attr, val);                                        \
    if (e_ != cudaSuccess) {                                                                     \
      set_error("cudaFuncSetAttribute(%s, %s, %d): %s", #fn, #attr, int(val), cudaGetErrorString(e_)); \
      return false;                                                                              \
    }                                                                                            \
  } while (0)

bool init_qr_attributes() {
  HG_QATTR(k_qr_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, qr_panel_smem(1024, 128));
  HG_QATTR(k_qr_panel_sp<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)QsSmem<128>::BYTES);
  HG_QATTR(k_qr_panel_sp<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)QsSmem<64>::BYTES);
  HG_QATTR(k_qr_apply<CfgQ64>, cudaFuncAttributeMaxDynamicSharedMemorySize, qr_apply_smem<CfgQ64>());
  HG_QATTR(k_qr_apply<CfgQ32>, cudaFuncAttributeMaxDynamicSharedMemorySize, qr_apply_smem<CfgQ32>());
  HG_QATTR(k_qr_apply<CfgQ16>, cudaFuncAttributeMaxDynamicSharedMemorySize, qr_apply_smem<CfgQ16>());
  HG_QATTR((k_qr_apply<CfgQ32, true>), cudaFuncAttributeMaxDynamicSharedMemorySize, qr_apply_smem<CfgQ32>());
  HG_QATTR((k_qr_apply<CfgQ4w, true, CfgQ4w1>), cudaFuncAttributeMaxDynamicSharedMemorySize,
           (qr_apply_smem<CfgQ4w, CfgQ4w1>()));
  HG_QATTR((k_qr_apply<CfgQ16, true>), cudaFuncAttributeMaxDynamicSharedMemorySize, qr_apply_smem<CfgQ16>());
  HG_QATTR(k_qr_apply_cl, cudaFuncAttributeMaxDynamicSharedMemorySize, qr_apply_cl_smem());
  return true;
}

// materialize_t (kernels.py:188-211): the T factor the panel left in the tile's side
// area is also written to the task's separate T block, so the DAG's T data block
// holds what the reference models it to hold
struct CopyParams {
  double* dst;
  const double* src;
  long long n;
};
__global__ void k_copy_doubles(CopyParams p) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < p.n; i += (long long)gridDim.x * blockDim.x)
    p.dst[i] = p.src[i];
}

bool build_qr_launches(int kind, const TaskOperands& o, std::vector<LaunchDesc>& out) {
  const int nb = o.nb, ib = o.ib;
  if (nb % 128 != 0 || nb > 1024 || ib != 128) {
    set_error("QR tile kernels need nb %% 128 == 0, nb <= 1024 and ib == 128; got nb=%d ib=%d", nb, ib);
    return false;
  }
  const size_t tile = size_t(nb) * nb;
  const int np = nb / ib;
  auto side = [&](int i) { return o.t[i] + tile; };
  // strip width: HG_QR_APPLY env ("cl" = 4-CTA cluster kernel, or 16 / 32 / 64)
  static const int mode_env = [] {
    const char* e = getenv("HG_QR_APPLY");
    if (!e) return 0;
    if (e[0] == 'c') return -1;
    return atoi(e);
  }();
  // HG_RED=0: C -= V W as load / subtract / store instead of L2 reductions (A/B)
  static const bool red = [] {
    const char* e = getenv("HG_RED");
    return !(e && e[0] == '0');
  }();
  auto push_apply = [&](const QrApplyParams& ap, int bn_default) {
    LaunchDesc d;
    const int bn = mode_env ? mode_env : bn_default;
    const int ncols = nb - ap.col0;
    if (bn < 0 && nb % (kQcCl * 128) == 0)
      d.set((const void*)k_qr_apply_cl, dim3(ncols / kQcBN * kQcCl), dim3(CfgQC::THREADS), qr_apply_cl_smem(), ap);
    else if (bn == 16)
      d.set(red ? (const void*)k_qr_apply<CfgQ16, true> : (const void*)k_qr_apply<CfgQ16>, dim3(ncols / 16),
            dim3(CfgQ16::THREADS), qr_apply_smem<CfgQ16>(), ap);
    else if (bn == 34 || (bn == 32 && red && mode_env == 0))
      d.set((const void*)k_qr_apply<CfgQ4w, true, CfgQ4w1>, dim3(ncols / 32), dim3(CfgQ4w::THREADS),
            qr_apply_smem<CfgQ4w, CfgQ4w1>(), ap);
    else if (bn == 32)
      d.set(red ? (const void*)k_qr_apply<CfgQ32, true> : (const void*)k_qr_apply<CfgQ32>, dim3(ncols / 32),
            dim3(CfgQ32::THREADS), qr_apply_smem<CfgQ32>(), ap);
    else
      d.set((const void*)k_qr_apply<CfgQ64>, dim3(ncols / 64), dim3(CfgQ64::THREADS), qr_apply_smem<CfgQ64>(), ap);
    out.push_back(d);
  };
  switch (kind) {
    case K_GEQRT:
    case K_TSQRT: {
      const bool ts = kind == K_TSQRT;
      double* A = ts ? o.t[1] : o.t[0];
      for (int P = 0; P < np; ++P) {
        QrPanelParams pp{A, ts ? o.t[0] : nullptr, ts ? side(1) : side(0), nb, ib, P * ib, ib,
                         ts ? QR_TSQRT : QR_GEQRT};
        LaunchDesc d;
        // HG_QR_PANEL=sp selects the sub-panel kernel: correct (tests pass) but measured
        // slower (745 vs 600 us per panel: ~1070 instructions per column per warp in the
        // shuffle reductions, I-cache misses of the unrolled column loop), so the
        // column-at-a-time kernel stays the default
        static const bool sp_panel = [] {
          const char* e = getenv("HG_QR_PANEL");
          return e && e[0] == 's';
        }();
        if (sp_panel && ib == kQsSB && (nb == 1024 || nb == 512))
          d.set(nb == 1024 ? (const void*)k_qr_panel_sp<128> : (const void*)k_qr_panel_sp<64>, dim3(kQrCl),
                dim3(kQsThreads), unsigned(nb == 1024 ? QsSmem<128>::BYTES : QsSmem<64>::BYTES), pp);
        else
          d.set((const void*)k_qr_panel, dim3(kQrCl), dim3(kQrThreads), qr_panel_smem(nb, ib), pp);
        out.push_back(d);
        if (P + 1 < np)
          push_apply(QrApplyParams{A, ts ? side(1) : side(0), ts ? o.t[0] : A, ts ? A : nullptr, nb, ib, P, P + 1,
                                   (P + 1) * ib, ts ? QR_TSQRT : QR_GEQRT}, 16);
      }
      const int t_idx = ts ? 2 : 1;  // materialized T block (GEQRT: kk, T; TSQRT: kk, ik, T)
      if (o.n_t > t_idx) {
        LaunchDesc d;
        d.set((const void*)k_copy_doubles, dim3(64), dim3(256), 0,
              CopyParams{o.t[t_idx], ts ? side(1) : side(0), (long long)ib * nb});
        out.push_back(d);
      }
      return true;
    }
    case K_UNMQR:
      push_apply(QrApplyParams{o.t[0], side(0), o.t[1], nullptr, nb, ib, 0, np, 0, QR_GEQRT}, o.urgent ? 16 : 32);
      return true;
    case K_TSMQR:
      push_apply(QrApplyParams{o.t[0], side(0), o.t[1], o.t[2], nb, ib, 0, np, 0, QR_TSQRT}, o.urgent ? 16 : 32);
      return true;
    default:
      set_error("kind %d is not a QR kind", kind);
      return false;
  }
}

}  // namespace hg
