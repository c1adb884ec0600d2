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
  PushList push;  // the task's last panel: producer-push of its output slots (tile + side)
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
  double* rrow = s + sb * LD;              // [2][sb] TSQRT: R row j
  double* wv = rrow + 2 * kQrMaxSb;        // [sb] reduced w / y
  double* vv = wv + kQrMaxSb;              // [R]  reflector entries of my rows for column jj
  double* ph = vv + kQrMaxSb;              // [2][sb] half-row partial sums
  // cross-CTA partials are PUSHED (remote stores before the barrier) into every CTA's local copy,
  // so nothing is loaded over DSMEM after a barrier (remote loads there cost ~1.5 us per column).
  // (The footprint stays <= 157 KB so that one 68 KB trailing-update strip CTA co-resides on each
  // of the cluster's SMs inside the DAG: staging the T columns / R rows too cost 5% of QR C4.)
  double* slotAll = ph + 2 * kQrMaxSb;    // [2][kQrCl][2] norm^2 partial, alpha
  double* pwAll = slotAll + 2 * kQrCl * 2;                // [2][kQrCl][sb] partial x^T [V | A]
  __shared__ double s_red[kQrThreads / 32];
  __shared__ double s_tau, s_beta, s_scal;
  // the two per-column exchanges are st.async messages completing on the receiver's mbarriers
  // (by column parity): bars[par] the (norm^2, alpha) messages, bars[2 + par] the partials
  __shared__ __align__(8) uint64_t bars[4];
  double* T = p.side + size_t(ii) * ib;    // this panel's ib x sb T block (ld = ib)
  double* A = p.A;

  for (int e = tid; e < sb * R; e += kQrThreads) {
    int c = e / R, r = e % R;
    int gr = row0 + r;
    s[c * LD + r] = (ts || gr >= ii) ? A[size_t(ii + c) * nb + gr] : 0.0;
  }
  if (tid == 0) {
    for (int b = 0; b < 4; ++b) mbar_init(&bars[b], 1);
    fence_mbar_init_cluster();
  }
  cl.sync();  // every CTA's barriers exist before the first message

  // partial ||x||^2 of column jj over my rows strictly below the diagonal row
  auto publish_norm = [&](int jj, int par, double rpre) {
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
    if (ts && tid < kQrMaxSb) rrow[par * kQrMaxSb + tid] = rpre;  // R row j, loaded a phase ahead
    if (tid == 0) mbar_arrive_tx(&bars[par], kQrCl * 16);     // this CTA's arrival for column jj
    __syncthreads();
    if (tid < kQrCl) {  // thread d sends this CTA's (norm^2 partial, alpha) to CTA d
      double t = 0.0;
      for (int w = 0; w < kQrThreads / 32; ++w) t += s_red[w];
      const double al = (!ts && j >= row0 && j < row0 + R) ? s[jj * LD + (j - row0)] : 0.0;
      st_async_v2f64(cluster_addr(slotAll + (par * kQrCl + q) * 2, tid), t, al, cluster_addr(&bars[par], tid));
    }
  };

  HG_STAMP(0);
  publish_norm(0, 0, (ts && tid < sb) ? p.R[size_t(ii + tid) * nb + ii] : 0.0);
  for (int jj = 0; jj < sb; ++jj) {
    const int j = ii + jj;
    const int par = jj & 1;
    if (jj < 16) HG_STAMP(300 + 8 * jj);
    if (jj < 16) HG_STAMP(301 + 8 * jj);
    if (tid < 32) {
      mbar_wait_cluster(&bars[par], (jj >> 1) & 1);  // the 8 (norm^2, alpha) messages of column jj
      double xn2 = 0.0, al = 0.0;
      if (tid < kQrCl) {
        const double* sl = slotAll + (par * kQrCl + tid) * 2;
        xn2 = sl[0];
        al = sl[1];  // only the owner of row j publishes a non-zero alpha
      }
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) {
        xn2 += __shfl_xor_sync(0xffffffffu, xn2, o);
        al += __shfl_xor_sync(0xffffffffu, al, o);
      }
      // dlarfg: beta = -sign(alpha) ||(alpha, x)||, tau = (beta - alpha) / beta, x *= 1 / (alpha - beta).
      // Lanes 0..7 hold the reduced (xn2, alpha); the two divisions run on different lanes, and
      // sqrt(alpha^2 + xn2) replaces dlapy2's overflow-safe hypot (xn2 is already a sum of squares;
      // the single-thread hypot + 2 divisions chain cost ~1.5 us per column)
      const double alpha = ts ? rrow[par * kQrMaxSb + jj] : al;
      if (xn2 != 0.0) {
        const double beta = -copysign(sqrt(fma(alpha, alpha, xn2)), alpha);
        if (tid == 0) s_tau = (beta - alpha) / beta;
        if (tid == 1) s_scal = 1.0 / (alpha - beta);
        if (tid == 2) s_beta = beta;
      } else if (tid == 0) {
        s_tau = 0.0;
        s_beta = alpha;
        s_scal = 1.0;
      }
    }
    __syncthreads();
    const double tau = s_tau, beta = s_beta, scal = s_scal;
    if (jj < 16) HG_STAMP(302 + 8 * jj);
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
    if (jj < 16) HG_STAMP(303 + 8 * jj);
    if (tid == 0) mbar_arrive_tx(&bars[2 + par], unsigned(kQrCl * sb * 8));
    {  // this CTA's partial of column c goes to every CTA: thread (c, half) covers 4 destinations
      const int c = tid % kQrMaxSb, h = tid / kQrMaxSb;
      if (c < sb) {
        const double v = ph[c] + ph[kQrMaxSb + c];
#pragma unroll
        for (int d = 0; d < kQrCl / 2; ++d) {
          const int dst = h * (kQrCl / 2) + d;
          st_async_f64(cluster_addr(pwAll + (par * kQrCl + q) * kQrMaxSb + c, dst), v,
                       cluster_addr(&bars[2 + par], dst));
        }
      }
    }
    mbar_wait_cluster(&bars[2 + par], (jj >> 1) & 1);  // the 8 partials of every column
    if (jj < 16) HG_STAMP(304 + 8 * jj);
    // R row j+1 for the next column's norm phase, issued now so it lands before barrier 1
    double rnext = 0.0;
    if (ts && tid < sb && jj + 1 < sb && tid >= jj + 1) rnext = p.R[size_t(ii + tid) * nb + j + 1];
    for (int c = tid; c < sb; c += kQrThreads) {
      double t = 0.0;
      if (c != jj) {
        double part[kQrCl];
#pragma unroll
        for (int c2 = 0; c2 < kQrCl; ++c2) part[c2] = pwAll[(par * kQrCl + c2) * kQrMaxSb + c];
#pragma unroll
        for (int c2 = 0; c2 < kQrCl; ++c2) t += part[c2];
      }
      if (ts && c > jj) t += rrow[par * kQrMaxSb + c];  // the unit of v_j sits in R row j
      wv[c] = t;
    }
    __syncthreads();
    if (jj < 16) HG_STAMP(305 + 8 * jj);
    // T column jj (y above the diagonal, tau on it) and the R row (TSQRT), by CTA jj % 8
    if (q == jj % kQrCl) {
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
    if (jj < 16) HG_STAMP(306 + 8 * jj);
    if (jj + 1 < sb) publish_norm(jj + 1, par ^ 1, rnext);
  }
  __syncthreads();
  for (int e = tid; e < sb * R; e += kQrThreads) {
    int c = e / R, r = e % R;
    int gr = row0 + r;
    if (ts || gr >= ii) A[size_t(ii + c) * nb + gr] = s[c * LD + r];
  }
  __threadfence();
  cl.sync();
  HG_STAMP(80);
  if (q == 0) {
    qr_t_from_y(T, ib, sb, s);
    HG_STAMP(82);
  }
  if (p.push.n) {  // producer-push: every kernel of the task is done once CTA 0's T is written
    __threadfence();
    cl.sync();
    push_slots(p.push, q, kQrCl);
  }
}

// ---------------------------------------------------------------------------
using CfgQ16 = GemmCfg<128, 16, 16, 32, 16, 3>;  // 4 warps: the in-panel trailing columns
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
  // M_MAJOR only: one warp's 32 slab rows [w0, w0 + 32) (warp-private rings of the C -= V W stream)
  HG_DEVICE void load_warp(double* s, int k0, int w0, int lane) const {
    static_assert(L == M_MAJOR, "warp-row loads are M_MAJOR");
    constexpr int BK = Cfg::BK, PAD = Cfg::PAD;
    const int rw = r0 + w0;
    // element-wise unless every row of the warp lies strictly below the slab's diagonal band
    // (rows entirely ABOVE it are zeros of the unit-lower V, not the stored R)
    if (!(masked && rw < ii + k0 + BK)) {
      load_slab_warp<Cfg, ROWS>(s, v, ld, r0, k0, w0, lane);
      return;
    }
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) s[kk * (ROWS + PAD) + w0 + lane] = val(rw + lane, k0 + kk);
  }
};

struct QrApplyParams {
  const double* V;     // factor tile (GEQRT: A_kk; TSQRT: A_ik)
  const double* side;  // its side area (T factors)
  double* top;         // UNMQR: the tile C (rows [ii, nb)); TSMQR: A_kj (rows [ii, ii+sb))
  double* bot;         // TSMQR: A_ij; UNMQR: unused
  int nb, ib, p0, p1, col0, mode;
#ifdef HG_PANEL_STAMPS
  int stamp;           // tools/ssssm_ab.cu (q mode): this task's CTA 0 records phase stamps
#endif
  PushList push;       // task-level launch: producer-push of the written tiles' columns of each strip
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
#ifdef HG_PANEL_STAMPS
  const int q = blockIdx.x == 0 && p.stamp ? 0 : -1;
#endif
  for (int P = p.p0; P < p.p1; ++P) {
    const int ii = P * ib;
    const double* Vp = p.V + size_t(ii) * nb;  // V(tr, pc) at Vp[pc*nb + tr]
    HG_STAMP(20 + 4 * (P - p.p0));
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
    HG_STAMP(20 + 4 * (P - p.p0) + 1);
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
    HG_STAMP(20 + 4 * (P - p.p0) + 2);
    // ---- C -= V W  (UNMQR rows [ii, nb))  |  bot -= V_B W (TSMQR)
    {
      VLoader<CfgQ, M_MAJOR, 128> la{Vp, nb, 0, ii, ts ? 0 : 1};
      gemm_sub_chunks_bsmem<CfgQ, decltype(la), false, 128, RED>(ring, la, W, kWld, 128, ts ? 0 : ii, nb,
                                                                  ts ? p.bot : p.top, nb, n0);
    }
    __syncthreads();
    HG_STAMP(20 + 4 * (P - p.p0) + 3);
  }
  if (p.push.n) {  // this strip's columns are final once its own L2 reductions landed
    __threadfence();
    __syncthreads();
    push_strip<kQrBN, CfgQ::THREADS>(p.push, n0, nb);
  }
}

// ---------------------------------------------------------------------------
static unsigned qr_panel_smem(int nb, int sb) {
  // the column loop's buffers follow the panel s[sb][R+1]; the end-of-panel T scratch
  // (qr_t_from_y, CTA 0) reuses the same region once they are dead
  const int R = nb / kQrCl;
  const size_t loop = size_t(sb) * (R + 1) + 6 * kQrMaxSb + 2 * kQrCl * 2 + 2 * kQrCl * kQrMaxSb;
  const size_t t = size_t(sb) * (sb + 1) + sb + 7 * 256;
  return unsigned((loop > t ? loop : t) * sizeof(double));
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
  HG_QATTR((k_qr_apply<CfgQ4w, true, CfgQ4w1>), cudaFuncAttributeMaxDynamicSharedMemorySize,
           (qr_apply_smem<CfgQ4w, CfgQ4w1>()));
  HG_QATTR((k_qr_apply<CfgQ16, true>), cudaFuncAttributeMaxDynamicSharedMemorySize, qr_apply_smem<CfgQ16>());
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
  // block-reflector applications: 16-column strips inside a panel task (few trailing columns),
  // 32-column strips of 4 warps at 3 CTAs / SM for UNMQR / TSMQR; C -= V W as L2 reductions
  auto push_apply = [&](QrApplyParams ap, int bn, bool push = false) {
    if (push) ap.push = resolve_push(o, false);  // the task-level strip launch pushes its columns
    LaunchDesc d;
    const int ncols = nb - ap.col0;
    if (bn == 16)
      d.set((const void*)k_qr_apply<CfgQ16, true>, dim3(ncols / 16), dim3(CfgQ16::THREADS),
            qr_apply_smem<CfgQ16>(), ap);
    else
      d.set((const void*)k_qr_apply<CfgQ4w, true, CfgQ4w1>, dim3(ncols / 32), dim3(CfgQ4w::THREADS),
            qr_apply_smem<CfgQ4w, CfgQ4w1>(), ap);
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
        if (P + 1 == np) pp.push = resolve_push(o, true);  // tile + side (T factors)
        LaunchDesc d;
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
      push_apply(QrApplyParams{o.t[0], side(0), o.t[1], nullptr, nb, ib, 0, np, 0, QR_GEQRT}, 32, true);
      return true;
    case K_TSMQR:
      push_apply(QrApplyParams{o.t[0], side(0), o.t[1], o.t[2], nb, ib, 0, np, 0, QR_TSQRT}, 32, true);
      return true;
    default:
      set_error("kind %d is not a QR kind", kind);
      return false;
  }
}

}  // namespace hg
