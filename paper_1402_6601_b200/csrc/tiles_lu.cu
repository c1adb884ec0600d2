// LU with incremental pivoting tile kernels for sm_100a:
// GETRF_INC, GESSM, TSTRF, SSSSM (reference kinds kernels.py:29-33, access
// lists kernels.py:156-167; semantics restated in oracle/tiles_lu_qr.py).
//
// Two kernels build every LU kind:
//
//  k_lu_panel  -- one ib-wide panel factorization (GETRF: partial pivoting
//                 over the tile rows >= j; TSTRF: pairwise pivoting between
//                 U(j,j) and the rows of A_ik).  A thread-block CLUSTER of 8
//                 CTAs keeps the panel resident in shared memory (CTA q owns
//                 rows [q*nb/8, (q+1)*nb/8)); each column costs ONE cluster
//                 barrier: every CTA publishes its local arg-max and that
//                 row's values (double-buffered by column parity), then all
//                 CTAs read the 8 candidates over DSMEM, agree on the pivot,
//                 and update their own rows.  The panel ends by inverting its
//                 unit-lower diagonal block L_uu into the tile's side area
//                 (so every later application is a DMMA product, no scalar
//                 substitution).
//  k_lu_apply  -- applies panels [p0, p1) of a factor to a column strip:
//                 row interchanges (gathered into smem, applied in order),
//                 top <- inv(L_uu) * top and bot -= L_a * top on the DMMA
//                 engine.  GESSM / SSSSM are one launch (all panels, all
//                 columns); GETRF / TSTRF call it after each panel on the
//                 trailing columns.
//
// Side area of a tile (after its nb*nb doubles): inv(L_uu) blocks, ib x nb
// column-major (panel p at columns [p*ib, p*ib+sb)), then int32 ipiv[nb]
// (GETRF: absolute row swapped with row j; TSTRF: A row swapped with U row j,
// or -1).
#include <cooperative_groups.h>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdlib>

#include "dgemm_dmma.cuh"
#include "tiles.h"

namespace cg = cooperative_groups;

namespace hg {

constexpr int kLuCl = 8;          // cluster size (portable)
constexpr int kLuThreads = 256;
constexpr int kLuMaxSb = 128;

enum { LU_GETRF = 0, LU_TSTRF = 1 };

struct LuPanelParams {
  double* A;      // panel tile (GETRF: A_kk, TSTRF: A_ik)
  double* U;      // TSTRF: A_kk (upper part holds U); GETRF: unused
  double* side;   // side area of A: inverse blocks (ib x nb), then ipiv
  int nb, ib, ii, sb, mode;
  int* status;
  PushList push;  // the task's last panel: producer-push of its output slots (tile + side)
};

__device__ __forceinline__ bool better(double v, int r, double bv, int br) {
  return v > bv || (v == bv && r < br);
}

// Register-resident panel: CTA q owns rows [q*R, (q+1)*R) of the panel; thread
// t owns row lr = t % R and the NC columns c = g + NG*m (g = t / R, NG = 256/R).
// Per column: 1 CTA barrier + 1 cluster barrier (local arg-max, candidate row
// published over DSMEM), then 2 CTA barriers (pivot row staged, multipliers
// published); the rank-1 update is NC independent register FMAs.
template <int R, int SB>
__global__ void __cluster_dims__(kLuCl, 1, 1) __launch_bounds__(kLuThreads) k_lu_panel(LuPanelParams p) {
  constexpr int NG = kLuThreads / R, NC = SB / NG;
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int q = (int)cl.block_rank();
  const int nb = p.nb, ii = p.ii, ib = p.ib;
  const int row0 = q * R;
  const int tid = threadIdx.x, lr = tid % R, grp = tid / R;
  const int gr = row0 + lr;
  const bool ts = p.mode == LU_TSTRF;
  double* cand = sm;                   // [2][SB]
  double* rowj = cand + 2 * SB;        // [2][SB]
  double* urow = rowj + 2 * SB;        // [2][SB]
  double* prow = urow + 2 * SB;        // [SB]
  double* lv = prow + SB;              // [R]
  double* slot_v = lv + R;             // [2]
  int* slot_r = reinterpret_cast<int*>(slot_v + 2);  // [2]
  double* Ls = sm;                     // reused after the sweep: [SB][SB+1]
  __shared__ double red_v[kLuThreads / 32];
  __shared__ int red_r[kLuThreads / 32];
  int* ipiv = reinterpret_cast<int*>(p.side + size_t(ib) * nb);
  double* inv = p.side + size_t(ii) * ib;
  double* A = p.A;
  const bool row_live = ts || gr >= ii;

  double a[NC];
#pragma unroll
  for (int m = 0; m < NC; ++m) a[m] = row_live ? A[size_t(ii + grp + NG * m) * nb + gr] : 0.0;
  if (ts && q == 0)
    for (int e = tid; e < ib * SB; e += kLuThreads) inv[e] = 0.0;  // dL written only for swapped rows
  __syncthreads();

  for (int jj = 0; jj < SB; ++jj) {
    const int j = ii + jj;
    const int par = jj & 1;
    const int gj = jj % NG, mj = jj / NG;
    if (ts)
      for (int c = tid; c < SB; c += kLuThreads) urow[par * SB + c] = c >= jj ? p.U[size_t(ii + c) * nb + j] : 0.0;
    // ---- phase A: local arg-max over column jj -------------------------------
    double bv = -1.0;
    int br = 0x7fffffff;
    if (grp == gj && (ts || gr >= j)) {
      double v = 0.0;
#pragma unroll
      for (int m = 0; m < NC; ++m)
        if (m == mj) v = a[m];
      bv = fabs(v);
      br = gr;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      int orr = __shfl_xor_sync(0xffffffffu, br, o);
      if (better(ov, orr, bv, br)) {
        bv = ov;
        br = orr;
      }
    }
    if ((tid & 31) == 0) {
      red_v[tid >> 5] = bv;
      red_r[tid >> 5] = br;
    }
    __syncthreads();
    {
      double v = red_v[0];
      int r = red_r[0];
#pragma unroll
      for (int w = 1; w < kLuThreads / 32; ++w)
        if (better(red_v[w], red_r[w], v, r)) {
          v = red_v[w];
          r = red_r[w];
        }
      if (tid == 0) {
        slot_v[par] = v;
        slot_r[par] = r;
      }
      if (gr == r) {
#pragma unroll
        for (int m = 0; m < NC; ++m) cand[par * SB + grp + NG * m] = a[m];
      }
      if (!ts && gr == j) {
#pragma unroll
        for (int m = 0; m < NC; ++m) rowj[par * SB + grp + NG * m] = a[m];
      }
    }
    cl.sync();
    // ---- phase B: global pivot (every warp resolves it) ---------------------
    int wr, wc;
    bool swap;
    {
      double v = -1.0;
      int r = 0x7fffffff, who = 0;
      const int l8 = tid & 31;
      if (l8 < kLuCl) {
        v = cl.map_shared_rank(slot_v, l8)[par];
        r = cl.map_shared_rank(slot_r, l8)[par];
        who = l8;
      }
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) {
        double ov = __shfl_xor_sync(0xffffffffu, v, o);
        int orr = __shfl_xor_sync(0xffffffffu, r, o);
        int ow = __shfl_xor_sync(0xffffffffu, who, o);
        if (better(ov, orr, v, r)) {
          v = ov;
          r = orr;
          who = ow;
        }
      }
      wr = __shfl_sync(0xffffffffu, r, 0);
      wc = __shfl_sync(0xffffffffu, who, 0);
      v = __shfl_sync(0xffffffffu, v, 0);
      swap = ts ? (v > fabs(urow[par * SB + jj])) : (wr != j);
    }
    const double* wcand = cl.map_shared_rank(cand, wc) + par * SB;
    for (int c = tid; c < SB; c += kLuThreads) prow[c] = (ts && !swap) ? urow[par * SB + c] : wcand[c];
    if (tid == 0 && q == 0) ipiv[j] = ts ? (swap ? wr : -1) : wr;
    if (swap) {
      if (ts) {
        if (gr == wr) {
#pragma unroll
          for (int m = 0; m < NC; ++m) {
            const int c = grp + NG * m;
            if (c < jj) {
              inv[size_t(c) * ib + jj] = a[m];  // dL(jj, c), inverted at the end
              a[m] = 0.0;
            } else {
              p.U[size_t(ii + c) * nb + j] = wcand[c];
              a[m] = urow[par * SB + c];
            }
          }
        }
      } else {
        if (gr == wr) {  // row p <- old row j
          const double* src = cl.map_shared_rank(rowj, j / R) + par * SB;
#pragma unroll
          for (int m = 0; m < NC; ++m) a[m] = src[grp + NG * m];
        }
        if (gr == j) {
#pragma unroll
          for (int m = 0; m < NC; ++m) a[m] = wcand[grp + NG * m];
        }
      }
    }
    __syncthreads();
    const double piv = prow[jj];
    const bool act = ts || gr > j;
    if (piv == 0.0) {
      if (tid == 0 && q == 0 && p.status) atomicOr(p.status, 2);
      continue;  // uniform across the cluster: nothing to eliminate
    }
    const double rcp = 1.0 / piv;
    if (grp == gj && act) {
      double v = 0.0;
#pragma unroll
      for (int m = 0; m < NC; ++m)
        if (m == mj) v = a[m];
      v *= rcp;
#pragma unroll
      for (int m = 0; m < NC; ++m)
        if (m == mj) a[m] = v;
      lv[lr] = v;
    }
    __syncthreads();
    if (act) {
      const double l = lv[lr];
      const double* pb = prow + grp;
#pragma unroll
      for (int m = 0; m < NC; ++m) {
        const double nv = fma(-l, pb[NG * m], a[m]);
        a[m] = (grp + NG * m > jj) ? nv : a[m];
      }
    }
  }
  // ---- write the panel back ----------------------------------------------------
  if (row_live) {
#pragma unroll
    for (int m = 0; m < NC; ++m) A[size_t(ii + grp + NG * m) * nb + gr] = a[m];
  }
  __threadfence();
  cl.sync();
  // ---- inv(L_uu) into the side area (columns distributed over the cluster) ----
  const int sb = SB;
  const int LL = sb + 1;
  for (int e = tid; e < sb * sb; e += kLuThreads) {
    int c = e / sb, r = e % sb;
    double v = 0.0;
    if (r > c) v = ts ? inv[size_t(c) * ib + r] : A[size_t(ii + c) * nb + ii + r];
    Ls[c * LL + r] = v;
  }
  __syncthreads();
  cl.sync();  // every CTA has its copy of dL before anyone overwrites it
  const int warp = tid >> 5, lane = tid & 31;
  for (int c = q * (kLuThreads / 32) + warp; c < sb; c += kLuCl * (kLuThreads / 32)) {
    double x[kLuMaxSb / 32];
#pragma unroll
    for (int m = 0; m < kLuMaxSb / 32; ++m) {
      int i = lane + 32 * m;
      x[m] = (i == c) ? 1.0 : 0.0;
    }
    for (int k = c; k < sb; ++k) {
      double xk = 0.0;
#pragma unroll
      for (int m = 0; m < kLuMaxSb / 32; ++m)
        if (m == k / 32) xk = x[m];
      xk = __shfl_sync(0xffffffffu, xk, k % 32);
#pragma unroll
      for (int m = 0; m < kLuMaxSb / 32; ++m) {
        int i = lane + 32 * m;
        if (i > k && i < sb) x[m] = fma(-Ls[k * LL + i], xk, x[m]);
      }
    }
#pragma unroll
    for (int m = 0; m < kLuMaxSb / 32; ++m) {
      int i = lane + 32 * m;
      if (i < sb) inv[size_t(c) * ib + i] = x[m];
    }
  }
}

// ---------------------------------------------------------------------------
template <int SB>
struct ApplyCfg {
  using G = GemmCfg<SB, 64, 16, 32, 32, 3>;  // SB x 64 CTA tiles
  static constexpr int BN = 64;
};

struct LuApplyParams {
  const double* L;      // factor tile (GETRF: A_kk; TSTRF: A_ik)
  const double* side;   // its side area (inverse blocks, ipiv)
  double* top;          // tile whose rows [ii, ii+sb) are transformed
  double* bot;          // GETRF-type: == top; TSTRF-type: the other tile
  int nb, ib, p0, p1, col0, mode;
  int swap_only;        // 1: row interchanges + inv(L_uu)*top only (the bot update is a separate wide GEMM)
#ifdef HG_PANEL_STAMPS
  int stamp;            // tools/ssssm_ab.cu: this task's CTA 0 records phase stamps
#endif
  PushList push;        // task-level launch: producer-push of the written tiles' columns of each strip
  alignas(64) CUtensorMap top_map;  // strip kernel: 2-D tensor map of `top` (128-row x BN-column boxes, TMA)
};

template <int SB>
__global__ void __launch_bounds__(ApplyCfg<SB>::G::THREADS) k_lu_apply(LuApplyParams p) {
  using G = typename ApplyCfg<SB>::G;
  constexpr int BN = ApplyCfg<SB>::BN;
  extern __shared__ double sm[];
  const int nb = p.nb, ib = p.ib;
  const int n0 = p.col0 + blockIdx.x * BN;
  const int tid = threadIdx.x;
  const bool ts = p.mode == LU_TSTRF;
  const int* ipiv = reinterpret_cast<const int*>(p.side + size_t(ib) * nb);
  // smem: swap buffer [2*SB][BN+1] + slot map [nb] ints, aliased with the GEMM ring
  double* buf = sm;
  constexpr int BLD = BN + 1;
  int* slot_of = reinterpret_cast<int*>(sm + 2 * SB * BLD);
  __shared__ int extra_row[SB];
  __shared__ int n_extra;
  for (int P = p.p0; P < p.p1; ++P) {
    const int ii = P * ib;
    // ---- 1) row interchanges of this panel, gathered into smem ----------------
    for (int r = tid; r < nb; r += blockDim.x) slot_of[r] = -1;
    __syncthreads();
    if (tid == 0) {
      int ne = 0;
      for (int jj = 0; jj < SB; ++jj) {
        int r = ipiv[ii + jj];
        bool sw = ts ? (r >= 0) : (r != ii + jj);
        if (!sw) continue;
        int key = ts ? r : r;  // bot row (TSTRF) / tile row (GETRF)
        bool in_top = !ts && r >= ii && r < ii + SB;
        if (!in_top && slot_of[key] < 0) {
          slot_of[key] = SB + ne;
          extra_row[ne++] = key;
        }
      }
      n_extra = ne;
    }
    __syncthreads();
    const int ne = n_extra;
    // gather top rows [ii, ii+SB) and the extra rows, column by column (coalesced)
    for (int e = tid; e < BN * (SB + ne); e += blockDim.x) {
      int c = e / (SB + ne), k = e % (SB + ne);
      double v;
      if (k < SB) v = p.top[size_t(n0 + c) * nb + ii + k];
      else v = (ts ? p.bot : p.top)[size_t(n0 + c) * nb + extra_row[k - SB]];
      buf[k * BLD + c] = v;
    }
    __syncthreads();
    if (tid < BN) {
      const int c = tid;
      for (int jj = 0; jj < SB; ++jj) {
        int r = ipiv[ii + jj];
        bool sw = ts ? (r >= 0) : (r != ii + jj);
        if (!sw) continue;
        int k2 = (!ts && r >= ii && r < ii + SB) ? (r - ii) : slot_of[r];
        double a = buf[jj * BLD + c];
        buf[jj * BLD + c] = buf[k2 * BLD + c];
        buf[k2 * BLD + c] = a;
      }
    }
    __syncthreads();
    for (int e = tid; e < BN * (SB + ne); e += blockDim.x) {
      int c = e / (SB + ne), k = e % (SB + ne);
      double v = buf[k * BLD + c];
      if (k < SB) p.top[size_t(n0 + c) * nb + ii + k] = v;
      else (ts ? p.bot : p.top)[size_t(n0 + c) * nb + extra_row[k - SB]] = v;
    }
    __threadfence();
    __syncthreads();
    // ---- 2) top <- inv(L_uu) * top (SB x BN, K = SB) -----------------------------
    {
      double acc[G::FM][G::FN][2];
      zero_acc<G>(acc);
      TileLoader<G, M_MAJOR, G::BM> la{p.side + size_t(ii) * ib, ib, 0};
      TileLoader<G, K_MAJOR, G::BN> lb{p.top + ii, nb, n0};
      gemm_mainloop<G>(acc, sm, la, lb, 0, SB);
      for_each_acc<G>(acc, [&](int r, int c, double v) { p.top[size_t(n0 + c) * nb + ii + r] = v; });
    }
    __threadfence();
    __syncthreads();
    if (p.swap_only) continue;
    // ---- 3) bot -= L_a * top ------------------------------------------------------
    const int m_begin = ts ? 0 : ii + SB;
    for (int m0 = m_begin; m0 < nb; m0 += SB) {
      double acc[G::FM][G::FN][2];
      zero_acc<G>(acc);
      TileLoader<G, M_MAJOR, G::BM> la{p.L + size_t(ii) * nb, nb, m0};
      TileLoader<G, K_MAJOR, G::BN> lb{p.top + ii, nb, n0};
      gemm_mainloop<G>(acc, sm, la, lb, 0, SB);
      sub_store<G>(acc, p.bot, nb, m0, n0);
    }
    __threadfence();
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// C -= A * B with A M_MAJOR (element (m, k) at A[k*lda + m]) and B K_MAJOR
// (element (n, k) at B[n*ldb + k]): the trailing "bot -= L_a * top" of one
// panel as a full-width DMMA GEMM (64x64 CTA tiles).
using CfgN = GemmCfg<64, 64, 16, 32, 32, 3>;

struct GemmNNParams {
  const double* A;
  const double* B;
  double* C;
  int lda, ldb, ldc, K;
};

__global__ void __launch_bounds__(CfgN::THREADS) k_gemm_nn(GemmNNParams p) {
  extern __shared__ double smem[];
  const int m0 = blockIdx.x * CfgN::BM, n0 = blockIdx.y * CfgN::BN;
  double acc[CfgN::FM][CfgN::FN][2];
  zero_acc<CfgN>(acc);
  TileLoader<CfgN, M_MAJOR, CfgN::BM> la{p.A, p.lda, m0};
  TileLoader<CfgN, K_MAJOR, CfgN::BN> lb{p.B, p.ldb, n0};
  gemm_mainloop<CfgN>(acc, smem, la, lb, 0, p.K);
  sub_store<CfgN>(acc, p.C, p.ldc, m0, n0);
}

static unsigned nn_smem() { return (unsigned)GemmSmem<CfgN, M_MAJOR, K_MAJOR>::BYTES; }

// ---------------------------------------------------------------------------
constexpr int kLcLd = kLuMaxSb + 4;             // smem [col][row] buffers of the strip kernel
constexpr int kLcMaxMoves = 2 * kLuMaxSb;

// Row moves of one panel (values before the panel -> positions after it).
// GETRF (rows of one tile): step j swaps rows j and p_j >= j.  Positions < j
// are final after step j, so with V(j) = the row pushed out of j at step j
//   V(j)            = V(j'') for the last j'' < j with p_j'' == j, else j
//   final row j     = V(j') for the last j' < j with p_j' == p_j, else p_j
//   final row x     = V(j') for the last j' with p_j' == x     (x >= ii+sb)
// TSTRF (top slot jj <-> bot row r_jj, or -1): with jp the last earlier step
// that swapped the same bot row,
//   final top jj    = T(jp) if jp exists else B(r_jj)
//   final bot r     = T(jj) for the last jj that swapped r.
// Encoding: bot rows >= 0, top slots -1-jj.  Returns the move count.
__device__ int lu_moves(const int* steps, int ii, int sb, bool ts, int* sp, int* mv_dst, int* mv_src,
                        int* cnt) {
  // steps[j]: pivot of step j (GETRF: absolute row p_j; TSTRF: bot row or -1);
  // ii: tile row of step 0 (GETRF)
  const int tid = threadIdx.x;
  if (tid == 0) *cnt = 0;
  for (int j = tid; j < sb; j += blockDim.x) sp[j] = steps[j];
  __syncthreads();
  if (ts) {
    for (int j = tid; j < sb; j += blockDim.x) {
      const int r = sp[j];
      if (r < 0) continue;
      // one pass over the pivot list, 4 entries per LDS.128 (sp is 16-byte aligned, sb % 4 == 0)
      int jp = -1;
      bool last = true;
      if ((reinterpret_cast<uintptr_t>(sp) & 15) || (sb & 3)) {
        for (int k = 0; k < j; ++k) jp = (sp[k] == r) ? k : jp;
        for (int k = j + 1; k < sb; ++k) last = last && (sp[k] != r);
      } else
      for (int k = 0; k < sb; k += 4) {
        const int4 q4 = *reinterpret_cast<const int4*>(sp + k);
        const int qv[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          jp = (k + u < j && qv[u] == r) ? k + u : jp;
          last = last && !(k + u > j && qv[u] == r);
        }
      }
      int n = atomicAdd(cnt, last ? 2 : 1);
      mv_dst[n] = -1 - j;
      mv_src[n] = jp >= 0 ? -1 - jp : r;
      if (last) {
        mv_dst[n + 1] = r;
        mv_src[n + 1] = -1 - j;
      }
    }
  } else {
    // pred[j]: last earlier step whose target is row j (panel rows only)
    int* pred = sp + sb;
    int* V = pred + sb;
    for (int j = tid; j < sb; j += blockDim.x) {
      int pr = -1;
      for (int k = 0; k < j; ++k) pr = (sp[k] == ii + j) ? k : pr;
      pred[j] = pr;
    }
    __syncthreads();
    for (int j = tid; j < sb; j += blockDim.x) {
      int k = j;
      while (pred[k] >= 0) k = pred[k];
      V[j] = ii + k;
    }
    __syncthreads();
    for (int j = tid; j < sb; j += blockDim.x) {
      const int pj = sp[j];
      int jl = -1;
      for (int k = 0; k < j; ++k) jl = (sp[k] == pj) ? k : jl;
      const int src = (pj == ii + j) ? V[j] : (jl >= 0 ? V[jl] : pj);
      if (src != ii + j) {
        int n = atomicAdd(cnt, 1);
        mv_dst[n] = ii + j;
        mv_src[n] = src;
      }
      if (pj >= ii + sb) {  // rows below the panel: the last step targeting them moves V into them
        bool last = true;
        for (int k = j + 1; k < sb; ++k) last = last && (sp[k] != pj);
        if (last) {
          int n = atomicAdd(cnt, 1);
          mv_dst[n] = pj;
          mv_src[n] = V[j];
        }
      }
    }
  }
  __syncthreads();
  return *cnt;
}

// ---------------------------------------------------------------------------
// k_lu_panel_sp -- one ib-wide panel factorisation (the GETRF / TSTRF
// semantics of k_lu_panel) blocked into W = 16-column sub-panels, so the
// per-column critical path only touches 16 registers per row:
//   * the 8-CTA cluster keeps the panel rows in shared memory (CTA q owns
//     rows [q*R, (q+1)*R), one row per thread);
//   * per column: local arg-max -> ONE cluster barrier -> every thread reads
//     the 8 candidates and the winner's 16 sub-panel values over DSMEM, swaps
//     and eliminates inside its registers (no further barrier);
//   * per sub-panel: the 16 row interchanges are applied to the panel columns
//     outside the sub-panel as one composed move list (lu_moves) over DSMEM;
//     TSTRF moves the swapped rows' earlier multipliers to dL; then the
//     right-hand columns get U12 = L11^-1 A12 (owner of the 16 pivot rows /
//     CTA 0 for TSTRF) and A22 -= L21 U12 (every row, registers x broadcast).
// Same outputs as k_lu_panel (ipiv, dL, panel values, inv(L_uu) in the side area).
constexpr int kSpW = 16;
constexpr int kSpThreads = 128;
constexpr int kSpSB = kLuMaxSb;

template <int R>
struct SpSmem {
  static constexpr int LDP = R + 1;
  static constexpr int PS = kSpSB * LDP;                  // panel [col][row]
  static constexpr int U12 = kSpW * kSpSB;                // [v][col] (the sub-panel's U block Ublk in the column loop)
  static constexpr int REC = 2 + kSpW;                    // column message: (value, row), candidate row
  static constexpr int INBOX = 2 * kLuCl * REC;           // [parity][sender] messages
  static constexpr int MISC = INBOX + 2 * kSpW + 2 * kSpW + 2 + kSpW * kSpW;
  // inbox, rowjIn[2][W], mycand/myrowj, 2 mbarriers, dlAll
  static constexpr int DOUBLES = PS + U12 + MISC;
  static constexpr int INTS = kSpSB + 4 * kSpW + 3 * kSpW;
  static constexpr size_t BYTES = size_t(DOUBLES) * 8 + size_t(INTS) * 4;
};

template <int R>
__global__ void __cluster_dims__(kLuCl, 1, 1) __launch_bounds__(kSpThreads) k_lu_panel_sp(LuPanelParams p) {
  constexpr int W = kSpW, SB = kSpSB;
  using S = SpSmem<R>;
  constexpr int LDP = S::LDP;
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int q = (int)cl.block_rank();
  const int nb = p.nb, ii = p.ii, ib = p.ib;
  const int row0 = q * R;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool ts = p.mode == LU_TSTRF;
  const bool mine = tid < R;
  const int gr = row0 + tid;
  const bool live = mine && (ts || gr >= ii);
  // Footprint <= 151 KB (nb = 1024) so that one 71 KB trailing-update strip CTA co-resides on each
  // of the cluster's SMs inside the DAG: no phase-S staging rows (moves go register -> remote Ps),
  // the sub-panel's U block lives in U12's space during the column loop.
  double* Ps = sm;
  double* U12 = Ps + S::PS;
  // per-column messages: every CTA pushes (local best |value|, its row, that row's W sub-panel
  // values) into every CTA's inbox with st.async, completing on the receiver's mbarrier -- no
  // cluster barrier per column.  GETRF: the owner of row j also pushes row j (rowjIn).
  double* inbox = U12 + S::U12;         // [2][kLuCl][REC]
  double* rowjIn = inbox + S::INBOX;    // [2][W]
  double* mycand = rowjIn + 2 * W;      // [W] staging of this CTA's candidate row
  double* myrowj = mycand + W;          // [W] staging of row j (its owner)
  uint64_t* bars = reinterpret_cast<uint64_t*>(myrowj + W);  // [2] by column parity
  double* Ublk = U12;                   // [W][W] during the column loop (U12 is idle then)
  double* dlAll = myrowj + W + 2;       // [W][W] CTA 0: the sub-panel's whole dL block (forward solve)
  int* swp = reinterpret_cast<int*>(sm + S::DOUBLES);  // [SB]
  int* mvd = swp + SB;                  // [2W]
  int* mvs = mvd + 2 * W;               // [2W]
  int* sp = mvs + 2 * W;                // [3W]
  __shared__ double red_v[kSpThreads / 32];
  __shared__ int red_r[kSpThreads / 32];
  __shared__ int n_mv;
  __shared__ __align__(8) uint64_t sbar;  // phase S: the moved values land with st.async (one phase per sub-panel)
  int* ipiv = reinterpret_cast<int*>(p.side + size_t(ib) * nb);
  double* inv = p.side + size_t(ii) * ib;  // dL(jj, c) at inv[c*ib + jj]
  double* A = p.A;
  HG_STAMP(0);

  for (int e = tid; e < SB * R; e += kSpThreads) {
    const int c = e / R, r = e % R;
    Ps[c * LDP + r] = (ts || row0 + r >= ii) ? A[size_t(ii + c) * nb + row0 + r] : 0.0;
  }
  if (ts && q == 0)
    for (int e = tid; e < ib * SB; e += kSpThreads) inv[e] = 0.0;
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_init(&sbar, 1);
    fence_mbar_init_cluster();
  }
  for (int e = tid; e < W * W; e += kSpThreads) dlAll[e] = 0.0;
  __threadfence();
  cl.sync();  // barriers initialised before any CTA pushes
  HG_STAMP(1);
  constexpr int REC = S::REC;
  const unsigned msg_bytes = unsigned(kLuCl * REC * 8 + (ts ? 0 : W * 8));

  for (int c0 = 0; c0 < SB; c0 += W) {
    HG_STAMP(2 + (c0 / W) * 8);
    if (ts) {
      for (int e = tid; e < W * W; e += kSpThreads) {
        const int u = e / W, v = e % W;
        Ublk[e] = v >= u ? __ldcg(p.U + size_t(ii + c0 + v) * nb + ii + c0 + u) : 0.0;
      }
    }
    double a[W];
#pragma unroll
    for (int v = 0; v < W; ++v) a[v] = mine ? Ps[(c0 + v) * LDP + tid] : 0.0;
    __syncthreads();
#pragma unroll
    for (int u = 0; u < W; ++u) {
      const int jj = c0 + u, j = ii + jj, par = jj & 1;
      // ---- A: local arg-max -> a message to every CTA (candidate row, + row j for GETRF) ----
      if (tid == 0) mbar_arrive_tx(&bars[par], msg_bytes);  // this CTA's one arrival of the phase
      double bv = -1.0;
      int br = 0x7fffffff;
      if (live && (ts || gr >= j)) {
        bv = fabs(a[u]);
        br = gr;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int orr = __shfl_xor_sync(0xffffffffu, br, o);
        if (better(ov, orr, bv, br)) {
          bv = ov;
          br = orr;
        }
      }
      if (lane == 0) {
        red_v[warp] = bv;
        red_r[warp] = br;
      }
      __syncthreads();
      if (c0 == 0) HG_STAMP(300 + 4 * u);
      double lv_ = red_v[0];
      int lr_ = red_r[0];
#pragma unroll
      for (int w = 1; w < kSpThreads / 32; ++w)
        if (better(red_v[w], red_r[w], lv_, lr_)) {
          lv_ = red_v[w];
          lr_ = red_r[w];
        }
      if (mine && gr == lr_) {
#pragma unroll
        for (int v2 = 0; v2 < W; ++v2) mycand[v2] = a[v2];
      }
      const bool own_j = !ts && j / R == q;
      if (own_j && mine && gr == j) {
#pragma unroll
        for (int v2 = 0; v2 < W; ++v2) myrowj[v2] = a[v2];
      }
      __syncthreads();
      {
        constexpr int NREC = kLuCl * (REC / 2);  // 16-byte pieces of the candidate messages
        const int nitems = NREC + (own_j ? kLuCl * (W / 2) : 0);
        for (int e = tid; e < nitems; e += kSpThreads) {
          int rcv, off;
          double x0, x1;
          double* dst;
          if (e < NREC) {
            rcv = e / (REC / 2);
            off = e % (REC / 2);
            x0 = off == 0 ? lv_ : mycand[2 * off - 2];
            x1 = off == 0 ? __longlong_as_double((long long)lr_) : mycand[2 * off - 1];
            dst = inbox + (par * kLuCl + q) * REC + 2 * off;
          } else {
            const int e2 = e - NREC;
            rcv = e2 / (W / 2);
            off = e2 % (W / 2);
            x0 = myrowj[2 * off];
            x1 = myrowj[2 * off + 1];
            dst = rowjIn + par * W + 2 * off;
          }
          st_async_v2f64(cluster_addr(dst, rcv), x0, x1, cluster_addr(&bars[par], rcv));
        }
      }
      if (c0 == 0) HG_STAMP(301 + 4 * u);
      mbar_wait_cluster(&bars[par], (jj >> 1) & 1);
      if (c0 == 0) HG_STAMP(302 + 4 * u);
      HG_STAMP(100 + jj);
      // ---- B: global pivot from the local inbox, pivot row, interchange --------------
      int wr = 0x7fffffff, wc = 0;
      double wv = -1.0;
#pragma unroll
      for (int w = 0; w < kLuCl; ++w) {
        const double* rec = inbox + (par * kLuCl + w) * REC;
        const double v = rec[0];
        const int r = (int)__double_as_longlong(rec[1]);
        if (better(v, r, wv, wr)) {
          wv = v;
          wr = r;
          wc = w;
        }
      }
      const bool swap = ts ? (wv > fabs(Ublk[u * W + u])) : (wr != j);
      const bool from_cand = !ts || swap;
      const double* cw = inbox + (par * kLuCl + wc) * REC + 2;
      double prow[W];
#pragma unroll
      for (int v2 = 0; v2 < W; ++v2) prow[v2] = 0.0;
#pragma unroll
      for (int v2 = u; v2 < W; ++v2) prow[v2] = from_cand ? cw[v2] : Ublk[u * W + v2];
      if (tid == 0) swp[jj] = ts ? (swap ? wr : -1) : wr;
      if (swap) {
        if (ts) {
          if (mine && gr == wr) {
            double* dl0 = cl.map_shared_rank(dlAll, 0) + u * W;  // CTA 0's forward solve reads it locally
#pragma unroll
            for (int v2 = 0; v2 < W; ++v2) {
              if (v2 < u) {
                inv[size_t(c0 + v2) * ib + jj] = a[v2];  // dL(jj, c0 + v2)
                dl0[v2] = a[v2];
                a[v2] = 0.0;
              } else {
                a[v2] = Ublk[u * W + v2];
              }
            }
          }
          // (no cluster barrier in the column loop: these global stores delay nothing)
          if (q == 0 && tid >= u && tid < W) p.U[size_t(ii + c0 + tid) * nb + j] = cw[tid];
        } else {
          if (mine && gr == wr) {
            const double* rj = rowjIn + par * W;
#pragma unroll
            for (int v2 = 0; v2 < W; ++v2) a[v2] = rj[v2];
          }
          if (mine && gr == j) {
#pragma unroll
            for (int v2 = 0; v2 < W; ++v2) a[v2] = cw[v2];
          }
        }
      }
      // ---- C: scale and eliminate inside the sub-panel -----------------------------
      const double piv = prow[u];
      if (piv == 0.0) {
        if (tid == 0 && q == 0 && p.status) atomicOr(p.status, 2);
        continue;
      }
      const double rcp = 1.0 / piv;
      if (live && (ts || gr > j)) {
        const double l = a[u] * rcp;
        a[u] = l;
#pragma unroll
        for (int v2 = u + 1; v2 < W; ++v2) a[v2] = fma(-l, prow[v2], a[v2]);
      }
      if (c0 == 0) HG_STAMP(303 + 4 * u);
    }
    if (mine) {
#pragma unroll
      for (int v = 0; v < W; ++v) Ps[(c0 + v) * LDP + tid] = a[v];
    }
    __syncthreads();
    HG_STAMP(2 + (c0 / W) * 8 + 1);
    // ---- S: the sub-panel's interchanges on the columns outside it ----------------------
    const int cR = c0 + W;  // first right-hand column
    if (q == 0 && tid < W) ipiv[ii + c0 + tid] = swp[c0 + tid];
    if (c0 == 16) HG_STAMP(400);
    if (ts) {
      // (i) a swapped A row's multipliers left of the sub-panel move to dL(jj, .) (first swap only)
      for (int u = 0; u < W; ++u) {
        const int r = swp[c0 + u];
        if (r < row0 || r >= row0 + R) continue;
        bool first = true;
        for (int u2 = 0; u2 < u; ++u2) first = first && (swp[c0 + u2] != r);
        if (!first) continue;
        for (int c = tid; c < c0; c += kSpThreads) {
          inv[size_t(c) * ib + c0 + u] = Ps[c * LDP + (r - row0)];
          Ps[c * LDP + (r - row0)] = 0.0;
        }
      }
    }
    if (c0 == 16) HG_STAMP(401);
    const int nm = lu_moves(swp + c0, ii + c0, W, ts, sp, mvd, mvs, &n_mv);
    if (c0 == 16) HG_STAMP(402);
    // moved values: GETRF rows, columns outside the sub-panel; TSTRF rows / U rows (top slots),
    // right-hand columns
    const int ncol_out = SB - W;
    auto out_col = [&](int k) { return k < c0 ? k : k + W; };
    if (ts && q == 0 && tid < SB - cR) {  // CTA 0: the sub-panel's U rows (right-hand columns) before the moves
#pragma unroll
      for (int v = 0; v < W; ++v) U12[v * SB + tid] = __ldcg(p.U + size_t(ii + cR + tid) * nb + ii + c0 + v);
    }
    // Moves in two steps separated by a cluster barrier: the CTA holding a move's source (a Ps
    // row, or for TSTRF a top slot: CTA 0's U12 prefetch) reads it into registers; after the
    // barrier it stores it straight into the destination (a Ps row of its owner over DSMEM, or a
    // U row: CTA 0's U12).  Remote stores, no remote loads, no staging rows.
    const int mcol = ts ? cR + tid : (tid < ncol_out ? out_col(tid) : -1);  // this thread's column
    const bool colok = ts ? (cR + tid < SB) : (tid < ncol_out);
    double mv[2 * W];
#pragma unroll
    for (int m = 0; m < 2 * W; ++m) {
      mv[m] = 0.0;
      if (m < nm && colok) {
        const int sidx = mvs[m];
        if (q == (sidx < 0 ? 0 : sidx / R)) mv[m] = sidx < 0 ? U12[(-1 - sidx) * SB + tid] : Ps[mcol * LDP + (sidx - row0)];
      }
    }
    if (c0 == 16) HG_STAMP(403);
    cl.sync();  // every source read before any destination is overwritten
    HG_STAMP(2 + (c0 / W) * 8 + 2);
    if (tid == 0) {  // this CTA's arrival: the bytes the moves will deliver into it
      const int ncv = ts ? SB - cR : ncol_out;
      int cnt = 0;
      for (int m = 0; m < nm; ++m) {
        const int d = mvd[m];
        cnt += (ts && d < 0) ? (q == 0) : (d / R == q);
      }
      mbar_arrive_tx(&sbar, unsigned(cnt * ncv * 8));
    }
#pragma unroll
    for (int m = 0; m < 2 * W; ++m) {
      if (m < nm && colok) {
        const int d = mvd[m], sidx = mvs[m];
        if (q == (sidx < 0 ? 0 : sidx / R)) {
          const bool top = ts && d < 0;  // a U row (right-hand columns): the forward solve writes it out
          const unsigned dst = top ? 0u : unsigned(d / R);
          double* loc = top ? U12 + (-1 - d) * SB + tid : Ps + mcol * LDP + (d % R);
          st_async_f64(cluster_addr(loc, dst), mv[m], cluster_addr(&sbar, dst));
        }
      }
    }
    mbar_wait_cluster(&sbar, (c0 / W) & 1);  // every move into this CTA has landed
    __syncthreads();
    HG_STAMP(2 + (c0 / W) * 8 + 3);
    if (cR >= SB) break;
    // ---- U: right-hand columns: U12 = L11^-1 A12, A22 -= L21 U12 --------------------------
    const int nR = SB - cR;
    // (no cluster barrier needed here: the owner reads only rows it wrote itself
    // and dL entries published before the phase-S barrier)
    const int owner = ts ? 0 : (ii + c0) / R;
    if (q == owner) {
      // forward substitution, one thread per right-hand column
      for (int c = tid; c < nR; c += kSpThreads) {
        double x[W];
#pragma unroll
        for (int v = 0; v < W; ++v) {
          double t = ts ? U12[v * SB + c] : Ps[(cR + c) * LDP + (ii + c0 + v - row0)];
#pragma unroll
          for (int w = 0; w < v; ++w) {
            const double l = ts ? dlAll[v * W + w] : Ps[(c0 + w) * LDP + (ii + c0 + v - row0)];
            t = fma(-l, x[w], t);
          }
          x[v] = t;
          U12[v * SB + c] = t;
          if (ts) p.U[size_t(ii + cR + c) * nb + ii + c0 + v] = t;
          else Ps[(cR + c) * LDP + (ii + c0 + v - row0)] = t;
        }
      }
      if (ts) {  // dlAll is rebuilt by the next sub-panel's winners (after the barriers below)
        __syncthreads();
        for (int e = tid; e < W * W; e += kSpThreads) dlAll[e] = 0.0;
      }
    }
    cl.sync();
    HG_STAMP(2 + (c0 / W) * 8 + 4);
    if (q != owner && tid < nR) {  // thread c copies column c of U12 (16 loads in flight)
      const double* src = cl.map_shared_rank(U12, owner);
      double v[W];
#pragma unroll
      for (int w = 0; w < W; ++w) v[w] = src[w * SB + tid];
#pragma unroll
      for (int w = 0; w < W; ++w) U12[w * SB + tid] = v[w];
    }
    __syncthreads();
    HG_STAMP(2 + (c0 / W) * 8 + 5);
    if (live && (ts || gr >= ii + cR)) {
      for (int c = 0; c < nR; c += 4) {  // nR % 16 == 0: four independent FMA chains
        double t[4];
#pragma unroll
        for (int x = 0; x < 4; ++x) t[x] = Ps[(cR + c + x) * LDP + tid];
#pragma unroll
        for (int v = 0; v < W; ++v)
#pragma unroll
          for (int x = 0; x < 4; ++x) t[x] = fma(-a[v], U12[v * SB + c + x], t[x]);
#pragma unroll
        for (int x = 0; x < 4; ++x) Ps[(cR + c + x) * LDP + tid] = t[x];
      }
    }
    cl.sync();  // U12 of the owner is not overwritten before every CTA copied it
    HG_STAMP(2 + (c0 / W) * 8 + 6);
  }
  // ---- write the panel back ------------------------------------------------------------
  for (int e = tid; e < SB * R; e += kSpThreads) {
    const int c = e / R, r = e % R;
    if (ts || row0 + r >= ii) A[size_t(ii + c) * nb + row0 + r] = Ps[c * LDP + r];
  }
  __threadfence();
  cl.sync();
  HG_STAMP(80);
  // ---- inv(L_uu) into the side area: CTA q computes block column q (16 columns) ----------
  // X = L^-1 of the unit-lower 128 x 128 L_uu by 16 x 16 blocks: X_ii = inv(L_ii) (one warp
  // each, lanes = columns), then down the block column X_ij = -X_ii sum_{k=j}^{i-1} L_ik X_kj.
  // L is kept packed (lower triangle by columns) so the scratch fits the panel's footprint.
  {
    constexpr int B = kSpW, NBK = SB / B;
    static_assert(NBK == kLuCl, "one block column per CTA");
    const int k0 = q * B;
    auto pk = [](int r, int c) { return c * SB - (c * (c - 1)) / 2 + (r - c); };  // r >= c
    double* Ls = sm;                          // packed lower L_uu (diagonal slot unused)
    double* Xd = Ls + SB * (SB + 1) / 2;      // [NBK][B][B] diagonal block inverses, Xd[bi*B*B + c*B + r]
    double* Xc = Xd + NBK * B * B;            // [SB][B] this block column of X, Xc[r * B + c]
    double* Tm = Xc + SB * B;                 // [B][B] Tm[c * B + m]
    const int tot = (SB - k0) * SB;
    for (int e0 = tid; e0 < tot; e0 += 16 * kSpThreads) {  // 16 L2 loads in flight per thread
      double v[16];
#pragma unroll
      for (int x = 0; x < 16; ++x) {
        const int e = e0 + x * kSpThreads;
        const int c = k0 + e / SB, r = e % SB;
        v[x] = 0.0;
        if (e < tot && r > c) v[x] = ts ? __ldcg(inv + size_t(c) * ib + r) : __ldcg(A + size_t(ii + c) * nb + ii + r);
      }
#pragma unroll
      for (int x = 0; x < 16; ++x) {
        const int e = e0 + x * kSpThreads;
        const int c = k0 + e / SB, r = e % SB;
        if (e < tot && r >= c) Ls[pk(r, c)] = v[x];
      }
    }
    __syncthreads();
    cl.sync();  // every CTA has read dL before any CTA overwrites it with the inverse
    HG_STAMP(81);
    for (int bi = q + warp; bi < NBK; bi += kSpThreads / 32) {
      if (lane < B) {
        double x[B];
#pragma unroll
        for (int r = 0; r < B; ++r) x[r] = r == lane ? 1.0 : 0.0;
#pragma unroll
        for (int k = 0; k < B; ++k)
#pragma unroll
          for (int r = k + 1; r < B; ++r) x[r] = fma(-Ls[pk(bi * B + r, bi * B + k)], x[k], x[r]);
#pragma unroll
        for (int r = 0; r < B; ++r) Xd[bi * B * B + lane * B + r] = x[r];
      }
    }
    __syncthreads();
    for (int e = tid; e < B * B; e += kSpThreads) {
      const int r = e % B, c = e / B;
      Xc[(k0 + r) * B + c] = Xd[q * B * B + c * B + r];
    }
    __syncthreads();
    for (int bi = q + 1; bi < NBK; ++bi) {
      for (int e = tid; e < B * B; e += kSpThreads) {  // Tm = sum_k L(bi*B + r, k) Xc(k, c), k in [k0, bi*B)
        const int r = e % B, c = e / B;
        double t[4] = {0.0, 0.0, 0.0, 0.0};
        for (int k = k0; k < bi * B; k += 4) {
#pragma unroll
          for (int x = 0; x < 4; ++x) t[x] = fma(Ls[pk(bi * B + r, k + x)], Xc[(k + x) * B + c], t[x]);
        }
        Tm[c * B + r] = (t[0] + t[1]) + (t[2] + t[3]);
      }
      __syncthreads();
      for (int e = tid; e < B * B; e += kSpThreads) {  // X_bi,q = -X_bi,bi Tm
        const int r = e % B, c = e / B;
        double x = 0.0;
#pragma unroll
        for (int m = 0; m < B; ++m) x = fma(Xd[bi * B * B + m * B + r], Tm[c * B + m], x);
        Xc[(bi * B + r) * B + c] = -x;
      }
      __syncthreads();
    }
    for (int e = tid; e < B * SB; e += kSpThreads) {
      const int c = e / SB, r = e % SB;
      inv[size_t(k0 + c) * ib + r] = r < k0 ? 0.0 : Xc[r * B + c];
    }
  }
  HG_STAMP(82);  if (p.push.n) {  // producer-push: every kernel of the task is done once the whole cluster is here
    __threadfence();
    cl.sync();
    push_slots(p.push, q, kLuCl);
  }
}

// ---------------------------------------------------------------------------
// k_lu_apply_strip -- the same panel application without a cluster: one CTA
// per BN-column strip owns every row of it (columns are independent), so the
// interchanges, top' = inv(L_uu) top (DMMA) and bot -= L_a top' (DMMA) need
// only CTA barriers.  Small shared-memory footprint (2 CTAs / SM), so it
// co-schedules with the other tile kernels of the DAG.
// RED: bot -= L_a top' as L2 reductions (red.global.add.f64 of -acc); every
// later read of bot inside the kernel goes through L2 (ld.cg / cp.async.cg).
// GU: the configuration of the bot -= L_a top' stream (default G); a GU with
// BM = 256 starts its first row chunk early and masks the rows above it.
template <class G, bool RED = false, class GU = G>
__global__ void __launch_bounds__(G::THREADS, G::THREADS == 128 ? 3 : (GU::BM == 256 ? 2 : 1))
k_lu_apply_strip(const __grid_constant__ LuApplyParams p) {
  static_assert(GU::THREADS == G::THREADS && GU::BN == G::BN, "update config");
  constexpr int BN = G::BN;
  constexpr int RING_T = G::STAGES * G::slab_mmaj(G::BM);  // only A streams (B is resident)
  constexpr int RING_U = GU::STAGES * GU::slab_mmaj(GU::BM);
  constexpr int RING = RING_T > RING_U ? RING_T : RING_U;
  constexpr int AREA = RING + BN * kLcLd;
  static_assert(RING >= BN * kLcLd, "the pristine top rows fit in the ring");
  extern __shared__ __align__(128) double sm[];  // the ring's first slot is a TMA destination
  double* ring = sm;
  double* Ts = sm + RING;                 // [BN][kLcLd] top rows after the moves, then top'
  double* Wt = Ts;                        // top' overwrites Ts once the product has read it
  int* mv_dst = reinterpret_cast<int*>(sm + AREA);
  int* mv_src = mv_dst + kLcMaxMoves;
  int* sp = mv_src + kLcMaxMoves;         // [3 * sb]
  __shared__ int n_moves;
  const int nb = p.nb, ib = p.ib, sb = ib;
  const int n0 = p.col0 + blockIdx.x * BN;
  const bool ts = p.mode == LU_TSTRF;
  const int tid = threadIdx.x;
  const int* ipiv = reinterpret_cast<const int*>(p.side + size_t(ib) * nb);
  double* top = p.top;
  double* bot = ts ? p.bot : p.top;
  __shared__ __align__(8) uint64_t tbar;  // the pristine top rows land by TMA (one phase per panel)
  if (tid == 0) {
    mbar_init(&tbar, 1);
    fence_proxy_async_smem();
  }
  __syncthreads();
#ifdef HG_PANEL_STAMPS
  const int q = blockIdx.x == 0 && p.stamp ? 0 : -1;  // tools/ssssm_ab.cu phase stamps (CTA 0 of one task)
#endif
  for (int P = p.p0; P < p.p1; ++P) {
    HG_STAMP(20 + 4 * (P - p.p0));
    const int ii = P * ib;
#ifdef HG_EXP_NO_MOVES  // tools/ssssm_ab.cu timing experiment only (wrong results)
    const int nm = 0;
#else
    const int nm = lu_moves(ipiv + ii, ii, sb, ts, sp, mv_dst, mv_src, &n_moves);
#endif
    // ---- the panel's row interchanges -------------------------------------------------
    // Each top slot jj (row ii + jj) takes its value from a bot row, another top slot or itself;
    // each bot row that receives a value receives a (pristine) top slot.  Only the bot side
    // touches global memory: bot-sourced slots are gathered straight into Ts (L2 loads), the top
    // rows' final values reach global memory through the top' epilogue below, and the bot rows
    // that received top slots are stored from a pristine smem copy (Pt) of the top rows.
    static_assert(G::THREADS == kLuMaxSb, "one thread per top slot");
    int* slot_src = sp;                     // [sb] >= 0: bot row; < 0: top slot -1-k (lu_moves' scratch is dead)
    int* bd_row = slot_src + kLuMaxSb;      // [sb] bot rows that receive a top slot
    int* bd_slot = bd_row + kLuMaxSb;       // [sb] ... namely this one
    __shared__ int n_bd;
    slot_src[tid] = -1 - tid;
    if (tid == 0) n_bd = 0;
    __syncthreads();
    for (int m = tid; m < nm; m += G::THREADS) {
      const int d = mv_dst[m], s = mv_src[m];
      // GETRF: rows inside the panel are its top slots; TSTRF: codes are already (bot row | -1-slot)
      const int dslot = ts ? (d < 0 ? -1 - d : -1) : (d >= ii && d < ii + sb ? d - ii : -1);
      const int scode = ts ? s : (s >= ii && s < ii + sb ? -1 - (s - ii) : s);
      if (dslot >= 0) {
        slot_src[dslot] = scode;
      } else {
        const int k = atomicAdd(&n_bd, 1);
        bd_row[k] = d;
        bd_slot[k] = -1 - scode;  // a bot row only ever receives a top slot
      }
    }
    __syncthreads();
    const int nbd = n_bd;
    // pristine top rows [ii, ii + 128) x [n0, n0 + BN): ONE tensor-map TMA box into the idle ring
    // (dense [BN][128]); it lands while the bot-sourced slots are gathered below
    constexpr int kPt = kLuMaxSb;
    double* Pt = ring;
    if (tid == 0) {
      fence_proxy_async_smem();  // the ring's generic-proxy reads of the previous panel come first
      mbar_arrive_tx(&tbar, unsigned(BN * kPt * sizeof(double)));
      tma_load_2d(Pt, &p.top_map, ii, n0, &tbar);
    }
    {
      const int sc = slot_src[tid];
      if (sc >= 0) {  // BN loads in flight, one bot row across the strip's columns
        double v[BN];
#pragma unroll
        for (int c = 0; c < BN; ++c) v[c] = __ldcg(bot + size_t(n0 + c) * nb + sc);
#pragma unroll
        for (int c = 0; c < BN; ++c) Ts[c * kLcLd + tid] = v[c];
      }
    }
    mbar_wait(&tbar, unsigned(P - p.p0) & 1u);
    __syncthreads();
    {
      const int sc = slot_src[tid];
      if (sc < 0) {
#pragma unroll 8
        for (int c = 0; c < BN; ++c) Ts[c * kLcLd + tid] = Pt[c * kPt + (-1 - sc)];
      }
      if (tid < nbd) {
        const int r = bd_row[tid], k = bd_slot[tid];
#pragma unroll 8
        for (int c = 0; c < BN; ++c) __stcg(bot + size_t(n0 + c) * nb + r, Pt[c * kPt + k]);
      }
    }
    __syncthreads();
    HG_STAMP(20 + 4 * (P - p.p0) + 1);
    {  // top' = inv(L_uu) top
      double acc[G::FM][G::FN][2];
      zero_acc<G>(acc);
      TileLoader<G, M_MAJOR, 128> la{p.side + size_t(ii) * ib, ib, 0};
      gemm_mainloop_bsmem<G, decltype(la), true>(acc, ring, la, Ts, kLcLd, 0, sb);  // inv(L_uu) lower
      for_each_acc<G>(acc, [&](int r, int c, double v) {
        Wt[c * kLcLd + r] = v;
        top[size_t(n0 + c) * nb + ii + r] = v;
      });
    }
    __syncthreads();
    HG_STAMP(20 + 4 * (P - p.p0) + 2);
    if (!p.swap_only) {
      TileLoader<GU, M_MAJOR, GU::BM> la{p.L + size_t(ii) * nb, nb, 0};
      const int m_mask = ts ? 0 : ii + sb;
      const int m_lo = nb - (nb - m_mask + GU::BM - 1) / GU::BM * GU::BM;
      gemm_sub_chunks_bsmem<GU, decltype(la), true, 128, RED>(ring, la, Wt, kLcLd, sb, m_lo, nb, bot, nb, n0,
                                                              m_mask);
    }
    __syncthreads();
    HG_STAMP(20 + 4 * (P - p.p0) + 3);
  }
  if (p.push.n) {  // this strip's columns are final once its own L2 reductions landed
    __threadfence();
    __syncthreads();
    push_strip<BN, G::THREADS>(p.push, n0, nb);
  }
}

using CfgLS16 = GemmCfg<128, 16, 16, 32, 16, 3>;  // 4 warps, 16-column strips: the in-panel trailing columns
using CfgLS4w = GemmCfg<128, 32, 8, 32, 32, 4>;     // 4 warps of 32x32, 8-wide k-slabs: 3 CTAs / SM (GESSM / SSSSM)

template <class G, class GU = G>
static unsigned lu_apply_strip_smem() {
  size_t ring = size_t(G::STAGES) * G::slab_mmaj(G::BM);
  const size_t ru = size_t(GU::STAGES) * GU::slab_mmaj(GU::BM);
  if (ru > ring) ring = ru;
  size_t d = ring + G::BN * kLcLd;
  size_t ints = 2 * kLcMaxMoves + 3 * kLuMaxSb;  // moves, lu_moves scratch (then the slot sources)
  return unsigned(d * sizeof(double) + ints * sizeof(int));
}

// ---------------------------------------------------------------------------
static unsigned sp_smem(int nb) {
  size_t b = nb == 1024 ? SpSmem<128>::BYTES
             : nb == 768 ? SpSmem<96>::BYTES
             : nb == 512 ? SpSmem<64>::BYTES
                         : SpSmem<32>::BYTES;
  // end-of-panel inverse scratch: packed L_uu, diagonal block inverses, one block column, a block product
  size_t ls = (size_t(kSpSB) * (kSpSB + 1) / 2 + 2 * size_t(kSpSB) * kSpW + size_t(kSpW) * kSpW) * 8;
  return unsigned(b > ls ? b : ls);
}

static unsigned panel_smem(int nb, int sb) {
  const int R = nb / kLuCl;
  size_t bufs = 7 * size_t(sb) + R + 4;
  size_t inv = size_t(sb) * (sb + 1);
  return unsigned((bufs > inv ? bufs : inv) * sizeof(double));
}

// ib = 128: the sub-panel kernel (nb in {256, 512, 768, 1024}: nb / 8 rows per CTA); ib = 64: the
// register-resident full-width panel kernel (nb in {512, 1024})
static bool use_sp_panel(int nb, int ib) { return ib == kSpSB && (nb == 1024 || nb == 768 || nb == 512 || nb == 256); }

static const void* panel_kernel(int nb, int ib) {
  if (use_sp_panel(nb, ib))
    return nb == 1024 ? (const void*)k_lu_panel_sp<128>
           : nb == 768 ? (const void*)k_lu_panel_sp<96>
           : nb == 512 ? (const void*)k_lu_panel_sp<64>
                       : (const void*)k_lu_panel_sp<32>;
  if (nb == 1024 && ib == 64) return (const void*)k_lu_panel<128, 64>;
  if (nb == 512 && ib == 64) return (const void*)k_lu_panel<64, 64>;
  return nullptr;
}

template <int SB>
static unsigned apply_smem(int nb) {
  using G = typename ApplyCfg<SB>::G;
  size_t swap = size_t(2 * SB) * (ApplyCfg<SB>::BN + 1) * 8 + size_t(nb) * 4;
  size_t ring = GemmSmem<G, M_MAJOR, K_MAJOR>::BYTES;
  return unsigned(swap > ring ? swap : ring);
}

#define HG_ATTR(fn, attr, val)                                                                   \
  do {                                                                                           \
    cudaError_t e_ = cudaFuncSetAttribute(fn, attr, val);                                        \
    if (e_ != cudaSuccess) {                                                                     \
      set_error("cudaFuncSetAttribute(%s, %s, %d): %s", #fn, #attr, int(val), cudaGetErrorString(e_)); \
      return false;                                                                              \
    }                                                                                            \
  } while (0)

bool init_lu_attributes() {
  HG_ATTR((k_lu_panel<128, 64>), cudaFuncAttributeMaxDynamicSharedMemorySize, panel_smem(1024, 128));
  HG_ATTR((k_lu_panel<64, 64>), cudaFuncAttributeMaxDynamicSharedMemorySize, panel_smem(1024, 128));
  HG_ATTR(k_lu_apply<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, apply_smem<64>(1024));
  HG_ATTR(k_gemm_nn, cudaFuncAttributeMaxDynamicSharedMemorySize, nn_smem());
  HG_ATTR((k_lu_apply_strip<CfgLS16, true>), cudaFuncAttributeMaxDynamicSharedMemorySize, lu_apply_strip_smem<CfgLS16>());
  HG_ATTR((k_lu_apply_strip<CfgLS4w, true>), cudaFuncAttributeMaxDynamicSharedMemorySize,
          lu_apply_strip_smem<CfgLS4w>());
  HG_ATTR(k_lu_panel_sp<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sp_smem(1024));
  HG_ATTR(k_lu_panel_sp<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sp_smem(512));
  HG_ATTR(k_lu_panel_sp<96>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sp_smem(768));
  HG_ATTR(k_lu_panel_sp<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sp_smem(256));
  return true;
}

static void push_apply(std::vector<LaunchDesc>& out, const LuApplyParams& ap) {  // ib = 64
  LaunchDesc d;
  const int ncols = ap.nb - ap.col0;
  d.set((const void*)k_lu_apply<64>, dim3(ncols / ApplyCfg<64>::BN), dim3(ApplyCfg<64>::G::THREADS),
        apply_smem<64>(ap.nb), ap);
  out.push_back(d);
}

// ib = 128: every panel application is the strip kernel (one CTA per 16 / 32-column strip,
// L2-reduction update).  ib = 64: narrow swap + inv(L_uu) kernel, then a wide GEMM.
static bool use_strip_apply(int nb, int ib) { return ib == kLuMaxSb && nb % 128 == 0; }

// Panels [P0, P1) applied to columns [col0, nb) by the strip kernel.
// The TMA tensor map of a tile's top rows: nb x nb column-major doubles, boxes of 128 rows x bn columns
// (cuTensorMapEncodeTiled through the runtime's driver entry point: no -lcuda link).
static bool top_rows_map(CUtensorMap* m, const double* tile, int nb, int bn) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  if (!encode) {
    set_error("cuTensorMapEncodeTiled is not available from the driver");
    return false;
  }
  const cuuint64_t dims[2] = {cuuint64_t(nb), cuuint64_t(nb)};
  const cuuint64_t strides[1] = {cuuint64_t(nb) * sizeof(double)};
  const cuuint32_t box[2] = {cuuint32_t(kLuMaxSb), cuuint32_t(bn)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(tile), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled(top rows, nb=%d, bn=%d) failed: %d", nb, bn, int(r));
    return false;
  }
  return true;
}

static bool push_apply_strip(std::vector<LaunchDesc>& out, const double* L, const double* side, double* top,
                             double* bot, int nb, int ib, int P0, int P1, int col0, int mode, int bn,
                             const PushList* push = nullptr) {
  LuApplyParams ap{L, side, top, bot, nb, ib, P0, P1, col0, mode, 0};
  if (push) ap.push = *push;
  if (!top_rows_map(&ap.top_map, top, nb, bn)) return false;
  LaunchDesc d;
  const int ncols = nb - col0;
  if (bn == 16)
    d.set((const void*)k_lu_apply_strip<CfgLS16, true>, dim3(ncols / 16), dim3(CfgLS16::THREADS),
          lu_apply_strip_smem<CfgLS16>(), ap);
  else
    d.set((const void*)k_lu_apply_strip<CfgLS4w, true>, dim3(ncols / 32), dim3(CfgLS4w::THREADS),
          lu_apply_strip_smem<CfgLS4w>(), ap);
  out.push_back(d);
  return true;
}

static bool push_panel_apply(std::vector<LaunchDesc>& out, int ib, const double* L, const double* side,
                             double* top, double* bot, int nb, int P, int col0, int mode) {
  if (use_strip_apply(nb, ib)) return push_apply_strip(out, L, side, top, bot, nb, ib, P, P + 1, col0, mode, 16);
  LuApplyParams ap{L, side, top, bot, nb, ib, P, P + 1, col0, mode, 1};
  push_apply(out, ap);
  const int ii = P * ib;
  const bool ts = mode == LU_TSTRF;
  const int m0 = ts ? 0 : ii + ib;
  const int M = nb - m0, N = nb - col0;
  if (M <= 0 || N <= 0) return true;
  GemmNNParams gp{L + size_t(ii) * nb + m0, top + size_t(col0) * nb + ii, bot + size_t(col0) * nb + m0, nb, nb, nb, ib};
  LaunchDesc d;
  d.set((const void*)k_gemm_nn, dim3(M / CfgN::BM, N / CfgN::BN), dim3(CfgN::THREADS), nn_smem(), gp);
  out.push_back(d);
  return true;
}

bool build_lu_launches(int kind, const TaskOperands& o, std::vector<LaunchDesc>& out) {
  const int nb = o.nb, ib = o.ib;
  if (!(ib == 128 && use_sp_panel(nb, ib)) && !(ib == 64 && (nb == 512 || nb == 1024))) {
    set_error("LU tile kernels need ib = 128 with nb in {256, 512, 768, 1024}, or ib = 64 with nb in {512, 1024}; "
              "got nb=%d ib=%d", nb, ib);
    return false;
  }
  const size_t tile = size_t(nb) * nb;
  const int np = nb / ib;
  auto side = [&](int i) { return o.t[i] + tile; };
  switch (kind) {
    case K_GETRF_INC:
    case K_TSTRF: {
      const bool ts = kind == K_TSTRF;
      double* A = ts ? o.t[1] : o.t[0];
      for (int P = 0; P < np; ++P) {
        LuPanelParams pp{A, ts ? o.t[0] : nullptr, ts ? side(1) : side(0), nb, ib, P * ib, ib,
                         ts ? LU_TSTRF : LU_GETRF, o.status};
        if (P + 1 == np && use_sp_panel(nb, ib)) pp.push = resolve_push(o, true);  // tile + side (dL, IPIV)
        LaunchDesc d;
        if (use_sp_panel(nb, ib))
          d.set(panel_kernel(nb, ib), dim3(kLuCl), dim3(kSpThreads), sp_smem(nb), pp);
        else
          d.set(panel_kernel(nb, ib), dim3(kLuCl), dim3(kLuThreads), panel_smem(nb, ib), pp);
        out.push_back(d);
        if (P + 1 < np && !push_panel_apply(out, ib, A, ts ? side(1) : side(0), ts ? o.t[0] : A, A, nb, P,
                                            (P + 1) * ib, ts ? LU_TSTRF : LU_GETRF))
          return false;
      }
      return true;
    }
    case K_GESSM:
      if (use_strip_apply(nb, ib)) {
        const PushList pl = resolve_push(o, false);
        return push_apply_strip(out, o.t[0], side(0), o.t[1], o.t[1], nb, ib, 0, np, 0, LU_GETRF, 32, &pl);
      }
      for (int P = 0; P < np; ++P)
        if (!push_panel_apply(out, ib, o.t[0], side(0), o.t[1], o.t[1], nb, P, 0, LU_GETRF)) return false;
      return true;
    case K_SSSSM:
      if (use_strip_apply(nb, ib)) {
        const PushList pl = resolve_push(o, false);
        return push_apply_strip(out, o.t[0], side(0), o.t[1], o.t[2], nb, ib, 0, np, 0, LU_TSTRF, 32, &pl);
      }
      for (int P = 0; P < np; ++P)
        if (!push_panel_apply(out, ib, o.t[0], side(0), o.t[1], o.t[2], nb, P, 0, LU_TSTRF)) return false;
      return true;
    default:
      set_error("kind %d is not an LU kind", kind);
      return false;
  }
}

}  // namespace hg
