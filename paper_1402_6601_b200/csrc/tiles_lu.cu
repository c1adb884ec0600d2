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
static unsigned panel_smem(int nb, int sb) {
  const int R = nb / kLuCl;
  size_t bufs = 7 * size_t(sb) + R + 4;
  size_t inv = size_t(sb) * (sb + 1);
  return unsigned((bufs > inv ? bufs : inv) * sizeof(double));
}

static const void* panel_kernel(int nb, int ib) {
  if (nb == 1024 && ib == 128) return (const void*)k_lu_panel<128, 128>;
  if (nb == 1024 && ib == 64) return (const void*)k_lu_panel<128, 64>;
  if (nb == 512 && ib == 128) return (const void*)k_lu_panel<64, 128>;
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
  HG_ATTR((k_lu_panel<128, 128>), cudaFuncAttributeMaxDynamicSharedMemorySize, panel_smem(1024, 128));
  HG_ATTR((k_lu_panel<128, 64>), cudaFuncAttributeMaxDynamicSharedMemorySize, panel_smem(1024, 128));
  HG_ATTR((k_lu_panel<64, 128>), cudaFuncAttributeMaxDynamicSharedMemorySize, panel_smem(1024, 128));
  HG_ATTR((k_lu_panel<64, 64>), cudaFuncAttributeMaxDynamicSharedMemorySize, panel_smem(1024, 128));
  HG_ATTR(k_lu_apply<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, apply_smem<128>(1024));
  HG_ATTR(k_lu_apply<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, apply_smem<64>(1024));
  HG_ATTR(k_gemm_nn, cudaFuncAttributeMaxDynamicSharedMemorySize, nn_smem());
  return true;
}

static void push_apply(std::vector<LaunchDesc>& out, int ib, const LuApplyParams& ap) {
  LaunchDesc d;
  const int ncols = ap.nb - ap.col0;
  if (ib == 128)
    d.set((const void*)k_lu_apply<128>, dim3(ncols / ApplyCfg<128>::BN), dim3(ApplyCfg<128>::G::THREADS),
          apply_smem<128>(ap.nb), ap);
  else
    d.set((const void*)k_lu_apply<64>, dim3(ncols / ApplyCfg<64>::BN), dim3(ApplyCfg<64>::G::THREADS),
          apply_smem<64>(ap.nb), ap);
  out.push_back(d);
}

// One panel applied to columns [col0, nb): narrow swap + inv(L_uu) kernel,
// then the wide bot -= L_a * top GEMM.
static void push_panel_apply(std::vector<LaunchDesc>& out, int ib, const double* L, const double* side,
                             double* top, double* bot, int nb, int P, int col0, int mode) {
  LuApplyParams ap{L, side, top, bot, nb, ib, P, P + 1, col0, mode, 1};
  push_apply(out, ib, ap);
  const int ii = P * ib;
  const bool ts = mode == LU_TSTRF;
  const int m0 = ts ? 0 : ii + ib;
  const int M = nb - m0, N = nb - col0;
  if (M <= 0 || N <= 0) return;
  GemmNNParams gp{L + size_t(ii) * nb + m0, top + size_t(col0) * nb + ii, bot + size_t(col0) * nb + m0, nb, nb, nb, ib};
  LaunchDesc d;
  d.set((const void*)k_gemm_nn, dim3(M / CfgN::BM, N / CfgN::BN), dim3(CfgN::THREADS), nn_smem(), gp);
  out.push_back(d);
}

bool build_lu_launches(int kind, const TaskOperands& o, std::vector<LaunchDesc>& out) {
  const int nb = o.nb, ib = o.ib;
  if ((nb != 512 && nb != 1024) || (ib != 64 && ib != 128)) {
    set_error("LU tile kernels need nb in {512, 1024} and ib in {64, 128}; got nb=%d ib=%d", nb, ib);
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
        LaunchDesc d;
        d.set(panel_kernel(nb, ib), dim3(kLuCl), dim3(kLuThreads), panel_smem(nb, ib), pp);
        out.push_back(d);
        if (P + 1 < np)
          push_panel_apply(out, ib, A, ts ? side(1) : side(0), ts ? o.t[0] : A, A, nb, P, (P + 1) * ib,
                           ts ? LU_TSTRF : LU_GETRF);
      }
      return true;
    }
    case K_GESSM:
      for (int P = 0; P < np; ++P) push_panel_apply(out, ib, o.t[0], side(0), o.t[1], o.t[1], nb, P, 0, LU_GETRF);
      return true;
    case K_SSSSM:
      for (int P = 0; P < np; ++P) push_panel_apply(out, ib, o.t[0], side(0), o.t[1], o.t[2], nb, P, 0, LU_TSTRF);
      return true;
    default:
      set_error("kind %d is not an LU kind", kind);
      return false;
  }
}

}  // namespace hg
