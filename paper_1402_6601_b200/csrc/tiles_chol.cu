// Cholesky tile kernels for sm_100a: POTRF, TRSM, SYRK, GEMM
// (reference kinds: kernels.py:23-27, access lists kernels.py:126-137).
//
// Tiles are nb x nb FP64, column-major, ld = nb (PLASMA tile layout).
//
//   GEMM  A_ij -= A_ik * A_jk^T            k_gemm_nt (full)      DMMA 64x64 CTA tiles
//   SYRK  A_ii -= A_ik * A_ik^T  (lower)   k_gemm_nt (lower)     DMMA, upper CTAs exit
//   TRSM  A_ik  = A_ik * L_kk^-T           k_trsm_rows           row strips, DMMA updates
//   POTRF A_kk  = L_kk (lower)             r=64 blocked right-looking chain:
//                                          k_potrf_diag -> k_trsm_rows -> k_gemm_nt(lower)
//
// POTRF leaves inv(L_JJ)^T of each 64x64 diagonal block in that block's
// strict upper triangle (the upper triangle of a Cholesky tile is never read
// by any other kind), so TRSM applies the diagonal-block inverses with DMMA
// instead of running a scalar substitution.  The upper triangle of diagonal
// tiles is therefore workspace, not input, after POTRF.
#include <cmath>
#include "dgemm_dmma.cuh"
#include "tiles.h"

namespace hg {

constexpr int kR = 64;  // inner blocking of POTRF / TRSM

using CfgG = GemmCfg<64, 64, 16, 32, 32, 3>;   // trailing updates
using CfgT = GemmCfg<32, 64, 16, 16, 32, 3>;   // TRSM row strips (32 rows)

// ---------------------------------------------------------------------------
// GEMM / SYRK: C[m0.., n0..] -= A * B^T, all M_MAJOR with a shared ld.
struct GemmNTParams {
  const double* A;
  const double* B;
  double* C;
  int ld, M, N, K;
  int lower;  // 1: update only C(i, j) with i >= j (SYRK)
};

__global__ void __launch_bounds__(CfgG::THREADS) k_gemm_nt(GemmNTParams p) {
  extern __shared__ double smem[];
  const int m0 = blockIdx.x * CfgG::BM, n0 = blockIdx.y * CfgG::BN;
  if (p.lower && m0 + CfgG::BM - 1 < n0) return;  // tile strictly above the diagonal
  double acc[CfgG::FM][CfgG::FN][2];
  zero_acc<CfgG>(acc);
  TileLoader<CfgG, M_MAJOR, CfgG::BM> la{p.A, p.ld, m0};
  TileLoader<CfgG, M_MAJOR, CfgG::BN> lb{p.B, p.ld, n0};
  gemm_mainloop<CfgG>(acc, smem, la, lb, 0, p.K);
  const bool diag = p.lower && (m0 == n0);
  double* C = p.C;
  const int ld = p.ld;
  for_each_acc<CfgG>(acc, [&](int r, int c, double v) {
    if (diag && r < c) return;
    size_t idx = size_t(n0 + c) * ld + m0 + r;
    C[idx] -= v;
  });
}

// ---------------------------------------------------------------------------
// Unblocked Cholesky of the 64x64 diagonal block at (j0, j0) + inverse.
// Writes L (lower) and inv(L)^T into the strict upper triangle of the block.
struct PotrfDiagParams {
  double* A;
  int ld, j0;
  int* status;
};

__global__ void __launch_bounds__(256) k_potrf_diag(PotrfDiagParams p) {
  __shared__ double s[kR][kR + 1];  // s[col][row]
  __shared__ double inv_diag[kR];
  double* blk = p.A + size_t(p.j0) * p.ld + p.j0;
  const int tid = threadIdx.x;
  for (int e = tid; e < kR * kR; e += blockDim.x) {
    int c = e / kR, r = e % kR;
    s[c][r] = blk[size_t(c) * p.ld + r];
  }
  __syncthreads();
  for (int j = 0; j < kR; ++j) {
    if (tid == 0) {
      double d = s[j][j];
      if (!(d > 0.0)) {
        if (p.status) atomicOr(p.status, 1);  // not positive definite
        d = 1.0;
      }
      d = sqrt(d);
      s[j][j] = d;
      inv_diag[j] = 1.0 / d;
    }
    __syncthreads();
    const double rd = inv_diag[j];
    for (int i = j + 1 + tid; i < kR; i += blockDim.x) s[j][i] *= rd;
    __syncthreads();
    // trailing update of columns c in (j, kR): s[c][i] -= s[j][i] * s[j][c], i >= c
    const int w = kR - j - 1;
    for (int e = tid; e < w * w; e += blockDim.x) {
      int c = j + 1 + e / w, i = j + 1 + e % w;
      if (i >= c) s[c][i] -= s[j][i] * s[j][c];
    }
    __syncthreads();
  }
  // write L back (lower incl. diagonal)
  for (int e = tid; e < kR * kR; e += blockDim.x) {
    int c = e / kR, r = e % kR;
    if (r >= c) blk[size_t(c) * p.ld + r] = s[c][r];
  }
  // inverse, one column per thread: L x = e_c (forward substitution)
  if (tid < kR) {
    const int c = tid;
    double x[kR];
#pragma unroll
    for (int i = 0; i < kR; ++i) x[i] = 0.0;
    x[c] = inv_diag[c];
    for (int i = c + 1; i < kR; ++i) {
      double acc = 0.0;
      for (int k = c; k < i; ++k) acc = fma(s[k][i], x[k], acc);
      x[i] = -acc * inv_diag[i];
    }
    // inv(i, c) for i > c goes to block position (row c, col i)
    for (int i = c + 1; i < kR; ++i) blk[size_t(i) * p.ld + c] = x[i];
  }
}

// ---------------------------------------------------------------------------
// Row-strip triangular solve X * L^T = B for column blocks [jb0, jb1):
//   X(:, J) = (B(:, J) - X(:, jb0..J) * L(J, jb0..J)^T) * inv(L_JJ)^T
// Rows are independent, so each CTA owns a 32-row strip and sweeps J; the
// update product runs on the DMMA engine, the inverse product from smem.
struct TrsmRowsParams {
  const double* L;  // tile holding L (and inv(L_JJ)^T in its diagonal blocks' upper triangles)
  double* B;        // tile solved in place; rows [row0, row0 + nrows)
  int ld, row0, jb0, jb1;
};

constexpr int kTrsmPipe = GemmSmem<CfgT, M_MAJOR, M_MAJOR>::DOUBLES;
constexpr int kTrsmS = kR * (CfgT::BM + 4);  // residual, M_MAJOR [k][row]
constexpr int kTrsmI = kR * (kR + 4);        // inv(L_JJ), [j][k]
constexpr int kTrsmSmemDoubles = (kTrsmPipe > kTrsmS + kTrsmI) ? kTrsmPipe : (kTrsmS + kTrsmI);

__global__ void __launch_bounds__(CfgT::THREADS) k_trsm_rows(TrsmRowsParams p) {
  extern __shared__ double smem[];
  double* sS = smem;
  double* sI = smem + kTrsmS;
  const int m0 = p.row0 + blockIdx.x * CfgT::BM;
  const int ld = p.ld;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int wm = (warp % CfgT::WARPS_M) * CfgT::WM;
  const int wn = (warp / CfgT::WARPS_M) * CfgT::WN;
  const int g = lane >> 2, t = lane & 3;
  for (int J = p.jb0; J < p.jb1; ++J) {
    const int c0 = J * kR;
    double acc[CfgT::FM][CfgT::FN][2];
    zero_acc<CfgT>(acc);
    if (J > p.jb0) {
      TileLoader<CfgT, M_MAJOR, CfgT::BM> la{p.B, ld, m0};
      TileLoader<CfgT, M_MAJOR, CfgT::BN> lb{p.L, ld, c0};
      gemm_mainloop<CfgT>(acc, smem, la, lb, p.jb0 * kR, c0);
    }
    // residual -> smem S[k][row]
    for_each_acc<CfgT>(acc, [&](int r, int c, double v) {
      sS[c * (CfgT::BM + 4) + r] = p.B[size_t(c0 + c) * ld + m0 + r] - v;
    });
    // inv(L_JJ): element (j, k) = inv(j, k), k < j stored at block (row k, col j)
    const double* Lb = p.L + size_t(c0) * ld + c0;
    for (int e = tid; e < kR * kR; e += CfgT::THREADS) {
      int j = e / kR, k = e % kR;
      double v;
      if (k < j) v = Lb[size_t(j) * ld + k];
      else if (k == j) v = 1.0 / Lb[size_t(j) * ld + j];
      else v = 0.0;
      sI[j * (kR + 4) + k] = v;
    }
    __syncthreads();
    // X(:, J) = S * inv^T : acc2(r, j) = sum_k S(r, k) inv(j, k)
    double acc2[CfgT::FM][CfgT::FN][2];
    zero_acc<CfgT>(acc2);
#pragma unroll 4
    for (int kk = 0; kk < kR; kk += 4) {
      double af[CfgT::FM], bf[CfgT::FN];
#pragma unroll
      for (int i = 0; i < CfgT::FM; ++i) af[i] = sS[(kk + t) * (CfgT::BM + 4) + wm + i * 8 + g];
#pragma unroll
      for (int j = 0; j < CfgT::FN; ++j) bf[j] = sI[(wn + j * 8 + g) * (kR + 4) + kk + t];
#pragma unroll
      for (int i = 0; i < CfgT::FM; ++i)
#pragma unroll
        for (int j = 0; j < CfgT::FN; ++j) dmma_8x8x4(acc2[i][j][0], acc2[i][j][1], af[i], bf[j]);
    }
    for_each_acc<CfgT>(acc2, [&](int r, int c, double v) { p.B[size_t(c0 + c) * ld + m0 + r] = v; });
    __threadfence();
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
static unsigned gemm_smem() { return (unsigned)GemmSmem<CfgG, M_MAJOR, M_MAJOR>::BYTES; }
static unsigned trsm_smem() { return (unsigned)(kTrsmSmemDoubles * sizeof(double)); }

bool init_chol_attributes() {
  if (cudaFuncSetAttribute(k_gemm_nt, cudaFuncAttributeMaxDynamicSharedMemorySize, gemm_smem()) != cudaSuccess)
    return false;
  if (cudaFuncSetAttribute(k_trsm_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, trsm_smem()) != cudaSuccess)
    return false;
  return true;
}

static void push_gemm(std::vector<LaunchDesc>& out, const double* A, const double* B, double* C,
                      int ld, int M, int N, int K, int lower) {
  LaunchDesc d;
  GemmNTParams p{A, B, C, ld, M, N, K, lower};
  d.set((const void*)k_gemm_nt, dim3(M / CfgG::BM, N / CfgG::BN), dim3(CfgG::THREADS), gemm_smem(), p);
  out.push_back(d);
}

static void push_trsm(std::vector<LaunchDesc>& out, const double* L, double* B, int ld, int row0, int nrows,
                      int jb0, int jb1) {
  LaunchDesc d;
  TrsmRowsParams p{L, B, ld, row0, jb0, jb1};
  d.set((const void*)k_trsm_rows, dim3(nrows / CfgT::BM), dim3(CfgT::THREADS), trsm_smem(), p);
  out.push_back(d);
}

bool build_chol_launches(int kind, const TaskOperands& o, std::vector<LaunchDesc>& out) {
  const int nb = o.nb;
  if (nb % kR != 0 || nb < kR) {
    set_error("Cholesky tile kernels need nb %% %d == 0, got nb=%d", kR, nb);
    return false;
  }
  const int nJ = nb / kR;
  switch (kind) {
    case K_POTRF: {
      double* A = o.t[0];
      for (int J = 0; J < nJ; ++J) {
        LaunchDesc d;
        PotrfDiagParams pd{A, nb, J * kR, o.status};
        d.set((const void*)k_potrf_diag, dim3(1), dim3(256), 0, pd);
        out.push_back(d);
        if (J + 1 < nJ) {
          const int r1 = (J + 1) * kR, rest = nb - r1;
          push_trsm(out, A, A, nb, r1, rest, J, J + 1);
          const double* panel = A + size_t(J) * kR * nb + r1;
          push_gemm(out, panel, panel, A + size_t(r1) * nb + r1, nb, rest, rest, kR, 1);
        }
      }
      return true;
    }
    case K_TRSM:
      push_trsm(out, o.t[0], o.t[1], nb, 0, nb, 0, nJ);
      return true;
    case K_SYRK:
      push_gemm(out, o.t[0], o.t[0], o.t[1], nb, nb, nb, nb, 1);
      return true;
    case K_GEMM:
      push_gemm(out, o.t[0], o.t[1], o.t[2], nb, nb, nb, nb, 0);
      return true;
    default:
      set_error("kind %d is not a Cholesky kind", kind);
      return false;
  }
}

}  // namespace hg
