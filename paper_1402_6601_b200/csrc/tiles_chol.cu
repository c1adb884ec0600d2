// Cholesky tile kernels for sm_100a: POTRF, TRSM, SYRK, GEMM
// (reference kinds: kernels.py:23-27, access lists kernels.py:126-137).
//
// Tiles are nb x nb FP64, column-major, ld = nb (PLASMA tile layout).
//
//   GEMM  A_ij -= A_ik * A_jk^T            k_gemm_nt (full)      DMMA 64x64 CTA tiles
//   SYRK  A_ii -= A_ik * A_ik^T  (lower)   k_gemm_nt (lower)     DMMA, upper CTAs exit
//   TRSM  A_ik  = A_ik * L_kk^-T           k_trsm_inv            DMMA product with M = L_kk^-1
//   POTRF A_kk  = L_kk (lower)             k_potrf_cluster: one 16-CTA cluster kernel,
//                                          r=64 right-looking blocked, lookahead diag,
//                                          also accumulates M = L_kk^-1 (upper triangle)
//
// POTRF leaves M^T = L_kk^-T in the strict upper triangle of the diagonal tile
// (the upper triangle of a Cholesky tile is never read by any other kind), so
// TRSM is a DMMA product instead of a substitution.  The upper triangle of
// diagonal tiles is therefore workspace, not input, after POTRF.
#include <cooperative_groups.h>

#include <cmath>
#include <utility>

#include "dgemm_dmma.cuh"
#include "tiles.h"

namespace cg = cooperative_groups;

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
  PushList push;  // producer-push destinations of C (runtime.cu), n = 0: none
};

using CfgG4 = GemmCfg<64, 64, 16, 32, 32, 4>;  // 4-stage ring, 3 CTAs / SM (default GEMM / SYRK tile)

template <class G = CfgG4, int MINB = 3>
__global__ void __launch_bounds__(G::THREADS, MINB) k_gemm_nt(const __grid_constant__ GemmNTParams p) {
  extern __shared__ double smem[];
  const int m0 = blockIdx.x * G::BM, n0 = blockIdx.y * G::BN;
  if (p.lower && m0 + G::BM - 1 < n0) return;  // tile strictly above the diagonal
  double acc[G::FM][G::FN][2];
  zero_acc<G>(acc);
  TileLoader<G, M_MAJOR, G::BM> la{p.A, p.ld, m0};
  TileLoader<G, M_MAJOR, G::BN> lb{p.B, p.ld, n0};
  gemm_mainloop<G>(acc, smem, la, lb, 0, p.K);
  sub_store<G>(acc, p.C, p.ld, m0, n0, p.lower != 0, false, p.push.n ? &p.push : nullptr);
}

// ---------------------------------------------------------------------------
// Unblocked Cholesky of the 64x64 diagonal block at (j0, j0) + its inverse,
// by one CTA of NT threads.  Writes L (lower) and inv(L)^T into the strict
// upper triangle of the block.  s is a [kR][kR+1] smem scratch (s[col][row]).
template <int NT>
__device__ void diag_factor_inverse(double* A, int ld, int j0, int* status, double (*s)[kR + 1],
                                    double* inv_diag) {
  double* blk = A + size_t(j0) * ld + j0;
  const int tid = threadIdx.x;
  for (int e = tid; e < kR * kR; e += NT) {
    int c = e / kR, r = e % kR;
    s[c][r] = __ldcg(blk + size_t(c) * ld + r);
  }
  __syncthreads();
  for (int j = 0; j < kR; ++j) {
    if (tid == 0) {
      double d = s[j][j];
      if (!(d > 0.0)) {
        if (status) atomicOr(status, 1);  // not positive definite
        d = 1.0;
      }
      d = sqrt(d);
      s[j][j] = d;
      inv_diag[j] = 1.0 / d;
    }
    __syncthreads();
    const double rd = inv_diag[j];
    for (int i = j + 1 + tid; i < kR; i += NT) s[j][i] *= rd;
    __syncthreads();
    // trailing update of columns c in (j, kR): s[c][i] -= s[j][i] * s[j][c], i >= c
    const int w = kR - j - 1;
    for (int e = tid; e < w * w; e += NT) {
      int c = j + 1 + e / w, i = j + 1 + e % w;
      if (i >= c) s[c][i] -= s[j][i] * s[j][c];
    }
    __syncthreads();
  }
  for (int e = tid; e < kR * kR; e += NT) {
    int c = e / kR, r = e % kR;
    if (r >= c) blk[size_t(c) * ld + r] = s[c][r];
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
    for (int i = c + 1; i < kR; ++i) blk[size_t(i) * ld + c] = x[i];
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Fast variant for 4 warps: the 64x64 block as a 2x2 recursion on 32x32
// leaves.  A leaf (Cholesky + inverse of a 32x32 block) runs in ONE warp with
// the block rows in registers and shuffles as the only communication (no
// __syncthreads inside); the off-diagonal products are spread over 128 threads.
//   L11, I11 = leaf(A11);  L21 = A21 I11^T;  A22 -= L21 L21^T;
//   L22, I22 = leaf(A22);  I21 = -I22 (L21 I11)
__device__ __noinline__ void leaf32(double* s, int lds, int r0, double* iv, int ldi, int* status) {
  // one warp; the 32x32 block stays in shared memory (B[c*lds + r] = element (r, c)),
  // loops stay rolled: small code, no local memory
  const int lane = threadIdx.x & 31;
  double* B = s + r0 * lds + r0;
  bool bad = false;
  for (int j = 0; j < 32; ++j) {
    double d = B[j * lds + j];
    if (!(d > 0.0)) {
      bad = true;
      d = 1.0;
    }
    d = sqrt(d);
    const double rd = 1.0 / d;
    const double lj = lane > j ? B[j * lds + lane] * rd : 0.0;
    __syncwarp();
    if (lane == j) B[j * lds + j] = d;
    if (lane > j) B[j * lds + lane] = lj;
    __syncwarp();
    for (int k = j + 1; k < 32; ++k) {
      const double lk = B[j * lds + k];
      if (lane >= k) B[k * lds + lane] = fma(-lj, lk, B[k * lds + lane]);
    }
    __syncwarp();
  }
  if (bad && lane == 0 && status) atomicOr(status, 1);
  // inverse: lane c computes column c of L^{-1} (stored iv[c*ldi + i] = inv(i, c))
  const int c = lane;
  double* x = iv + c * ldi;
  for (int i = 0; i < 32; ++i) {
    const double rli = 1.0 / B[i * lds + i];
    double v = 0.0;
    if (i == c) v = rli;
    else if (i > c) {
      double acc = 0.0;
      for (int k = c; k < i; ++k) acc = fma(B[k * lds + i], x[k], acc);
      v = -acc * rli;
    }
    x[i] = v;
  }
  __syncwarp();
}

// 32x32x32 product on DMMA by 4 warps (warp w owns the 16x16 quadrant
// (w&1, w>>1)); a(i, k), b(c, k) fetch operands, out(i, c, v) consumes results.
template <class FA, class FB, class FO>
__device__ __forceinline__ void mma32(FA a, FB b, FO out) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp >= 4) return;
  const int g = lane >> 2, t = lane & 3;
  const int i0 = (warp & 1) * 16, c0 = (warp >> 1) * 16;
  double acc[2][2][2] = {};
#pragma unroll
  for (int k0 = 0; k0 < 32; k0 += 4) {
    double af[2], bf[2];
#pragma unroll
    for (int m = 0; m < 2; ++m) af[m] = a(i0 + m * 8 + g, k0 + t);
#pragma unroll
    for (int n = 0; n < 2; ++n) bf[n] = b(c0 + n * 8 + g, k0 + t);
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int n = 0; n < 2; ++n) dmma_8x8x4(acc[m][n][0], acc[m][n][1], af[m], bf[n]);
  }
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int n = 0; n < 2; ++n) {
      out(i0 + m * 8 + g, c0 + n * 8 + 2 * t, acc[m][n][0]);
      out(i0 + m * 8 + g, c0 + n * 8 + 2 * t + 1, acc[m][n][1]);
    }
}

template <int NT>
__device__ void diag_factor_inverse_fast(double* A, int ld, int j0, int* status, double (*s)[kR + 1],
                                         double (*iv)[kR + 1], double (*tm)[33]) {
  double* blk = A + size_t(j0) * ld + j0;
  const int tid = threadIdx.x, warp = tid >> 5;
  double* S = &s[0][0];
  double* IV = &iv[0][0];
  constexpr int L = kR + 1;
  for (int e = tid; e < kR * kR; e += NT) {
    int c = e / kR, r = e % kR;
    s[c][r] = __ldcg(blk + size_t(c) * ld + r);
  }
  __syncthreads();
  if (warp == 0) leaf32(S, L, 0, IV, L, status);
  __syncthreads();
  // L21 = A21 I11^T : out(i, c) = sum_k A21(i, k) I11(c, k), I11(c, k) = iv[k][c]
  mma32([&](int i, int k) { return s[k][32 + i]; }, [&](int c, int k) { return iv[k][c]; },
        [&](int i, int c, double v) { tm[c][i] = v; });
  __syncthreads();
  for (int e = tid; e < 32 * 32; e += NT) s[e / 32][32 + e % 32] = tm[e / 32][e % 32];
  __syncthreads();
  // A22 -= L21 L21^T (lower)
  mma32([&](int i, int k) { return s[k][32 + i]; }, [&](int c, int k) { return s[k][32 + c]; },
        [&](int i, int c, double v) {
          if (i >= c) s[32 + c][32 + i] -= v;
        });
  __syncthreads();
  if (warp == 0) leaf32(S, L, 32, IV + 32 * L + 32, L, status);
  __syncthreads();
  // T = L21 I11 : T(i, c) = sum_k L21(i, k) I11(k, c), I11(k, c) = iv[c][k]
  mma32([&](int i, int k) { return s[k][32 + i]; }, [&](int c, int k) { return iv[c][k]; },
        [&](int i, int c, double v) { tm[c][i] = v; });
  __syncthreads();
  // I21 = -I22 T : I21(i, c) = -sum_k I22(i, k) T(k, c), I22(i, k) = iv[32 + k][32 + i]
  mma32([&](int i, int k) { return iv[32 + k][32 + i]; }, [&](int c, int k) { return tm[c][k]; },
        [&](int i, int c, double v) { iv[c][32 + i] = -v; });
  __syncthreads();
  // L (lower) and inv^T (strict upper: inv(i, c), i > c, at block (row c, col i))
  for (int e = tid; e < kR * kR; e += NT) {
    int c = e / kR, r = e % kR;
    if (r >= c) blk[size_t(c) * ld + r] = s[c][r];
    else blk[size_t(c) * ld + r] = iv[r][c];
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// 64x64 Cholesky + inverse by 128 threads, register resident.  Thread t owns
// row i = t/2, columns k = 2m + (t&1) (m < 32) of both A (-> L) and R (-> X =
// L^{-1}; R = I initially).  Per column j, two barriers:
//   1: column-j owners scale L(i, j) = A(i, j) / sqrt(A(j, j)) and publish it;
//      the two owners of row j publish X(j, :) = R(j, :) / L(j, j)
//   2: every thread updates its registers from the published column / row
//      (independent smem loads), the owner of (j+1, j+1) publishes the next pivot.
// Broadcast buffers are double-buffered by column parity.
__device__ void diag64_reg(double* A, int ld, int j0, int* status, double* bufs) {
  double* blk = A + size_t(j0) * ld + j0;
  const int tid = threadIdx.x;
  const int i = tid >> 1, h = tid & 1;
  double* colj = bufs;              // [2][64]
  double* rowx = bufs + 2 * kR;     // [2][64]
  double* diag = bufs + 4 * kR;     // [2]
  double a[32], r[32];
#pragma unroll
  for (int m = 0; m < 32; ++m) {
    const int k = 2 * m + h;
    a[m] = (k <= i) ? __ldcg(blk + size_t(k) * ld + i) : 0.0;
    r[m] = (k == i) ? 1.0 : 0.0;
  }
  if (tid == 0) diag[0] = a[0];
  bool bad = false;
  __syncthreads();
  for (int j = 0; j < kR; ++j) {
    const int par = j & 1;
    double djj = diag[par];
    if (!(djj > 0.0)) {
      bad = true;
      djj = 1.0;
    }
    const double rj = rsqrt(djj);
    if (h == (j & 1)) {
#pragma unroll
      for (int m = 0; m < 32; ++m)
        if (2 * m + h == j) {
          if (i > j) {
            a[m] *= rj;
            colj[par * kR + i] = a[m];
          } else if (i == j) {
            a[m] = djj * rj;
          }
        }
    }
    if (i == j) {
#pragma unroll
      for (int m = 0; m < 32; ++m)
        if (2 * m + h <= j) {
          r[m] *= rj;
          rowx[par * kR + 2 * m + h] = r[m];
        }
    }
    __syncthreads();
    if (i > j) {
      // one base register + immediate offsets, unconditional loads, selects: the
      // upper part (k > i) of a[] is never read back, so only k > j matters
      const double li = colj[par * kR + i];
      const double* cb = colj + par * kR + h;
      const double* rb = rowx + par * kR + h;
#pragma unroll
      for (int m = 0; m < 32; ++m) {
        const double cv = cb[2 * m], rv = rb[2 * m];
        const bool up = (2 * m + h) > j;
        const double am = fma(-li, cv, a[m]), rm = fma(-li, rv, r[m]);
        a[m] = up ? am : a[m];
        r[m] = up ? r[m] : rm;
      }
    }
    if (i == j + 1 && h == ((j + 1) & 1)) {
#pragma unroll
      for (int m = 0; m < 32; ++m)
        if (2 * m + h == j + 1) diag[par ^ 1] = a[m];
    }
    __syncthreads();
  }
  if (bad && tid == 0 && status) atomicOr(status, 1);
  // L (lower) and X^T in the strict upper triangle: position (row c, col i) <- X(i, c), c < i
#pragma unroll
  for (int m = 0; m < 32; ++m) {
    const int k = 2 * m + h;
    if (k <= i) blk[size_t(k) * ld + i] = a[m];
    if (k < i) blk[size_t(i) * ld + k] = r[m];
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// 64x64 Cholesky + inverse by 128 threads, register resident, with the column
// loop FULLY UNROLLED so every register index is a compile-time constant (the
// runtime-j variant above pays ~1100 instructions per column in index
// selects and divergent branches).  Thread t owns row i = t/2 and columns
// k = 2m + (t&1) of A (-> L) and R (-> X = L^-1, R = I initially).  ONE
// barrier per column: at the end of step j the owners of column j+1 publish
// it, and the two owners of row j+1 of R publish that row (both final after
// step j), into the buffer of the other parity; step j+1 then reads
//   d = A(j+1, j+1), A(i, j+1), A(k, j+1), R(j+1, k)
// and updates its registers with no further synchronisation.
template <int J>
__device__ __forceinline__ void diag64_step(double (&a)[32], double (&r)[32], double* colb, double* rowb, int i, int h,
                                            bool& bad) {
  constexpr int par = J & 1;
  const double* cj = colb + par * kR;
  const double* rj = rowb + par * kR;
  double d = cj[J];
  if (!(d > 0.0)) {
    bad = true;
    d = 1.0;
  }
  const double rs = rsqrt(d);
  const double lij = cj[i] * rs;  // L(i, J) (meaningful for i > J)
  const bool below = i > J, diag = i == J;
#pragma unroll
  for (int m = 0; m < 32; ++m) {
    const int k = 2 * m + h;
    if (2 * m > J) {  // k > J: trailing column of A
      a[m] = fma(-lij, cj[k] * rs, a[m]);
    } else if (2 * m + 1 < J) {  // k < J: R columns of earlier pivots
      const double x = rj[k] * rs;
      r[m] = below ? fma(-lij, x, r[m]) : (diag ? x : r[m]);
    } else {  // the pair {2m, 2m+1} holds column J
      if (k == J) {
        a[m] = below ? lij : (diag ? d * rs : a[m]);
        const double x = rj[k] * rs;
        r[m] = below ? fma(-lij, x, r[m]) : (diag ? x : r[m]);
      } else if (k > J) {
        a[m] = fma(-lij, cj[k] * rs, a[m]);
      } else {
        const double x = rj[k] * rs;
        r[m] = below ? fma(-lij, x, r[m]) : (diag ? x : r[m]);
      }
    }
  }
  if constexpr (J + 1 < kR) {
    double* cn = colb + (par ^ 1) * kR;
    double* rn = rowb + (par ^ 1) * kR;
    constexpr int mn = (J + 1) >> 1;
    if (h == ((J + 1) & 1)) cn[i] = a[mn];
    if (i == J + 1) {
#pragma unroll
      for (int m = 0; m < 32; ++m)
        if (2 * m <= J + 1 && 2 * m + h <= J + 1) rn[2 * m + h] = r[m];
    }
  }
  __syncthreads();
}

template <int... Js>
__device__ __forceinline__ void diag64_steps(double (&a)[32], double (&r)[32], double* colb, double* rowb, int i,
                                             int h, bool& bad, std::integer_sequence<int, Js...>) {
  (diag64_step<Js>(a, r, colb, rowb, i, h, bad), ...);
}

// ---------------------------------------------------------------------------
// 64x64 Cholesky + inverse by 128 threads, register resident, with the column
// loop unrolled at compile time (diag64_step<J>) so every register index is a
// constant (the runtime-j variant above pays ~1100 instructions per column in
// index selects and divergent branches; a shifted-window runtime loop was
// measured 4x slower still).  Thread t owns row i = t/2 and columns
// k = 2m + (t&1) of A (-> L) and R (-> X = L^-1, R = I initially).  ONE
// barrier per column: at the end of step j the owners of column j+1 publish
// it and the two owners of row j+1 of R publish that row (both final after
// step j) into the buffer of the other parity; step j+1 then reads
// d = A(j+1, j+1), A(i, j+1), A(k, j+1), R(j+1, k) with no further barrier.
// Measured (tools/potrf_micro): 94 us -> 57 us per 64x64 block.
__device__ __noinline__ void diag64_fast(double* A, int ld, int j0, int* status, double* bufs) {
  double* blk = A + size_t(j0) * ld + j0;
  const int tid = threadIdx.x;
  const int i = tid >> 1, h = tid & 1;
  double* colb = bufs;           // [2][64]: column j of A
  double* rowb = bufs + 2 * kR;  // [2][64]: row j of R (unscaled)
  double a[32], r[32];
#pragma unroll
  for (int m = 0; m < 32; ++m) {
    const int k = 2 * m + h;
    a[m] = (k <= i) ? __ldcg(blk + size_t(k) * ld + i) : 0.0;
    r[m] = (k == i) ? 1.0 : 0.0;
  }
  if (h == 0) colb[i] = a[0];
  if (tid == 0) rowb[0] = 1.0;
  bool bad = false;
  __syncthreads();
  diag64_steps(a, r, colb, rowb, i, h, bad, std::make_integer_sequence<int, kR>{});
  if (bad && tid == 0 && status) atomicOr(status, 1);
#pragma unroll
  for (int m = 0; m < 32; ++m) {
    const int k = 2 * m + h;
    if (k <= i) blk[size_t(k) * ld + i] = a[m];
    if (k < i) blk[size_t(i) * ld + k] = r[m];
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// 64x64 Cholesky + inverse, BLOCKED (4 x 16-column blocks) so the serial
// part is a 16-column warp leaf and everything else is DMMA:
//   for J in 0..3:
//     leaf (warp 0, registers + shuffles): L_JJ, T = L_JJ^-1      (16 serial columns)
//     L(I,J) = A(I,J) T^T (I > J);  M(J,K) <- T M(J,K) (K < J), M(J,J) = T     (DMMA)
//     A(I,K) -= L(I,J) L(K,J)^T (J < K <= I);  M(I,K) -= L(I,J) M(J,K) (K <= J)  (DMMA)
// with M = L^-1 accumulated exactly as the cluster kernel does per 64-block.
// The 64 serial columns of the unblocked variants (~1700 cycles each) become
// 4 leaves of 16 columns plus 8 small DMMA products.
constexpr int kBL = 68;  // smem column stride (conflict-free DMMA fragment loads)

// C(8x8 tile at (r0, c0)) op= sum_k A(r0+i, k) * B(c0+j, k) over k in [0, K) (K % 4 == 0),
// operands fetched by functors fa(row, k), fb(col, k).
template <class FA, class FB>
__device__ __forceinline__ void tile8_dmma(double& c0, double& c1, int K, FA&& fa, FB&& fb) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  for (int k0 = 0; k0 < K; k0 += 4) dmma_8x8x4(c0, c1, fa(g, k0 + t), fb(g, k0 + t));
}

// One column step of the warp leaf (J compile-time, so a[] / r[] stay in registers).
template <int J>
__device__ __forceinline__ void leaf16_step(double (&a)[16], double (&r)[16], int i, bool& ok) {
  double d = __shfl_sync(0xffffffffu, a[J], J);
  if (!(d > 0.0)) {
    ok = false;
    d = 1.0;
  }
  const double rs = rsqrt(d);
  const double lij = a[J] * rs;  // L(i, J) for i > J
  if (i > J) a[J] = lij;
  else if (i == J) a[J] = d * rs;
#pragma unroll
  for (int k = J + 1; k < 16; ++k) {
    const double lkj = __shfl_sync(0xffffffffu, a[J], k);  // L(k, J) (lane k, already scaled)
    if (i >= k) a[k] = fma(-lij, lkj, a[k]);
  }
#pragma unroll
  for (int k = 0; k <= J; ++k) {
    const double xjk = __shfl_sync(0xffffffffu, r[k], J) * rs;  // X(J, k) = R(J, k) / L(J, J)
    if (i > J) r[k] = fma(-lij, xjk, r[k]);
    else if (i == J) r[k] = xjk;
  }
}

template <int... Js>
__device__ __forceinline__ void leaf16_steps(double (&a)[16], double (&r)[16], int i, bool& ok,
                                             std::integer_sequence<int, Js...>) {
  (leaf16_step<Js>(a, r, i, ok), ...);
}

// Warp-level 16x16 Cholesky + inverse: lanes 0..15 own the rows (16..31 mirror them).
// In: sA block (lower).  Out: L in sA (lower), T = L^-1 in sT[c*17 + r] (lower).
// Returns false on a non-positive pivot.
__device__ __forceinline__ bool leaf16(double* sA, int r0, double* sT) {
  const int lane = threadIdx.x & 31;
  const int i = lane & 15;
  double a[16], r[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    a[k] = (k <= i) ? sA[(r0 + k) * kBL + r0 + i] : 0.0;
    r[k] = (k == i) ? 1.0 : 0.0;
  }
  bool ok = true;
  leaf16_steps(a, r, i, ok, std::make_integer_sequence<int, 16>{});
  if (lane < 16) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (k <= i) sA[(r0 + k) * kBL + r0 + i] = a[k];
      sT[k * 17 + i] = (k <= i) ? r[k] : 0.0;
    }
  }
  return ok;
}

__device__ __noinline__ void diag64_blocked(double* A, int ld, int j0, int* status, double* work) {
  double* blk = A + size_t(j0) * ld + j0;
  double* sA = work;               // [64][kBL]: A -> L, sA[c*kBL + r]
  double* sM = work + kR * kBL;    // [64][kBL]: M = L^-1
  double* sT = sM + kR * kBL;      // [16][17]: leaf inverse
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  constexpr int NW = CfgG::THREADS / 32;
  // the whole 64x64 block with cp.async (16-byte chunks of a column), so all the
  // L2 round trips overlap; the strict upper part is never read as L
  for (int e = tid; e < kR * (kR / 2); e += CfgG::THREADS) {
    const int c = e / (kR / 2), r = (e % (kR / 2)) * 2;
    cp_async16(sA + c * kBL + r, blk + size_t(c) * ld + r);
  }
  cp_async_commit();
  for (int e = tid; e < kR * kR; e += CfgG::THREADS) {
    const int c = e / kR, r = e % kR;
    sM[c * kBL + r] = (r == c) ? 1.0 : 0.0;
  }
  cp_async_wait<0>();
  __syncthreads();
  bool ok = true;
  for (int J = 0; J < 4; ++J) {
    const int b0 = 16 * J;
    if (warp == 0) ok = leaf16(sA, b0, sT) && ok;
    __syncthreads();
    // ---- L(I,J) = A(I,J) T^T for rows [b0+16, 64); M(J,K) <- T M(J,K), M(J,J) = T ----------
    {
      const int nr = (kR - b0 - 16) / 8;  // 8-row tiles below the block
      const int n_panel = nr * 2;           // x 2 column tiles
      const int n_mrow = 2 * (b0 / 8);      // M(J, K<J): 2 row tiles x b0/8 column tiles
      double acc[4][2];
      int tiles[4];
      int nt = 0;
      for (int w = warp; w < n_panel + n_mrow; w += NW) {
        double c0 = 0.0, c1 = 0.0;
        if (w < n_panel) {
          const int r0 = b0 + 16 + (w >> 1) * 8, cc = (w & 1) * 8;
          tile8_dmma(c0, c1, 16, [&](int gg, int k) { return sA[(b0 + k) * kBL + r0 + gg]; },
                     [&](int gg, int k) { return sT[k * 17 + cc + gg]; });  // T^T(k, c) = T(c, k)
        } else {
          const int w2 = w - n_panel;
          const int rr = (w2 & 1) * 8, c0m = (w2 >> 1) * 8;
          tile8_dmma(c0, c1, 16, [&](int gg, int k) { return sT[k * 17 + rr + gg]; },           // T(r, k)
                     [&](int gg, int k) { return sM[(c0m + gg) * kBL + b0 + k]; });         // M(b0+k, c)
        }
        acc[nt][0] = c0;
        acc[nt][1] = c1;
        tiles[nt++] = w;
      }
      __syncthreads();
      for (int q2 = 0; q2 < nt; ++q2) {
        const int w = tiles[q2];
        if (w < n_panel) {
          const int r0 = b0 + 16 + (w >> 1) * 8, cc = b0 + (w & 1) * 8;
          sA[(cc + 2 * t) * kBL + r0 + g] = acc[q2][0];
          sA[(cc + 2 * t + 1) * kBL + r0 + g] = acc[q2][1];
        } else {
          const int w2 = w - n_panel;
          const int rr = b0 + (w2 & 1) * 8, c0m = (w2 >> 1) * 8;
          sM[(c0m + 2 * t) * kBL + rr + g] = acc[q2][0];
          sM[(c0m + 2 * t + 1) * kBL + rr + g] = acc[q2][1];
        }
      }
      // M(J,J) = T
      for (int e = tid; e < 256; e += CfgG::THREADS) {
        const int c = e >> 4, r = e & 15;
        sM[(b0 + c) * kBL + b0 + r] = sT[c * 17 + r];
      }
    }
    __syncthreads();
    if (J == 3) break;
    // ---- trailing: A(r,c) -= L(r,J) L(c,J)^T (c <= r, both >= b0+16); M(r,K) -= L(r,J) M(J,K) --------
    {
      const int m0 = b0 + 16;
      const int nt8 = (kR - m0) / 8;
      const int n_tr = nt8 * (nt8 + 1) / 2;  // lower tiles incl. diagonal tiles
      const int n_mu = nt8 * ((b0 + 16) / 8);
      // outputs (columns / rows >= m0) are disjoint from the inputs (block column / row J): write in place
      for (int w = warp; w < n_tr + n_mu; w += NW) {
        double c0 = 0.0, c1 = 0.0;
        if (w < n_tr) {
          int ti = 0, rem = w;
          while (rem > ti) { rem -= ti + 1; ++ti; }  // (ti, tj = rem), tj <= ti
          const int r0 = m0 + ti * 8, cl0 = m0 + rem * 8;
          tile8_dmma(c0, c1, 16, [&](int gg, int k) { return sA[(b0 + k) * kBL + r0 + gg]; },
                     [&](int gg, int k) { return sA[(b0 + k) * kBL + cl0 + gg]; });
          sA[(cl0 + 2 * t) * kBL + r0 + g] -= c0;
          sA[(cl0 + 2 * t + 1) * kBL + r0 + g] -= c1;
        } else {
          const int w2 = w - n_tr;
          const int ti = w2 % nt8, tj = w2 / nt8;
          const int r0 = m0 + ti * 8, cm = tj * 8;
          tile8_dmma(c0, c1, 16, [&](int gg, int k) { return sA[(b0 + k) * kBL + r0 + gg]; },  // L(r, b0+k)
                     [&](int gg, int k) { return sM[(cm + gg) * kBL + b0 + k]; });           // M(b0+k, c)
          sM[(cm + 2 * t) * kBL + r0 + g] -= c0;
          sM[(cm + 2 * t + 1) * kBL + r0 + g] -= c1;
        }
      }
    }
    __syncthreads();
  }
  if (!ok && tid == 0 && status) atomicOr(status, 1);
  // L (lower) and M^T into the strict upper triangle: (row c, col i) <- M(i, c), c < i
  for (int e = tid; e < kR * kR; e += CfgG::THREADS) {
    const int c = e / kR, r = e % kR;
    if (r >= c) blk[size_t(c) * ld + r] = sA[c * kBL + r];
    else blk[size_t(c) * ld + r] = sM[r * kBL + c];
  }
  __syncthreads();
}

struct PotrfDiagParams {
  double* A;
  int ld, j0;
  int* status;
};

__global__ void __launch_bounds__(256) k_potrf_diag(PotrfDiagParams p) {
  __shared__ double s[kR][kR + 1];
  __shared__ double inv_diag[kR];
  diag_factor_inverse<256>(p.A, p.ld, p.j0, p.status, s, inv_diag);
}

// ---------------------------------------------------------------------------
// POTRF of a whole nb x nb tile as ONE thread-block-cluster kernel (16 CTAs,
// non-portable size), r = 64 right-looking blocked Cholesky that ALSO
// accumulates M = L^{-1} (stored transposed in the tile's strict upper
// triangle, diagonal implicit 1/L(j,j)) so that every TRSM of this column is
// a plain DMMA product X = B M^T.  Per step J (cluster barriers between):
//   P: L(I,J) = A(I,J) inv(L_JJ)^T (I > J)   and   M(J,K) <- inv(L_JJ) M(J,K) (K < J)
//   U: A(I,K) -= L(I,J) L(K,J)^T (J < K <= I) and   M(I,K) -= L(I,J) M(J,K) (I > J, K <= J)
// CTA 0 updates the next diagonal block first and factors it (lookahead) while
// the other CTAs finish U.  M starts as the identity, so M(I,J) for K == J is
// initialised (=) instead of accumulated.
constexpr int kPotrfCl = 16;

struct PotrfParams {
  double* A;
  int nb;
  int* status;
  PushList push;  // producer-push: the finished tile is also copied to these slots
};

constexpr int kSolveS = kR * (kR + 4);
constexpr int kPotrfSmemDoubles =
    (2 * kSolveS > GemmSmem<CfgG, M_MAJOR, M_MAJOR>::DOUBLES) ? 2 * kSolveS : GemmSmem<CfgG, M_MAJOR, M_MAJOR>::DOUBLES;
constexpr int kPotrfDynDoubles = kPotrfSmemDoubles + 2 * kR * (kR + 1) + 32 * 33;

// blk (64x64, ld) <- blk * inv(L_JJ)^T in place; inv(L_JJ)(j, k), k < j, sits at
// diagonal-block position (row k, col j), its diagonal is 1/L(j, j).
__device__ void apply_inv_right(double* blk, int ld, const double* Lb, double* smem) {
  double* sS = smem;            // [k][row], ld kR+4
  double* sI = smem + kSolveS;  // [j][k],  ld kR+4
  const int tid = threadIdx.x;
  // both 64x64 blocks are column-contiguous in global: stage them with cp.async
  for (int e = tid; e < kR * (kR / 2); e += CfgG::THREADS) {
    int c = e / (kR / 2), r = (e % (kR / 2)) * 2;
    cp_async16(sS + c * (kR + 4) + r, blk + size_t(c) * ld + r);
    cp_async16(sI + c * (kR + 4) + r, Lb + size_t(c) * ld + r);  // row j=c holds inv(j, k<j) at k=r
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  // the raw rows hold L(k, j) for k >= j: diagonal -> 1/L(j, j), below -> 0
  for (int e = tid; e < kR * kR; e += CfgG::THREADS) {
    int j = e / kR, k = e % kR;
    if (k >= j) {
      double* q = sI + j * (kR + 4) + k;
      *q = (k == j) ? 1.0 / *q : 0.0;
    }
  }
  __syncthreads();
  const int warp = tid >> 5, lane = tid & 31;
  const int wm = (warp % CfgG::WARPS_M) * CfgG::WM;
  const int wn = (warp / CfgG::WARPS_M) * CfgG::WN;
  const int g = lane >> 2, t = lane & 3;
  double acc[CfgG::FM][CfgG::FN][2];
  zero_acc<CfgG>(acc);
#pragma unroll 4
  for (int kk = 0; kk < kR; kk += 4) {
    double af[CfgG::FM], bf[CfgG::FN];
#pragma unroll
    for (int i = 0; i < CfgG::FM; ++i) af[i] = sS[(kk + t) * (kR + 4) + wm + i * 8 + g];
#pragma unroll
    for (int j = 0; j < CfgG::FN; ++j) bf[j] = sI[(wn + j * 8 + g) * (kR + 4) + kk + t];
#pragma unroll
    for (int i = 0; i < CfgG::FM; ++i)
#pragma unroll
      for (int j = 0; j < CfgG::FN; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
  }
  for_each_acc<CfgG>(acc, [&](int r, int c, double v) { blk[size_t(c) * ld + r] = v; });
  __syncthreads();
}

// inv(L_JJ)^T as an M_MAJOR operand: element (r, k) = inv(k, r): k > r stored at
// (row r, col k), k == r -> 1/L(r, r), k < r -> 0
template <class Cfg, int ROWS>
struct InvTLoader {
  static constexpr int layout = M_MAJOR;
  static constexpr int rows = ROWS;
  const double* blk;  // diagonal block base, ld
  int ld;
  HG_DEVICE void load(double* s, int k0) const {
    for (int e = threadIdx.x; e < ROWS * Cfg::BK; e += Cfg::THREADS) {
      int kk = e / ROWS, rr = e % ROWS;
      int k = k0 + kk;
      double v;
      if (k > rr) v = __ldcg(blk + size_t(k) * ld + rr);
      else if (k == rr) v = 1.0 / __ldcg(blk + size_t(rr) * ld + rr);
      else v = 0.0;
      s[kk * (ROWS + Cfg::PAD) + rr] = v;
    }
  }
};

// C(64x64 at Cp, ld) (-)= A_op * B_op^T, optional lower mask / initialisation
template <class LdA, class LdB>
__device__ void block_update(double* Cp, int ld, const LdA& la, const LdB& lb, bool lower, bool init,
                             double* smem) {
  double acc[CfgG::FM][CfgG::FN][2];
  zero_acc<CfgG>(acc);
  gemm_mainloop<CfgG>(acc, smem, la, lb, 0, kR);
  sub_store<CfgG>(acc, Cp, ld, 0, 0, lower, init);
  __syncthreads();
}

__global__ void __cluster_dims__(kPotrfCl, 1, 1) __launch_bounds__(CfgG::THREADS) k_potrf_cluster(const __grid_constant__ PotrfParams p) {
  extern __shared__ double smem[];
  // dynamic smem: [GEMM ring / solve buffers | s 64x65 | iv 64x65 | tm 32x33]
  auto s = reinterpret_cast<double(*)[kR + 1]>(smem + kPotrfSmemDoubles);
  auto iv = reinterpret_cast<double(*)[kR + 1]>(smem + kPotrfSmemDoubles + kR * (kR + 1));
  auto tm = reinterpret_cast<double(*)[33]>(smem + kPotrfSmemDoubles + 2 * kR * (kR + 1));
  cg::cluster_group cl = cg::this_cluster();
  const int q = (int)cl.block_rank();
  const int nb = p.nb, nJ = nb / kR, ld = nb;
  double* A = p.A;
  auto blk = [&](int I, int K) { return A + size_t(K) * kR * ld + size_t(I) * kR; };  // block (I, K)
  if (q == 0) diag64_blocked(A, nb, 0, p.status, &s[0][0]);
  __threadfence();
  cl.sync();
  for (int J = 0; J < nJ; ++J) {
    // ---- P: panel solve (I > J) and M row scaling (K < J): nJ-1 tasks -------------
    for (int t = q; t < nJ - 1; t += kPotrfCl) {
      if (t < nJ - 1 - J) apply_inv_right(blk(J + 1 + t, J), ld, blk(J, J), smem);
      else apply_inv_right(blk(t - (nJ - 1 - J), J), ld, blk(J, J), smem);  // upper block (K, J) = M(J,K)^T
    }
    __threadfence();
    cl.sync();
    if (J + 1 == nJ) break;
    // ---- U: trailing lower tiles + M accumulation tiles ----------------------------
    if (q == 0) {
      TileLoader<CfgG, M_MAJOR, kR> la{blk(0, J), ld, (J + 1) * kR};
      block_update(blk(J + 1, J + 1), ld, la, la, true, false, smem);
      __threadfence();
      diag64_blocked(A, nb, (J + 1) * kR, p.status, &s[0][0]);
    } else {
      int t = 0;
      const int others = kPotrfCl - 1;
      // (iii) A(I,K) -= L(I,J) L(K,J)^T, J < K <= I, skipping (J+1, J+1)
      for (int I = J + 1; I < nJ; ++I)
        for (int K = J + 1; K <= I; ++K) {
          if (I == J + 1 && K == J + 1) continue;
          if (t++ % others != q - 1) continue;
          TileLoader<CfgG, M_MAJOR, kR> la{blk(0, J), ld, I * kR};
          TileLoader<CfgG, M_MAJOR, kR> lb{blk(0, J), ld, K * kR};
          block_update(blk(I, K), ld, la, lb, I == K, false, smem);
        }
      // (iv) M(I,K)^T (upper block (K, I)) -= M(J,K)^T L(I,J)^T, I > J, K <= J
      for (int I = J + 1; I < nJ; ++I)
        for (int K = 0; K <= J; ++K) {
          if (t++ % others != q - 1) continue;
          TileLoader<CfgG, M_MAJOR, kR> lb{blk(0, J), ld, I * kR};
          if (K == J) {
            InvTLoader<CfgG, kR> la{blk(J, J), ld};
            block_update(blk(K, I), ld, la, lb, false, true, smem);
          } else {
            TileLoader<CfgG, M_MAJOR, kR> la{blk(0, J), ld, K * kR};  // upper block (K, J) rows
            block_update(blk(K, I), ld, la, lb, false, false, smem);
          }
        }
    }
    __threadfence();
    cl.sync();
  }
  // producer-push: the finished tile (L_kk and M^T) streamed to the consumer GPUs' slots by the
  // cluster that produced it (the last phase ended with a release/acquire cluster barrier)
  if (p.push.n) {
    const size_t n2 = size_t(nb) * nb / 2;
    const double2* src = reinterpret_cast<const double2*>(A);
    for (size_t e = size_t(q) * CfgG::THREADS + threadIdx.x; e < n2; e += size_t(kPotrfCl) * CfgG::THREADS) {
      const double2 v = __ldcg(src + e);
      for (int d = 0; d < p.push.n; ++d) __stcg(reinterpret_cast<double2*>(p.push.dst[d]) + e, v);
    }
  }
}

// ---------------------------------------------------------------------------
// TRSM  B <- B L^{-T} = B M^T with M = L^{-1} from POTRF (upper triangle of the
// diagonal tile, transposed; diagonal 1/L(j,j)).  A plain DMMA product per
// 64x64 block X(I, J) = sum_{K <= J} B(I, K) M(J, K)^T.  In place: X(I, J)
// may only be written once every CTA of row strip I has finished reading B,
// so each CTA computes two blocks (J, nJ-1-J: equal work), then meets the
// other CTAs of its strip at a cluster barrier, then writes.  The P CTAs of a
// strip form one thread-block cluster, which the hardware makes co-resident
// all-or-nothing: a global-memory strip barrier could deadlock once many TRSMs
// run at once (63 concurrent TRSMs at N=65536 leave every SM slot spinning on a
// strip whose remaining CTAs cannot be scheduled).
struct TrsmInvParams {
  const double* L;  // diagonal tile after POTRF (M^T in its upper triangle)
  double* B;
  int* count;       // unused (the strip barrier is a cluster barrier); kept for the param layout
  int ld;
  PushList push;    // producer-push destinations of B
};

template <class Cfg, int ROWS>
struct MRowLoader {  // rows j in [j0, j0+ROWS): element (j, k) = M(j, k)
  static constexpr int layout = K_MAJOR;
  static constexpr int rows = ROWS;
  const double* L;
  int ld, j0;
  HG_DEVICE void load(double* s, int k0) const {
    if (k0 + Cfg::BK <= j0) {  // strictly left of the diagonal block: plain upper-triangle rows
      load_slab<Cfg, K_MAJOR, ROWS>(s, L, ld, j0, k0);
      return;
    }
    for (int e = threadIdx.x; e < ROWS * Cfg::BK; e += Cfg::THREADS) {
      int rr = e / Cfg::BK, kk = e % Cfg::BK;
      int j = j0 + rr, k = k0 + kk;
      double v;
      if (k < j) v = __ldcg(L + size_t(j) * ld + k);
      else if (k == j) v = 1.0 / __ldcg(L + size_t(j) * ld + j);
      else v = 0.0;
      s[Cfg::kmaj(rr, kk)] = v;
    }
  }
};

template <int P>
__global__ void __cluster_dims__(P, 1, 1) __launch_bounds__(CfgG::THREADS, 3) k_trsm_inv(const __grid_constant__ TrsmInvParams p) {
  extern __shared__ double smem[];
  const int ld = p.ld, nJ = ld / kR;
  // strip-major ids: the P CTAs of row strip I are one cluster (rank = pair)
  const int I = blockIdx.x / P, pair = blockIdx.x % P;
  const int Js[2] = {pair, nJ - 1 - pair};
  double acc0[CfgG::FM][CfgG::FN][2], acc1[CfgG::FM][CfgG::FN][2];
  zero_acc<CfgG>(acc0);
  zero_acc<CfgG>(acc1);
  TileLoader<CfgG, M_MAJOR, kR> la{p.B, ld, I * kR};
  {
    MRowLoader<CfgG, kR> lb{p.L, ld, Js[0] * kR};
    gemm_mainloop<CfgG>(acc0, smem, la, lb, 0, (Js[0] + 1) * kR);
  }
  {
    MRowLoader<CfgG, kR> lb{p.L, ld, Js[1] * kR};
    gemm_mainloop<CfgG>(acc1, smem, la, lb, 0, (Js[1] + 1) * kR);
  }
  // all reads of B by this CTA are complete (mainloop ends with wait_group 0 + barrier);
  // the cluster barrier (release / acquire) extends that to the whole strip
  cg::this_cluster().sync();
  double* B = p.B;
  const int np = p.push.n;
  for_each_acc<CfgG>(acc0, [&](int r, int c, double v) {
    const size_t o = size_t(Js[0] * kR + c) * ld + I * kR + r;
    B[o] = v;
    for (int d = 0; d < np; ++d) __stcg(p.push.dst[d] + o, v);
  });
  for_each_acc<CfgG>(acc1, [&](int r, int c, double v) {
    const size_t o = size_t(Js[1] * kR + c) * ld + I * kR + r;
    B[o] = v;
    for (int d = 0; d < np; ++d) __stcg(p.push.dst[d] + o, v);
  });
}

// ---------------------------------------------------------------------------
static unsigned trsm_smem() { return (unsigned)GemmSmem<CfgG, M_MAJOR, K_MAJOR>::BYTES; }

#define HG_ATTR(fn, attr, val)                                                                   \
  do {                                                                                           \
    cudaError_t e_ = cudaFuncSetAttribute(fn, attr, val);                                        \
    if (e_ != cudaSuccess) {                                                                     \
      set_error("cudaFuncSetAttribute(%s, %s, %d): %s", #fn, #attr, int(val), cudaGetErrorString(e_)); \
      return false;                                                                              \
    }                                                                                            \
  } while (0)

bool init_chol_attributes() {
  HG_ATTR((k_gemm_nt<CfgG4, 3>), cudaFuncAttributeMaxDynamicSharedMemorySize,
          (int)(GemmSmem<CfgG4, M_MAJOR, M_MAJOR>::BYTES));
  HG_ATTR(k_trsm_inv<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, trsm_smem());
  HG_ATTR(k_trsm_inv<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, trsm_smem());
  HG_ATTR(k_trsm_inv<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, trsm_smem());
  HG_ATTR(k_trsm_inv<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, trsm_smem());
  HG_ATTR(k_trsm_inv<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, trsm_smem());
  HG_ATTR(k_trsm_inv<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, trsm_smem());
  HG_ATTR(k_trsm_inv<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, trsm_smem());
  HG_ATTR(k_trsm_inv<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, trsm_smem());
  HG_ATTR(k_potrf_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kPotrfDynDoubles * sizeof(double)));
  HG_ATTR(k_potrf_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  return true;
}

static void push_gemm(std::vector<LaunchDesc>& out, const double* A, const double* B, double* C,
                      int ld, int M, int N, int K, int lower, const PushList& push) {
  LaunchDesc d;
  GemmNTParams p{A, B, C, ld, M, N, K, lower, push};
  d.set((const void*)k_gemm_nt<CfgG4, 3>, dim3(M / CfgG4::BM, N / CfgG4::BN), dim3(CfgG4::THREADS),
        (unsigned)GemmSmem<CfgG4, M_MAJOR, M_MAJOR>::BYTES, p);
  out.push_back(d);
}

int chol_scratch_ints(int kind, int nb) {
  (void)kind;
  (void)nb;
  return 0;  // the TRSM strip barrier is a cluster barrier: no per-task counters
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
      LaunchDesc d;
      PotrfParams pp{o.t[0], nb, o.status, o.push};
      d.set((const void*)k_potrf_cluster, dim3(kPotrfCl), dim3(CfgG::THREADS),
            unsigned(kPotrfDynDoubles * sizeof(double)), pp);
      out.push_back(d);
      return true;
    }
    case K_TRSM: {
      const int P = nJ / 2;  // CTAs per row strip = cluster size (portable: <= 8)
      if (nJ % 2 || P < 1 || P > 8) {
        set_error("TRSM needs nb a multiple of %d up to 1024 (nb=%d)", 2 * kR, nb);
        return false;
      }
      LaunchDesc d;
      TrsmInvParams tp{o.t[0], o.t[1], o.scratch, nb, o.push};
      static const void* const kTrsm[9] = {nullptr,
                                           (const void*)k_trsm_inv<1>, (const void*)k_trsm_inv<2>,
                                           (const void*)k_trsm_inv<3>, (const void*)k_trsm_inv<4>,
                                           (const void*)k_trsm_inv<5>, (const void*)k_trsm_inv<6>,
                                           (const void*)k_trsm_inv<7>, (const void*)k_trsm_inv<8>};
      const void* f = kTrsm[P];
      d.set(f, dim3(nJ * P), dim3(CfgG::THREADS), trsm_smem(), tp);
      out.push_back(d);
      return true;
    }
    case K_SYRK:
      push_gemm(out, o.t[0], o.t[0], o.t[1], nb, nb, nb, nb, 1, o.push);
      return true;
    case K_GEMM:
      push_gemm(out, o.t[0], o.t[1], o.t[2], nb, nb, nb, nb, 0, o.push);
      return true;
    default:
      set_error("kind %d is not a Cholesky kind", kind);
      return false;
  }
}

}  // namespace hg
