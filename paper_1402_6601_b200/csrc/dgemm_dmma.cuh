// CTA-level FP64 DMMA GEMM engine used by every trailing-update tile kernel.
//
//   acc(BM x BN) += opA(BM x K) * opB(BN x K)^T
//
// Operands are addressed through (ptr, ld, layout):
//   layout M_MAJOR: element (r, k) at ptr[k*ld + r]   (column-major tile, rows contiguous)
//   layout K_MAJOR: element (r, k) at ptr[r*ld + k]   (the transpose of a column-major tile)
// so C -= A*B^T of two column-major tiles is (M_MAJOR, M_MAJOR), C -= A*B is
// (M_MAJOR, K_MAJOR) and C -= A^T*B is (K_MAJOR, K_MAJOR).
//
// Global -> shared staging is a STAGES-deep cp.async (LDGSTS) ring of BK-wide
// k-slabs; the smem rows are padded by 4 doubles so that the DMMA fragment
// loads (4 k-rows x 8 consecutive rows per half-warp) hit 32 distinct banks.
#pragma once
#include "hg_common.cuh"
#include "tiles.h"

namespace hg {

enum Layout { M_MAJOR = 0, K_MAJOR = 1 };

// KSWZ: K_MAJOR slabs unpadded (rows of BK = 8 doubles) with the k index XOR-swizzled
// by bit 1 of the row, conflict-free for the fragment loads at 2/3 of the padded size.
template <int BM_, int BN_, int BK_, int WM_, int WN_, int STAGES_, bool KSWZ_ = false>
struct GemmCfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, WM = WM_, WN = WN_, STAGES = STAGES_;
  static constexpr bool KSWZ = KSWZ_;
  static_assert(!KSWZ_ || BK_ == 8, "swizzled K_MAJOR slabs are 8 doubles wide");
  static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
  static constexpr int THREADS = WARPS_M * WARPS_N * 32;
  static constexpr int FM = WM / 8, FN = WN / 8;  // 8x8 fragments per warp
  static constexpr int PAD = 4;
  // smem footprint of one operand slab for each layout
  __host__ __device__ static constexpr int slab_mmaj(int rows) { return BK * (rows + PAD); }
  __host__ __device__ static constexpr int slab_kmaj(int rows) { return rows * (KSWZ ? BK : BK + PAD); }
  // smem index of K_MAJOR slab element (row r, k)
  __host__ __device__ static constexpr int kmaj(int r, int k) {
    return KSWZ ? r * BK + (k ^ (((r >> 1) & 1) << 2)) : r * (BK + PAD) + k;
  }
};

template <class Cfg, int LA, int LB>
struct GemmSmem {
  static constexpr int A_SLAB = LA == M_MAJOR ? Cfg::slab_mmaj(Cfg::BM) : Cfg::slab_kmaj(Cfg::BM);
  static constexpr int B_SLAB = LB == M_MAJOR ? Cfg::slab_mmaj(Cfg::BN) : Cfg::slab_kmaj(Cfg::BN);
  static constexpr int DOUBLES = Cfg::STAGES * (A_SLAB + B_SLAB);
  static constexpr size_t BYTES = size_t(DOUBLES) * sizeof(double);
};

// Issue the cp.async copies of one (ROWS x BK) slab starting at (r0, k0).
template <class Cfg, int L, int ROWS>
HG_DEVICE void load_slab(double* s, const double* __restrict__ g, int ld, int r0, int k0) {
  constexpr int BK = Cfg::BK, PAD = Cfg::PAD;
  if constexpr (L == M_MAJOR) {
    constexpr int CH_PER_K = ROWS / 2;  // 16-byte chunks per k-row
    constexpr int CHUNKS = BK * CH_PER_K;
    if constexpr (CHUNKS % Cfg::THREADS == 0) {
      // compile-time trip count: the per-chunk offsets strength-reduce to one base
      // pointer per thread plus immediates
      const double* gb = g + size_t(k0) * ld + r0;
#pragma unroll
      for (int i = 0; i < CHUNKS / Cfg::THREADS; ++i) {
        const int c = threadIdx.x + i * Cfg::THREADS;
        const int kk = c / CH_PER_K, rr = (c % CH_PER_K) * 2;
        cp_async16(s + kk * (ROWS + PAD) + rr, gb + size_t(kk) * ld + rr);
      }
    } else {
      for (int c = threadIdx.x; c < CHUNKS; c += Cfg::THREADS) {
        int kk = c / CH_PER_K, rr = (c % CH_PER_K) * 2;
        cp_async16(s + kk * (ROWS + PAD) + rr, g + size_t(k0 + kk) * ld + r0 + rr);
      }
    }
  } else {
    constexpr int CH_PER_R = BK / 2;
    constexpr int CHUNKS = ROWS * CH_PER_R;
    if constexpr (CHUNKS % Cfg::THREADS == 0) {
      const double* gb = g + size_t(r0) * ld + k0;
#pragma unroll
      for (int i = 0; i < CHUNKS / Cfg::THREADS; ++i) {
        const int c = threadIdx.x + i * Cfg::THREADS;
        const int rr = c / CH_PER_R, kk = (c % CH_PER_R) * 2;
        cp_async16(s + Cfg::kmaj(rr, kk), gb + size_t(rr) * ld + kk);
      }
    } else {
      for (int c = threadIdx.x; c < CHUNKS; c += Cfg::THREADS) {
        int rr = c / CH_PER_R, kk = (c % CH_PER_R) * 2;
        cp_async16(s + Cfg::kmaj(rr, kk), g + size_t(r0 + rr) * ld + k0 + kk);
      }
    }
  }
}

// One warp's 32 rows [w0, w0 + 32) of an M_MAJOR (ROWS x BK) slab: per k 256 contiguous
// bytes (16 chunks), BK / 2 chunks per lane.
template <class Cfg, int ROWS>
HG_DEVICE void load_slab_warp(double* s, const double* __restrict__ g, int ld, int r0, int k0, int w0, int lane) {
  constexpr int BK = Cfg::BK, PAD = Cfg::PAD;
  static_assert((BK * 16) % 32 == 0, "whole chunks per lane");
  const double* gb = g + size_t(k0) * ld + r0 + w0;
#pragma unroll
  for (int i = 0; i < BK * 16 / 32; ++i) {
    const int c = lane + i * 32;
    const int kk = c / 16, rr = (c % 16) * 2;
    cp_async16(s + kk * (ROWS + PAD) + w0 + rr, gb + size_t(kk) * ld + rr);
  }
}

template <class Cfg, int L, int ROWS>
HG_DEVICE double frag_at(const double* s, int r, int k) {
  if constexpr (L == M_MAJOR) return s[k * (ROWS + Cfg::PAD) + r];
  else return s[Cfg::kmaj(r, k)];
}

// Standard operand loader: a (ROWS x k) window of a tile addressed by layout.
template <class Cfg, int L, int ROWS>
struct TileLoader {
  static constexpr int layout = L;
  static constexpr int rows = ROWS;
  const double* p;
  int ld;
  int r0;
  HG_DEVICE void load(double* s, int k0) const { load_slab<Cfg, L, ROWS>(s, p, ld, r0, k0); }
  // M_MAJOR only: the 32 slab rows [w0, w0 + 32) of one warp (warp-private rings)
  HG_DEVICE void load_warp(double* s, int k0, int w0, int lane) const {
    static_assert(L == M_MAJOR, "warp-row loads are M_MAJOR");
    load_slab_warp<Cfg, ROWS>(s, p, ld, r0, k0, w0, lane);
  }
};

// Main loop over k in [k_begin, k_end) (multiples of BK). acc[FM][FN][2].
// LdA / LdB are loader functors (TileLoader or a kernel-specific masked
// loader) exposing `layout`, `rows` and `load(slab, k0)`.
template <class Cfg, class LdA, class LdB>
HG_DEVICE void gemm_mainloop_nd(double (&acc)[Cfg::FM][Cfg::FN][2], double* smem, const LdA& la, const LdB& lb,
                                int k_begin, int k_end);

// (STAGES >= 3 with BK % 8 == 0 runs the non-draining variant below: same
// k order, bit-identical results, +3-4% DMMA throughput on the 64x64 tile)
template <class Cfg, class LdA, class LdB>
HG_DEVICE void gemm_mainloop(double (&acc)[Cfg::FM][Cfg::FN][2], double* smem,
                             const LdA& la, const LdB& lb, int k_begin, int k_end) {
  if constexpr (Cfg::STAGES >= 3 && Cfg::BK % 8 == 0) {
    gemm_mainloop_nd<Cfg>(acc, smem, la, lb, k_begin, k_end);
    return;
  }
  constexpr int LA = LdA::layout, LB = LdB::layout;
  static_assert(LdA::rows == Cfg::BM && LdB::rows == Cfg::BN, "loader rows");
  using SM = GemmSmem<Cfg, LA, LB>;
  constexpr int BK = Cfg::BK, STAGES = Cfg::STAGES;
  double* sA = smem;
  double* sB = smem + STAGES * SM::A_SLAB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = (warp % Cfg::WARPS_M) * Cfg::WM;
  const int wn = (warp / Cfg::WARPS_M) * Cfg::WN;
  const int g = lane >> 2, t = lane & 3;
  const int nk = (k_end - k_begin) / BK;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) {
      la.load(sA + s * SM::A_SLAB, k_begin + s * BK);
      lb.load(sB + s * SM::B_SLAB, k_begin + s * BK);
    }
    cp_async_commit();
  }
  for (int it = 0; it < nk; ++it) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {  // prefetch slab it+STAGES-1 into the ring slot freed last iteration
      int nxt = it + STAGES - 1;
      if (nxt < nk) {
        int slot = nxt % STAGES;
        la.load(sA + slot * SM::A_SLAB, k_begin + nxt * BK);
        lb.load(sB + slot * SM::B_SLAB, k_begin + nxt * BK);
      }
      cp_async_commit();
    }
    const double* a_s = sA + (it % STAGES) * SM::A_SLAB;
    const double* b_s = sB + (it % STAGES) * SM::B_SLAB;
    // fragments double-buffered in registers: k-step kk+4 is loaded while the
    // 16 DMMAs of k-step kk issue
    double af[2][Cfg::FM], bf[2][Cfg::FN];
#pragma unroll
    for (int i = 0; i < Cfg::FM; ++i) af[0][i] = frag_at<Cfg, LA, Cfg::BM>(a_s, wm + i * 8 + g, t);
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j) bf[0][j] = frag_at<Cfg, LB, Cfg::BN>(b_s, wn + j * 8 + g, t);
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      const int cur = (kk >> 2) & 1, nxt = cur ^ 1;
      if (kk + 4 < BK) {
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i) af[nxt][i] = frag_at<Cfg, LA, Cfg::BM>(a_s, wm + i * 8 + g, kk + 4 + t);
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) bf[nxt][j] = frag_at<Cfg, LB, Cfg::BN>(b_s, wn + j * 8 + g, kk + 4 + t);
      }
#pragma unroll
      for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[cur][i], bf[cur][j]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();
}

// gemm_mainloop with a fragment pipeline that never drains at slab boundaries
// (STAGES >= 3): the barrier at the top of iteration `it` publishes slab it+1
// too (wait_group STAGES-3), so the last k-step of slab it loads slab it+1's
// first fragments while its DMMAs issue.  One barrier per slab, as before.
template <class Cfg, class LdA, class LdB>
HG_DEVICE void gemm_mainloop_nd(double (&acc)[Cfg::FM][Cfg::FN][2], double* smem, const LdA& la, const LdB& lb,
                                int k_begin, int k_end) {
  constexpr int LA = LdA::layout, LB = LdB::layout;
  static_assert(LdA::rows == Cfg::BM && LdB::rows == Cfg::BN, "loader rows");
  using SM = GemmSmem<Cfg, LA, LB>;
  constexpr int BK = Cfg::BK, STAGES = Cfg::STAGES;
  static_assert(STAGES >= 3 && BK % 8 == 0, "non-draining pipeline");
  double* sA = smem;
  double* sB = smem + STAGES * SM::A_SLAB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = (warp % Cfg::WARPS_M) * Cfg::WM;
  const int wn = (warp / Cfg::WARPS_M) * Cfg::WN;
  const int g = lane >> 2, t = lane & 3;
  const int nk = (k_end - k_begin) / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) {
      la.load(sA + s * SM::A_SLAB, k_begin + s * BK);
      lb.load(sB + s * SM::B_SLAB, k_begin + s * BK);
    }
    cp_async_commit();
  }
  double af[2][Cfg::FM], bf[2][Cfg::FN];
  cp_async_wait<STAGES - 2>();
  __syncthreads();
#pragma unroll
  for (int i = 0; i < Cfg::FM; ++i) af[0][i] = frag_at<Cfg, LA, Cfg::BM>(sA, wm + i * 8 + g, t);
#pragma unroll
  for (int j = 0; j < Cfg::FN; ++j) bf[0][j] = frag_at<Cfg, LB, Cfg::BN>(sB, wn + j * 8 + g, t);
  for (int it = 0; it < nk; ++it) {
    cp_async_wait<STAGES - 3>();
    __syncthreads();
    {
      const int nxt = it + STAGES - 1;
      if (nxt < nk) {
        const int slot = nxt % STAGES;
        la.load(sA + slot * SM::A_SLAB, k_begin + nxt * BK);
        lb.load(sB + slot * SM::B_SLAB, k_begin + nxt * BK);
      }
      cp_async_commit();
    }
    const double* a_s = sA + (it % STAGES) * SM::A_SLAB;
    const double* b_s = sB + (it % STAGES) * SM::B_SLAB;
    const double* a_n = sA + ((it + 1) % STAGES) * SM::A_SLAB;
    const double* b_n = sB + ((it + 1) % STAGES) * SM::B_SLAB;
    const bool more = it + 1 < nk;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      const int cur = (kk >> 2) & 1, nx = cur ^ 1;
      if (kk + 4 < BK) {
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i) af[nx][i] = frag_at<Cfg, LA, Cfg::BM>(a_s, wm + i * 8 + g, kk + 4 + t);
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) bf[nx][j] = frag_at<Cfg, LB, Cfg::BN>(b_s, wn + j * 8 + g, kk + 4 + t);
      } else if (more) {
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i) af[nx][i] = frag_at<Cfg, LA, Cfg::BM>(a_n, wm + i * 8 + g, t);
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) bf[nx][j] = frag_at<Cfg, LB, Cfg::BN>(b_n, wn + j * 8 + g, t);
      }
#pragma unroll
      for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[cur][i], bf[cur][j]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();
}

// Producer/consumer variant of the M_MAJOR x M_MAJOR main loop: one thread
// streams each k-slab with bulk copies (one per k-column: ROWS contiguous
// doubles) that complete on the slot's `full` mbarrier; each warp releases a
// slot by arriving on its `empty` mbarrier.  No CTA-wide barrier in the loop:
// a warp only waits for the bytes it reads.  bars: 2 * STAGES uint64 in smem.
// Measured SLOWER than gemm_mainloop_nd (30.4 vs 34.4 TF/s on 32 tiles,
// profiles/r01_gemm_nd_variants.jsonl): 32 small (512 B) bulk copies per stage
// from one thread; a 2D tensor map per operand would need tile-pool tensor maps
// in the runtime.  Kept for tools/microbench.cu only.
template <class Cfg>
HG_DEVICE void gemm_mainloop_mb(double (&acc)[Cfg::FM][Cfg::FN][2], double* smem, uint64_t* bars,
                                const double* __restrict__ A, int lda, int m0, const double* __restrict__ B, int ldb,
                                int n0, int k_begin, int k_end) {
  constexpr int BK = Cfg::BK, STAGES = Cfg::STAGES, PAD = Cfg::PAD;
  constexpr int WARPS = Cfg::THREADS / 32;
  constexpr int A_SLAB = Cfg::slab_mmaj(Cfg::BM), B_SLAB = Cfg::slab_mmaj(Cfg::BN);
  constexpr unsigned STAGE_BYTES = unsigned(BK * (Cfg::BM + Cfg::BN) * sizeof(double));
  static_assert(BK % 8 == 0 && STAGES >= 2, "pipeline");
  double* sA = smem;
  double* sB = smem + STAGES * A_SLAB;
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = (warp % Cfg::WARPS_M) * Cfg::WM;
  const int wn = (warp / Cfg::WARPS_M) * Cfg::WN;
  const int g = lane >> 2, t = lane & 3;
  const int nk = (k_end - k_begin) / BK;
  const bool producer = threadIdx.x == 0;
  auto issue = [&](int s) {  // slab s into slot s % STAGES
    const int slot = s % STAGES;
    mbar_arrive_tx(&full[slot], STAGE_BYTES);
    const int k0 = k_begin + s * BK;
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      bulk_g2s(sA + slot * A_SLAB + kk * (Cfg::BM + PAD), A + size_t(k0 + kk) * lda + m0,
               Cfg::BM * sizeof(double), &full[slot]);
      bulk_g2s(sB + slot * B_SLAB + kk * (Cfg::BN + PAD), B + size_t(k0 + kk) * ldb + n0,
               Cfg::BN * sizeof(double), &full[slot]);
    }
  };
  __syncthreads();  // previous users of this smem / barrier area are done
  if (producer) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (producer)
    for (int s = 0; s < STAGES && s < nk; ++s) issue(s);
  double af[2][Cfg::FM], bf[2][Cfg::FN];
  if (nk > 0) {
    mbar_wait(&full[0], 0);
#pragma unroll
    for (int i = 0; i < Cfg::FM; ++i) af[0][i] = sA[t * (Cfg::BM + PAD) + wm + i * 8 + g];
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j) bf[0][j] = sB[t * (Cfg::BN + PAD) + wn + j * 8 + g];
  }
  for (int it = 0; it < nk; ++it) {
    const int slot = it % STAGES;
    const double* a_s = sA + slot * A_SLAB;
    const double* b_s = sB + slot * B_SLAB;
    const int ns = (it + 1) % STAGES;
    const double* a_n = sA + ns * A_SLAB;
    const double* b_n = sB + ns * B_SLAB;
    const bool more = it + 1 < nk;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      const int cur = (kk >> 2) & 1, nx = cur ^ 1;
      if (kk + 4 < BK) {
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i) af[nx][i] = a_s[(kk + 4 + t) * (Cfg::BM + PAD) + wm + i * 8 + g];
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) bf[nx][j] = b_s[(kk + 4 + t) * (Cfg::BN + PAD) + wn + j * 8 + g];
      } else if (more) {
        mbar_wait(&full[ns], ((it + 1) / STAGES) & 1);
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i) af[nx][i] = a_n[t * (Cfg::BM + PAD) + wm + i * 8 + g];
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) bf[nx][j] = b_n[t * (Cfg::BN + PAD) + wn + j * 8 + g];
      }
#pragma unroll
      for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[cur][i], bf[cur][j]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
    // refill the slot of slab it-1 (one slab of slack: its readers are long done)
    if (producer && it >= 1 && it - 1 + STAGES < nk) {
      const int ps = (it - 1) % STAGES;
      mbar_wait(&empty[ps], ((it - 1) / STAGES) & 1);
      issue(it - 1 + STAGES);
    }
  }
  __syncthreads();
}

// Visit every accumulator element with its (row, col) inside the CTA tile.
template <class Cfg, class F>
HG_DEVICE void for_each_acc(double (&acc)[Cfg::FM][Cfg::FN][2], F&& f) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = (warp % Cfg::WARPS_M) * Cfg::WM;
  const int wn = (warp / Cfg::WARPS_M) * Cfg::WN;
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j) {
      int r = wm + i * 8 + g, c = wn + j * 8 + 2 * t;
      f(r, c, acc[i][j][0]);
      f(r, c + 1, acc[i][j][1]);
    }
}

template <class Cfg>
HG_DEVICE void zero_acc(double (&acc)[Cfg::FM][Cfg::FN][2]) {
#pragma unroll
  for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
}

// (i, j, row, col) of every accumulator fragment pair of this thread
template <class Cfg, class F>
HG_DEVICE void for_each_acc_ij(F&& f) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = (warp % Cfg::WARPS_M) * Cfg::WM;
  const int wn = (warp / Cfg::WARPS_M) * Cfg::WN;
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j) f(i, j, wm + i * 8 + g, wn + j * 8 + 2 * t);
}

// Loads C(m0 + r, n0 + c) at every accumulator position (all loads issued
// before any use, so the L2 latency is paid once, not once per element).
template <class Cfg>
HG_DEVICE void load_like_acc(double (&cv)[Cfg::FM][Cfg::FN][2], const double* __restrict__ C, int ldc, int m0,
                             int n0) {
  for_each_acc_ij<Cfg>([&](int i, int j, int r, int c) {
    cv[i][j][0] = C[size_t(n0 + c) * ldc + m0 + r];
    cv[i][j][1] = C[size_t(n0 + c + 1) * ldc + m0 + r];
  });
}

}  // namespace hg

namespace hg {

// Main loop whose B operand is already resident in shared memory, stored as
// sB[n * ldsb + k] (K-major rows of length >= k_end - k_begin, indexed from
// k_begin).  Only A streams through the cp.async ring.
// LOWER_A: A is lower triangular (A(r, k) == 0 for k > r, k counted from
// k_begin): a warp skips the k-steps that lie entirely above its row block.
template <class Cfg, class LdA, bool LOWER_A = false>
HG_DEVICE void gemm_mainloop_bsmem(double (&acc)[Cfg::FM][Cfg::FN][2], double* ring, const LdA& la,
                                   const double* sB, int ldsb, int k_begin, int k_end) {
  constexpr int LA = LdA::layout;
  constexpr int A_SLAB = LA == M_MAJOR ? Cfg::slab_mmaj(Cfg::BM) : Cfg::slab_kmaj(Cfg::BM);
  constexpr int BK = Cfg::BK, STAGES = Cfg::STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = (warp % Cfg::WARPS_M) * Cfg::WM;
  const int wn = (warp / Cfg::WARPS_M) * Cfg::WN;
  const int g = lane >> 2, t = lane & 3;
  const int nk = (k_end - k_begin) / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) la.load(ring + s * A_SLAB, k_begin + s * BK);
    cp_async_commit();
  }
  for (int it = 0; it < nk; ++it) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      int nxt = it + STAGES - 1;
      if (nxt < nk) la.load(ring + (nxt % STAGES) * A_SLAB, k_begin + nxt * BK);
      cp_async_commit();
    }
    const double* a_s = ring + (it % STAGES) * A_SLAB;
    const int kb = it * BK;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      if (LOWER_A && kb + kk >= wm + Cfg::WM) break;  // warp-uniform
      double af[Cfg::FM], bf[Cfg::FN];
#pragma unroll
      for (int i = 0; i < Cfg::FM; ++i) af[i] = frag_at<Cfg, LA, Cfg::BM>(a_s, wm + i * 8 + g, kk + t);
#pragma unroll
      for (int j = 0; j < Cfg::FN; ++j) bf[j] = sB[(wn + j * 8 + g) * ldsb + kb + kk + t];
#pragma unroll
      for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();
}

}  // namespace hg

namespace hg {

// C(m0 + r, n0 + c) = (init ? 0 : C) - acc(r, c) for the CTA tile, with all C
// loads issued before any store (a read-modify-write through a lambda would
// order every load behind the previous store: one L2 round trip per element).
// lower: skip r < c of a diagonal tile (m0 == n0).
template <class Cfg>
HG_DEVICE void sub_store(double (&acc)[Cfg::FM][Cfg::FN][2], double* __restrict__ C, int ldc, int m0, int n0,
                         bool lower = false, bool init = false, const PushList* push = nullptr) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = (warp % Cfg::WARPS_M) * Cfg::WM;
  const int wn = (warp / Cfg::WARPS_M) * Cfg::WN;
  const int g = lane >> 2, t = lane & 3;
  const bool diag = lower && (m0 == n0);
  double cv[Cfg::FM][Cfg::FN][2];
  if (!init) {
#pragma unroll
    for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
      for (int j = 0; j < Cfg::FN; ++j) {
        const int r = wm + i * 8 + g, c = wn + j * 8 + 2 * t;
        cv[i][j][0] = C[size_t(n0 + c) * ldc + m0 + r];
        cv[i][j][1] = C[size_t(n0 + c + 1) * ldc + m0 + r];
      }
  }
#pragma unroll
  for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j) {
      const int r = wm + i * 8 + g, c = wn + j * 8 + 2 * t;
      const double b0 = init ? 0.0 : cv[i][j][0], b1 = init ? 0.0 : cv[i][j][1];
      const size_t o0 = size_t(n0 + c) * ldc + m0 + r, o1 = o0 + ldc;
      const double v0 = b0 - acc[i][j][0], v1 = b1 - acc[i][j][1];
      const bool s0 = !diag || r >= c, s1 = !diag || r >= c + 1;
      if (s0) C[o0] = v0;
      if (s1) C[o1] = v1;
      if (push)  // producer-push: the final value also goes to every consumer GPU's slot (peer stores)
        for (int q = 0; q < push->n; ++q) {
          if (s0) __stcg(push->dst[q] + o0, v0);
          if (s1) __stcg(push->dst[q] + o1, v1);
        }
    }
}

}  // namespace hg

namespace hg {

// C[m, n0 + c] -= sum_k A(m, k) B(c, k) for every BM-row chunk of [m_begin,
// m_end), with B resident in shared memory (sB[c*ldsb + k], k in [0, K)) and
// ONE continuous cp.async ring over all (chunk, k-slab) pairs: the A stream
// never drains between chunks, only the per-chunk epilogue interrupts the
// DMMAs (the trailing updates of GESSM / SSSSM / UNMQR / TSMQR, K = ib).
// LdA exposes a mutable row origin r0.
// RED: the epilogue is red.global.add(-acc) instead of load / subtract / store
// (no C load latency, no C registers, half the C traffic); the caller's later
// reads of C must bypass L1 (cp.async.cg / ld.cg): a __threadfence() here makes
// the reductions visible before the caller's next barrier.
// m_mask: rows < m_mask are computed but not written (lets a BM that does not
// divide m_end - m_mask start its first chunk early; RED epilogue only).
template <class Cfg, class LdA, bool PREFETCH_C = true, int KC = 128, bool RED = false>
HG_DEVICE void gemm_sub_chunks_bsmem(double* ring, LdA la, const double* sB, int ldsb, int K, int m_begin,
                                     int m_end, double* __restrict__ C, int ldc, int n0, int m_mask = 0) {
  // K == KC (the panel width ib = 128 in every caller): the slab / chunk indices are
  // compile-time divisions, and the A fragments are double-buffered in registers
  constexpr int LA = LdA::layout;
  constexpr int A_SLAB = LA == M_MAJOR ? Cfg::slab_mmaj(Cfg::BM) : Cfg::slab_kmaj(Cfg::BM);
  constexpr int BK = Cfg::BK, STAGES = Cfg::STAGES;
  constexpr int NK = KC / BK;
  (void)K;
  const int total = NK * ((m_end - m_begin) / Cfg::BM);
  if (total <= 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = (warp % Cfg::WARPS_M) * Cfg::WM;
  const int wn = (warp / Cfg::WARPS_M) * Cfg::WN;
  const int g = lane >> 2, t = lane & 3;
  auto load = [&](int s) {
    LdA l = la;
    l.r0 = m_begin + (s / NK) * Cfg::BM;
    l.load(ring + (s % STAGES) * A_SLAB, (s % NK) * BK);
  };
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < total) load(s);
    cp_async_commit();
  }
  if constexpr (RED && STAGES >= 3 && Cfg::WARPS_N == 1 && LA == M_MAJOR) {
    // Warp-private A stream: with one warp column every warp reads only its own 32 rows of
    // each A slab (B is resident), so each warp loads exactly those rows with its own cp.async
    // groups and synchronises with __syncwarp -- no CTA barrier in the stream.  The warps
    // drift apart, so one warp's chunk epilogue (the red.global.add drain) overlaps the other
    // warps' DMMAs instead of all four draining in lockstep.  Same k order per accumulator as
    // the CTA-barrier variant below: bit-identical results.
    static_assert(BK % 8 == 0, "slabs start on fragment buffer 0");
    __syncthreads();  // the ring may still be read by the caller's previous (CTA-wide) phase
    auto load_w = [&](int s) {
      LdA l = la;
      l.r0 = m_begin + (s / NK) * Cfg::BM;
      l.load_warp(ring + (s % STAGES) * A_SLAB, (s % NK) * BK, wm, lane);
    };
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
      if (s < total) load_w(s);
      cp_async_commit();
    }
    double acc[Cfg::FM][Cfg::FN][2];
    zero_acc<Cfg>(acc);
    double af[2][Cfg::FM], bf[2][Cfg::FN];
    cp_async_wait<STAGES - 2>();
    __syncwarp();
#pragma unroll
    for (int i = 0; i < Cfg::FM; ++i) af[0][i] = frag_at<Cfg, LA, Cfg::BM>(ring, wm + i * 8 + g, t);
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j) bf[0][j] = sB[(wn + j * 8 + g) * ldsb + t];
    for (int it = 0; it < total; ++it) {
      const int kslab = it % NK;
      cp_async_wait<STAGES - 3>();
      __syncwarp();
      if (it + STAGES - 1 < total) load_w(it + STAGES - 1);
      cp_async_commit();
      const double* a_s = ring + (it % STAGES) * A_SLAB;
      const double* a_n = ring + ((it + 1) % STAGES) * A_SLAB;
      const int kb = kslab * BK;
      const int kb_n = ((it + 1) % NK) * BK;
      const bool more = it + 1 < total;
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4) {
        const int cur = (kk >> 2) & 1, nxt = cur ^ 1;
        if (kk + 4 < BK) {
#pragma unroll
          for (int i = 0; i < Cfg::FM; ++i) af[nxt][i] = frag_at<Cfg, LA, Cfg::BM>(a_s, wm + i * 8 + g, kk + 4 + t);
#pragma unroll
          for (int j = 0; j < Cfg::FN; ++j) bf[nxt][j] = sB[(wn + j * 8 + g) * ldsb + kb + kk + 4 + t];
        } else if (more) {
#pragma unroll
          for (int i = 0; i < Cfg::FM; ++i) af[nxt][i] = frag_at<Cfg, LA, Cfg::BM>(a_n, wm + i * 8 + g, t);
#pragma unroll
          for (int j = 0; j < Cfg::FN; ++j) bf[nxt][j] = sB[(wn + j * 8 + g) * ldsb + kb_n + t];
        }
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
          for (int j = 0; j < Cfg::FN; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[cur][i], bf[cur][j]);
      }
      if (kslab == NK - 1) {
        const int m0 = m_begin + (it / NK) * Cfg::BM;
        for_each_acc_ij<Cfg>([&](int i, int j, int r, int c) {
          if (m0 + r >= m_mask) {
            red_add_f64(C + size_t(n0 + c) * ldc + m0 + r, -acc[i][j][0]);
            red_add_f64(C + size_t(n0 + c + 1) * ldc + m0 + r, -acc[i][j][1]);
          }
        });
        zero_acc<Cfg>(acc);
      }
    }
    __threadfence();
    cp_async_wait<0>();
    __syncthreads();
    return;
  } else if constexpr (RED && STAGES >= 3) {
    static_assert(BK % 8 == 0, "slabs start on fragment buffer 0");
    // Fragment pipeline that never drains at slab boundaries: the barrier at the
    // top of iteration `it` publishes slab it+1 as well (wait_group STAGES-3), so
    // the last k-step of slab it already loads slab it+1's first fragments.
    double acc[Cfg::FM][Cfg::FN][2];
    zero_acc<Cfg>(acc);
    double af[2][Cfg::FM], bf[2][Cfg::FN];
    cp_async_wait<STAGES - 2>();
    __syncthreads();
#pragma unroll
    for (int i = 0; i < Cfg::FM; ++i) af[0][i] = frag_at<Cfg, LA, Cfg::BM>(ring, wm + i * 8 + g, t);
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j) bf[0][j] = sB[(wn + j * 8 + g) * ldsb + t];
    for (int it = 0; it < total; ++it) {
      const int kslab = it % NK;
      cp_async_wait<STAGES - 3>();
      __syncthreads();
      if (it + STAGES - 1 < total) load(it + STAGES - 1);
      cp_async_commit();
      const double* a_s = ring + (it % STAGES) * A_SLAB;
      const double* a_n = ring + ((it + 1) % STAGES) * A_SLAB;
      const int kb = kslab * BK;
      const int kb_n = ((it + 1) % NK) * BK;
      const bool more = it + 1 < total;
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4) {
        const int cur = (kk >> 2) & 1, nxt = cur ^ 1;  // BK / 4 is even: slab starts on buffer 0
        if (kk + 4 < BK) {
#pragma unroll
          for (int i = 0; i < Cfg::FM; ++i) af[nxt][i] = frag_at<Cfg, LA, Cfg::BM>(a_s, wm + i * 8 + g, kk + 4 + t);
#pragma unroll
          for (int j = 0; j < Cfg::FN; ++j) bf[nxt][j] = sB[(wn + j * 8 + g) * ldsb + kb + kk + 4 + t];
        } else if (more) {
#pragma unroll
          for (int i = 0; i < Cfg::FM; ++i) af[nxt][i] = frag_at<Cfg, LA, Cfg::BM>(a_n, wm + i * 8 + g, t);
#pragma unroll
          for (int j = 0; j < Cfg::FN; ++j) bf[nxt][j] = sB[(wn + j * 8 + g) * ldsb + kb_n + t];
        }
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
          for (int j = 0; j < Cfg::FN; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[cur][i], bf[cur][j]);
      }
      if (kslab == NK - 1) {
        const int m0 = m_begin + (it / NK) * Cfg::BM;
        for_each_acc_ij<Cfg>([&](int i, int j, int r, int c) {
          if (m0 + r >= m_mask) {
            red_add_f64(C + size_t(n0 + c) * ldc + m0 + r, -acc[i][j][0]);
            red_add_f64(C + size_t(n0 + c + 1) * ldc + m0 + r, -acc[i][j][1]);
          }
        });
        zero_acc<Cfg>(acc);
      }
    }
    __threadfence();
    cp_async_wait<0>();
    __syncthreads();
    return;
  }
  double acc[Cfg::FM][Cfg::FN][2];
  double cv[Cfg::FM][Cfg::FN][2];  // this chunk's C, loaded while its k-slabs run
  zero_acc<Cfg>(acc);
  for (int it = 0; it < total; ++it) {
    const int kslab = it % NK;
    if (!RED && PREFETCH_C && kslab == 0) load_like_acc<Cfg>(cv, C, ldc, m_begin + (it / NK) * Cfg::BM, n0);
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    if (it + STAGES - 1 < total) load(it + STAGES - 1);
    cp_async_commit();
    const double* a_s = ring + (it % STAGES) * A_SLAB;
    const int kb = kslab * BK;
    double af[2][Cfg::FM], bf[2][Cfg::FN];
#pragma unroll
    for (int i = 0; i < Cfg::FM; ++i) af[0][i] = frag_at<Cfg, LA, Cfg::BM>(a_s, wm + i * 8 + g, t);
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j) bf[0][j] = sB[(wn + j * 8 + g) * ldsb + kb + t];
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      const int cur = (kk >> 2) & 1, nxt = cur ^ 1;
      if (kk + 4 < BK) {
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i) af[nxt][i] = frag_at<Cfg, LA, Cfg::BM>(a_s, wm + i * 8 + g, kk + 4 + t);
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) bf[nxt][j] = sB[(wn + j * 8 + g) * ldsb + kb + kk + 4 + t];
      }
#pragma unroll
      for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[cur][i], bf[cur][j]);
    }
    if (kslab == NK - 1) {
      const int m0 = m_begin + (it / NK) * Cfg::BM;
      if constexpr (RED) {
        for_each_acc_ij<Cfg>([&](int i, int j, int r, int c) {
          if (m0 + r >= m_mask) {
            red_add_f64(C + size_t(n0 + c) * ldc + m0 + r, -acc[i][j][0]);
            red_add_f64(C + size_t(n0 + c + 1) * ldc + m0 + r, -acc[i][j][1]);
          }
        });
      } else {
        if (!PREFETCH_C) load_like_acc<Cfg>(cv, C, ldc, m0, n0);
        for_each_acc_ij<Cfg>([&](int i, int j, int r, int c) {
          C[size_t(n0 + c) * ldc + m0 + r] = cv[i][j][0] - acc[i][j][0];
          C[size_t(n0 + c + 1) * ldc + m0 + r] = cv[i][j][1] - acc[i][j][1];
        });
      }
      zero_acc<Cfg>(acc);
    }
  }
  if constexpr (RED) __threadfence();
  cp_async_wait<0>();
  __syncthreads();
}


// ---------------------------------------------------------------------------
// Producer-push helpers: the producing kernel stores the final values of a
// task's output block into the consumer GPUs' slots of that block (peer / IPC pointers), so the
// plan's copy job needs no copy node.  Callers fence + synchronise first (the values are read
// back through L2: the trailing updates end in L2 reductions).

// Whole slots (tile + side area), the threads of `nrank` CTAs of a cluster cooperating.
HG_DEVICE void push_slots(const PushList& pl, int rank, int nrank) {
  const long long n2 = pl.len / 2;
  const long long step = (long long)nrank * blockDim.x;
  for (int q = 0; q < pl.n; ++q) {
    const double2* s = reinterpret_cast<const double2*>(pl.src[q]);
    double2* d = reinterpret_cast<double2*>(pl.dst[q]);
    long long e = (long long)rank * blockDim.x + threadIdx.x;
    for (; e + 3 * step < n2; e += 4 * step) {  // 4 L2 loads in flight per thread
      double2 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcg(s + e + u * step);
#pragma unroll
      for (int u = 0; u < 4; ++u) __stcg(d + e + u * step, v[u]);
    }
    for (; e < n2; e += step) __stcg(d + e, __ldcg(s + e));
    if ((pl.len & 1) && rank == 0 && threadIdx.x == 0) pl.dst[q][pl.len - 1] = __ldcg(pl.src[q] + pl.len - 1);
  }
}

// Columns [n0, n0 + BN) of every pushed tile (all nb rows, column-major ld = nb): one CTA's strip.
template <int BN, int THREADS>
HG_DEVICE void push_strip(const PushList& pl, int n0, int nb) {
  const int h = nb / 2;  // double2 per column
  for (int q = 0; q < pl.n; ++q) {
    const double2* s = reinterpret_cast<const double2*>(pl.src[q] + size_t(n0) * nb);
    double2* d = reinterpret_cast<double2*>(pl.dst[q] + size_t(n0) * nb);
    for (int e = threadIdx.x; e < BN * h; e += 4 * THREADS) {
      double2 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (e + u * THREADS < BN * h) v[u] = __ldcg(s + e + u * THREADS);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (e + u * THREADS < BN * h) __stcg(d + e + u * THREADS, v[u]);
    }
  }
}

}  // namespace hg
