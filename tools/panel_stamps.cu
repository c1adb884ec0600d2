// Phase timeline of one k_lu_panel_sp launch (TSTRF or GETRF panel 0, nb=1024, ib=128) from the
// kernel's own %globaltimer stamps (HG_PANEL_STAMPS).  Build + run on a B200:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DHG_PANEL_STAMPS \
//        -I paper_1402_6601_b200/csrc -I include tools/panel_stamps.cu -o /tmp/panel_stamps && /tmp/panel_stamps
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1402_6601_b200/csrc/tiles_lu.cu"

namespace hg {
void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vfprintf(stderr, fmt, ap);
  va_end(ap);
  fputc('\n', stderr);
}
}  // namespace hg

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e = (x);                                                               \
    if (e != cudaSuccess) {                                                            \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));       \
      exit(1);                                                                         \
    }                                                                                  \
  } while (0)

int main(int argc, char** argv) {
  const int nb = 1024, ib = 128;
  const bool ts = argc < 2 || argv[1][0] == 't';
  const size_t tile = size_t(nb) * nb, slot = tile + size_t(ib) * nb + nb;
  std::vector<double> h(tile);
  srand(1);
  double *A, *U;
  CK(cudaMalloc(&A, slot * 8));
  CK(cudaMalloc(&U, slot * 8));
  CK(cudaMemset(A, 0, slot * 8));
  CK(cudaMemset(U, 0, slot * 8));
  for (size_t i = 0; i < tile; ++i) h[i] = rand() / double(RAND_MAX) - 0.5;
  CK(cudaMemcpy(A, h.data(), tile * 8, cudaMemcpyHostToDevice));
  for (int c = 0; c < nb; ++c)
    for (int r = 0; r < nb; ++r) h[size_t(c) * nb + r] = r > c ? 0.0 : (r == c ? 0.2 : rand() / double(RAND_MAX) - 0.5);
  CK(cudaMemcpy(U, h.data(), tile * 8, cudaMemcpyHostToDevice));
  if (!hg::init_lu_attributes()) return 1;
  hg::LuPanelParams pp{A, ts ? U : nullptr, A + tile, nb, ib, 0, ib, ts ? hg::LU_TSTRF : hg::LU_GETRF, nullptr};
  for (int rep = 0; rep < 3; ++rep) {
    hg::k_lu_panel_sp<128><<<hg::kLuCl, hg::kSpThreads, hg::sp_smem(nb)>>>(pp);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
  }
  unsigned long long st[8][512];
  CK(cudaMemcpyFromSymbol(st, hg::g_panel_stamps, sizeof(st)));
  auto us = [&](int q, int k) { return (st[q][k] - st[0][0]) * 1e-3; };
  printf("{\"mode\": \"%s\", \"total_us\": %.1f, \"setup_us\": %.1f", ts ? "tstrf" : "getrf", us(0, 82), us(0, 1));
  double col = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0, s5 = 0, s6 = 0;
  for (int s = 0; s < 8; ++s) {
    const int b = 2 + s * 8;
    col += us(0, b + 1) - us(0, b);
    s1 += us(0, b + 2) - us(0, b + 1);
    s2 += us(0, b + 3) - us(0, b + 2);
    if (s == 7) {  // the last sub-panel has no right-hand columns
      s6 += us(0, 80) - us(0, b + 3);
      continue;
    }
    s3 += us(0, b + 4) - us(0, b + 3);
    s4 += us(0, b + 5) - us(0, b + 4);
    s5 += us(0, b + 6) - us(0, b + 5);
    s6 += us(0, b + 8) - us(0, b + 6);
  }
  printf(", \"column_loops_us\": %.1f, \"S_read_bar_us\": %.1f, \"S_write_us\": %.1f, \"U12_fwd_bar_us\": %.1f, "
         "\"U12_copy_us\": %.1f, \"A22_bar_us\": %.1f, \"gap_us\": %.1f, \"writeback_us\": %.1f, \"inverse_us\": %.1f",
         col, s1, s2, s3, s4, s5, s6, us(0, 80) - us(0, 2 + 7 * 8 + 3), us(0, 82) - us(0, 80));
  printf(", \"first_subpanel_phases_ns\": [");  // per column: argmax+sync, push, wait, pivot+update
  for (int u = 1; u < 16; ++u)
    printf("%s[%llu, %llu, %llu, %llu]", u > 1 ? ", " : "", st[0][300 + 4 * u] - st[0][303 + 4 * (u - 1)],
           st[0][301 + 4 * u] - st[0][300 + 4 * u], st[0][302 + 4 * u] - st[0][301 + 4 * u],
           st[0][303 + 4 * u] - st[0][302 + 4 * u]);
  printf("]");
  printf(", \"subpanel1_by_cta_ns\": [");  // per CTA: column loop end, S read barrier, S write, fwd barrier, copy, A22 barrier
  for (int q = 0; q < 8; ++q) {
    const int b = 2 + 1 * 8;
    printf("%s[", q ? ", " : "");
    for (int k = 1; k <= 6; ++k) printf("%s%llu", k > 1 ? ", " : "", st[q][b + k] - st[0][b]);
    printf("]");
  }
  printf("]");
  printf(", \"s_phase_ns\": [%llu, %llu, %llu, %llu, %llu]", st[0][400] - st[0][2 + 8 + 1], st[0][401] - st[0][400],
         st[0][402] - st[0][401], st[0][403] - st[0][402], st[0][2 + 8 + 2] - st[0][403]);
  printf(", \"per_column_us\": [");
  for (int j = 1; j < 128; ++j) printf("%s%.2f", j > 1 ? ", " : "", us(0, 100 + j) - us(0, 100 + j - 1));
  printf("]}\n");
  return 0;
}
