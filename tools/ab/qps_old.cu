// Phase timeline of one k_qr_panel launch (TSQRT or GEQRT panel 0, nb=1024, ib=128) from the
// kernel's own %globaltimer stamps (HG_PANEL_STAMPS).  Build + run on a B200:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DHG_PANEL_STAMPS \
//        -I paper_1402_6601_b200/csrc -I include tools/qr_panel_stamps.cu -o /tmp/qps && /tmp/qps t
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tiles_qr_old.cu"

namespace hg {
void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vfprintf(stderr, fmt, ap);
  va_end(ap);
  fputc('\n', stderr);
}
}  // namespace hg

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e = (x);                                                         \
    if (e != cudaSuccess) {                                                      \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
      exit(1);                                                                   \
    }                                                                            \
  } while (0)

static unsigned long long zero_stamps[16][512];

int main(int argc, char** argv) {
  const int nb = 1024, ib = 128;
  const bool ts = argc < 2 || argv[1][0] == 't';
  const size_t tile = size_t(nb) * nb, slot = tile + size_t(ib) * nb + nb;
  std::vector<double> h(tile);
  srand(1);
  double *A, *R;
  CK(cudaMalloc(&A, slot * 8));
  CK(cudaMalloc(&R, slot * 8));
  CK(cudaMemset(A, 0, slot * 8));
  for (size_t i = 0; i < tile; ++i) h[i] = rand() / double(RAND_MAX) - 0.5;
  CK(cudaMemcpy(A, h.data(), tile * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(R, h.data(), tile * 8, cudaMemcpyHostToDevice));
  if (!hg::init_qr_attributes()) return 1;
  hg::QrPanelParams pp{A, ts ? R : nullptr, A + tile, nb, ib, 0, ib, ts ? hg::QR_TSQRT : hg::QR_GEQRT};
  for (int rep = 0; rep < 3; ++rep) {  // fresh operands every time (the panel factors in place)
    CK(cudaMemcpy(A, h.data(), tile * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(R, h.data(), tile * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpyToSymbol(hg::g_panel_stamps, zero_stamps, sizeof(zero_stamps)));
    hg::k_qr_panel<<<hg::kQrCl, hg::kQrThreads, hg::qr_panel_smem(nb, ib)>>>(pp);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
  }
  unsigned long long st[16][512];
  CK(cudaMemcpyFromSymbol(st, hg::g_panel_stamps, sizeof(st)));
  auto ns = [&](int q, int k) { return (long long)(st[q][k] - st[0][0]); };
  printf("{\"mode\": \"%s\", \"total_us\": %.1f, \"loop_us\": %.1f, \"t_factor_us\": %.1f, \"phases_ns\": [",
         ts ? "tsqrt" : "geqrt", ns(0, 82) * 1e-3, ns(0, 80) * 1e-3, (ns(0, 82) - ns(0, 80)) * 1e-3);
  // per column: barrier1 wait, tau, scale+products, pw+barrier2, reduce w, T/R+apply, next norm
  for (int j = 1; j < 15; ++j) {
    const int b = 300 + 8 * j;
    printf("%s[%lld, %lld, %lld, %lld, %lld, %lld, %lld]", j > 1 ? ", " : "", ns(0, b + 1) - ns(0, b),
           ns(0, b + 2) - ns(0, b + 1), ns(0, b + 3) - ns(0, b + 2), ns(0, b + 4) - ns(0, b + 3),
           ns(0, b + 5) - ns(0, b + 4), ns(0, b + 6) - ns(0, b + 5), ns(0, b + 8) - ns(0, b + 6));
  }
  printf("], \"tsqrt_exact_norm_columns\": %llu}\n", st[0][500]);
  return 0;
}
