// SSSSM strip-kernel throughput with 32 concurrent tasks, for timing experiments:
//   nvcc ... [-DHG_EXP_RED_AS_STORE] [-DHG_EXP_NO_MOVES] tools/ssssm_ab.cu -o /tmp/ab && /tmp/ab
// (the experiment macros break the results; the product build never defines them)
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1402_6601_b200/csrc/tiles_lu.cu"
#include "../paper_1402_6601_b200/csrc/tiles_qr.cu"

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

int main(int argc, char** argv) {
  const bool qr = argc > 1 && argv[1][0] == 'q';  // TSMQR instead of SSSSM
  const int nb = 1024, ib = 128, conc = 32, reps = 5;
  const size_t tile = size_t(nb) * nb, slot = tile + size_t(ib) * nb + nb;
  if (!hg::init_lu_attributes() || !hg::init_qr_attributes()) return 1;
  std::vector<double> h(slot);
  srand(3);
  std::vector<double*> L(conc), T(conc), B(conc);
  std::vector<cudaStream_t> st(conc);
  for (int i = 0; i < conc; ++i) {
    for (size_t e = 0; e < tile; ++e) h[e] = (rand() / double(RAND_MAX) - 0.5) * 0.1;
    for (int c = 0; c < nb; ++c)  // side: identity inverse blocks, random bot-row pivots (TSTRF-like)
      for (int r = 0; r < ib; ++r) h[tile + size_t(c) * ib + r] = (r == c % ib) ? 1.0 : 0.0;
    int* piv = reinterpret_cast<int*>(h.data() + tile + size_t(ib) * nb);
    for (int j = 0; j < nb; ++j) piv[j] = rand() % nb;
    CK(cudaMalloc(&L[i], slot * 8));
    CK(cudaMalloc(&T[i], slot * 8));
    CK(cudaMalloc(&B[i], slot * 8));
    CK(cudaMemcpy(L[i], h.data(), slot * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(T[i], h.data(), tile * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(B[i], h.data(), tile * 8, cudaMemcpyHostToDevice));
    CK(cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking));
  }
  std::vector<hg::LaunchDesc> ld;
  auto run = [&](int r) {
    for (int rep = 0; rep < r; ++rep)
      for (int i = 0; i < conc; ++i) {
        hg::TaskOperands o;
        o.nb = nb;
        o.ib = ib;
        o.t[0] = L[i];
        o.t[1] = T[i];
        o.t[2] = B[i];
        o.n_t = 3;
        ld.clear();
        if (!(qr ? hg::build_qr_launches(hg::K_TSMQR, o, ld) : hg::build_lu_launches(hg::K_SSSSM, o, ld))) exit(1);
        for (auto& d : ld) {
#ifdef HG_PANEL_STAMPS
          if (qr) reinterpret_cast<hg::QrApplyParams*>(d.params)->stamp = (i == conc / 2 && rep == r - 1);
          else reinterpret_cast<hg::LuApplyParams*>(d.params)->stamp = (i == conc / 2 && rep == r - 1);
#endif
          void* args[1] = {d.params};
          CK(cudaLaunchKernel(d.func, d.grid, d.block, args, d.smem, st[i]));
        }
      }
  };
  run(1);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0));
  for (int i = 0; i < conc; ++i) CK(cudaStreamWaitEvent(st[i], e0));
  run(reps);
  for (int i = 0; i < conc; ++i) {
    cudaEvent_t ev;
    CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CK(cudaEventRecord(ev, st[i]));
    CK(cudaStreamWaitEvent(0, ev));
  }
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  const double fl = (qr ? 4.0 : 2.0) * nb * double(nb) * nb;
  printf("{\"kind\": \"%s\", \"tflops\": %.2f, \"ms\": %.2f", qr ? "TSMQR" : "SSSSM", conc * reps * fl / (ms * 1e-3) / 1e12, ms);
#ifdef HG_PANEL_STAMPS
  unsigned long long stp[16][512];
  CK(cudaMemcpyFromSymbol(stp, hg::g_panel_stamps, sizeof(stp)));
  double mv = 0, tr = 0, up = 0;
  for (int P = 0; P < 8; ++P) {
    const int b = 20 + 4 * P;
    mv += (stp[0][b + 1] - stp[0][b]) * 1e-3;
    tr += (stp[0][b + 2] - stp[0][b + 1]) * 1e-3;
    up += ((P < 7 ? stp[0][b + 4] : stp[0][b + 3]) - stp[0][b + 2]) * 1e-3;
  }
  printf(qr ? ", \"cta0_us\": {\"W=top+VtB\": %.1f, \"TtW\": %.1f, \"update\": %.1f}"
            : ", \"cta0_us\": {\"moves\": %.1f, \"trsm\": %.1f, \"update\": %.1f}", mv, tr, up);
#endif
  printf("}\n");
  return 0;
}
