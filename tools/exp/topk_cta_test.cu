// Standalone check of launch_topk_cta against a CPU reference (not part of the library).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <numeric>
#include <cstring>
#include "../../paper_2510_24273_b200/csrc/kernels.h"
using namespace sals;
#ifdef SALS_TKC_TRACE
namespace sals { namespace tkc { extern __device__ long long g_tkc_t[16]; } }
#endif
#ifdef SALS_TOPK_DBG3
namespace sals { namespace tkc { extern __device__ int g_d3[12][1024]; } }
#endif
static uint32_t fkey(float f) { f += 0.0f; uint32_t u; memcpy(&u, &f, 4); return (u & 0x80000000u) ? ~u : (u | 0x80000000u); }
int main(int argc, char** argv) {
  int fails = 0;
  srand(1);
  for (int trial = 0; trial < 40; ++trial) {
    const int B = 1 + trial % 3;
    const int n = (trial < 30) ? 32 + rand() % 8000 : 8192 + rand() % 120000;
    const int k = 1 + rand() % n;
    const int stride = (n + 3) / 4 * 4;
    std::vector<float> sc(B * stride, 0.f);
    for (auto& v : sc) v = (float)((rand() % 2000) - 1000) / ((trial % 4 == 0) ? 1.f : 37.f);
    std::vector<uint32_t> h(B * kH0Bins, 0);
    for (int b = 0; b < B; ++b) for (int i = 0; i < n; ++i) h[b * kH0Bins + (fkey(sc[b * stride + i]) >> kH0Shift)]++;
    float* dsc; uint32_t* dh; int *dsel, *dlen, *dcnt;
    cudaMalloc(&dsc, sc.size() * 4); cudaMalloc(&dh, h.size() * 4); cudaMalloc(&dsel, B * k * 4); cudaMalloc(&dlen, B * 4); cudaMalloc(&dcnt, B * 4);
    cudaMemcpy(dsc, sc.data(), sc.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dh, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    std::vector<int> len(B, n);
    cudaMemcpy(dlen, len.data(), B * 4, cudaMemcpyHostToDevice);
    TopkArgs a{};
    a.scores = dsc; a.score_stride = stride; a.seq_len = dlen; a.k = k; a.mode = 0;
    a.sel_out = dsel; a.sel_stride = k; a.sel_count = dcnt; a.pad_to = k; a.hist0 = dh;
    cudaError_t e = launch_topk_cta(a, B, n, 0);
    cudaError_t e2 = cudaDeviceSynchronize();
#ifdef SALS_TOPK_DBG3
    if (trial == 39) {
      static int d3[12][1024]; cudaMemcpyFromSymbol(d3, sals::tkc::g_d3, sizeof(d3));
      FILE* f = fopen("gpurun_out/d3.bin", "wb"); fwrite(d3, 4, 12 * 1024, f); fclose(f);
      FILE* g = fopen("gpurun_out/d3_scores.bin", "wb"); fwrite(sc.data(), 4, stride, g); fclose(g);
      printf("dumped trial 39 n %d k %d\n", n, k);
    }
#endif
    std::vector<int> sel(B * k);
    cudaMemcpy(sel.data(), dsel, B * k * 4, cudaMemcpyDeviceToHost);
    for (int b = 0; b < B; ++b) {
      std::vector<int> idx(n);
      std::iota(idx.begin(), idx.end(), 0);
      const float* r = &sc[b * stride];
      std::stable_sort(idx.begin(), idx.end(), [&](int x, int y) { return fkey(r[x]) > fkey(r[y]); });
      std::vector<int> ref(idx.begin(), idx.begin() + k);
      std::sort(ref.begin(), ref.end());
      bool ok = std::equal(ref.begin(), ref.end(), sel.begin() + b * k);
      int cnt = -1; cudaMemcpy(&cnt, dcnt + b, 4, cudaMemcpyDeviceToHost);
      int inter = 0; for (int i = 0; i < k; ++i) inter += std::binary_search(ref.begin(), ref.end(), sel[b * k + i]);
      if (!ok) printf("   count %d k %d overlap %d\n", cnt, k, inter);
      if (!ok) { ++fails; printf("trial %d b %d n %d k %d MISMATCH (gpu %d %d %d .. ref %d %d %d) err %d %d\n", trial, b, n, k, sel[b*k], sel[b*k+1], sel[b*k+2], ref[0], ref[1], ref[2], (int)e, (int)e2); }
    }
    cudaFree(dsc); cudaFree(dh); cudaFree(dsel); cudaFree(dlen); cudaFree(dcnt);
  }
  printf("fails %d\n", fails);
  {   // timing: c2-like (B = 8, n = 4096, k = 512), 200 back-to-back launches
    const int B = 8, n = 4096, k = 512, stride = 4096;
    std::vector<float> sc(B * stride);
    for (auto& v : sc) v = (float)((rand() % 200000) - 100000) / 7777.f;
    std::vector<uint32_t> h(B * kH0Bins, 0);
    for (int b = 0; b < B; ++b) for (int i = 0; i < n; ++i) h[b * kH0Bins + (fkey(sc[b * stride + i]) >> kH0Shift)]++;
    float* dsc; uint32_t* dh; int *dsel, *dlen, *dcnt;
    cudaMalloc(&dsc, sc.size() * 4); cudaMalloc(&dh, h.size() * 4); cudaMalloc(&dsel, B * k * 4); cudaMalloc(&dlen, B * 4); cudaMalloc(&dcnt, B * 4);
    cudaMemcpy(dsc, sc.data(), sc.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dh, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    std::vector<int> len(B, n);
    cudaMemcpy(dlen, len.data(), B * 4, cudaMemcpyHostToDevice);
    TopkArgs a{};
    a.scores = dsc; a.score_stride = stride; a.seq_len = dlen; a.k = k; a.mode = 0;
    a.sel_out = dsel; a.sel_stride = k; a.sel_count = dcnt; a.pad_to = k; a.hist0 = dh;
    cudaStream_t st; cudaStreamCreate(&st);
    for (int i = 0; i < 20; ++i) launch_topk_cta(a, B, n, st);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
    for (int i = 0; i < 200; ++i) launch_topk_cta(a, B, n, st);
    cudaEventRecord(e1, st); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("c2-like topk_cta: %.2f us per launch\n", ms * 1000 / 200);
#ifdef SALS_TKC_TRACE
    long long t[16]; cudaMemcpyFromSymbol(t, sals::tkc::g_tkc_t, sizeof(t));
    for (int i = 1; i < 7; ++i) printf("  stamp %d: +%lld cycles\n", i, t[i] - t[0]);
#endif
  }
  return fails != 0;
}
