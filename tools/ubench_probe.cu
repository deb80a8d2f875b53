// Microbenchmark: the random-probe rate a top-down BFS level is bounded by.
// Random 4 B accesses into an L2-resident bitmap (8 MB = RMAT-26's visited
// set), indices streamed coalesced from HBM like `col` is.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o ubench_probe tools/ubench_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

template <int MODE>
__global__ void probe(const uint32_t* __restrict__ idx, size_t n, uint32_t* bm, uint32_t* out) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const uint32_t v = __ldcs(&idx[i]);
    if (MODE == 0) acc ^= __ldcg(&bm[v >> 5]);
    if (MODE == 1) acc ^= __ldca(&bm[v >> 5]);
    if (MODE == 2) atomicOr(&bm[v >> 5], 1u << (v & 31));  // RED (result unused)
    if (MODE == 3) acc ^= atomicOr(&bm[v >> 5], 0u);        // ATOM with return
  }
  if (acc == 0x12345678u) out[0] = acc;
}

template <int MODE, int U>
__global__ void probe_ilp(const uint32_t* __restrict__ idx, size_t n, uint32_t* bm, uint32_t* out) {
  uint32_t acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride * U) {
    uint32_t v[U], w[U];
#pragma unroll
    for (int k = 0; k < U; ++k) v[k] = __ldcs(&idx[i + k * stride < n ? i + k * stride : i]);
#pragma unroll
    for (int k = 0; k < U; ++k) w[k] = MODE == 0 ? __ldcg(&bm[v[k] >> 5]) : __ldca(&bm[v[k] >> 5]);
#pragma unroll
    for (int k = 0; k < U; ++k) acc ^= w[k];
  }
  if (acc == 0x12345678u) out[0] = acc;
}

int main() {
  const size_t n = 1ull << 30;            // 1 Gi probes
  const uint32_t nv = 1u << 26;           // vertices (8 MB bitmap)
  std::vector<uint32_t> h(n);
  std::mt19937 rng(1);
  // RMAT-like skew: each id bit is 1 with p = 0.24 (as RMAT endpoints), or uniform.
  for (int skew = 0; skew < 2; ++skew) {
    for (size_t i = 0; i < n; ++i) {
      uint32_t v = 0;
      if (skew) {
        for (int b = 0; b < 26; ++b) v = (v << 1) | ((rng() % 100) < 24);
      } else {
        v = rng() % nv;
      }
      h[i] = v;
    }
    uint32_t *idx, *bm, *out;
    cudaMalloc(&idx, n * 4);
    cudaMalloc(&bm, nv / 8);
    cudaMalloc(&out, 4);
    cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
    cudaMemset(bm, 0, nv / 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char* names[] = {"ld.cg", "ld.ca", "red.or", "atom.or", "ld.cg x8", "ld.ca x8"};
    for (int mode = 0; mode < 6; ++mode) {
      for (int occ : {148 * 8, 148 * 16}) {
        float best = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
          cudaEventRecord(a);
          if (mode == 0) probe<0><<<occ, 256>>>(idx, n, bm, out);
          if (mode == 1) probe<1><<<occ, 256>>>(idx, n, bm, out);
          if (mode == 2) probe<2><<<occ, 256>>>(idx, n, bm, out);
          if (mode == 3) probe<3><<<occ, 256>>>(idx, n, bm, out);
          if (mode == 4) probe_ilp<0, 8><<<occ, 256>>>(idx, n, bm, out);
          if (mode == 5) probe_ilp<1, 8><<<occ, 256>>>(idx, n, bm, out);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          best = ms < best ? ms : best;
        }
        printf("%s %-9s grid=%5d: %7.2f G probes/s  (%.3f ms for 1 Gi)\n", skew ? "rmat" : "unif",
               names[mode], occ, n / (best * 1e-3) / 1e9, best);
      }
    }
    cudaFree(idx);
    cudaFree(bm);
    cudaFree(out);
  }
  return 0;
}
