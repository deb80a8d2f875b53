// Microbenchmark: cost of one grid-wide barrier inside a persistent kernel
// with the traversal kernel's geometry (3 x 256-thread CTAs per SM). A
// small BFS level is ~2 such barriers plus a few L2 round trips, so this is
// the floor of the per-level latency on deep graphs (the 4096^2 mesh).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o ubench_barrier tools/ubench_barrier.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;
constexpr int kGroups = 16;

struct Ctl {
  unsigned long long top;
  unsigned long long pad0[15];
  unsigned long long sub[kGroups][16];
  unsigned long long flat;
  unsigned long long pad1[15];
};

__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long atom_add_release(unsigned long long* p,
                                                               unsigned long long x) {
  unsigned long long old;
  asm volatile("atom.add.release.gpu.global.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(x) : "memory");
  return old;
}
__device__ __forceinline__ void red_add_release(unsigned long long* p, unsigned long long x) {
  asm volatile("red.add.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(x) : "memory");
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

template <int MODE>
__global__ void __launch_bounds__(256, 3) bar_loop(Ctl* ctl, int iters, unsigned* sink) {
  unsigned long long k = 0;
  unsigned acc = 0;
  for (int it = 0; it < iters; ++it) {
    // A token of per-level work: one global write per CTA.
    if (threadIdx.x == 0) sink[blockIdx.x] = it;
    if (MODE == 4) {
      cg::this_grid().sync();
      acc += sink[(blockIdx.x + 1) % gridDim.x];
      continue;
    }
    __syncthreads();
    ++k;
    if (threadIdx.x == 0) {
      if (MODE == 0) {  // two-level, sc fences, relaxed poll + nanosleep (current)
        const unsigned g = blockIdx.x % kGroups;
        const unsigned long long size = (gridDim.x - g + kGroups - 1) / kGroups;
        __threadfence();
        const unsigned long long old = atomicAdd(&ctl->sub[g][0], 1ull);
        if (old == k * size - 1) atomicAdd(&ctl->top, 1ull);
        while (ld_relaxed(&ctl->top) < k * kGroups) __nanosleep(32);
        __threadfence();
      } else if (MODE == 1) {  // flat, release arrive, relaxed spin, acq_rel fence
        atom_add_release(&ctl->flat, 1ull);
        while (ld_relaxed(&ctl->flat) < k * gridDim.x) {
        }
        fence_acq_rel();
      } else if (MODE == 2) {  // flat, red.release arrive, acquire spin
        red_add_release(&ctl->flat, 1ull);
        while (ld_acquire(&ctl->flat) < k * gridDim.x) {
        }
      } else if (MODE == 3) {  // two-level, release/acquire, no sleep
        const unsigned g = blockIdx.x % kGroups;
        const unsigned long long size = (gridDim.x - g + kGroups - 1) / kGroups;
        const unsigned long long old = atom_add_release(&ctl->sub[g][0], 1ull);
        if (old == k * size - 1) {
          fence_acq_rel();
          red_add_release(&ctl->top, 1ull);
        }
        while (ld_relaxed(&ctl->top) < k * kGroups) {
        }
        fence_acq_rel();
      } else if (MODE == 5) {  // flat, red.release arrive, relaxed spin + nanosleep(20), fence
        red_add_release(&ctl->flat, 1ull);
        while (ld_relaxed(&ctl->flat) < k * gridDim.x) __nanosleep(20);
        fence_acq_rel();
      } else if (MODE == 7) {  // flat 32-bit flip-bit counter, atom.release, acquire spin
        unsigned* c = reinterpret_cast<unsigned*>(&ctl->flat);
        const unsigned nb = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u;
        unsigned old, cur;
        asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(c), "r"(nb) : "memory");
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(c) : "memory");
        } while (((old ^ cur) & 0x80000000u) == 0);
      } else if (MODE == 6) {  // flat, red.release arrive, relaxed spin, fence
        red_add_release(&ctl->flat, 1ull);
        while (ld_relaxed(&ctl->flat) < k * gridDim.x) {
        }
        fence_acq_rel();
      }
    }
    __syncthreads();
    acc += sink[(blockIdx.x + 1) % gridDim.x];
  }
  if (acc == 0xdeadbeefu) sink[0] = acc;
}

template <int MODE>
void run(const char* name, int blocks_per_sm) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * blocks_per_sm;
  Ctl* ctl;
  unsigned* sink;
  cudaMalloc(&ctl, sizeof(Ctl));
  cudaMalloc(&sink, grid * sizeof(unsigned));
  const int iters = 20000;
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(ctl, 0, sizeof(Ctl));
    int it = iters;
    void* args[] = {&ctl, &it, &sink};
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaError_t e = cudaLaunchCooperativeKernel((void*)bar_loop<MODE>, grid, 256, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) {
      printf("%s: launch failed: %s\n", name, cudaGetErrorString(e));
      return;
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  printf("%-52s grid %4d: %.3f us per barrier\n", name, grid, best * 1e3f / iters);
  cudaFree(ctl);
  cudaFree(sink);
}

int main() {
  for (int bps : {3, 1}) {
    run<0>("two-level, sc fences, relaxed poll + nanosleep(32)", bps);
    run<3>("two-level, release/acquire, spin", bps);
    run<1>("flat, atom.release, relaxed spin, fence", bps);
    run<6>("flat, red.release, relaxed spin, fence", bps);
    run<5>("flat, red.release, relaxed spin + nanosleep(20)", bps);
    run<2>("flat, red.release, acquire spin", bps);
    run<7>("flat u32 flip bit, atom.release, acquire spin", bps);
    run<4>("cooperative_groups grid.sync()", bps);
  }
  return 0;
}
