// Grid-barrier microbenchmark (148 CTAs x 512 threads, cooperative launch):
// K-way sharded monotonic counters. CTA b release-adds counter (b % K) (or its
// SM's die half when K == -2); lanes 0..K-1 of warp 0 acquire-poll one counter
// each until it reaches epoch * (CTAs mapped to it).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/microbench_bar scripts/microbench_bar.cu
#include <algorithm>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

__device__ __forceinline__ unsigned ld_rlx(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_vol(const unsigned* p) {
  unsigned v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// mode 0: red.relaxed + ld.relaxed (no ordering), 1: fence.acq_rel + red.relaxed + ld.relaxed + fence,
// 2: red.release + ld.acquire, 3: red.relaxed + ld.acquire, 4: red.release + ld.relaxed + fence.acquire-ish
// (fence.acq_rel after the spin), 5: atom.add.release (returns) + ld.acquire
__global__ void bar_modes(unsigned* ctr, int mode, int iters, int nstores, double* buf, long long* out) {
  const int G = gridDim.x, b = blockIdx.x;
  long long t0 = clock64();
  for (int l = 1; l <= iters; ++l) {
    for (int i = threadIdx.x; i < nstores; i += blockDim.x) buf[((size_t)b * nstores + i) * 5 % (G * nstores)] = l;
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned target = (unsigned)l * G;
      if (mode == 0) {
        asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        while (ld_rlx(ctr) < target) {
        }
      } else if (mode == 1) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        while (ld_rlx(ctr) < target) {
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      } else if (mode == 2) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        while (ld_acq(ctr) < target) {
        }
      } else if (mode == 3) {
        asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        while (ld_acq(ctr) < target) {
        }
      } else if (mode == 4) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        while (ld_rlx(ctr) < target) {
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      } else if (mode == 5) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        while (ld_vol(ctr) < target) {
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[b] = (t1 - t0) / iters;
}

__global__ void bar_sharded(unsigned* ctr, int K, int iters, int work, long long* out, double* sink) {
  const int G = gridDim.x, b = blockIdx.x;
  const int slot = (K > 0) ? b % K : 0;
  const int KK = K > 0 ? K : 1;
  __shared__ double red[16];
  double acc = b;
  long long t0 = clock64();
  for (int l = 1; l <= iters; ++l) {
    // a little work so arrivals are not perfectly aligned
    for (int i = 0; i < work; ++i) acc = acc * 1.0000001 + 1e-9;
    __syncthreads();
    if (threadIdx.x == 0)
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr + 32 * slot) : "memory");
    if (threadIdx.x < 32) {
      const int c = threadIdx.x;
      if (c < KK) {
        const unsigned n_c = (unsigned)((G - c + KK - 1) / KK);  // CTAs with b % K == c
        const unsigned target = (unsigned)l * n_c;
        while (ld_acq(ctr + 32 * c) < target) {
        }
      }
      __syncwarp();
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[b] = (t1 - t0) / iters;
  if (threadIdx.x < 16) red[threadIdx.x] = acc;
  sink[b] = red[0];
}

int main() {
  const int G = 148;
  long long* d_out;
  cudaMalloc(&d_out, 8 * G);
  double* sink;
  cudaMalloc(&sink, 8 * G);
  unsigned* ctr;
  cudaMalloc(&ctr, 4 * 32 * 64);
  std::vector<long long> h(G);
  double* buf;
  cudaMalloc(&buf, 8 * 148 * 1024);
  for (int ns : {0, 800}) {
    for (int mode = 0; mode < 6; ++mode) {
      cudaMemset(ctr, 0, 4 * 32 * 64);
      int it = 3000, m = mode, n = ns;
      void* args[] = {&ctr, &m, &it, &n, &buf, &d_out};
      cudaError_t e = cudaLaunchCooperativeKernel((void*)bar_modes, dim3(G), dim3(512), args, 0, 0);
      cudaError_t e2 = cudaDeviceSynchronize();
      cudaMemcpy(h.data(), d_out, 8 * G, cudaMemcpyDeviceToHost);
      long long mn = *std::min_element(h.begin(), h.end()), mx = *std::max_element(h.begin(), h.end());
      printf("stores %3d mode %d: %lld..%lld cycles per iteration (%s/%s)\n", ns, mode, mn, mx, cudaGetErrorString(e),
             cudaGetErrorString(e2));
    }
  }
  for (int work : {0}) {
    for (int K : {1, 2, 4, 8, 16, 32}) {
      cudaMemset(ctr, 0, 4 * 32 * 64);
      int it = 3000, k = K, w = work;
      void* args[] = {&ctr, &k, &it, &w, &d_out, &sink};
      cudaError_t e = cudaLaunchCooperativeKernel((void*)bar_sharded, dim3(G), dim3(512), args, 0, 0);
      cudaError_t e2 = cudaDeviceSynchronize();
      cudaMemcpy(h.data(), d_out, 8 * G, cudaMemcpyDeviceToHost);
      long long mn = *std::min_element(h.begin(), h.end()), mx = *std::max_element(h.begin(), h.end());
      printf("work %3d K=%2d: %lld..%lld cycles per iteration (%s/%s)\n", work, K, mn, mx, cudaGetErrorString(e),
             cudaGetErrorString(e2));
    }
  }
  return 0;
}
