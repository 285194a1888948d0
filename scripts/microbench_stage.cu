// Staging microbenchmark: per iteration every CTA loads S 32-byte sectors of a
// ~1 MB vector written by the other CTAs (after a grid barrier) into shared
// memory. Variants: 2x16B loads, one 32B load, sorted sector lists, TMA bulk
// copies, single active CTA.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/microbench_stage scripts/microbench_stage.cu
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void barrier(unsigned* ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    while (ld_acq(ctr) < target) {
    }
  }
  __syncthreads();
}
__device__ __forceinline__ double4 ld_sector(const double* p) {
  double4 r;
  asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(p)
               : "memory");
  return r;
}

__global__ void stage(unsigned* ctr, double* v0, double* v1, const unsigned* secs, int S, int per_cta, int iters,
                      int variant, int active, long long* out, double* sink) {
  extern __shared__ __align__(128) double xs[];
  __shared__ __align__(8) unsigned long long mbar;
  long long t_stage = 0;
  double acc = 0.0;
  const int T = blockDim.x, tid = threadIdx.x;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&mbar)));
  }
  __syncthreads();
  unsigned phase = 0;
  for (int l = 1; l <= iters; ++l) {
    double* vw = (l & 1) ? v1 : v0;
    const double* vr = (l & 1) ? v0 : v1;
    for (int i = tid; i < per_cta; i += T) vw[blockIdx.x * per_cta + i] = l + i;
    barrier(ctr, (unsigned)l * gridDim.x);
    long long bt = clock64();
    const unsigned* my = secs + (size_t)blockIdx.x * S;
    if (blockIdx.x < active) {
      if (variant == 0) {
        const double2* src = reinterpret_cast<const double2*>(vr);
        double2* dst = reinterpret_cast<double2*>(xs);
        for (int j = tid; j < S; j += T) {
          const size_t s = my[j];
          dst[2 * j] = src[2 * s];
          dst[2 * j + 1] = src[2 * s + 1];
        }
      } else if (variant == 1) {
        double4* dst = reinterpret_cast<double4*>(xs);
        for (int j0 = tid; j0 < S; j0 += 4 * T) {
          double4 r[4];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (j0 + u * T < S) r[u] = ld_sector(vr + 4 * (size_t)my[j0 + u * T]);
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (j0 + u * T < S) dst[j0 + u * T] = r[u];
        }
      } else if (variant == 2) {  // TMA bulk copies, 32 B each
        const unsigned mb = (unsigned)__cvta_generic_to_shared(&mbar);
        if (tid == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(mb), "r"((unsigned)(32 * S))
                       : "memory");
        __syncthreads();
        for (int j = tid; j < S; j += T) {
          const unsigned d = (unsigned)__cvta_generic_to_shared(xs + 4 * j);
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 32, [%2];" ::"r"(d),
              "l"(vr + 4 * (size_t)my[j]), "r"(mb)
              : "memory");
        }
        // wait for the phase
        unsigned done = 0;
        while (!done) {
          asm volatile(
              "{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
              : "=r"(done)
              : "r"(mb), "r"(phase)
              : "memory");
        }
        phase ^= 1;
      } else if (variant == 3) {  // 2 sectors per thread-load pair via 64-byte rows (v4 x2 when adjacent)
        double4* dst = reinterpret_cast<double4*>(xs);
        for (int j0 = tid; j0 < S; j0 += 8 * T) {
          double4 r[8];
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (j0 + u * T < S) r[u] = ld_sector(vr + 4 * (size_t)my[j0 + u * T]);
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (j0 + u * T < S) dst[j0 + u * T] = r[u];
        }
      }
    }
    __syncthreads();
    long long c = clock64();
    t_stage += c - bt;
    if (tid < 2 * S) acc += xs[tid];
  }
  if (tid == 0) out[blockIdx.x] = t_stage / iters;
  sink[blockIdx.x * blockDim.x + tid] = acc;
}

int main() {
  const int G = 148, per_cta = 830, nv = G * per_cta;
  long long* d_out;
  cudaMalloc(&d_out, 8 * G);
  std::vector<long long> h(G);
  unsigned* d_ctr;
  cudaMalloc(&d_ctr, 64);
  double *v0, *v1, *sink;
  cudaMalloc(&v0, (nv + 8) * 8);
  cudaMalloc(&v1, (nv + 8) * 8);
  cudaMalloc(&sink, G * 512 * 8);
  cudaFuncSetAttribute((void*)stage, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  srand(7);
  for (int S : {300, 650, 900, 1800}) {
    for (int sorted = 0; sorted < 2; ++sorted) {
      std::vector<unsigned> secs((size_t)G * S);
      for (int g = 0; g < G; ++g) {
        std::vector<unsigned> s;
        while ((int)s.size() < S) {
          s.push_back(rand() % (nv / 4));
        }
        if (sorted) std::sort(s.begin(), s.end());
        std::copy(s.begin(), s.end(), secs.begin() + (size_t)g * S);
      }
      unsigned* d_secs;
      cudaMalloc(&d_secs, secs.size() * 4);
      cudaMemcpy(d_secs, secs.data(), secs.size() * 4, cudaMemcpyHostToDevice);
      for (int variant = 0; variant < 4; ++variant) {
        for (int active : {G, 1}) {
          if (active == 1 && variant != 1) continue;
          cudaMemset(d_ctr, 0, 64);
          int it = 500, pc = per_cta, Sx = S, var = variant, act = active;
          void* args[] = {&d_ctr, &v0, &v1, &d_secs, &Sx, &pc, &it, &var, &act, &d_out, &sink};
          cudaError_t e = cudaLaunchCooperativeKernel((void*)stage, dim3(G), dim3(512), args, 32 * S, 0);
          cudaError_t e2 = cudaDeviceSynchronize();
          cudaMemcpy(h.data(), d_out, 8 * G, cudaMemcpyDeviceToHost);
          double m = 0;
          long long mx = 0;
          for (int g = 0; g < active; ++g) { m += h[g]; mx = std::max(mx, h[g]); }
          printf("S=%4d %s variant %d active %3d: staging mean %6.0f max %6lld cycles (%s/%s)\n", S,
                 sorted ? "sorted  " : "unsorted", variant, active, m / active, mx, cudaGetErrorString(e),
                 cudaGetErrorString(e2));
        }
      }
      cudaFree(d_secs);
    }
  }
  return 0;
}
