// Grid-barrier variants for the resident kernel (148 CTAs x 512 threads, one per SM).
// Every iteration each CTA stores `nstores` doubles (its v_next rows), publishes
// three partial doubles, signals, waits for all CTAs and then warp 0 reads all
// G partials (as the resident kernel's decision does).
//   mode 0: one monotonic counter, red.release + ld.acquire poll (current kernel)
//   mode 1: per-CTA flag words packed (148 x u32), st.release; warp 0 polls with
//           ld.relaxed (<=5 flags per lane) + __all_sync, then fence.acq_rel
//   mode 2: per-CTA flags, one 32-byte sector each, same polling as 1
//   mode 3: as 1 but the poll loads are ld.acquire
//   mode 4: per-CTA flag = the epoch stored into the partial record itself
//           (st.release of the u32 epoch after the 3 doubles, same sector); warp 0
//           polls the epochs of all records and then reads the doubles
//   mode 5: cluster pairs: barrier.cluster arrive/wait, leader red.release on a
//           counter of 74 arrivals, poll, cluster barrier again
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/microbench_bar2 scripts/microbench_bar2.cu
#include <algorithm>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_rlx(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int MODE>
__global__ void bar(unsigned* ctr, unsigned* flags, double* part, int iters, int nstores, double* buf,
                    long long* out, double* sink) {
  const int G = gridDim.x, b = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ double tot;
  double acc = 0.0;
  long long t0 = 0;
  for (int l = 1; l <= iters; ++l) {
    if (l == 2) t0 = clock64();
    for (int i = threadIdx.x; i < nstores; i += blockDim.x) buf[(size_t)b * nstores + i] = l + acc;
    __syncthreads();
    if (MODE == 5) {
      asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    }
    if (threadIdx.x == 0) {
      double* q = part + (size_t)b * 4;
      q[0] = l;
      q[1] = b;
      q[2] = acc;
      if (MODE == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        while (ld_acq(ctr) < (unsigned)l * G) {
        }
      } else if (MODE == 1 || MODE == 3) {
        st_rel(flags + b, l);
      } else if (MODE == 2) {
        st_rel(flags + 8 * b, l);
      } else if (MODE == 4) {
        st_rel(reinterpret_cast<unsigned*>(q + 3), l);
      } else if (MODE == 5) {
        unsigned rank;
        asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
        if (rank == 0) {
          asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
          while (ld_acq(ctr) < (unsigned)l * (G / 2)) {
          }
        }
      }
    }
    if (MODE >= 1 && MODE <= 4 && warp == 0) {
      bool done = false;
      while (!done) {
        bool ok = true;
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const int g = lane + 32 * k;
          if (g < G) {
            unsigned f;
            if (MODE == 1) f = ld_rlx(flags + g);
            else if (MODE == 2) f = ld_rlx(flags + 8 * g);
            else if (MODE == 3) f = ld_acq(flags + g);
            else f = ld_rlx(reinterpret_cast<const unsigned*>(part + (size_t)g * 4 + 3));
            ok = ok && (f >= (unsigned)l);
          }
        }
        done = __all_sync(0xffffffffu, ok);
      }
      if (MODE != 3) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    if (MODE == 5) {
      asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    }
    if (warp == 0) {  // read all partials
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        const int g = lane + 32 * k;
        if (g < G) s += __ldcg(part + (size_t)g * 4 + 2) + __ldcg(part + (size_t)g * 4 + 0);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) tot = s;
    }
    __syncthreads();
    acc = tot * 1e-30;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) {
    out[b] = (t1 - t0) / (iters - 1);
    sink[b] = acc;
  }
}

template <int MODE>
void run(int nstores, unsigned* ctr, unsigned* flags, double* part, double* buf, long long* d_out, double* sink) {
  const int G = 148;
  cudaMemset(ctr, 0, 4 * 64);
  cudaMemset(flags, 0, 4 * 8 * 256);
  cudaMemset(part, 0, 8 * 4 * 256);
  int it = 2000;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(512);
  cudaLaunchAttribute at[2];
  int na = 0;
  at[na].id = cudaLaunchAttributeCooperative;
  at[na].val.cooperative = 1;
  ++na;
  if (MODE == 5) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = 2;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  cudaError_t e = cudaLaunchKernelEx(&cfg, bar<MODE>, ctr, flags, part, it, nstores, buf, d_out, sink);
  cudaError_t e2 = cudaDeviceSynchronize();
  std::vector<long long> h(G);
  cudaMemcpy(h.data(), d_out, 8 * G, cudaMemcpyDeviceToHost);
  long long mn = *std::min_element(h.begin(), h.end()), mx = *std::max_element(h.begin(), h.end());
  printf("stores %4d mode %d: %lld..%lld cycles per iteration (%s/%s)\n", nstores, MODE, mn, mx,
         cudaGetErrorString(e), cudaGetErrorString(e2));
}

int main() {
  long long* d_out;
  double *sink, *part, *buf;
  unsigned *ctr, *flags;
  cudaMalloc(&d_out, 8 * 256);
  cudaMalloc(&sink, 8 * 256);
  cudaMalloc(&part, 8 * 4 * 256);
  cudaMalloc(&buf, 8 * 148 * 2048);
  cudaMalloc(&ctr, 4 * 64);
  cudaMalloc(&flags, 4 * 8 * 256);
  for (int ns : {0, 832}) {
    run<0>(ns, ctr, flags, part, buf, d_out, sink);
    run<1>(ns, ctr, flags, part, buf, d_out, sink);
    run<2>(ns, ctr, flags, part, buf, d_out, sink);
    run<3>(ns, ctr, flags, part, buf, d_out, sink);
    run<4>(ns, ctr, flags, part, buf, d_out, sink);
    run<5>(ns, ctr, flags, part, buf, d_out, sink);
  }
  return 0;
}
