// Microbenchmarks that bound the resident iteration kernel on B200:
//   (a) dependent-load latency to L2 (pointer chase, one warp)
//   (b) grid barrier round trip (release-add counter + acquire spin), 148 CTAs
//   (c) barrier + per-CTA staging of S random 32-byte sectors written by other CTAs
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb scripts/microbench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_rel(unsigned* p) {
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}
__device__ __forceinline__ void barrier(unsigned* ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    red_rel(ctr);
    while (ld_acq(ctr) < target) {
    }
  }
  __syncthreads();
}

__device__ __forceinline__ unsigned ld_rlx(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// variant 1: relaxed red + relaxed spin + acq_rel fences
__device__ __forceinline__ void barrier_v1(unsigned* ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    while (ld_rlx(ctr) < target) {
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}
// variant 2: per-CTA flags, warp 0 polls all flags in parallel
__device__ __forceinline__ void barrier_v2(unsigned* flags, unsigned epoch) {
  __syncthreads();
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) st_rel(flags + blockIdx.x * 32, epoch);
    for (;;) {
      bool ok = true;
      for (int k = 0; k < 5; ++k) {
        const int g = threadIdx.x + 32 * k;
        if (g < (int)gridDim.x) ok &= ld_rlx(flags + g * 32) >= epoch;
      }
      if (__all_sync(0xffffffffu, ok)) break;
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}
// variant 3: CTA 0 collects, then releases one go word
__device__ __forceinline__ void barrier_v3(unsigned* ctr, unsigned* go, unsigned epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    red_rel(ctr);
    if (blockIdx.x == 0) {
      while (ld_acq(ctr) < epoch * gridDim.x) {
      }
      st_rel(go, epoch);
    } else {
      while (ld_acq(go) < epoch) {
      }
    }
  }
  __syncthreads();
}
__global__ void bar_var(unsigned* ctr, unsigned* flags, int iters, int var, long long* out) {
  long long t0 = clock64();
  for (int l = 1; l <= iters; ++l) {
    if (var == 1) barrier_v1(ctr, (unsigned)l * gridDim.x);
    else if (var == 2) barrier_v2(flags, (unsigned)l);
    else barrier_v3(ctr, flags, (unsigned)l);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / iters;
}

__global__ void fp64_lat(double* io, long long* out, int n) {
  double a = io[0], b = io[1], c = io[2];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = __dadd_rn(a, b);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) c = __dmul_rn(c, b);
  long long t2 = clock64();
  double d = a;
  for (int i = 0; i < n; ++i) d = __ddiv_rn(d, b);
  long long t3 = clock64();
  double e = c + 2.0;
  for (int i = 0; i < n; ++i) e = __dsqrt_rn(e) + 1.0;
  long long t4 = clock64();
  io[3] = a + c + d + e;
  if (threadIdx.x == 0) { out[0] = (t1 - t0) / n; out[1] = (t2 - t1) / n; out[2] = (t3 - t2) / n; out[3] = (t4 - t3) / n; }
}

// SELL row dots out of shared memory: 512 threads, rows of `len` entries,
// x gathered at random smem offsets (like xs / vown in the resident kernel)
__global__ void rowdot_bench(int len, int nx, long long* out, double* sink) {
  extern __shared__ double smd[];
  double* sv = smd;                          // [len*512]
  unsigned* mp = (unsigned*)(sv + len * 512);  // [len*512]
  double* xs = (double*)(mp + len * 512 + (len * 512) % 2);
  const int T = blockDim.x, tid = threadIdx.x;
  unsigned seed = 12345u + tid;
  for (int i = tid; i < len * 512; i += T) {
    seed = seed * 1664525u + 1013904223u;
    sv[i] = 1.0 + (i & 7);
    mp[i] = seed % nx;
  }
  for (int i = tid; i < nx; i += T) xs[i] = 0.5 * i;
  __syncthreads();
  double acc = 0.0;
  long long t0 = clock64();
  for (int rep = 0; rep < 16; ++rep) {
    const int base = tid;
    int k = 0;
    for (; k + 4 <= len; k += 4) {
      double a[4], x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = base + 512 * (k + u);
        a[u] = sv[i];
        x[u] = xs[mp[i]];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) acc = __dadd_rn(acc, __dmul_rn(a[u], x[u]));
    }
    for (; k < len; ++k) acc = __dadd_rn(acc, __dmul_rn(sv[base + 512 * k], xs[mp[base + 512 * k]]));
  }
  __syncthreads();
  long long t1 = clock64();
  sink[tid] = acc;
  if (tid == 0) out[0] = (t1 - t0) / 16;
}

__global__ void chase(const unsigned* next, int steps, long long* out) {
  unsigned i = 0;
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) i = next[i];
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / steps + (i == 0xffffffff);
}

__global__ void bar_only(unsigned* ctr, int iters, long long* out) {
  long long t0 = clock64();
  for (int l = 1; l <= iters; ++l) barrier(ctr, (unsigned)l * gridDim.x);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / iters;
}

// each iteration: write own slice of v, barrier, load S sectors of other CTAs' slices
__global__ void bar_stage(unsigned* ctr, double* v0, double* v1, const unsigned* secs, int S, int per_cta, int iters,
                          long long* out, double* sink) {
  extern __shared__ double xs[];
  long long t_stage = 0, t_bar = 0;
  double acc = 0.0;
  for (int l = 1; l <= iters; ++l) {
    double* vw = (l & 1) ? v1 : v0;
    const double* vr = (l & 1) ? v0 : v1;
    for (int i = threadIdx.x; i < per_cta; i += blockDim.x) vw[blockIdx.x * per_cta + i] = l + i;
    long long a = clock64();
    barrier(ctr, (unsigned)l * gridDim.x);
    long long bt = clock64();
    const double2* src = reinterpret_cast<const double2*>(vr);
    double2* dst = reinterpret_cast<double2*>(xs);
    for (int j = threadIdx.x; j < S; j += blockDim.x) {
      const size_t s = secs[blockIdx.x * S + j];
      dst[2 * j] = src[2 * s];
      dst[2 * j + 1] = src[2 * s + 1];
    }
    __syncthreads();
    long long c = clock64();
    t_bar += bt - a;
    t_stage += c - bt;
    if (threadIdx.x < 2 * S) acc += xs[threadIdx.x];
  }
  if (threadIdx.x == 0) {
    out[2 * blockIdx.x] = t_bar / iters;
    out[2 * blockIdx.x + 1] = t_stage / iters;
  }
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  long long* d_out;
  cudaMalloc(&d_out, 1 << 20);
  std::vector<long long> h(4096);
  // (a) pointer chase over 16 MB (L2-resident after a warm pass)
  const int N = 4 << 20;
  std::vector<unsigned> nx(N);
  {
    std::vector<unsigned> perm(N);
    for (int i = 0; i < N; ++i) perm[i] = i;
    srand(1);
    for (int i = N - 1; i > 0; --i) { int j = rand() % (i + 1); std::swap(perm[i], perm[j]); }
    for (int i = 0; i < N; ++i) nx[perm[i]] = perm[(i + 1) % N];
  }
  unsigned* d_nx;
  cudaMalloc(&d_nx, N * 4);
  cudaMemcpy(d_nx, nx.data(), N * 4, cudaMemcpyHostToDevice);
  chase<<<1, 32>>>(d_nx, 1 << 16, d_out);
  chase<<<1, 32>>>(d_nx, 1 << 16, d_out);
  cudaMemcpy(h.data(), d_out, 8, cudaMemcpyDeviceToHost);
  printf("L2 dependent-load latency: %lld cycles\n", h[0]);
  {
    double* io;
    cudaMalloc(&io, 64);
    double hv[4] = {1.0, 1.0000001, 3.0, 0.0};
    cudaMemcpy(io, hv, 32, cudaMemcpyHostToDevice);
    fp64_lat<<<1, 32>>>(io, d_out, 4096);
    cudaMemcpy(h.data(), d_out, 32, cudaMemcpyDeviceToHost);
    printf("fp64 dependent latency: DADD %lld, DMUL %lld, DDIV %lld, DSQRT(+DADD) %lld cycles\n", h[0], h[1], h[2], h[3]);
  }
  for (int len : {4, 16, 45}) {
    double* sink;
    cudaMalloc(&sink, 512 * 8);
    const int nx = 3000;
    const size_t smb = (size_t)len * 512 * 12 + 16 + nx * 8;
    cudaFuncSetAttribute((void*)rowdot_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    rowdot_bench<<<1, 512, smb>>>(len, nx, d_out, sink);
    cudaDeviceSynchronize();
    cudaMemcpy(h.data(), d_out, 8, cudaMemcpyDeviceToHost);
    printf("row dot from smem, 512 rows x %d entries: %lld cycles (%s)\n", len, h[0], cudaGetErrorString(cudaGetLastError()));
    cudaFree(sink);
  }
  // (b) barrier only
  unsigned* d_ctr;
  cudaMalloc(&d_ctr, 64);
  for (int threads : {32, 512}) {
    cudaMemset(d_ctr, 0, 64);
    int G = 148, it = 2000;
    void* args[] = {&d_ctr, &it, &d_out};
    cudaLaunchCooperativeKernel((void*)bar_only, dim3(G), dim3(threads), args, 0, 0);
    cudaDeviceSynchronize();
    cudaMemcpy(h.data(), d_out, 8 * G, cudaMemcpyDeviceToHost);
    long long mn = h[0], mx = h[0];
    for (int g = 0; g < G; ++g) { mn = std::min(mn, h[g]); mx = std::max(mx, h[g]); }
    printf("barrier only (148 CTAs x %d thr): %lld..%lld cycles per barrier\n", threads, mn, mx);
  }
  for (int var = 1; var <= 3; ++var) {
    unsigned* d_flags;
    cudaMalloc(&d_flags, 148 * 128 + 64);
    cudaMemset(d_flags, 0, 148 * 128 + 64);
    cudaMemset(d_ctr, 0, 64);
    int G = 148, it = 2000;
    void* args[] = {&d_ctr, &d_flags, &it, &var, &d_out};
    cudaError_t e = cudaLaunchCooperativeKernel((void*)bar_var, dim3(G), dim3(512), args, 0, 0);
    cudaDeviceSynchronize();
    cudaMemcpy(h.data(), d_out, 8 * G, cudaMemcpyDeviceToHost);
    long long mn = h[0], mx = h[0];
    for (int g = 0; g < G; ++g) { mn = std::min(mn, h[g]); mx = std::max(mx, h[g]); }
    printf("barrier variant %d: %lld..%lld cycles (%s)\n", var, mn, mx, cudaGetErrorString(e));
    cudaFree(d_flags);
  }
  // (c) barrier + staging of S sectors per CTA from a 1 MB vector
  const int G = 148, per_cta = 830, nv = G * per_cta;
  double *v0, *v1, *sink;
  cudaMalloc(&v0, (nv + 8) * 8);
  cudaMalloc(&v1, (nv + 8) * 8);
  cudaMalloc(&sink, G * 512 * 8);
  for (int S : {0, 300, 900, 2000}) {
    std::vector<unsigned> secs(G * std::max(S, 1));
    for (auto& x : secs) x = rand() % (nv / 4);
    unsigned* d_secs;
    cudaMalloc(&d_secs, secs.size() * 4);
    cudaMemcpy(d_secs, secs.data(), secs.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(d_ctr, 0, 64);
    int it = 1000, pc = per_cta;
    void* args[] = {&d_ctr, &v0, &v1, &d_secs, &S, &pc, &it, &d_out, &sink};
    cudaFuncSetAttribute((void*)bar_stage, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    cudaError_t e = cudaLaunchCooperativeKernel((void*)bar_stage, dim3(G), dim3(512), args, 32 * std::max(S, 1), 0);
    cudaDeviceSynchronize();
    cudaMemcpy(h.data(), d_out, 16 * G, cudaMemcpyDeviceToHost);
    double mb = 0, ms = 0;
    for (int g = 0; g < G; ++g) { mb += h[2 * g]; ms += h[2 * g + 1]; }
    printf("S=%4d sectors/CTA: barrier %.0f cycles, staging %.0f cycles (err=%s)\n", S, mb / G, ms / G,
           cudaGetErrorString(e));
    cudaFree(d_secs);
  }
  return 0;
}
