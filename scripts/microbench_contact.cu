// Latency of the per-contact one-shot (frame apply, trial impulse, strict
// projection, J_c^T scatter) for one lane per contact, 4 warps, data in smem.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -I paper_2201_09212_b200/csrc \
//        -o scripts/microbench_contact scripts/microbench_contact.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "vfpi_math.cuh"
using vfpi::frame_apply; using vfpi::frame_apply_t; using vfpi::trial_impulse; using vfpi::project_strict;
#define dsub vfpi::dsub
#define dadd vfpi::dadd
#define dmul vfpi::dmul

__global__ void oneshot_bench(const double* g_fr, const double* g_par, const double* g_vs, int C, int reps,
                              long long* out, double* sink) {
  __shared__ double fr[9 * 128], par[4 * 128], vs[6 * 128], lam_o[3 * 128], jt[6 * 128];
  const int k = threadIdx.x;
  for (int t = 0; t < 9; ++t) fr[9 * k + t] = g_fr[9 * k + t];
  for (int t = 0; t < 4; ++t) par[4 * k + t] = g_par[4 * k + t];
  for (int t = 0; t < 6; ++t) vs[6 * k + t] = g_vs[6 * k + t];
  __syncthreads();
  long long t_tr = 0, t_pr = 0, t_sc = 0;
  double th = 0.0;
  for (int r = 0; r < reps; ++r) {
    __syncthreads();
    long long a = clock64();
    const double* R9 = fr + 9 * k;
    double rel[3], eta[3], lam[3], wv[3];
    for (int t = 0; t < 3; ++t) rel[t] = dsub(vs[6 * k + t], vs[6 * k + 3 + t]);
    frame_apply(R9, rel, eta);
    trial_impulse(eta, par[4 * k + 2], par[4 * k + 3], lam);
    __syncwarp();
    long long b = clock64();
    project_strict(lam, par[4 * k + 0]);
    __syncwarp();
    long long c = clock64();
    for (int t = 0; t < 3; ++t) lam_o[3 * k + t] = lam[t];
    frame_apply_t(R9, lam, wv);
    for (int a2 = 0; a2 < 3; ++a2) {
      const double oi = dadd(0.0, wv[a2]);
      jt[6 * k + a2] = oi;
      const double vn = dadd(vs[6 * k + a2], dmul(0.3, oi));
      const double d = dsub(vn, vs[6 * k + a2]);
      th = dadd(th, dmul(d, d));
      const double oj = dsub(0.0, wv[a2]);
      jt[6 * k + 3 + a2] = oj;
      const double vn2 = dadd(vs[6 * k + 3 + a2], dmul(0.3, oj));
      const double d2 = dsub(vn2, vs[6 * k + 3 + a2]);
      th = dadd(th, dmul(d2, d2));
    }
    __syncwarp();
    long long d = clock64();
    t_tr += b - a;
    t_pr += c - b;
    t_sc += d - c;
    vs[6 * k] = dadd(vs[6 * k], 1e-300 * th);  // keep the chain alive
  }
  if (k == 0) {
    out[0] = t_tr / reps;
    out[1] = t_pr / reps;
    out[2] = t_sc / reps;
  }
  sink[k] = th + jt[6 * k] + lam_o[3 * k];
}

int main() {
  const int C = 128;
  double h_fr[9 * C], h_par[4 * C], h_vs[6 * C];
  srand(3);
  for (int k = 0; k < C; ++k) {
    double n[3] = {rand() / (double)RAND_MAX - 0.5, rand() / (double)RAND_MAX - 0.5, rand() / (double)RAND_MAX + 0.2};
    double nn = sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
    for (int t = 0; t < 9; ++t) h_fr[9 * k + t] = (t < 3 ? n[t] / nn : (rand() / (double)RAND_MAX - 0.5));
    h_par[4 * k + 0] = 0.5;
    h_par[4 * k + 1] = 0.5;
    h_par[4 * k + 2] = 0.0;
    h_par[4 * k + 3] = 3.7e-5 + 1e-6 * k;
    for (int t = 0; t < 6; ++t) h_vs[6 * k + t] = rand() / (double)RAND_MAX - 0.5;
  }
  double *d_fr, *d_par, *d_vs, *sink;
  long long* d_out;
  cudaMalloc(&d_fr, sizeof h_fr);
  cudaMalloc(&d_par, sizeof h_par);
  cudaMalloc(&d_vs, sizeof h_vs);
  cudaMalloc(&sink, 8 * C);
  cudaMalloc(&d_out, 64);
  cudaMemcpy(d_fr, h_fr, sizeof h_fr, cudaMemcpyHostToDevice);
  cudaMemcpy(d_par, h_par, sizeof h_par, cudaMemcpyHostToDevice);
  cudaMemcpy(d_vs, h_vs, sizeof h_vs, cudaMemcpyHostToDevice);
  for (int threads : {32, 128}) {
    oneshot_bench<<<1, threads>>>(d_fr, d_par, d_vs, C, 200, d_out, sink);
    cudaDeviceSynchronize();
    long long h[3];
    cudaMemcpy(h, d_out, 24, cudaMemcpyDeviceToHost);
    printf("%3d lanes: trial %lld, project %lld, scatter %lld cycles (%s)\n", threads, h[0], h[1], h[2],
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
