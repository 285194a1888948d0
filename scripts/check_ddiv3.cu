// Bit-exactness check of vfpi::ddiv3 (shared-reciprocal division, csrc/vfpi_math.cuh)
// against __ddiv_rn on random and special operands. Prints mismatches; exit 1 on any.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 -I paper_2201_09212_b200/csrc \
//        -o /tmp/check_ddiv3 scripts/check_ddiv3.cu && /tmp/check_ddiv3
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <vector>
#include <random>
#include "vfpi_math.cuh"

__global__ void k(const double* a, const double* b, int n, unsigned long long* bad, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double aa[3] = {a[3 * i], a[3 * i + 1], a[3 * i + 2]};
  double q[3];
  vfpi::ddiv3(aa, b[i], q);
  for (int t = 0; t < 3; ++t) {
    const double r = __ddiv_rn(aa[t], b[i]);
    if (__double_as_longlong(r) != __double_as_longlong(q[t])) {
      const unsigned long long k = atomicAdd(bad, 1ull);
      if (k < 8) { out[3 * k] = aa[t]; out[3 * k + 1] = b[i]; out[3 * k + 2] = q[t]; }
    }
  }
}

static double pick(std::mt19937_64& g) {
  static const double sp[] = {0.0, -0.0, 1.0, -1.0, 1e-320, -4.9e-324, 2.2250738585072014e-308, 1.7976931348623157e308,
                              INFINITY, -INFINITY, NAN, 3.0, 1e-300, 1e300, 0x1p-1022, 0x1p1023, 0x1p-1074};
  const unsigned c = g() % 16;
  if (c == 0) return sp[g() % (sizeof(sp) / sizeof(sp[0]))];
  if (c == 1) { uint64_t u = g(); double d; memcpy(&d, &u, 8); return d; }  // any bit pattern
  std::uniform_real_distribution<double> U(-1.0, 1.0);
  const int e = (c < 8) ? (int)(g() % 40) - 20 : (int)(g() % 2100) - 1050;
  return ldexp(U(g), e);
}

int main() {
  const int n = 1 << 22;
  std::mt19937_64 g(2201);
  std::vector<double> a(3 * (size_t)n), b(n);
  for (auto& x : a) x = pick(g);
  for (auto& x : b) x = pick(g);
  double *da, *db, *dout;
  unsigned long long* dbad;
  cudaMalloc(&da, 8 * a.size()); cudaMalloc(&db, 8 * b.size()); cudaMalloc(&dout, 8 * 24); cudaMalloc(&dbad, 8);
  cudaMemcpy(da, a.data(), 8 * a.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), 8 * b.size(), cudaMemcpyHostToDevice);
  unsigned long long bad = 0, total = 0;
  for (int rep = 0; rep < 8; ++rep) {
    if (rep) {
      for (auto& x : a) x = pick(g);
      for (auto& x : b) x = pick(g);
      cudaMemcpy(da, a.data(), 8 * a.size(), cudaMemcpyHostToDevice);
      cudaMemcpy(db, b.data(), 8 * b.size(), cudaMemcpyHostToDevice);
    }
    cudaMemset(dbad, 0, 8);
    k<<<(n + 255) / 256, 256>>>(da, db, n, dbad, dout);
    unsigned long long nb = 0;
    cudaMemcpy(&nb, dbad, 8, cudaMemcpyDeviceToHost);
    if (nb && !bad) {
      double o[24];
      cudaMemcpy(o, dout, 8 * 24, cudaMemcpyDeviceToHost);
      for (unsigned k2 = 0; k2 < nb && k2 < 8; ++k2) printf("mismatch a=%a b=%a got=%a\n", o[3 * k2], o[3 * k2 + 1], o[3 * k2 + 2]);
    }
    bad += nb;
    total += 3ull * n;
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("ddiv3 vs __ddiv_rn: %llu quotients, %llu mismatches, %s\n", total, bad, cudaGetErrorString(e));
  return (bad || e != cudaSuccess) ? 1 : 0;
}
