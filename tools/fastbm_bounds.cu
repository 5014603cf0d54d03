// Exhaustive error survey of single-precision Box-Muller pieces against the fp64 contract
// (NC-3) over every 32-bit word: the radius word a (r = sqrt(-2 zlog((a+1) 2^-32))) and the
// angle word b (sin, cos of 2 pi b 2^-32).  Prints per-octave maxima of |r_f - r| as JSON.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -I paper_2208_06102_b200/csrc
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "contract.cuh"
using namespace zs;

constexpr int NB = 48;   // octave buckets of r: [2^(k-40), 2^(k-39)), k = 0..47
__device__ unsigned int g_dmax[NB], g_d2max[NB], g_rmin[NB];
__device__ unsigned int g_cnt[NB], g_dmaxB[NB];
__device__ unsigned int g_ang[4];   // max |c_f - c|, |s_f - s|, max r_f (bits), spare

__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2_approx(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__global__ void radius_kernel(const double2 *logtab, uint64_t begin, uint64_t n) {
  __shared__ double2 tab[kLogTab];
  for (int i = threadIdx.x; i < kLogTab; i += blockDim.x) tab[i] = logtab[i];
  __syncthreads();
  for (uint64_t i = begin + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < begin + n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t a = (uint32_t)i;
    const double u1 = (double)((unsigned long long)a + 1ull) * 0x1p-32;
    const double r2 = -2.0 * zlog(u1, tab);
    const double r = sqrt(r2);
    const float uf = fmaf(__uint2float_rn(a), 0x1p-32f, 0x1p-32f);
    const float r2f = lg2_approx(uf) * -1.3862943611198906f;
    const float rf = sqrt_approx(r2f);
    const double d = fabs((double)rf - r);
    // variant B: -ln(1 - d) by its series when d = 1 - u1 = (~a) 2^-32 < 2^-6
    const float dd = __uint2float_rn(~a) * 0x1p-32f;
    const float pser = fmaf(dd, fmaf(dd, fmaf(dd, 0.25f, 0.33333334f), 0.5f), 1.0f);
    const float r2B = (~a < (1u << 26)) ? 2.0f * dd * pser : r2f;
    const float rB = sqrt_approx(r2B);
    atomicMax(&g_dmaxB[(r > 0 ? min(max((int)floor(log2(r)) + 40, 0), NB - 1) : 0)],
              __float_as_uint((float)fabs((double)rB - r)));
    const double d2 = fabs((double)r2f - r2);
    int k = r > 0 ? (int)floor(log2(r)) + 40 : 0;
    k = k < 0 ? 0 : (k >= NB ? NB - 1 : k);
    atomicMax(&g_dmax[k], __float_as_uint((float)d));
    atomicMax(&g_d2max[k], __float_as_uint((float)d2));
    atomicMin(&g_rmin[k], __float_as_uint(rf));
    atomicAdd(&g_cnt[k], 1u);
    atomicMax(&g_ang[2], __float_as_uint(rf));
  }
}

__global__ void angle_kernel(uint64_t begin, uint64_t n) {
  for (uint64_t i = begin + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < begin + n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t b = (uint32_t)i;
    double s, c;
    zsincospi_b32(b, s, c);
    const float x = (float)(int)b * 1.4629180792671596e-09f;   // 2 pi 2^-32
    float sf, cf;
    __sincosf(x, &sf, &cf);
    atomicMax(&g_ang[0], __float_as_uint((float)fabs((double)cf - c)));
    atomicMax(&g_ang[1], __float_as_uint((float)fabs((double)sf - s)));
  }
}

int main() {
  double2 *tab;
  cudaMalloc(&tab, kLogTab * sizeof(double2));
  log_table_kernel<<<1, 128>>>(tab);
  unsigned int init[NB];
  for (int i = 0; i < NB; ++i) init[i] = 0x7f800000u;
  cudaMemcpyToSymbol(g_rmin, init, sizeof(init));
  const uint64_t N = 1ull << 32, chunk = 1ull << 30;
  for (uint64_t b = 0; b < N; b += chunk) {
    radius_kernel<<<148 * 8, 256>>>(tab, b, chunk);
    angle_kernel<<<148 * 8, 256>>>(b, chunk);
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { fprintf(stderr, "%s\n", cudaGetErrorString(e)); return 1; }
  unsigned int dmaxB[NB], dmax[NB], d2max[NB], rmin[NB], cnt[NB], ang[4];
  cudaMemcpyFromSymbol(dmax, g_dmax, sizeof(dmax));
  cudaMemcpyFromSymbol(dmaxB, g_dmaxB, sizeof(dmaxB));
  cudaMemcpyFromSymbol(d2max, g_d2max, sizeof(d2max));
  cudaMemcpyFromSymbol(rmin, g_rmin, sizeof(rmin));
  cudaMemcpyFromSymbol(cnt, g_cnt, sizeof(cnt));
  cudaMemcpyFromSymbol(ang, g_ang, sizeof(ang));
  auto f = [](unsigned int u) { float x; memcpy(&x, &u, 4); return x; };
  printf("{\"angle_cos_max\": %.6e, \"angle_sin_max\": %.6e, \"r_f_max\": %.9g, \"buckets\": [\n",
         f(ang[0]), f(ang[1]), f(ang[2]));
  bool first = true;
  for (int k = 0; k < NB; ++k) {
    if (!cnt[k]) continue;
    printf("%s {\"r_lo\": %.6e, \"count\": %u, \"rf_min\": %.6e, \"d_max\": %.6e, \"d2_max\": %.6e, \"dB_max\": %.6e}",
           first ? "" : ",\n", ldexp(1.0, k - 40), cnt[k], f(rmin[k]), f(dmax[k]), f(d2max[k]), f(dmaxB[k]));
    first = false;
  }
  printf("\n]}\n");
  return 0;
}
