// peaks.cu -- B200 ALU peaks and latencies for the replay's roofline.
//
// Throughput kernels: every SM full of warps, each thread running 8 independent
// chains of one instruction type; result in lane-instructions per second.
// Latency kernels: one thread, one dependent chain, timed with clock64().
// Build + run:  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peaks tools/peaks.cu && ./peaks
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e)); return 1; } } while (0)

constexpr int kIters = 4096;

__global__ void dfma_tput(double *out, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.0) out[0] = s;
}

__global__ void dmul_tput(double *out, double a) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i + 1;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = x[i] * a;
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.0) out[0] = s;
}

// INT throughput: one PTX instruction per op, each a single SASS instruction (checked with
// cuobjdump: 1024 LOP3 / IMAD / IMAD.HI per unrolled loop body and nothing else but the loop
// counter), 8 independent chains per thread, operands in registers so nothing folds.  (A chain
// of add.u32 is folded by ptxas into one IMAD, so the ALU pipe is measured with LOP3 only.)
constexpr int kUnroll = 4;
#define INT_TPUT(NAME, ASM)                                                                  \
  __global__ void NAME(uint32_t *out, uint32_t a, uint32_t b) {                              \
    uint32_t x[8];                                                                           \
    _Pragma("unroll") for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 7 + i;                \
    for (int it = 0; it < kIters / kUnroll; ++it) {                                          \
      _Pragma("unroll") for (int u = 0; u < kUnroll; ++u)                                    \
      _Pragma("unroll") for (int i = 0; i < 8; ++i) asm volatile(ASM : "+r"(x[i]) : "r"(a), "r"(b)); \
    }                                                                                        \
    uint32_t s = 0;                                                                          \
    _Pragma("unroll") for (int i = 0; i < 8; ++i) s ^= x[i];                                 \
    if (s == 12345u) out[0] = s;                                                             \
  }
INT_TPUT(lop3_tput, "lop3.b32 %0, %0, %1, %2, 0x96;")          // LOP3.LUT (alu pipe)
INT_TPUT(imad_tput, "mad.lo.u32 %0, %0, %1, %2;")               // IMAD (fma pipe)
INT_TPUT(imadhi_tput, "mad.hi.u32 %0, %0, %1, %2;")             // IMAD.HI (fma pipe)

__global__ void dfma_lat(double *out, long long *cyc, double a, double b) {
  double x = threadIdx.x;
  const long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) x = fma(x, a, b);
  const long long t1 = clock64();
  out[0] = x;
  cyc[0] = t1 - t0;
}

__global__ void ddiv_lat(double *out, long long *cyc, double a) {
  double x = threadIdx.x + 1.5;
  const long long t0 = clock64();
  for (int it = 0; it < 256; ++it) x = a / x;
  const long long t1 = clock64();
  out[0] = x;
  cyc[0] = t1 - t0;
}

__global__ void imad_lat(uint32_t *out, long long *cyc, uint32_t m) {
  uint32_t x = threadIdx.x + 3;
  const long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) x = __umulhi(x, m) ^ it;
  const long long t1 = clock64();
  out[0] = x;
  cyc[0] = t1 - t0;
}

template <class F>
double time_ms(F launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / 5.0;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  double *d;
  uint32_t *u;
  long long *c;
  CK(cudaMalloc(&d, 64));
  CK(cudaMalloc(&u, 64));
  CK(cudaMalloc(&c, 64));
  const int sms = p.multiProcessorCount, tpb = 256, blocks = sms * 8;
  const double threads = (double)blocks * tpb;
  const double ops = threads * kIters * 8;
  double ms_dfma = time_ms([&] { dfma_tput<<<blocks, tpb>>>(d, 0.999999, 1e-9); });
  double ms_dmul = time_ms([&] { dmul_tput<<<blocks, tpb>>>(d, 0.999999); });
  double ms_lop = time_ms([&] { lop3_tput<<<blocks, tpb>>>(u, 0x9E3779B9u, 0x10u); });
  double ms_imad = time_ms([&] { imad_tput<<<blocks, tpb>>>(u, 0xD2511F53u, 0x10u); });
  double ms_imadhi = time_ms([&] { imadhi_tput<<<blocks, tpb>>>(u, 0xD2511F53u, 0x10u); });
  CK(cudaGetLastError());
  long long h[3];
  dfma_lat<<<1, 1>>>(d, c, 0.999999, 1e-9);
  CK(cudaMemcpy(&h[0], c, 8, cudaMemcpyDeviceToHost));
  ddiv_lat<<<1, 1>>>(d, c, 1.000001);
  CK(cudaMemcpy(&h[1], c, 8, cudaMemcpyDeviceToHost));
  imad_lat<<<1, 1>>>(u, c, 0xD2511F53u);
  CK(cudaMemcpy(&h[2], c, 8, cudaMemcpyDeviceToHost));
  printf("{\"device\": \"%s\", \"sms\": %d, \"clock_rate_mhz\": %.0f, "
         "\"dfma_lane_per_s\": %.4e, \"dmul_lane_per_s\": %.4e, \"lop3_lane_per_s\": %.4e, "
         "\"imad_lane_per_s\": %.4e, \"imad_hi_lane_per_s\": %.4e, "
         "\"dfma_latency_cyc\": %.2f, \"ddiv_latency_cyc\": %.1f, \"imad_hi_xor_latency_cyc\": %.2f}\n",
         p.name, sms, clk_khz / 1e3, ops / (ms_dfma * 1e-3), ops / (ms_dmul * 1e-3),
         ops / (ms_lop * 1e-3), ops / (ms_imad * 1e-3),
         ops / (ms_imadhi * 1e-3), (double)h[0] / kIters, (double)h[1] / 256, (double)h[2] / kIters);
  return 0;
}
