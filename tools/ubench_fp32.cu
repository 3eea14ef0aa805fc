// Microbenchmarks behind the beamform kernel's "alu" roofline (bench.py peak_basis):
// per-SM throughput of FFMA, FADD, FMUL, packed FFMA2 / FADD2 (fma.rn.f32x2 / add.rn.f32x2), LDS.32 /
// LDS.64 / LDS.128 shared-memory loads, and MUFU square root -- measured in SM clock cycles with
// clock64(), so the figures do not depend on the clock the GPU runs at.
//
// One CTA of 1024 threads (32 warps) per SM, every thread running independent dependency chains so
// the pipes, not latency, bound the loop.  Rate per SM = operations (lanes) of one CTA / its cycles.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_fp32 tools/ubench_fp32.cu
//   ./ubench_fp32            -> one JSON object on stdout (tools/ubench.py writes profiles/r02/ubench.json)

#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int THREADS = 1024;
constexpr int ITERS = 4096;
constexpr int CHAINS = 8;

__device__ unsigned long long g_cycles[1024];
__device__ float g_sink[1024 * THREADS];

__device__ __forceinline__ void publish(unsigned long long t0, float v) {
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  g_sink[blockIdx.x * THREADS + threadIdx.x] = v;
}

__global__ void __launch_bounds__(THREADS, 1) k_ffma(float a, float b) {
  float x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-3f + c;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fmaf(x[c], a, b);
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  publish(t0, s);
}

__global__ void __launch_bounds__(THREADS, 1) k_fadd(float a) {
  float x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-3f + c;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = __fadd_rn(x[c], a);
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  publish(t0, s);
}

__global__ void __launch_bounds__(THREADS, 1) k_fmul(float a) {
  float x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-3f + c;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = __fmul_rn(x[c], a);
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  publish(t0, s);
}

// packed FP32x2: one instruction, two lanes of work per thread
__global__ void __launch_bounds__(THREADS, 1) k_ffma2(float a, float b) {
  unsigned long long x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) {
    const float lo = threadIdx.x * 1e-3f + c, hi = lo + 0.5f;
    x[c] = ((unsigned long long)__float_as_uint(hi) << 32) | __float_as_uint(lo);
  }
  const unsigned long long av = ((unsigned long long)__float_as_uint(a) << 32) | __float_as_uint(a);
  const unsigned long long bv = ((unsigned long long)__float_as_uint(b) << 32) | __float_as_uint(b);
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[c]) : "l"(av), "l"(bv));
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += __uint_as_float((unsigned)x[c]) + __uint_as_float((unsigned)(x[c] >> 32));
  publish(t0, s);
}

__global__ void __launch_bounds__(THREADS, 1) k_fadd2(float a) {
  unsigned long long x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) {
    const float lo = threadIdx.x * 1e-3f + c, hi = lo + 0.5f;
    x[c] = ((unsigned long long)__float_as_uint(hi) << 32) | __float_as_uint(lo);
  }
  const unsigned long long av = ((unsigned long long)__float_as_uint(a) << 32) | __float_as_uint(a);
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(x[c]) : "l"(av));
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += __uint_as_float((unsigned)x[c]) + __uint_as_float((unsigned)(x[c] >> 32));
  publish(t0, s);
}

__global__ void __launch_bounds__(THREADS, 1) k_mufu_sqrt(float a) {
  float x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-3f + c + 1.f;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int i = 0; i < ITERS / 8; ++i)
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) asm volatile("sqrt.approx.f32 %0, %0;" : "+f"(x[c]));
  float s = a;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  publish(t0, s);
}

// shared-memory loads of W bytes per lane, consecutive lanes on consecutive words (conflict-free)
template <int W>
__global__ void __launch_bounds__(THREADS, 1) k_lds(int stride) {
  extern __shared__ __align__(16) uint8_t sm[];
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += THREADS) reinterpret_cast<float*>(sm)[i] = i;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm) + (uint32_t)((warp & 7) * 32 * W + lane * W);
  float acc = 0.f;
  const unsigned long long t0 = clock64();
  for (int i = 0; i < ITERS / 4; ++i) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint32_t a = base + (uint32_t)(c * stride * 8);       // immediate offsets: no address math
      if (W == 4) {
        float v;
        asm volatile("ld.volatile.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
        acc += v;
      } else if (W == 8) {
        float v0, v1;
        asm volatile("ld.volatile.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v0), "=f"(v1) : "r"(a));
        acc += v0 + v1;
      } else {
        float v0, v1, v2, v3;
        asm volatile("ld.volatile.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v0), "=f"(v1), "=f"(v2), "=f"(v3) : "r"(a));
        acc += (v0 + v1) + (v2 + v3);
      }
    }
  }
  publish(t0, acc);
}

static double run(const char* name, void (*launch)(int), int sm, double ops_per_block, bool first) {
  launch(sm);   // warm-up
  cudaDeviceSynchronize();
  launch(sm);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    fprintf(stderr, "%s: %s\n", name, cudaGetErrorString(e));
    return -1;
  }
  unsigned long long cyc[1024];
  cudaMemcpyFromSymbol(cyc, g_cycles, sizeof(unsigned long long) * sm);
  unsigned long long mx = 0;
  double mean = 0;
  for (int i = 0; i < sm; ++i) {
    mx = cyc[i] > mx ? cyc[i] : mx;
    mean += (double)cyc[i] / sm;
  }
  const double rate = ops_per_block / mean;
  printf("%s  \"%s\": {\"per_sm_per_clk\": %.2f, \"cycles_mean\": %.0f, \"cycles_max\": %llu}", first ? "" : ",\n",
         name, rate, mean, mx);
  return rate;
}

int main() {
  int sm = 0, clk = 0;
  cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaFuncSetAttribute(k_lds<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  cudaFuncSetAttribute(k_lds<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  cudaFuncSetAttribute(k_lds<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  const double lanes = (double)THREADS * ITERS * CHAINS;
  printf("{\n  \"sm_count\": %d, \"clock_rate_khz\": %d,\n", sm, clk);
  printf("  \"note\": \"1 CTA x 1024 threads per SM, 8 independent chains per thread; per_sm_per_clk = lanes (FP32 "
         "ops: one per lane, a packed x2 op counts 2) or bytes (LDS) or MUFU ops per SM per SM clock\",\n");
  run("ffma_lanes", [](int g) { k_ffma<<<g, THREADS>>>(1.0001f, 1e-7f); }, sm, lanes, true);
  run("fadd_lanes", [](int g) { k_fadd<<<g, THREADS>>>(1e-7f); }, sm, lanes, false);
  run("fmul_lanes", [](int g) { k_fmul<<<g, THREADS>>>(1.0000001f); }, sm, lanes, false);
  run("ffma2_lanes", [](int g) { k_ffma2<<<g, THREADS>>>(1.0001f, 1e-7f); }, sm, 2 * lanes, false);
  run("fadd2_lanes", [](int g) { k_fadd2<<<g, THREADS>>>(1e-7f); }, sm, 2 * lanes, false);
  run("mufu_sqrt_ops", [](int g) { k_mufu_sqrt<<<g, THREADS>>>(0.f); }, sm, (double)THREADS * (ITERS / 8) * CHAINS,
      false);
  run("lds32_bytes", [](int g) { k_lds<4><<<g, THREADS, 48 * 1024>>>(4 * 32); }, sm, (double)THREADS * ITERS * 4, false);
  run("lds64_bytes", [](int g) { k_lds<8><<<g, THREADS, 48 * 1024>>>(8 * 32); }, sm, (double)THREADS * ITERS * 8, false);
  run("lds128_bytes", [](int g) { k_lds<16><<<g, THREADS, 48 * 1024>>>(16 * 32); }, sm, (double)THREADS * ITERS * 16,
      false);
  printf("\n}\n");
  return 0;
}
