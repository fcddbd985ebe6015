// ubench_fp.cu -- issue rate of the FP32 instruction forms the butterflies use
// (scalar FFMA/FADD, packed FFMA2/FADD2/FMUL2; register, uniform-register and
// immediate operands), measured as warp instructions per cycle per SM.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o ubench_fp tools/ubench_fp.cu
// Run:   ./ubench_fp  (one line per form; check the forms with cuobjdump -sass)
#include <cuda_runtime.h>

#include <cstdio>

constexpr int ACC = 12;    // independent chains per thread
constexpr int ITERS = 2048;

enum Kind { FFMA_RRR, FFMA_RIR, FFMA_RUR, FADD_RR, FFMA2_RIR, FFMA2_RUR, FFMA2_RRR, FADD2_RR, FMUL2_RI, MIX_2D, MIX_HALF, MIX_SCALAR_HALF };

template <int K>
__global__ void __launch_bounds__(256) kern(float* out, float ku, float kv) {
  const float kr = ku + threadIdx.x * 1e-30f;  // a per-thread (vector register) value
  if constexpr (K <= FADD_RR || K == MIX_SCALAR_HALF) {
    float a[ACC];
#pragma unroll
    for (int i = 0; i < ACC; ++i) a[i] = threadIdx.x * 0.001f + i;
#pragma unroll 1
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
      for (int i = 0; i < ACC; ++i) {
        if constexpr (K == FFMA_RRR) a[i] = fmaf(a[i], kr, a[(i + 1) % ACC]);
        if constexpr (K == FFMA_RIR) a[i] = fmaf(a[i], 0.70710677f, a[(i + 1) % ACC]);
        if constexpr (K == FFMA_RUR) a[i] = fmaf(a[i], ku, a[(i + 1) % ACC]);
        if constexpr (K == FADD_RR) a[i] = a[i] + a[(i + 1) % ACC];
        if constexpr (K == MIX_SCALAR_HALF) {
          if (i % 2 == 0) a[i] = a[i] + a[(i + 1) % ACC];
          else a[i] = fmaf(a[i], 0.70710677f, a[(i + 1) % ACC]);
        }
      }
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < ACC; ++i) s += a[i];
    if (s == 1234.5f) out[threadIdx.x] = s;
  } else {
    float2 a[ACC];
#pragma unroll
    for (int i = 0; i < ACC; ++i) a[i] = make_float2(threadIdx.x * 0.001f + i, i * 0.5f);
    const float2 kr2 = make_float2(kr, kr), ku2 = make_float2(ku, ku), ki2 = make_float2(0.70710677f, 0.70710677f);
#pragma unroll 1
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
      for (int i = 0; i < ACC; ++i) {
        if constexpr (K == FFMA2_RIR) a[i] = __ffma2_rn(a[i], ki2, a[(i + 1) % ACC]);
        if constexpr (K == FFMA2_RUR) a[i] = __ffma2_rn(a[i], ku2, a[(i + 1) % ACC]);
        if constexpr (K == FFMA2_RRR) a[i] = __ffma2_rn(a[i], kr2, a[(i + 1) % ACC]);
        if constexpr (K == FADD2_RR) a[i] = __fadd2_rn(a[i], a[(i + 1) % ACC]);
        if constexpr (K == FMUL2_RI) a[i] = __fmul2_rn(a[i], ki2);
        if constexpr (K == MIX_HALF) {  // 1 FADD2 : 1 FFMA2-imm (do they share a pipe?)
          if (i % 2 == 0) a[i] = __fadd2_rn(a[i], a[(i + 1) % ACC]);
          else a[i] = __ffma2_rn(a[i], ki2, a[(i + 1) % ACC]);
        }
        if constexpr (K == MIX_2D) {  // butterfly-like: add / sub / ffma-imm alternating
          if (i % 3 == 0) a[i] = __fadd2_rn(a[i], a[(i + 1) % ACC]);
          else if (i % 3 == 1) a[i] = __fadd2_rn(a[i], make_float2(-a[(i + 1) % ACC].x, -a[(i + 1) % ACC].y));
          else a[i] = __ffma2_rn(a[i], ki2, a[(i + 1) % ACC]);
        }
      }
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < ACC; ++i) s += a[i].x + a[i].y;
    if (s == 1234.5f) out[threadIdx.x] = s;
  }
}

template <int K>
void run(const char* name, float* out, int sms, int clk_khz) {
  const int threads = 256, per_sm = 4;  // 32 warps / SM (8 per SMSP)
  const int grid = sms * per_sm;
  kern<K><<<grid, threads>>>(out, 0.999f, 0.5f);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) kern<K><<<grid, threads>>>(out, 0.999f, 0.5f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double winst = double(reps) * grid * (threads / 32) * ITERS * ACC;
  const double cycles = ms * 1e-3 * clk_khz * 1e3;
  std::printf("%-10s %.3f warp-instr / cycle / SM (%.3f per SMSP; rt %.2f), %.3f ms\n", name,
              winst / cycles / sms, winst / cycles / sms / 4, 4.0 * cycles * sms / winst, ms / reps);
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  std::printf("%s, %d SMs, clock attr %d kHz\n", p.name, p.multiProcessorCount, clk);
  float* out;
  cudaMalloc(&out, 4096);
  run<FFMA_RRR>("FFMA rrr", out, p.multiProcessorCount, clk);
  run<FFMA_RIR>("FFMA rir", out, p.multiProcessorCount, clk);
  run<FFMA_RUR>("FFMA rur", out, p.multiProcessorCount, clk);
  run<FADD_RR>("FADD rr", out, p.multiProcessorCount, clk);
  run<FFMA2_RIR>("FFMA2 rir", out, p.multiProcessorCount, clk);
  run<FFMA2_RUR>("FFMA2 rur", out, p.multiProcessorCount, clk);
  run<FFMA2_RRR>("FFMA2 rrr", out, p.multiProcessorCount, clk);
  run<FADD2_RR>("FADD2 rr", out, p.multiProcessorCount, clk);
  run<FMUL2_RI>("FMUL2 ri", out, p.multiProcessorCount, clk);
  run<MIX_2D>("mix2", out, p.multiProcessorCount, clk);
  run<MIX_HALF>("FADD2+FFMA2", out, p.multiProcessorCount, clk);
  run<MIX_SCALAR_HALF>("FADD+FFMA", out, p.multiProcessorCount, clk);
  cudaError_t e = cudaDeviceSynchronize();
  std::printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
