// Throughput probe: legacy warp-level mma.sync m16n8k8 TF32 (fp32 accumulate)
// on sm_100a, 4 independent accumulator chains per warp.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(float *out, int iters) {
  unsigned a0 = threadIdx.x, a1 = a0 ^ 1, a2 = a0 ^ 2, a3 = a0 ^ 3, b0 = a0 * 3, b1 = a0 * 5;
  float c[4][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float *out; cudaMalloc(&out, 148 * 8 * 256 * 4);
  int iters = 20000;
  for (int warps : {4, 8, 16}) {
    probe<<<148 * 2, warps * 32>>>(out, 10);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    probe<<<148 * 2, warps * 32>>>(out, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double flops = 2.0 * 16 * 8 * 8 * 4.0 * iters * warps * 148 * 2;
    printf("mma.sync tf32 m16n8k8: %d warps/CTA x 2 CTA/SM: %.1f TFLOP/s\n", warps, flops / ms / 1e9);
  }
  return 0;
}
