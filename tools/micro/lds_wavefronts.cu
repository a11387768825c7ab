// Microbenchmark: shared-memory wavefronts per LUT lookup for the access
// patterns a warp's classify() produces (LUT path).  Run under
//   ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,
//       smsp__inst_executed_op_shared_ld.sum ./lds_wavefronts
// one launch per (layout, pattern); wavefronts / instruction is the answer.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ int pick(int pattern, int lane, int it, int base) {
  switch (pattern) {
    case 0: return base;                              // uniform
    case 1: return base + (lane & 1);                 // 2 entries
    case 2: return base + (lane & 3);                 // 4 consecutive
    case 3: return base + (lane & 7);                 // 8 consecutive (one 128-B row if aligned)
    case 4: return base + (lane >> 2);                // 8 consecutive, lanes grouped by 4
    case 5: return base + (lane & 15);                // 16 consecutive
    case 6: return base + lane;                       // 32 consecutive
    case 7: return (lane * 37 + it * 101) & 255;      // scattered
    case 8: return base + ((lane & 15) >> 1);         // paired lanes l, l+16 same, 8 entries
    default: return base;
  }
}

// AoS float4 LUT: one LDS.128 per entry (the kernel's classify reads two).
__global__ void aos128(int pattern, int iters, float* out) {
  __shared__ float4 lut[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) lut[i] = make_float4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    int base = ((it * 29) & 0xF8) + (threadIdx.x >> 5);  // vary per warp/iter, 8-aligned + warp offset
    base = min(base, 256 - 33);
    int idx = pick(pattern, lane, it, base);
    idx = (idx + (int)(acc * 0.0f)) & 255;
    const float4 v = lut[idx];
    acc += v.x + v.y + v.z + v.w;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// Planar LUT: four LDS.32, one per channel.
__global__ void planar32(int pattern, int iters, float* out) {
  __shared__ float lut[4][256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    for (int c = 0; c < 4; ++c) lut[c][i] = i + c;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    int base = ((it * 29) & 0xF8) + (threadIdx.x >> 5);
    base = min(base, 256 - 33);
    int idx = pick(pattern, lane, it, base);
    idx = (idx + (int)(acc * 0.0f)) & 255;
    acc += lut[0][idx] + lut[1][idx] + lut[2][idx] + lut[3][idx];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// Pair-packed float2 per channel: (c_i, c_{i+1}) -> four LDS.64 give both lerp ends.
__global__ void pair64(int pattern, int iters, float* out) {
  __shared__ float2 lut[4][256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    for (int c = 0; c < 4; ++c) lut[c][i] = make_float2(i + c, i + c + 1);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    int base = ((it * 29) & 0xF8) + (threadIdx.x >> 5);
    base = min(base, 256 - 33);
    int idx = pick(pattern, lane, it, base);
    idx = (idx + (int)(acc * 0.0f)) & 255;
    float2 a = lut[0][idx], b = lut[1][idx], c = lut[2][idx], d = lut[3][idx];
    acc += a.x + a.y + b.x + b.y + c.x + c.y + d.x + d.y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 256 * sizeof(float));
  const int iters = 256;
  for (int p = 0; p <= 8; ++p) {
    aos128<<<148, 256>>>(p, iters, out);
    planar32<<<148, 256>>>(p, iters, out);
    pair64<<<148, 256>>>(p, iters, out);
  }
  cudaDeviceSynchronize();
  printf("done: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
