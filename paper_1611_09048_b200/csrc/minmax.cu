// K4: per-source normalisation -- (min, max) of the float32-chained first
// component over a brick's interior (guard excluded).  There is no reference
// function for this (value ranges are scene state, scene.py:188,
// runtime.py:154-157); it feeds the auto value range of a transfer function.
//
// Streaming reduction: each warp walks whole x-rows (coalesced loads: 16-byte
// loads for contiguous float32 rows, else 16 scalar loads per lane in flight
// for memory-level parallelism), reduces with warp shuffles, then one
// shared-memory pass per CTA and two ordered-integer atomicMax per CTA; the
// last CTA writes the result (one memset + one kernel per call).  min/max are
// exact, so the result is
// bit-identical to the oracle regardless of reduction order.
#include "common.cuh"
#include "sample.cuh"

namespace isc {

__device__ __forceinline__ unsigned int order_key(float f) {
  const unsigned int u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float from_key(unsigned int k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

#ifndef ISC_MINMAX_UNROLL
#define ISC_MINMAX_UNROLL 16
#endif
constexpr int kUnroll = ISC_MINMAX_UNROLL;

// Streaming read (each element is read once): evict-first.
template <bool F32>
__device__ __forceinline__ float load_stream(const isc_source& s, long long idx) {
#ifdef ISC_MINMAX_LDG
  return load_as<F32>(s, idx);
#else
  if constexpr (F32) return __ldcs(reinterpret_cast<const float*>(s.data) + idx);
  else return load_elem(s, idx);
#endif
}

// Accumulators of one call (the caller's 4-word buffer, zeroed by one
// memset): word 0 counts finished CTAs (the last one writes the result over
// it), words 2 / 3 hold ~key(min) / key(max) -- both grow by atomicMax from
// 0, so zero is the identity of both and no init kernel is needed.

// float4 body of one contiguous float32 row [e0, e0 + n): scalar head up to
// a 16-byte boundary, 16-byte loads (evict-first), scalar tail.
template <typename V>
__device__ __forceinline__ void row_f32_vec(const float* __restrict__ base, long long e0, int n, int lane, V& visit) {
  const int head = min(n, (int)((4 - (e0 & 3)) & 3));
  if (lane < head) visit(__ldcs(base + e0 + lane));
  const long long b0 = e0 + head;
  const int nv = (n - head) >> 2;
  const float4* v4 = reinterpret_cast<const float4*>(base + b0);
  // batches of 4 predicated 16-byte loads per lane, all issued before any is
  // used (a partial last batch must not fall back to one load per trip)
  for (int i0 = 0; i0 < nv; i0 += 32 * 4) {
    float4 q[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + lane + 32 * u;
      q[u] = i < nv ? __ldcs(v4 + i) : make_float4(CUDART_NAN_F, CUDART_NAN_F, CUDART_NAN_F, CUDART_NAN_F);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {  // NaN padding is ignored by visit
      visit(q[u].x);
      visit(q[u].y);
      visit(q[u].z);
      visit(q[u].w);
    }
  }
  const int done = head + 4 * nv;
  if (lane < n - done) visit(__ldcs(base + b0 + 4 * nv + lane));
}

template <int DIM, bool F32>
__global__ void __launch_bounds__(256) minmax_kernel(const __grid_constant__ isc_source s, int sx, int sy, int sz,
                                                      int g, unsigned int* keys, float* out) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const long long rows = (long long)sy * sz;
  float lo = CUDART_INF_F, hi = -CUDART_INF_F;
  bool any = false;
  auto visit = [&](float r) {
    if (r == r) {
      lo = fminf(lo, r);
      hi = fmaxf(hi, r);
      any = true;
    }
  };
  // scalar float32 source with contiguous rows and no chain: 16-byte loads
  const bool vec = DIM == 1 && F32 && s.n_steps == 0 && s.stride[2] == 1;
  for (long long row = warp; row < rows; row += nwarps) {
    const int y = (int)(row % sy), z = (int)(row / sy);
    const long long base = (long long)(z + g) * s.stride[0] + (long long)(y + g) * s.stride[1] + (long long)g * s.stride[2];
    if (vec) {
      // a 16-byte aligned base pointer and the row's element offset from it
      const float* f = reinterpret_cast<const float*>(s.data);
      const int shift = (int)((reinterpret_cast<uintptr_t>(f) >> 2) & 3);
      row_f32_vec(f - shift, base + shift, sx, lane, visit);
      continue;
    }
    // kUnroll independent loads per lane in flight (memory-level parallelism)
    int x = lane;
    for (; x + 32 * (kUnroll - 1) < sx; x += 32 * kUnroll) {
      float v[kUnroll][4];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const long long e = base + (long long)(x + 32 * u) * s.stride[2];
#pragma unroll
        for (int c = 0; c < DIM; ++c) v[u][c] = load_stream<F32>(s, e + c * s.stride[3]);
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) visit(run_chain(s, v[u], DIM));
    }
    for (; x < sx; x += 32) {
      const long long e = base + (long long)x * s.stride[2];
      float v[4];
#pragma unroll
      for (int c = 0; c < DIM; ++c) v[c] = load_stream<F32>(s, e + c * s.stride[3]);
      visit(run_chain(s, v, DIM));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    any |= __shfl_xor_sync(0xffffffffu, (int)any, o) != 0;
  }
  __shared__ float slo[8], shi[8];
  __shared__ int sany[8];
  const int wib = threadIdx.x >> 5;
  if (lane == 0) {
    slo[wib] = lo;
    shi[wib] = hi;
    sany[wib] = any;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    bool b = false;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
      if (!sany[i]) continue;
      lo = b ? fminf(lo, slo[i]) : slo[i];
      hi = b ? fmaxf(hi, shi[i]) : shi[i];
      b = true;
    }
    if (b) {
      atomicMax(keys, ~order_key(lo));
      atomicMax(keys + 1, order_key(hi));
    }
    // the last CTA to finish turns the keys into (min, max)
    __threadfence();
    unsigned int* done = reinterpret_cast<unsigned int*>(out);
    if (atomicAdd(done, 1u) == gridDim.x - 1) {
      __threadfence();
      const unsigned int kmin = ~atomicAdd(keys, 0u), kmax = atomicAdd(keys + 1, 0u);
      const bool empty = kmax == 0u;
      out[0] = empty ? CUDART_NAN_F : from_key(kmin);
      out[1] = empty ? CUDART_NAN_F : from_key(kmax);
    }
  }
}

}  // namespace isc

using namespace isc;

extern "C" int isc_value_range(const isc_source* src, const int32_t brick_size[3], int32_t guard,
                               float* out_minmax, void* stream) {
  if (!src || !src->data || !out_minmax || !brick_size) return fail(ISC_E_VALUE, "null argument");
  if (src->feature_dim < 1 || src->feature_dim > 4) return fail(ISC_E_FIELD, "feature_dim must be 1..4");
  if (src->n_steps < 0 || src->n_steps > ISC_MAX_CHAIN) return fail(ISC_E_CHAIN, "chain too long");
  for (int i = 0; i < 3; ++i)
    if (brick_size[i] <= 0) return fail(ISC_E_FIELD, "brick size must be positive");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // out_minmax holds 4 words: [0], [1] = min, max (float); [2], [3] = scratch keys.
  unsigned int* keys = reinterpret_cast<unsigned int*>(out_minmax) + 2;
  int dev = 0;
  ISC_CUDA_CHECK(cudaGetDevice(&dev));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long rows = (long long)brick_size[1] * brick_size[2];
  const long long want = (rows + 7) / 8;  // 8 warps per CTA, >= 1 row per warp
  const int grid = (int)(want < (long long)sms * 8 ? (want > 0 ? want : 1) : (long long)sms * 8);
  ISC_CUDA_CHECK(cudaMemsetAsync(out_minmax, 0, 4 * sizeof(float), s));
  const int bx = brick_size[0], by = brick_size[1], bz = brick_size[2];
  if (src->dtype == ISC_F32) {
    switch (src->feature_dim) {
      case 1: minmax_kernel<1, true><<<grid, 256, 0, s>>>(*src, bx, by, bz, guard, keys, out_minmax); break;
      case 2: minmax_kernel<2, true><<<grid, 256, 0, s>>>(*src, bx, by, bz, guard, keys, out_minmax); break;
      case 3: minmax_kernel<3, true><<<grid, 256, 0, s>>>(*src, bx, by, bz, guard, keys, out_minmax); break;
      default: minmax_kernel<4, true><<<grid, 256, 0, s>>>(*src, bx, by, bz, guard, keys, out_minmax); break;
    }
  } else {
    switch (src->feature_dim) {
      case 1: minmax_kernel<1, false><<<grid, 256, 0, s>>>(*src, bx, by, bz, guard, keys, out_minmax); break;
      case 2: minmax_kernel<2, false><<<grid, 256, 0, s>>>(*src, bx, by, bz, guard, keys, out_minmax); break;
      case 3: minmax_kernel<3, false><<<grid, 256, 0, s>>>(*src, bx, by, bz, guard, keys, out_minmax); break;
      default: minmax_kernel<4, false><<<grid, 256, 0, s>>>(*src, bx, by, bz, guard, keys, out_minmax); break;
    }
  }
  ISC_CUDA_CHECK(cudaGetLastError());
  return ISC_OK;
}
