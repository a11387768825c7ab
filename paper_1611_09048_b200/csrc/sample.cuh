// Field sampling, functor chains and transfer-function classification on the
// device (float32 arithmetic on values, float64 for positions/indices).
//
//   guard / clamp contract   fields.py:218-246  (guard reads legal only when
//                            has_guard && interpolation; else clamp per index)
//   trilinear                raycast.py:182-199 (8 corners, floor + frac)
//   nearest                  raycast.py:174-178 (floor, clamp)
//   chain                    functors.py:102-147, 212-222; first component
//                            functors.py:239-240
//   classify                 scene.py:139-152   (clip, x = 255 t, lerp LUT,
//                            non-finite -> transparent)
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"

namespace isc {

struct Brick {
  int size[3];
  int guard;
  double offset[3];
};

__device__ __forceinline__ float load_elem(const isc_source& s, long long idx) {
  switch (s.dtype) {
    case ISC_F64: return (float)__ldg(reinterpret_cast<const double*>(s.data) + idx);
    case ISC_F16: return __half2float(reinterpret_cast<const __half*>(s.data)[idx]);
    case ISC_BF16: return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(s.data)[idx]);
    default: return __ldg(reinterpret_cast<const float*>(s.data) + idx);
  }
}

template <bool F32>
__device__ __forceinline__ float load_as(const isc_source& s, long long idx) {
  if constexpr (F32) return __ldg(reinterpret_cast<const float*>(s.data) + idx);
  else return load_elem(s, idx);
}

// Integer local index of one axis for the corner pair (i, i+1) under the
// guard/clamp contract.  Returns false on a guard-contract violation (the
// indices are then clamped into the halo so the read stays in bounds).
__device__ __forceinline__ bool corner_pair(int i, int size, int g, bool guarded, int& i0, int& i1) {
  if (guarded) {
    bool ok = (i >= -g) && (i + 1 < size + g);
    i0 = min(max(i, -g), size + g - 1);
    i1 = min(max(i + 1, -g), size + g - 1);
    return ok;
  }
  i0 = min(max(i, 0), size - 1);
  i1 = min(max(i + 1, 0), size - 1);
  return true;
}

// Sample a source at a LOCAL position (global - offset) -> dim components.
template <bool F32, int DIM>
__device__ __forceinline__ void sample_local(const isc_source& s, const Brick& b, const double l[3],
                                             bool interp, float v[4], uint32_t* err) {
  const int g = b.guard;
  const double fx0 = floor(l[0]), fy0 = floor(l[1]), fz0 = floor(l[2]);
  const int ix = (int)fx0, iy = (int)fy0, iz = (int)fz0;
  const int dim = DIM > 0 ? DIM : s.feature_dim;
  if (!interp) {
    const int cx = min(max(ix, 0), b.size[0] - 1);
    const int cy = min(max(iy, 0), b.size[1] - 1);
    const int cz = min(max(iz, 0), b.size[2] - 1);
    const long long base = (long long)(cz + g) * s.stride[0] + (long long)(cy + g) * s.stride[1] +
                           (long long)(cx + g) * s.stride[2];
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (c < dim) v[c] = load_as<F32>(s, base + c * s.stride[3]);
    return;
  }
  const bool guarded = s.has_guard != 0;
  int x0, x1, y0, y1, z0, z1;
  bool ok = corner_pair(ix, b.size[0], g, guarded, x0, x1);
  ok &= corner_pair(iy, b.size[1], g, guarded, y0, y1);
  ok &= corner_pair(iz, b.size[2], g, guarded, z0, z1);
  if (!ok && err) atomicAdd(err, 1u);
  const float fx = (float)dsub(l[0], fx0), fy = (float)dsub(l[1], fy0), fz = (float)dsub(l[2], fz0);
  const long long ox0 = (long long)(x0 + g) * s.stride[2], ox1 = (long long)(x1 + g) * s.stride[2];
  const long long oy0 = (long long)(y0 + g) * s.stride[1], oy1 = (long long)(y1 + g) * s.stride[1];
  const long long oz0 = (long long)(z0 + g) * s.stride[0], oz1 = (long long)(z1 + g) * s.stride[0];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    if (c >= dim) break;
    const long long cc = c * s.stride[3];
    const float v000 = load_as<F32>(s, oz0 + oy0 + ox0 + cc), v100 = load_as<F32>(s, oz0 + oy0 + ox1 + cc);
    const float v010 = load_as<F32>(s, oz0 + oy1 + ox0 + cc), v110 = load_as<F32>(s, oz0 + oy1 + ox1 + cc);
    const float v001 = load_as<F32>(s, oz1 + oy0 + ox0 + cc), v101 = load_as<F32>(s, oz1 + oy0 + ox1 + cc);
    const float v011 = load_as<F32>(s, oz1 + oy1 + ox0 + cc), v111 = load_as<F32>(s, oz1 + oy1 + ox1 + cc);
    const float a0 = fmaf(fx, v100 - v000, v000), a1 = fmaf(fx, v110 - v010, v010);
    const float a2 = fmaf(fx, v101 - v001, v001), a3 = fmaf(fx, v111 - v011, v011);
    const float b0 = fmaf(fy, a1 - a0, a0), b1 = fmaf(fy, a3 - a2, a2);
    v[c] = fmaf(fz, b1 - b0, b0);
  }
}

// Functor chain on up to 4 components; returns the first component
// (reduce_to_scalar_array).  Sums and norms use explicit round-to-nearest
// adds/multiplies so the float32 value-range kernel is bit-exact with the
// oracle's float32 restatement.
__device__ __forceinline__ float run_chain(const isc_source& s, float v[4], int dim) {
  for (int i = 0; i < s.n_steps; ++i) {
    const isc_chain_step& st = s.steps[i];
    switch (st.op) {
      case ISC_OP_ADD:
#pragma unroll
        for (int c = 0; c < 4; ++c) if (c < dim) v[c] = fadd(v[c], st.arg[c]);
        break;
      case ISC_OP_MUL:
#pragma unroll
        for (int c = 0; c < 4; ++c) if (c < dim) v[c] = fmul(v[c], st.arg[c]);
        break;
      case ISC_OP_POW:
#pragma unroll
        for (int c = 0; c < 4; ++c) if (c < dim) v[c] = powf(v[c], st.arg[c]);
        break;
      case ISC_OP_LENGTH: {
        float acc = fmul(v[0], v[0]);
#pragma unroll
        for (int c = 1; c < 4; ++c) if (c < dim) acc = fadd(acc, fmul(v[c], v[c]));
        v[0] = __fsqrt_rn(acc);
        dim = 1;
      } break;
      case ISC_OP_SUM: {
        float acc = v[0];
#pragma unroll
        for (int c = 1; c < 4; ++c) if (c < dim) acc = fadd(acc, v[c]);
        v[0] = acc;
        dim = 1;
      } break;
      case ISC_OP_SQRT:
#pragma unroll
        for (int c = 0; c < 4; ++c) if (c < dim) v[c] = __fsqrt_rn(v[c]);
        break;
      case ISC_OP_ABS:
#pragma unroll
        for (int c = 0; c < 4; ++c) if (c < dim) v[c] = fabsf(v[c]);
        break;
      case ISC_OP_NEG:
#pragma unroll
        for (int c = 0; c < 4; ++c) if (c < dim) v[c] = -v[c];
        break;
      case ISC_OP_EXP:
#pragma unroll
        for (int c = 0; c < 4; ++c) if (c < dim) v[c] = expf(v[c]);
        break;
      case ISC_OP_LOG:
#pragma unroll
        for (int c = 0; c < 4; ++c) if (c < dim) v[c] = logf(v[c]);
        break;
      case ISC_OP_MIN:
#pragma unroll
        for (int c = 0; c < 4; ++c) if (c < dim) v[c] = (v[c] != v[c]) ? v[c] : fminf(v[c], st.arg[c]);
        break;
      case ISC_OP_MAX:
#pragma unroll
        for (int c = 0; c < 4; ++c) if (c < dim) v[c] = (v[c] != v[c]) ? v[c] : fmaxf(v[c], st.arg[c]);
        break;
      default: break;
    }
  }
  return v[0];
}

// One dimension-preserving chain step other than add / mul (pow, sqrt, abs,
// neg, exp, log, min, max): out of line, the kernels' hot loops only carry
// the common steps.
static __device__ __noinline__ void chain_step_rare(const isc_chain_step& st, float* v, int dim) {
  isc_source one{};
  one.n_steps = 1;
  one.steps[0] = st;
  float w[4] = {v[0], v[1], v[2], v[3]};
  run_chain(one, w, dim);
#pragma unroll
  for (int c = 0; c < 4; ++c) v[c] = w[c];
}

// run_chain for a source whose input has D components (compile time): the
// common steps (add, mul, length, sum) are tested first with uniform
// branches and no per-component dimension tests; results are identical to
// run_chain (same float32 operations in the same order).  After a reducing
// step only component 0 is meaningful; the others keep being computed and are
// ignored.
// The step loop is unrolled to ISC_MAX_CHAIN so every step's opcode and
// arguments are read at a compile-time offset of the kernel parameters
// (immediate constant-bank operands, no indexed constant loads).
template <int D>
__device__ __forceinline__ float run_chain_fast(const isc_source& s, float v[4]) {
  bool reduced = (D == 1);
  const unsigned ops = s.step_ops;
#pragma unroll
  for (int i = 0; i < ISC_MAX_CHAIN; ++i) {
    if (i >= s.n_steps) break;
    const isc_chain_step& st = s.steps[i];
    const int op = (int)((ops >> (4 * i)) & 0xFu);
    if (op == ISC_OP_ADD) {
#pragma unroll
      for (int c = 0; c < D; ++c) v[c] = fadd(v[c], st.arg[c]);
    } else if (op == ISC_OP_MUL) {
#pragma unroll
      for (int c = 0; c < D; ++c) v[c] = fmul(v[c], st.arg[c]);
    } else if (op == ISC_OP_LENGTH || op == ISC_OP_SUM) {
      const bool len = op == ISC_OP_LENGTH;
      float acc = len ? fmul(v[0], v[0]) : v[0];
      if (!reduced) {
#pragma unroll
        for (int c = 1; c < D; ++c) acc = fadd(acc, len ? fmul(v[c], v[c]) : v[c]);
      }
      v[0] = len ? __fsqrt_rn(acc) : acc;
      reduced = true;
    } else {
      chain_step_rare(st, v, reduced ? 1 : D);
    }
  }
  return v[0];
}

// Straight RGBA from a float4 LUT in global memory (iso-hit shading, once per hit).
__device__ __forceinline__ float4 classify_aos(const float4* lut, float lo, float inv_span, float v) {
  if (!isfinite(v)) return make_float4(0.f, 0.f, 0.f, 0.f);
  float t = (v - lo) * inv_span;
  t = fminf(fmaxf(t, 0.0f), 1.0f);
  const float x = t * (float)(ISC_LUT_ENTRIES - 1);
  const int i0 = min((int)x, ISC_LUT_ENTRIES - 1);
  const int i1 = min(i0 + 1, ISC_LUT_ENTRIES - 1);
  const float w = x - (float)i0;
  const float4 a = lut[i0], b = lut[i1];
  return make_float4(fmaf(w, b.x - a.x, a.x), fmaf(w, b.y - a.y, a.y), fmaf(w, b.z - a.z, a.z),
                     fmaf(w, b.w - a.w, a.w));
}

// Shared-memory LUTs are held planar, one 256-float table per channel
// (lut_fill): a lookup is eight LDS.32 (both lerp ends of four channels).  A
// warp's lookups touch a few neighbouring entries, so each LDS.32 is ~1
// data-pipe wavefront (1.08 measured on C4), while the float4 entry layout's
// two LDS.128 cost 7.0 each (entries 8 apart share a bank group): C4 LUT path
// 5.33 -> 4.87 ms, images bit-identical (tools/micro/).
constexpr int kLutWords = 4 * ISC_LUT_ENTRIES;  // floats per source

// Fill one source's planar table from its float4 LUT (all threads of the CTA;
// the caller syncs).
__device__ __forceinline__ void lut_fill(float* dst, const float4* src) {
  for (int i = threadIdx.x; i < ISC_LUT_ENTRIES; i += blockDim.x) {
    const float4 c = src[i];
    dst[0 * ISC_LUT_ENTRIES + i] = c.x;
    dst[1 * ISC_LUT_ENTRIES + i] = c.y;
    dst[2 * ISC_LUT_ENTRIES + i] = c.z;
    dst[3 * ISC_LUT_ENTRIES + i] = c.w;
  }
}

// lut_fill for n sources (tables back to back).
__device__ __forceinline__ void lut_fill_sources(float* dst, const isc_render_args& a, int n) {
  for (int i = threadIdx.x; i < n * ISC_LUT_ENTRIES; i += blockDim.x) {
    const float4 c = reinterpret_cast<const float4*>(a.src[i >> 8].lut)[i & (ISC_LUT_ENTRIES - 1)];
    float* t = dst + (i >> 8) * kLutWords + (i & (ISC_LUT_ENTRIES - 1));
    t[0 * ISC_LUT_ENTRIES] = c.x;
    t[1 * ISC_LUT_ENTRIES] = c.y;
    t[2 * ISC_LUT_ENTRIES] = c.z;
    t[3 * ISC_LUT_ENTRIES] = c.w;
  }
}

// Straight RGBA from a planar LUT in shared memory (scene.py:139-152).
__device__ __forceinline__ float4 classify(const float* tab, float lo, float inv_span, float v) {
  if (!isfinite(v)) return make_float4(0.f, 0.f, 0.f, 0.f);
  float t = (v - lo) * inv_span;
  t = fminf(fmaxf(t, 0.0f), 1.0f);
  const float x = t * (float)(ISC_LUT_ENTRIES - 1);
  const int i0 = min((int)x, ISC_LUT_ENTRIES - 1);
  const int i1 = min(i0 + 1, ISC_LUT_ENTRIES - 1);
  const float w = x - (float)i0;
  float c[4];
#pragma unroll
  for (int ch = 0; ch < 4; ++ch) {
    const float a = tab[ch * ISC_LUT_ENTRIES + i0], b = tab[ch * ISC_LUT_ENTRIES + i1];
    c[ch] = fmaf(w, b - a, a);
  }
  return make_float4(c[0], c[1], c[2], c[3]);
}

__device__ __forceinline__ float4 premultiply(float4 c) {
  return make_float4(c.x * c.w, c.y * c.w, c.z * c.w, c.w);
}

// Straight RGBA of a transfer function whose LUT lerp is piecewise linear
// with L-1 slope changes (isc_source.lut_linear / lut_kinks):
//   base + slope*x + sum_k dslope_k * max(x - x_k, 0),
// identical to the LUT lerp, no shared-memory lookup (the coefficients are
// kernel-parameter constants, free FFMA operands).  Returns the
// PREMULTIPLIED colour; a non-finite value gets alpha 0 (and so rgb 0)
// through a select instead of a branch.
// L = kLineRuntime: 4 to ISC_MAX_LUT_KINKS kinks, count read at run time
// (warp-uniform; one instantiation instead of one per count).
constexpr int kLineRuntime = ISC_MAX_LUT_KINKS + 1;
template <int L>
__device__ __forceinline__ float4 classify_line_premul(const isc_source& s, float lo, float inv_span, float v) {
  const float x = fminf(fmaxf((v - lo) * inv_span, 0.0f), 1.0f) * (float)(ISC_LUT_ENTRIES - 1);
  float c[4];
#pragma unroll
  for (int ch = 0; ch < 4; ++ch) c[ch] = fmaf(s.lut_slope[ch], x, s.lut_base[ch]);
#pragma unroll
  for (int k = 0; k < L - 1; ++k) {
    if (L == kLineRuntime && k >= 3 && k >= s.lut_kinks) break;
    const float h = fmaxf(x - s.lut_kink_x[k], 0.0f);
#pragma unroll
    for (int ch = 0; ch < 4; ++ch) c[ch] = fmaf(s.lut_kink_dslope[k][ch], h, c[ch]);
  }
  const float a = isfinite(v) ? c[3] : 0.0f;
  return make_float4(c[0] * a, c[1] * a, c[2] * a, a);
}

// Premultiplied colour of a source whose transfer function has the analytic
// piecewise-linear form (isc_source.lut_linear, lut_kinks at run time; see
// march.cu classify_line_premul for the compile-time variant), else the
// shared-memory LUT.  Warp-uniform branches.
__device__ __forceinline__ float4 classify_src_premul(const isc_source& s, const float* lut, float inv_span,
                                                     float v) {
  if (!s.lut_linear) return premultiply(classify(lut, s.range_lo, inv_span, v));
  const float x = fminf(fmaxf((v - s.range_lo) * inv_span, 0.0f), 1.0f) * (float)(ISC_LUT_ENTRIES - 1);
  float c[4];
#pragma unroll
  for (int ch = 0; ch < 4; ++ch) c[ch] = fmaf(s.lut_slope[ch], x, s.lut_base[ch]);
#pragma unroll
  for (int k = 0; k < ISC_MAX_LUT_KINKS; ++k) {
    if (k >= s.lut_kinks) break;
    const float h = fmaxf(x - s.lut_kink_x[k], 0.0f);
#pragma unroll
    for (int ch = 0; ch < 4; ++ch) c[ch] = fmaf(s.lut_kink_dslope[k][ch], h, c[ch]);
  }
  const float a = isfinite(v) ? c[3] : 0.0f;
  return make_float4(c[0] * a, c[1] * a, c[2] * a, a);
}

}  // namespace isc
