// Device helpers shared by the march kernels (march.cu, march_multi.cu):
// 32-bit field views, exact cell selection, trilinear / nearest gathers, the
// persistent tile scheduler's Morton decode and pair shuffles.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"
#include "raysetup.cuh"

namespace isc {

constexpr int kTile = 16;
constexpr int kThreads = kTile * kTile;

struct FastField {
  const void* __restrict__ f;   // element type: the kernel's T (float, double, __half, __nv_bfloat16)
  int sx, sy, sz;        // element strides
  int sc;                // component stride (feature_dim > 1)
  int lo[3];             // brick offset - guard (global cell of array index 0)
  int hi[3];             // largest legal base index (guarded) / size-1 (clamped)
  int g;
  // split iso + volume render (march.cu launch_split): the iso probe's
  // per-pixel station counts and shaded hit colours; a ray marches only the
  // stations before its iso hit and composites the hit colour behind them.
  // Null in a plain render.
  const uint32_t* stop_counts;
  const float4* stop_shade;
};

// floor(p) as an exact double and as an int without conversion instructions:
// rounding p + 1.5*2^52 toward -inf leaves floor(p) in the low mantissa bits
// (exact for |p| < 2^51), so the XU pipe only sees the final float conversion.
__device__ __forceinline__ double floor_split(double p, int& i) {
  constexpr double kMagic = 6755399441055744.0;  // 2^52 + 2^51
  const double t = __dadd_rd(p, kMagic);
  i = __double2loint(t);
  return __dsub_rn(t, kMagic);
}

// Guard contract of a trilinear gather at p (fields.py:218-238): the base
// cell must lie in [0, hi] of the guarded array on every axis.
__device__ __forceinline__ bool guard_ok(const FastField& F, const double p[3]) {
  int ix, iy, iz;
  floor_split(p[0], ix);
  floor_split(p[1], iy);
  floor_split(p[2], iz);
  return (unsigned)(ix - F.lo[0]) <= (unsigned)F.hi[0] && (unsigned)(iy - F.lo[1]) <= (unsigned)F.hi[1] &&
         (unsigned)(iz - F.lo[2]) <= (unsigned)F.hi[2];
}

// One field element as float32 (read-only path).
__device__ __forceinline__ float ldf(const float* p) { return __ldg(p); }
__device__ __forceinline__ float ldf(const __half* p) { return __half2float(__ldg(p)); }
__device__ __forceinline__ float ldf(const __nv_bfloat16* p) { return __bfloat162float(__ldg(p)); }
__device__ __forceinline__ float ldf(const double* p) { return (float)__ldg(p); }

#ifndef ISC_PTR_ADDR
#define ISC_PTR_ADDR 1
#endif
// p + off bytes as one 64-bit add the compiler cannot re-associate into
// (index + stride) * sizeof(T) address arithmetic.
template <typename T>
__device__ __forceinline__ const T* padd(const T* p, long long off) {
  const T* r;
  asm("add.s64 %0, %1, %2;" : "=l"(r) : "l"(p), "l"(off));
  return r;
}

// CHECK = false: the caller has proven the guard contract for this sample
// (see march_fast_kernel: endpoint check per ray).
template <bool INTERP, bool GUARDED, bool CHECK = true, typename T = float>
__device__ __forceinline__ float fast_sample(const FastField& F, const double p[3], uint32_t* err) {
  const T* __restrict__ fld = reinterpret_cast<const T*>(F.f);
  int ix, iy, iz;
  const double flx = floor_split(p[0], ix), fly = floor_split(p[1], iy), flz = floor_split(p[2], iz);
  if constexpr (!INTERP) {
    // nearest: clamp the local cell into the brick (fields.py:240-242)
    const int x = min(max(ix - F.lo[0] - F.g, 0), F.hi[0]) + F.g;
    const int y = min(max(iy - F.lo[1] - F.g, 0), F.hi[1]) + F.g;
    const int z = min(max(iz - F.lo[2] - F.g, 0), F.hi[2]) + F.g;
    return ldf(fld + (z * F.sz + y * F.sy + x * F.sx));
  } else {
    const float fx = (float)dsub(p[0], flx), fy = (float)dsub(p[1], fly), fz = (float)dsub(p[2], flz);
    int x0, y0, z0, dx, dy, dz;
    if constexpr (GUARDED) {
      x0 = ix - F.lo[0];
      y0 = iy - F.lo[1];
      z0 = iz - F.lo[2];
      if (CHECK &&
          ((unsigned)x0 > (unsigned)F.hi[0] || (unsigned)y0 > (unsigned)F.hi[1] || (unsigned)z0 > (unsigned)F.hi[2])) {
        if (err) atomicAdd(err, 1u);
        x0 = min(max(x0, 0), F.hi[0]);
        y0 = min(max(y0, 0), F.hi[1]);
        z0 = min(max(z0, 0), F.hi[2]);
      }
      dx = F.sx;
      dy = F.sy;
      dz = F.sz;
    } else {
      // clamp each corner index into the brick (fields.py:240-242)
      const int lx = ix - F.lo[0] - F.g, ly = iy - F.lo[1] - F.g, lz = iz - F.lo[2] - F.g;
      x0 = min(max(lx, 0), F.hi[0]);
      y0 = min(max(ly, 0), F.hi[1]);
      z0 = min(max(lz, 0), F.hi[2]);
      dx = (min(max(lx + 1, 0), F.hi[0]) - x0) * F.sx;
      dy = (min(max(ly + 1, 0), F.hi[1]) - y0) * F.sy;
      dz = (min(max(lz + 1, 0), F.hi[2]) - z0) * F.sz;
      x0 += F.g;
      y0 += F.g;
      z0 += F.g;
    }
    const T* b = fld + (z0 * F.sz + y0 * F.sy + x0 * F.sx);
#if ISC_PTR_ADDR
    // corner addresses as 64-bit pointer adds of byte strides (2 instructions
    // each) instead of re-forming base + (index + stride) * sizeof(T) per corner
    const long long bx = (long long)dx * sizeof(T), by = (long long)dy * sizeof(T), bz = (long long)dz * sizeof(T);
    const T* py = padd(b, by);
    const T* pz = padd(b, bz);
    const T* pyz = padd(pz, by);
    const float v000 = ldf(b), v100 = ldf(padd(b, bx)), v010 = ldf(py), v110 = ldf(padd(py, bx));
    const float v001 = ldf(pz), v101 = ldf(padd(pz, bx)), v011 = ldf(pyz), v111 = ldf(padd(pyz, bx));
#else
    const float v000 = ldf(b), v100 = ldf(b + dx), v010 = ldf(b + dy), v110 = ldf(b + dy + dx);
    const T* c = b + dz;
    const float v001 = ldf(c), v101 = ldf(c + dx), v011 = ldf(c + dy), v111 = ldf(c + dy + dx);
#endif
    const float a0 = fmaf(fx, v100 - v000, v000), a1 = fmaf(fx, v110 - v010, v010);
    const float a2 = fmaf(fx, v101 - v001, v001), a3 = fmaf(fx, v111 - v011, v011);
    const float b0 = fmaf(fy, a1 - a0, a0), b1 = fmaf(fy, a3 - a2, a2);
    return fmaf(fz, b1 - b0, b0);
  }
}

// DIM-component trilinear gather with the guard contract already proven for
// this station (march_fast_kernel's per-ray check): v[c] for c < DIM.
template <int DIM, typename T = float>
__device__ __forceinline__ void fast_gather(const FastField& F, const double p[3], float v[4]) {
  const T* __restrict__ fld = reinterpret_cast<const T*>(F.f);
  int ix, iy, iz;
  const double flx = floor_split(p[0], ix), fly = floor_split(p[1], iy), flz = floor_split(p[2], iz);
  const float fx = (float)dsub(p[0], flx), fy = (float)dsub(p[1], fly), fz = (float)dsub(p[2], flz);
  const int x0 = ix - F.lo[0], y0 = iy - F.lo[1], z0 = iz - F.lo[2];
  const T* b = fld + (z0 * F.sz + y0 * F.sy + x0 * F.sx);
  const int dx = F.sx, dy = F.sy, dz = F.sz;
#pragma unroll
  for (int c = 0; c < DIM; ++c) {
    const T* q0 = b + c * F.sc;
    const float v000 = ldf(q0), v100 = ldf(q0 + dx), v010 = ldf(q0 + dy), v110 = ldf(q0 + dy + dx);
    const T* q1 = q0 + dz;
    const float v001 = ldf(q1), v101 = ldf(q1 + dx), v011 = ldf(q1 + dy), v111 = ldf(q1 + dy + dx);
    const float a0 = fmaf(fx, v100 - v000, v000), a1 = fmaf(fx, v110 - v010, v010);
    const float a2 = fmaf(fx, v101 - v001, v001), a3 = fmaf(fx, v111 - v011, v011);
    const float b0 = fmaf(fy, a1 - a0, a0), b1 = fmaf(fy, a3 - a2, a2);
    v[c] = fmaf(fz, b1 - b0, b0);
  }
}

// fast_gather<3> for the standard AoS float3 layout (x contiguous,
// components interleaved: sx == 3, sc == 1, even row / slice strides, an
// 8-byte aligned base): the 6 floats of a corner row (x0 and x0 + 1, three
// components each) come from 3 aligned 8-byte loads when x0 is even, and
// from the 8-byte words around them (+ one 4-byte load of the last float)
// when x0 is odd -- 16 load requests per station instead of 24 (each request
// touches the same cache lines either way).  Same arithmetic as fast_gather.
__device__ __forceinline__ void fast_gather_aos3(const FastField& F, const double p[3], float v[4]) {
  const float* __restrict__ fld = reinterpret_cast<const float*>(F.f);
  int ix, iy, iz;
  const double flx = floor_split(p[0], ix), fly = floor_split(p[1], iy), flz = floor_split(p[2], iz);
  const float fx = (float)dsub(p[0], flx), fy = (float)dsub(p[1], fly), fz = (float)dsub(p[2], flz);
  const int x0 = ix - F.lo[0], y0 = iy - F.lo[1], z0 = iz - F.lo[2];
  const bool odd = (x0 & 1) != 0;  // parity of the element offset (even strides)
  const float* r00 = fld + ((z0 * F.sz + y0 * F.sy + 3 * x0) & ~1);
  const float* rows[4] = {r00, r00 + F.sy, r00 + F.sz, r00 + F.sz + F.sy};
  float c[4][6];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const float2* q = reinterpret_cast<const float2*>(rows[r]);
    const float2 w0 = __ldg(q), w1 = __ldg(q + 1), w2 = __ldg(q + 2);
    float t = 0.f;
    if (odd) t = __ldg(rows[r] + 6);
    c[r][0] = odd ? w0.y : w0.x;
    c[r][1] = odd ? w1.x : w0.y;
    c[r][2] = odd ? w1.y : w1.x;
    c[r][3] = odd ? w2.x : w1.y;
    c[r][4] = odd ? w2.y : w2.x;
    c[r][5] = odd ? t : w2.y;
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float a0 = fmaf(fx, c[0][3 + k] - c[0][k], c[0][k]), a1 = fmaf(fx, c[1][3 + k] - c[1][k], c[1][k]);
    const float a2 = fmaf(fx, c[2][3 + k] - c[2][k], c[2][k]), a3 = fmaf(fx, c[3][3 + k] - c[3][k], c[3][k]);
    const float b0 = fmaf(fy, a1 - a0, a0), b1 = fmaf(fy, a3 - a2, a2);
    v[k] = fmaf(fz, b1 - b0, b0);
  }
}

// Host: conservative pixel rectangle [x0, x1) x [y0, y1) outside which no
// primary ray can hit the brick -- the bounding box of the pinhole projection
// of the brick's 8 corners (the image of a box in front of the camera is the
// convex hull of its projected corners), widened by 2 px against rounding.
// False (no culling) when a corner is not strictly in front of the camera,
// for explicit ray lists, and when per-pixel debug outputs are requested
// (they are defined for every pixel).
// stations_internal: out_stations is the split render's scratch (read back
// only inside the same screen rectangle), so it does not force a full raster.
inline bool brick_screen_rect(const isc_render_args* a, int& x0, int& y0, int& x1, int& y1,
                              bool stations_internal = false) {
  if (a->ray_dirs || (a->out_stations && !stations_internal) || a->out_hit || a->out_t || a->out_krange)
    return false;
  const isc_camera& c = a->camera;
  double xmin = 1e300, xmax = -1e300, ymin = 1e300, ymax = -1e300;
  for (int corner = 0; corner < 8; ++corner) {
    double v[3];
    for (int i = 0; i < 3; ++i)
      v[i] = a->brick_offset[i] + ((corner >> i) & 1 ? a->brick_size[i] : 0) - c.origin[i];
    const double depth = v[0] * c.fwd[0] + v[1] * c.fwd[1] + v[2] * c.fwd[2];
    const double len = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    if (!(depth > 1e-6 * len) || !(depth > 0.0)) return false;
    const double col = (v[0] * c.right[0] + v[1] * c.right[1] + v[2] * c.right[2]) / (depth * c.tan_half * c.aspect);
    const double row = (v[0] * c.up[0] + v[1] * c.up[1] + v[2] * c.up[2]) / (depth * c.tan_half);
    const double px = (col + 1.0) * 0.5 * c.width - 0.5, py = (1.0 - row) * 0.5 * c.height - 0.5;
    xmin = fmin(xmin, px);
    xmax = fmax(xmax, px);
    ymin = fmin(ymin, py);
    ymax = fmax(ymax, py);
  }
  auto clampi = [](double v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : (int)v); };
  x0 = clampi(floor(xmin) - 2.0, 0, c.width);
  y0 = clampi(floor(ymin) - 2.0, 0, c.height);
  x1 = clampi(ceil(xmax) + 3.0, 0, c.width);
  y1 = clampi(ceil(ymax) + 3.0, 0, c.height);
  if (x1 < x0) x1 = x0;
  if (y1 < y0) y1 = y0;
  return true;
}

// Host: resident CTAs per SM of `kernel` at `threads` threads and no dynamic
// shared memory, queried once per (kernel, device) -- the occupancy query
// costs microseconds on every frame otherwise.
template <auto Kernel>
inline int cached_blocks_per_sm(int threads) {
  static int cache[64] = {};  // one per kernel instantiation (Kernel is a template argument)
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (cache[dev] == 0) {
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, Kernel, threads, 0);
    cache[dev] = n > 0 ? n : 1;
  }
  return cache[dev];
}

// Host: SM count of the current device (cached per device).
inline int cached_sm_count() {
  static int cache[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (cache[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 148;
  }
  return cache[dev];
}

// The culled rectangle is the whole image: the kernel writes every pixel, so
// the canvas needs no clearing first.
inline bool rect_is_whole(const isc_render_args* a, int x0, int y0, int x1, int y1) {
  return x0 == 0 && y0 == 0 && x1 == a->camera.width && y1 == a->camera.height;
}

__device__ __forceinline__ int morton3(int w, int shift) {
  return ((w >> shift) & 1) | (((w >> (shift + 2)) & 1) << 1) | (((w >> (shift + 4)) & 1) << 2);
}

// Lane l receives lane l + n's value (full mask; lanes past 31 - n keep their own).
__device__ __forceinline__ float4 shfl_down_n(float4 v, int n) {
  return make_float4(__shfl_down_sync(0xffffffffu, v.x, n), __shfl_down_sync(0xffffffffu, v.y, n),
                     __shfl_down_sync(0xffffffffu, v.z, n), __shfl_down_sync(0xffffffffu, v.w, n));
}

// Lanes 0-15 receive lane + 16's value (full mask; lanes 16-31 get their own).
__device__ __forceinline__ float4 shfl_down16(float4 v) {
  return make_float4(__shfl_down_sync(0xffffffffu, v.x, 16), __shfl_down_sync(0xffffffffu, v.y, 16),
                     __shfl_down_sync(0xffffffffu, v.z, 16), __shfl_down_sync(0xffffffffu, v.w, 16));
}

}  // namespace isc
