// K1: per-pixel ray setup in float64, reproducing the reference's numpy
// evaluation order so hit masks and station ranges are bit-exact.
//
//   direction   scene.py:55-70      d = (fwd + xs*right) + ys*up,
//                                   xs = (px*tan)*aspect, ys = py*tan,
//                                   d /= sqrt((dx*dx + dy*dy) + dz*dz)
//   slab test   raycast.py:100-120
//   clip planes raycast.py:123-143  dn = dirs @ n evaluated as the OpenBLAS
//                                   dgemv_t tail does: fma(dz,nz, fma(dx,nx, dy*ny))
//   hit         raycast.py:522      (t1 > max(t0, 0)) & (t1 > 0)
//   stations    raycast.py:316-324  [ceil(max(t0,0)/step), ceil(max(t1,0)/step))
#pragma once

#include <math_constants.h>

#include "common.cuh"

namespace isc {

struct Ray {
  double d[3];          // unit direction
  double t_in, t_out;   // brick interval after clipping
  double g_in, g_out;   // global-volume interval after clipping
  long long k_lo, k_hi, kg_lo, kg_hi;
  bool hit;
};

__device__ __forceinline__ void ray_direction(const isc_camera& c, int px, int py, double d[3]) {
  const double w = (double)c.width, h = (double)c.height;
  // (arange + 0.5) / w * 2.0 - 1.0   and   1.0 - (arange + 0.5) / h * 2.0
  const double col = dsub(dmul(ddiv(dadd((double)px, 0.5), w), 2.0), 1.0);
  const double row = dsub(1.0, dmul(ddiv(dadd((double)py, 0.5), h), 2.0));
  const double xs = dmul(dmul(col, c.tan_half), c.aspect);
  const double ys = dmul(row, c.tan_half);
#pragma unroll
  for (int a = 0; a < 3; ++a) d[a] = dadd(dadd(c.fwd[a], dmul(xs, c.right[a])), dmul(ys, c.up[a]));
  const double len = __dsqrt_rn(dadd(dadd(dmul(d[0], d[0]), dmul(d[1], d[1])), dmul(d[2], d[2])));
#pragma unroll
  for (int a = 0; a < 3; ++a) d[a] = ddiv(d[a], len);
}

__device__ __forceinline__ void slab(const double o[3], const double d[3], const double lo[3],
                                     const double hi[3], double& t0, double& t1) {
  t0 = -CUDART_INF;
  t1 = CUDART_INF;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double near_, far_;
    if (d[a] == 0.0) {
      const bool inside = (o[a] >= lo[a]) && (o[a] <= hi[a]);
      near_ = inside ? -CUDART_INF : CUDART_INF;
      far_ = inside ? CUDART_INF : -CUDART_INF;
    } else {
      const double ta = ddiv(dsub(lo[a], o[a]), d[a]);
      const double tb = ddiv(dsub(hi[a], o[a]), d[a]);
      near_ = dmin(ta, tb);
      far_ = dmax(ta, tb);
    }
    t0 = dmax(t0, near_);
    t1 = dmin(t1, far_);
  }
}

__device__ __forceinline__ void clip_planes(const isc_render_args& a, const double d[3], double& t0,
                                            double& t1) {
  for (int p = 0; p < a.n_clip; ++p) {
    const isc_clip_plane& pl = a.clip[p];
    const double dn = __fma_rn(d[2], pl.normal[2], __fma_rn(d[0], pl.normal[0], dmul(d[1], pl.normal[1])));
    const double tc = ddiv(-pl.f0, dn);
    if (dn > 0.0) t0 = dmax(t0, tc);
    if (dn < 0.0) t1 = dmin(t1, tc);
    if (dn == 0.0 && pl.f0 < 0.0) t1 = -CUDART_INF;
  }
}

__device__ __forceinline__ long long station_ceil(double t, double step) {
  return (long long)ceil(ddiv(dmax(t, 0.0), step));
}

__device__ __forceinline__ void setup_ray(const isc_render_args& a, int px, int py, Ray& r) {
  if (a.ray_dirs) {  // ray-list mode (march_rays): direction and intervals given
    const long long i = (long long)py * a.camera.width + px;
#pragma unroll
    for (int k = 0; k < 3; ++k) r.d[k] = a.ray_dirs[3 * i + k];
    r.t_in = a.ray_intervals[4 * i];
    r.t_out = a.ray_intervals[4 * i + 1];
    r.g_in = a.ray_intervals[4 * i + 2];
    r.g_out = a.ray_intervals[4 * i + 3];
    r.hit = true;
    r.k_lo = station_ceil(r.t_in, a.step);
    r.k_hi = station_ceil(r.t_out, a.step);
    r.kg_lo = station_ceil(r.g_in, a.step);
    r.kg_hi = station_ceil(r.g_out, a.step);
    if (r.k_hi < r.k_lo) r.k_hi = r.k_lo;
    return;
  }
  const isc_camera& c = a.camera;
  ray_direction(c, px, py, r.d);
  double lo[3], hi[3], glo[3], ghi[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    lo[i] = (double)a.brick_offset[i];
    hi[i] = dadd(lo[i], (double)a.brick_size[i]);
    glo[i] = 0.0;
    ghi[i] = (double)a.volume_size[i];
  }
  slab(c.origin, r.d, lo, hi, r.t_in, r.t_out);
  clip_planes(a, r.d, r.t_in, r.t_out);
  slab(c.origin, r.d, glo, ghi, r.g_in, r.g_out);
  clip_planes(a, r.d, r.g_in, r.g_out);
  r.hit = (r.t_out > dmax(r.t_in, 0.0)) && (r.t_out > 0.0);
  if (r.hit) {
    r.k_lo = station_ceil(r.t_in, a.step);
    r.k_hi = station_ceil(r.t_out, a.step);
    r.kg_lo = station_ceil(r.g_in, a.step);
    r.kg_hi = station_ceil(r.g_out, a.step);
  } else {
    r.k_lo = r.k_hi = r.kg_lo = r.kg_hi = 0;
  }
}

// Global position of station k: origin + (k*step)*d  (raycast.py:346).
__device__ __forceinline__ void station_pos(const double o[3], const double d[3], double tk,
                                            double p[3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i) p[i] = dadd(o[i], dmul(tk, d[i]));
}

}  // namespace isc
