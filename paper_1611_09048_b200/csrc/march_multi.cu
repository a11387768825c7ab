// Multi-source march (C3: scalar iso surface + float3 volume with a functor
// chain, and any 1-4 float32 sources): the per-station loop of
// raycast.march_rays (raycast.py:336-380) with every active source sampled in
// source-id order, iso detection (_iso_detect, raycast.py:384-468) and
// gradient shading (raycast.py:210-242, 351-369).
//
// Versus the generic kernel (march.cu): persistent warps on the Morton tile
// scheduler, the exact float64 cell / fraction computed ONCE per station and
// shared by all sources (they share the brick, raycast.py:86), 32-bit element
// offsets, float32 loads without per-load dtype dispatch, the source loop
// unrolled at compile time (NS = 1..4) so per-source iso state lives in
// registers.  Iso side-samples (entry pair, exit pair, 6 gradient taps) are
// rare and go through one out-of-line point sampler.
#include <cstdlib>

#include "march_common.cuh"
#include "sample.cuh"

namespace isc {

struct MultiSrc {
  const float* __restrict__ f;
  int sx, sy, sz, sc;   // element strides: x, y, z, component
  int dim;
  int guarded;          // has_guard && interpolation
  int hi[3];            // guarded: size + 2g - 2 ; clamped: size - 1
};

struct MultiField {
  MultiSrc s[4];
  int lo[3];            // brick offset - guard
  int g;
};

// dim components of one source at the cell (ix, iy, iz) + fractions.
template <bool INTERP>
__device__ __forceinline__ void multi_sample(const MultiSrc& S, const MultiField& M, int ix, int iy, int iz,
                                             float fx, float fy, float fz, float v[4], uint32_t* err) {
  const int g = M.g;
  if constexpr (!INTERP) {
    const int x = min(max(ix - M.lo[0] - g, 0), S.hi[0]) + g;
    const int y = min(max(iy - M.lo[1] - g, 0), S.hi[1]) + g;
    const int z = min(max(iz - M.lo[2] - g, 0), S.hi[2]) + g;
    const float* b = S.f + (z * S.sz + y * S.sy + x * S.sx);
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (c < S.dim) v[c] = __ldg(b + c * S.sc);
    return;
  } else {
    int x0, y0, z0, dx, dy, dz;
    if (S.guarded) {
      x0 = ix - M.lo[0];
      y0 = iy - M.lo[1];
      z0 = iz - M.lo[2];
      if ((unsigned)x0 > (unsigned)S.hi[0] || (unsigned)y0 > (unsigned)S.hi[1] || (unsigned)z0 > (unsigned)S.hi[2]) {
        if (err) atomicAdd(err, 1u);
        x0 = min(max(x0, 0), S.hi[0]);
        y0 = min(max(y0, 0), S.hi[1]);
        z0 = min(max(z0, 0), S.hi[2]);
      }
      dx = S.sx;
      dy = S.sy;
      dz = S.sz;
    } else {
      const int lx = ix - M.lo[0] - g, ly = iy - M.lo[1] - g, lz = iz - M.lo[2] - g;
      x0 = min(max(lx, 0), S.hi[0]);
      y0 = min(max(ly, 0), S.hi[1]);
      z0 = min(max(lz, 0), S.hi[2]);
      dx = (min(max(lx + 1, 0), S.hi[0]) - x0) * S.sx;
      dy = (min(max(ly + 1, 0), S.hi[1]) - y0) * S.sy;
      dz = (min(max(lz + 1, 0), S.hi[2]) - z0) * S.sz;
      x0 += g;
      y0 += g;
      z0 += g;
    }
    const float* b = S.f + (z0 * S.sz + y0 * S.sy + x0 * S.sx);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (c >= S.dim) break;
      const float* p = b + c * S.sc;
      const float v000 = __ldg(p), v100 = __ldg(p + dx), v010 = __ldg(p + dy), v110 = __ldg(p + dy + dx);
      const float* q = p + dz;
      const float v001 = __ldg(q), v101 = __ldg(q + dx), v011 = __ldg(q + dy), v111 = __ldg(q + dy + dx);
      const float a0 = fmaf(fx, v100 - v000, v000), a1 = fmaf(fx, v110 - v010, v010);
      const float a2 = fmaf(fx, v101 - v001, v001), a3 = fmaf(fx, v111 - v011, v011);
      const float b0 = fmaf(fy, a1 - a0, a0), b1 = fmaf(fy, a3 - a2, a2);
      v[c] = fmaf(fz, b1 - b0, b0);
    }
  }
}

__device__ __forceinline__ void cell_of(const double p[3], int& ix, int& iy, int& iz, float& fx, float& fy,
                                        float& fz) {
  const double flx = floor_split(p[0], ix), fly = floor_split(p[1], iy), flz = floor_split(p[2], iz);
  fx = (float)dsub(p[0], flx);
  fy = (float)dsub(p[1], fly);
  fz = (float)dsub(p[2], flz);
}

// Cell, float32 fractions and the exact float64 fractions (iso_exact sources).
__device__ __forceinline__ void cell_of_d(const double p[3], int& ix, int& iy, int& iz, double& fxd, double& fyd,
                                          double& fzd) {
  const double flx = floor_split(p[0], ix), fly = floor_split(p[1], iy), flz = floor_split(p[2], iz);
  fxd = dsub(p[0], flx);
  fyd = dsub(p[1], fly);
  fzd = dsub(p[2], flz);
}

// The reference's float64 trilinear (raycast.py:182-199) from the 8 corners
// (x fastest: v000 v100 v010 v110 v001 v101 v011 v111): out starts at 0 and
// accumulates ((wx*wy)*wz)*corner over dz, dy, dx in that order, w = f or
// 1 - f -- the same roundings as numpy, so the value is bit-identical.
__device__ __forceinline__ double trilinear_d(const float c[8], double fx, double fy, double fz) {
  double out = 0.0;
#pragma unroll
  for (int dz = 0; dz < 2; ++dz) {
    const double wz = dz ? fz : dsub(1.0, fz);
#pragma unroll
    for (int dy = 0; dy < 2; ++dy) {
      const double wy = dy ? fy : dsub(1.0, fy);
#pragma unroll
      for (int dx = 0; dx < 2; ++dx) {
        const double wx = dx ? fx : dsub(1.0, fx);
        out = dadd(out, dmul(dmul(dmul(wx, wy), wz), (double)c[dz * 4 + dy * 2 + dx]));
      }
    }
  }
  return out;
}

// float64 add / mul chain of an iso_exact source (functors.py:212-222).
__device__ __forceinline__ double run_chain_d(const isc_source& s, double v) {
  const unsigned ops = s.step_ops;
#pragma unroll
  for (int i = 0; i < ISC_MAX_CHAIN; ++i) {
    if (i >= s.n_steps) break;
    const isc_chain_step& st = s.steps[i];
    v = ((ops >> (4 * i)) & 0xFu) == ISC_OP_ADD ? dadd(v, st.arg_d[0]) : dmul(v, st.arg_d[0]);
  }
  return v;
}

// The 8 corners of a guarded scalar source at base cell (x0, y0, z0).
__device__ __forceinline__ void corners_guarded(const MultiSrc& S, int x0, int y0, int z0, float c[8]) {
  const float* p = S.f + (z0 * S.sz + y0 * S.sy + x0 * S.sx);
  const int dx = S.sx, dy = S.sy, dz = S.sz;
  c[0] = __ldg(p);
  c[1] = __ldg(p + dx);
  c[2] = __ldg(p + dy);
  c[3] = __ldg(p + dy + dx);
  const float* q = p + dz;
  c[4] = __ldg(q);
  c[5] = __ldg(q + dx);
  c[6] = __ldg(q + dy);
  c[7] = __ldg(q + dy + dx);
}

// float32 trilinear of 8 corners (the kernels' usual arithmetic).
__device__ __forceinline__ float lerp8(const float c[8], float fx, float fy, float fz) {
  const float a0 = fmaf(fx, c[1] - c[0], c[0]), a1 = fmaf(fx, c[3] - c[2], c[2]);
  const float a2 = fmaf(fx, c[5] - c[4], c[4]), a3 = fmaf(fx, c[7] - c[6], c[6]);
  const float b0 = fmaf(fy, a1 - a0, a0), b1 = fmaf(fy, a3 - a2, a2);
  return fmaf(fz, b1 - b0, b0);
}

// Iso value of source si at a global position, as a double: the exact
// float64 value for an iso_exact source (guarded), else the float32 chain.
template <bool INTERP>
__device__ __noinline__ double iso_point_value(const MultiSrc& S, const MultiField& M, const isc_source& src,
                                               const double p[3], uint32_t* err);

// Chained scalar of one source at an arbitrary global position (iso extras).
template <bool INTERP>
__device__ __noinline__ float point_scalar(const MultiSrc& S, const MultiField& M, const isc_source& src,
                                           const double p[3], uint32_t* err) {
  int ix, iy, iz;
  float fx, fy, fz;
  cell_of(p, ix, iy, iz, fx, fy, fz);
  float v[4] = {0.f, 0.f, 0.f, 0.f};
  multi_sample<INTERP>(S, M, ix, iy, iz, fx, fy, fz, v, err);
  return run_chain(src, v, S.dim);
}

template <bool INTERP>
__device__ __noinline__ double iso_point_value(const MultiSrc& S, const MultiField& M, const isc_source& src,
                                               const double p[3], uint32_t* err) {
  if (INTERP && src.iso_exact && S.guarded && S.dim == 1) {
    int ix, iy, iz;
    double fx, fy, fz;
    cell_of_d(p, ix, iy, iz, fx, fy, fz);
    int x0 = ix - M.lo[0], y0 = iy - M.lo[1], z0 = iz - M.lo[2];
    if ((unsigned)x0 > (unsigned)S.hi[0] || (unsigned)y0 > (unsigned)S.hi[1] || (unsigned)z0 > (unsigned)S.hi[2]) {
      if (err) atomicAdd(err, 1u);
      x0 = min(max(x0, 0), S.hi[0]);
      y0 = min(max(y0, 0), S.hi[1]);
      z0 = min(max(z0, 0), S.hi[2]);
    }
    float c[8];
    corners_guarded(S, x0, y0, z0, c);
    return run_chain_d(src, trilinear_d(c, fx, fy, fz));
  }
  return (double)point_scalar<INTERP>(S, M, src, p, err);
}

__device__ __forceinline__ bool reach(const double off[3], const double size[3], int g, const double p[3]) {
  bool ok = true;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double lo = dsub(off[i], (double)g);
    const double hi = dsub(dadd(dadd(off[i], size[i]), (double)g), 1.0);
    ok &= (p[i] >= lo) && (p[i] < hi);
  }
  return ok;
}

template <bool INTERP>
__device__ __noinline__ float3 multi_normal(const MultiSrc& S, const MultiField& M, const isc_source& src,
                                            const double off[3], const int size[3], const double p[3],
                                            const double d[3], uint32_t* err) {
  const int g = S.guarded ? M.g : 0;
  float grad[3];
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    const double lo = dsub(off[ax], (double)g);
    const double hi = dsub(dsub(dadd(dadd(lo, (double)size[ax]), (double)(2 * g)), 1.0), 1e-9);
    double pp[3] = {p[0], p[1], p[2]}, pm[3] = {p[0], p[1], p[2]};
    pp[ax] = dmin(dmax(dadd(p[ax], 1.0), lo), hi);
    pm[ax] = dmin(dmax(dsub(p[ax], 1.0), lo), hi);
    double span = dsub(pp[ax], pm[ax]);
    if (span == 0.0) span = 1.0;
    const float sp = point_scalar<INTERP>(S, M, src, pp, err);
    const float sm = point_scalar<INTERP>(S, M, src, pm, err);
    grad[ax] = (float)((double)(sp - sm) / span);
  }
  const float mag = sqrtf((grad[0] * grad[0] + grad[1] * grad[1]) + grad[2] * grad[2]);
  if (mag < 1e-12f) {
    const double dm = sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
    return make_float3((float)(-d[0] / dm), (float)(-d[1] / dm), (float)(-d[2] / dm));
  }
  return make_float3(grad[0] / mag, grad[1] / mag, grad[2] / mag);
}

// Rare iso pair tests of source si, out of line (see iso_hit_color): the
// entry pair's earlier value (station k-1 through the guard) and the forward
// exit pair (the next brick cannot reach back), raycast.py:384-468.
__device__ __noinline__ double iso_entry_value(const isc_render_args& a, const MultiField& M, int si, double d0,
                                               double d1, double d2, int k, uint32_t* err) {
  const double d[3] = {d0, d1, d2};
  double off[3], bsz[3], pq[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    off[i] = (double)a.brick_offset[i];
    bsz[i] = (double)a.brick_size[i];
  }
  station_pos(a.camera.origin, d, dmul((double)(k - 1), a.step), pq);
  return reach(off, bsz, M.g, pq) ? iso_point_value<true>(M.s[si], M, a.src[si], pq, err) : (double)CUDART_NAN_F;
}

__device__ __noinline__ bool iso_exit_pair(const isc_render_args& a, const MultiField& M, int si, double d0,
                                           double d1, double d2, int k, double p0, double p1, double p2, double sb,
                                           double* tau, uint32_t* err) {
  const double d[3] = {d0, d1, d2}, p[3] = {p0, p1, p2};
  double off[3], bsz[3], vb[3], pn[3], noff[3];
  station_pos(a.camera.origin, d, dmul((double)(k + 1), a.step), pn);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    off[i] = (double)a.brick_offset[i];
    bsz[i] = (double)a.brick_size[i];
    vb[i] = ddiv((double)a.volume_size[i], (double)a.decomposition[i]);  // raycast.py:283-285
    double c = floor(ddiv(pn[i], vb[i]));
    c = dmin(dmax(c, 0.0), (double)(a.decomposition[i] - 1));
    noff[i] = dmul(c, vb[i]);
  }
  if (reach(off, bsz, M.g, pn) && !reach(noff, vb, M.g, p)) {
    const double sn = dsub(iso_point_value<true>(M.s[si], M, a.src[si], pn, err), a.src[si].iso_threshold_d);
    if ((sb < 0.0) != (sn < 0.0)) {
      const double den = dsub(sb, sn);
      *tau = den != 0.0 ? ddiv(sb, den) : 1.0;
      return true;
    }
  }
  return false;
}

template <bool INTERP = true>
__device__ __noinline__ float4 iso_hit_color(const isc_render_args& a, const MultiField& M, int si, double d0,
                                             double d1, double d2, double p0, double p1, double p2, double tau,
                                             double back, uint32_t* err) {
  const double d[3] = {d0, d1, d2}, p[3] = {p0, p1, p2};
  const isc_source& s = a.src[si];
  double hp[3], off[3];
  int isz[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    off[i] = (double)a.brick_offset[i];
    isz[i] = a.brick_size[i];
  }
  const double tt = dmul(dadd(tau, back), a.step);
#pragma unroll
  for (int i = 0; i < 3; ++i) hp[i] = dadd(p[i], dmul(tt, d[i]));
  const float3 nrm = multi_normal<INTERP>(M.s[si], M, s, off, isz, hp, d, err);
  const float shade = fabsf(nrm.x * (float)d[0] + nrm.y * (float)d[1] + nrm.z * (float)d[2]);
  const float4 base = classify_aos(reinterpret_cast<const float4*>(s.lut), s.range_lo, 1.0f / (s.range_hi - s.range_lo),
                               s.iso_threshold);
  return make_float4(base.x * shade, base.y * shade, base.z * shade, 1.0f);
}

template <int NS, bool INTERP, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) march_multi_kernel(const __grid_constant__ isc_render_args a,
                                                               const __grid_constant__ MultiField M, int tiles_x,
                                                               int tiles_y, int super_x, int n_codes) {
  __shared__ float lut_s[NS * kLutWords];
  lut_fill_sources(lut_s, a, NS);
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const bool gate_alpha = a.alpha_stop < 1.0;
  const float stop_f = __double2float_ru(a.alpha_stop);  // w >= stop_f <=> (double)w >= alpha_stop
  const double* o = a.camera.origin;
  const double step = a.step;
  uint32_t* err = a.error_word;
  double off[3], bsz[3], vb[3];
  int isz[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    off[i] = (double)a.brick_offset[i];
    bsz[i] = (double)a.brick_size[i];
    isz[i] = a.brick_size[i];
    vb[i] = ddiv((double)a.volume_size[i], (double)a.decomposition[i]);  // raycast.py:283-285
  }
  float inv[NS];
#pragma unroll
  for (int si = 0; si < NS; ++si) inv[si] = 1.0f / (a.src[si].range_hi - a.src[si].range_lo);
  unsigned long long warp_stations = 0;

  for (;;) {
    int t = 0;
    if (lane == 0) t = (int)atomicAdd(a.work_counter, 1u);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= n_codes) break;
    const int sblk = t >> 6, w = t & 63;
    const int tx = (sblk % super_x) * 8 + morton3(w, 0);
    const int ty = (sblk / super_x) * 8 + morton3(w, 1);
    if (tx >= tiles_x || ty >= tiles_y) continue;
    const int px = tx * 8 + (lane & 7), py = ty * 4 + (lane >> 3);
    if (px >= a.camera.width || py >= a.camera.height) continue;

    Ray r;
    setup_ray(a, px, py, r);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    uint32_t stations = 0;
    int hit_si = -1;                     // first iso source hit (shaded after the loop)
    long long hit_k = 0;
    double hit_tau = 0.0, hit_back = 0.0;
    float4 hit_front = make_float4(0.f, 0.f, 0.f, 0.f);
    if (r.hit) {
      float prev[NS];
#pragma unroll
      for (int si = 0; si < NS; ++si) prev[si] = CUDART_NAN_F;
      for (long long k = r.k_lo; k < r.k_hi; ++k) {
        ++stations;
        double p[3];
        station_pos(o, r.d, dmul((double)k, step), p);
        int ix, iy, iz;
        float fx, fy, fz;
        cell_of(p, ix, iy, iz, fx, fy, fz);
        float4 st = make_float4(0.f, 0.f, 0.f, 0.f);
        bool stop = false;
#pragma unroll
        for (int si = 0; si < NS; ++si) {
          const isc_source& s = a.src[si];
          const MultiSrc& S = M.s[si];
          float v[4] = {0.f, 0.f, 0.f, 0.f};
          multi_sample<INTERP>(S, M, ix, iy, iz, fx, fy, fz, v, err);
          const float cur = s.n_steps ? run_chain(s, v, S.dim) : v[0];
          const float* lut = lut_s + si * kLutWords;
          if (s.mode != ISC_ISO) {
            st = over4(st, premultiply(classify(lut, s.range_lo, inv[si], cur)));
            continue;
          }
          // ---- iso: raycast.py:384-468 ----
          const float thr = s.iso_threshold;
          const bool exact = S.guarded != 0;
          float before = prev[si];
          if (k == r.k_lo && k - 1 >= r.kg_lo) {  // entry pair: sample k-1 through the guard
            double pq[3];
            station_pos(o, r.d, dmul((double)(k - 1), step), pq);
            before = (!exact || reach(off, bsz, M.g, pq)) ? point_scalar<INTERP>(S, M, s, pq, err) : CUDART_NAN_F;
          }
          const float sa = before - thr, sb = cur - thr;
          bool hit = isfinite(sa) && ((sa < 0.f) != (sb < 0.f));
          double tau = 0.0, back = 0.0;
          if (hit) {
            const float den = sa - sb;
            tau = den != 0.f ? (double)(sa / den) : 1.0;
            back = -1.0;
          }
          if (exact && !hit && k == r.k_hi - 1 && k + 1 < r.kg_hi) {  // exit pair, checked forward
            double pn[3], noff[3];
            station_pos(o, r.d, dmul((double)(k + 1), step), pn);
#pragma unroll
            for (int i = 0; i < 3; ++i) {
              double c = floor(ddiv(pn[i], vb[i]));
              c = dmin(dmax(c, 0.0), (double)(a.decomposition[i] - 1));
              noff[i] = dmul(c, vb[i]);
            }
            if (reach(off, bsz, M.g, pn) && !reach(noff, vb, M.g, p)) {
              const float sn = point_scalar<INTERP>(S, M, s, pn, err) - thr;
              if ((sb < 0.f) != (sn < 0.f)) {
                const float den = sb - sn;
                tau = den != 0.f ? (double)(sb / den) : 1.0;
                back = 0.0;
                hit = true;
              }
            }
          }
          prev[si] = cur;
          if (hit && !stop) {  // shaded after the loop; later sources sit behind the hit
            hit_si = si;
            hit_k = k;
            hit_tau = tau;
            hit_back = back;
            hit_front = st;
            stop = true;
          }
        }
        if (stop) break;
        acc = over4(acc, st);
        if (gate_alpha && acc.w >= stop_f) break;
      }
    }
    if (hit_si >= 0) {  // all hitting lanes of the warp shade together
      double ph[3];
      station_pos(o, r.d, dmul((double)hit_k, step), ph);
      const float4 c = iso_hit_color<INTERP>(a, M, hit_si, r.d[0], r.d[1], r.d[2], ph[0], ph[1], ph[2], hit_tau,
                                             hit_back, err);
      acc = over4(acc, over4(hit_front, c));
    }
    const long long pix = (long long)py * a.camera.width + px;
    reinterpret_cast<float4*>(a.out_rgba)[pix] = acc;
    warp_stations += stations;
    if (a.out_stations) a.out_stations[pix] = stations;
    if (a.out_hit) a.out_hit[pix] = r.hit ? 1 : 0;
    if (a.out_t) {
      a.out_t[2 * pix] = r.t_in;
      a.out_t[2 * pix + 1] = r.t_out;
    }
    if (a.out_krange)
      reinterpret_cast<int4*>(a.out_krange)[pix] = make_int4((int)r.k_lo, (int)r.k_hi, (int)r.kg_lo, (int)r.kg_hi);
  }
  if (a.out_station_total) {
#pragma unroll
    for (int off2 = 16; off2 > 0; off2 >>= 1) warp_stations += __shfl_xor_sync(0xffffffffu, warp_stations, off2);
    if (lane == 0 && warp_stations) atomicAdd(a.out_station_total, warp_stations);
  }
}

// ---------------------------------------------------------------------------
// Specialised multi-source march: trilinear, every source guarded
// (has_guard), component counts known at compile time (DIMS packs one base-5
// digit per source).  Versus march_multi_kernel: the guard contract is proven
// once per ray from its end stations (cell indices are monotone in k, see
// march_fast_kernel), so the per-station gathers of all sources carry no
// checks or clamps and are issued back to back; component loops are fully
// unrolled.  A ray whose end station fails the check is marched with the
// per-station check instead: an iso hit or early termination may stop it
// before the bad station, and the reference only raises on a gather it
// performs.  Iso side samples reuse the generic out-of-line point sampler.
template <int DIMS, int SI>
__host__ __device__ constexpr int dim_at() {
  return SI == 0 ? DIMS % 5 : SI == 1 ? (DIMS / 5) % 5 : SI == 2 ? (DIMS / 25) % 5 : (DIMS / 125) % 5;
}

template <int D>
__device__ __forceinline__ void gather_guarded(const MultiSrc& S, int x0, int y0, int z0, float fx, float fy,
                                               float fz, float v[4]) {
  const float* b = S.f + (z0 * S.sz + y0 * S.sy + x0 * S.sx);
  const int dx = S.sx, dy = S.sy, dz = S.sz;
#pragma unroll
  for (int c = 0; c < D; ++c) {
    const float* p = b + c * S.sc;
    const float v000 = __ldg(p), v100 = __ldg(p + dx), v010 = __ldg(p + dy), v110 = __ldg(p + dy + dx);
    const float* q = p + dz;
    const float v001 = __ldg(q), v101 = __ldg(q + dx), v011 = __ldg(q + dy), v111 = __ldg(q + dy + dx);
    const float a0 = fmaf(fx, v100 - v000, v000), a1 = fmaf(fx, v110 - v010, v010);
    const float a2 = fmaf(fx, v101 - v001, v001), a3 = fmaf(fx, v111 - v011, v011);
    const float b0 = fmaf(fy, a1 - a0, a0), b1 = fmaf(fy, a3 - a2, a2);
    v[c] = fmaf(fz, b1 - b0, b0);
  }
}

// Standard zero-copy layout (x contiguous, components interleaved: sx ==
// D, sc == 1 -- a C-contiguous (z, y, x[, c]) array): one 64-bit base per
// (y, z) corner row, the x+1 corner and every component at an immediate
// offset (the general form computes a 64-bit address per corner and
// component from the runtime strides).
template <int D>
__device__ __forceinline__ void gather_contig(const MultiSrc& S, int x0, int y0, int z0, float fx, float fy,
                                              float fz, float v[4]) {
  const float* r00 = S.f + (z0 * S.sz + y0 * S.sy + x0 * D);
  const float* r10 = r00 + S.sy;
  const float* r01 = r00 + S.sz;
  const float* r11 = r01 + S.sy;
#pragma unroll
  for (int c = 0; c < D; ++c) {
    const float v000 = __ldg(r00 + c), v100 = __ldg(r00 + D + c), v010 = __ldg(r10 + c), v110 = __ldg(r10 + D + c);
    const float v001 = __ldg(r01 + c), v101 = __ldg(r01 + D + c), v011 = __ldg(r11 + c), v111 = __ldg(r11 + D + c);
    const float a0 = fmaf(fx, v100 - v000, v000), a1 = fmaf(fx, v110 - v010, v010);
    const float a2 = fmaf(fx, v101 - v001, v001), a3 = fmaf(fx, v111 - v011, v011);
    const float b0 = fmaf(fy, a1 - a0, a0), b1 = fmaf(fy, a3 - a2, a2);
    v[c] = fmaf(fz, b1 - b0, b0);
  }
}

__device__ __forceinline__ void corners_contig(const MultiSrc& S, int x0, int y0, int z0, float c[8]) {
  const float* r00 = S.f + (z0 * S.sz + y0 * S.sy + x0);
  const float* r10 = r00 + S.sy;
  const float* r01 = r00 + S.sz;
  const float* r11 = r01 + S.sy;
  c[0] = __ldg(r00);
  c[1] = __ldg(r00 + 1);
  c[2] = __ldg(r10);
  c[3] = __ldg(r10 + 1);
  c[4] = __ldg(r01);
  c[5] = __ldg(r01 + 1);
  c[6] = __ldg(r11);
  c[7] = __ldg(r11 + 1);
}

__device__ __forceinline__ bool cell_guard_ok(const MultiField& M, const double p[3]) {
  int ix, iy, iz;
  floor_split(p[0], ix);
  floor_split(p[1], iy);
  floor_split(p[2], iz);
  const MultiSrc& S = M.s[0];  // every source of this kernel is guarded: same halo bounds
  return (unsigned)(ix - M.lo[0]) <= (unsigned)S.hi[0] && (unsigned)(iy - M.lo[1]) <= (unsigned)S.hi[1] &&
         (unsigned)(iz - M.lo[2]) <= (unsigned)S.hi[2];
}

// Shaded colour of an iso hit on source si (gradient normal, raycast.py:
// 210-242, 351-369), out of line so the station loop keeps its registers;
// direction and position by value so the caller's Ray stays in registers.
#ifndef ISC_MULTI_FAST_MINB
#define ISC_MULTI_FAST_MINB 2
#endif
#ifndef ISC_MULTI_FAST_THREADS
#define ISC_MULTI_FAST_THREADS 256
#endif
constexpr int kMultiFastThreads = ISC_MULTI_FAST_THREADS;

template <int NS, int DIMS, bool CONTIG>
__global__ void __launch_bounds__(kMultiFastThreads, ISC_MULTI_FAST_MINB)
    march_multi_fast_kernel(const __grid_constant__ isc_render_args a, const __grid_constant__ MultiField M,
                            int tiles_x, int tiles_y, int super_x, int n_codes, int tile_x0, int tile_y0,
                            int tw_log2) {
  __shared__ float lut_s[NS * kLutWords];
  lut_fill_sources(lut_s, a, NS);
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const bool gate_alpha = a.alpha_stop < 1.0;
  const float stop_f = __double2float_ru(a.alpha_stop);  // w >= stop_f <=> (double)w >= alpha_stop
  const double* o = a.camera.origin;
  const double step = a.step;
  uint32_t* err = a.error_word;
  unsigned long long warp_stations = 0;
  float inv_span[NS];
#pragma unroll
  for (int si = 0; si < NS; ++si) inv_span[si] = 1.0f / (a.src[si].range_hi - a.src[si].range_lo);

  for (;;) {
    int t = 0;
    if (lane == 0) t = (int)atomicAdd(a.work_counter, 1u);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= n_codes) break;
    const int sblk = t >> 6, w = t & 63;
    const int tx = (sblk % super_x) * 8 + morton3(w, 0);
    const int ty = (sblk / super_x) * 8 + morton3(w, 1);
    if (tx >= tiles_x || ty >= tiles_y) continue;
    const int px = ((tx + tile_x0) << tw_log2) + (lane & ((1 << tw_log2) - 1));
    const int py = (ty + tile_y0) * (32 >> tw_log2) + (lane >> tw_log2);
    if (px >= a.camera.width || py >= a.camera.height) continue;

    Ray r;
    setup_ray(a, px, py, r);
    const long long pix = (long long)py * a.camera.width + px;
    // parity / debug outputs first: the slab intervals are then dead during the march
    if (a.out_hit) a.out_hit[pix] = r.hit ? 1 : 0;
    if (a.out_t) {
      a.out_t[2 * pix] = r.t_in;
      a.out_t[2 * pix + 1] = r.t_out;
    }
    if (a.out_krange)
      reinterpret_cast<int4*>(a.out_krange)[pix] = make_int4((int)r.k_lo, (int)r.k_hi, (int)r.kg_lo, (int)r.kg_hi);
    // station indices as int for the march (a ray holds < 2^31 stations)
    const int k_lo = (int)r.k_lo, k_hi = (int)r.k_hi, kg_lo = (int)r.kg_lo, kg_hi = (int)r.kg_hi;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    uint32_t stations = 0;
    // Stations whose gathers honour the guard form one interval (each cell
    // index is monotone in k).  A bad first station is gathered by any hit
    // ray: error.  A bad last station: binary-search the last good one and
    // stop there; reaching that point without an iso hit / early stop is
    // the reference's GuardContractError (fields.py:230-238).
    long long kend = r.k_hi;
    bool bad_tail = false;
    if (r.hit && r.k_hi > r.k_lo) {  // a hit ray can hold no station (t_in, t_out in one step)
      double pa[3], pb[3];
      station_pos(o, r.d, dmul((double)r.k_lo, step), pa);
      station_pos(o, r.d, dmul((double)(r.k_hi - 1), step), pb);
      if (!cell_guard_ok(M, pa)) {
        if (err) atomicAdd(err, 1u);
        kend = r.k_lo;
      } else if (!cell_guard_ok(M, pb)) {
        long long good = r.k_lo, bad = r.k_hi - 1;
        while (bad - good > 1) {
          const long long mid = good + ((bad - good) >> 1);
          double pm[3];
          station_pos(o, r.d, dmul((double)mid, step), pm);
          if (cell_guard_ok(M, pm)) good = mid;
          else bad = mid;
        }
        kend = bad;
        bad_tail = true;
      }
    }
    bool stopped = false;
    int hit_si = -1;                     // first iso source hit (shaded after the loop)
    int hit_k = 0;
    double hit_tau = 0.0;
    double hit_sb = 0.0;                 // backward pairs: s at the hit station (tau after the loop)
    bool hit_behind = false;             // crossing between k-1 and k (back = -1) rather than k and k+1
    float4 hit_front = make_float4(0.f, 0.f, 0.f, 0.f);  // the station's sources in front of it
    if (r.hit) {
      double prev[NS];   // previous station's iso value (float64: the reference's sign tests)
#pragma unroll
      for (int si = 0; si < NS; ++si) prev[si] = (double)CUDART_NAN_F;
      double kd = (double)r.k_lo;
      const double kendd = (double)kend;
      for (; kd < kendd; kd = dadd(kd, 1.0)) {
        ++stations;
        double p[3];
        station_pos(o, r.d, dmul(kd, step), p);
        int ix, iy, iz;
        double fxd, fyd, fzd;
        cell_of_d(p, ix, iy, iz, fxd, fyd, fzd);
        const float fx = (float)fxd, fy = (float)fyd, fz = (float)fzd;
        const int x0 = ix - M.lo[0], y0 = iy - M.lo[1], z0 = iz - M.lo[2];
        float v[NS][4];
        float cr[NS][8];   // raw corners of scalar sources (iso_exact float64 path)
        // all gathers of the station first (they are independent)
#pragma unroll
        for (int si = 0; si < NS; ++si) {
          constexpr int kDims[4] = {dim_at<DIMS, 0>(), dim_at<DIMS, 1>(), dim_at<DIMS, 2>(), dim_at<DIMS, 3>()};
          if (kDims[si] == 1) {
            if constexpr (CONTIG) corners_contig(M.s[si], x0, y0, z0, cr[si]);
            else corners_guarded(M.s[si], x0, y0, z0, cr[si]);
            v[si][0] = lerp8(cr[si], fx, fy, fz);
          } else if constexpr (CONTIG) {
            if (si == 0) gather_contig<dim_at<DIMS, 0>()>(M.s[0], x0, y0, z0, fx, fy, fz, v[0]);
            else if (si == 1) gather_contig<dim_at<DIMS, 1>()>(M.s[1], x0, y0, z0, fx, fy, fz, v[1]);
            else if (si == 2) gather_contig<dim_at<DIMS, 2>()>(M.s[2], x0, y0, z0, fx, fy, fz, v[2]);
            else gather_contig<dim_at<DIMS, 3>()>(M.s[3], x0, y0, z0, fx, fy, fz, v[3]);
          } else if (si == 0) {
            gather_guarded<dim_at<DIMS, 0>()>(M.s[0], x0, y0, z0, fx, fy, fz, v[0]);
          } else if (si == 1) {
            gather_guarded<dim_at<DIMS, 1>()>(M.s[1], x0, y0, z0, fx, fy, fz, v[1]);
          } else if (si == 2) {
            gather_guarded<dim_at<DIMS, 2>()>(M.s[2], x0, y0, z0, fx, fy, fz, v[2]);
          } else {
            gather_guarded<dim_at<DIMS, 3>()>(M.s[3], x0, y0, z0, fx, fy, fz, v[3]);
          }
        }
        float4 st = make_float4(0.f, 0.f, 0.f, 0.f);
        bool stop = false;
#pragma unroll
        for (int si = 0; si < NS; ++si) {
          const isc_source& s = a.src[si];
          float cur;
          if (si == 0) cur = run_chain_fast<dim_at<DIMS, 0>()>(s, v[0]);
          else if (si == 1) cur = run_chain_fast<dim_at<DIMS, 1>()>(s, v[1]);
          else if (si == 2) cur = run_chain_fast<dim_at<DIMS, 2>()>(s, v[2]);
          else cur = run_chain_fast<dim_at<DIMS, 3>()>(s, v[3]);
          const float* lut = lut_s + si * kLutWords;
          const float inv = inv_span[si];
          if (s.mode != ISC_ISO) {
            st = over4(st, classify_src_premul(s, lut, inv, cur));
            continue;
          }
          // ---- iso: raycast.py:384-468 (every source here is guarded: "exact") ----
          // iso_exact: the value, sign test and tau in the reference's float64
          constexpr int kDimsI[4] = {dim_at<DIMS, 0>(), dim_at<DIMS, 1>(), dim_at<DIMS, 2>(), dim_at<DIMS, 3>()};
          double cur_d = (double)cur;
          const double thr = s.iso_threshold_d;
          if (kDimsI[si] == 1 && s.iso_exact) {
            if (s.n_steps == 0) {
              // identity chain: the float32 trilinear is within 2^-20 max|corner|
              // of the float64 one (3 lerp levels, each <= 2.5 * 2^-23 M), so
              // its sign against the threshold is the reference's outside a
              // 4x wider band; inside it (rare) take the float64 value
              float m = fabsf(cr[si][0]);
#pragma unroll
              for (int c = 1; c < 8; ++c) m = fmaxf(m, fabsf(cr[si][c]));
              if (!(fabs(dsub(cur_d, thr)) > (double)m * 0x1p-18)) cur_d = trilinear_d(cr[si], fxd, fyd, fzd);
            } else {
              cur_d = run_chain_d(s, trilinear_d(cr[si], fxd, fyd, fzd));
            }
          }
          double before = prev[si];
          const int k = (int)kd;
          if (k == k_lo && k - 1 >= kg_lo)  // entry pair: sample k-1 through the guard
            before = iso_entry_value(a, M, si, r.d[0], r.d[1], r.d[2], k, err);
          const double sa = dsub(before, thr), sb = dsub(cur_d, thr);
          bool hit = isfinite(sa) && ((sa < 0.0) != (sb < 0.0));
          double tau = 0.0, back = 0.0;
          if (hit) {  // tau = sa / (sa - sb) once, after the loop (hit_sa / hit_den)
            tau = sa;
            back = -1.0;
          }
          if (!hit && k == k_hi - 1 && k + 1 < kg_hi) {  // exit pair, checked forward
            double tx = 0.0;
            if (iso_exit_pair(a, M, si, r.d[0], r.d[1], r.d[2], k, p[0], p[1], p[2], sb, &tx, err)) {
              tau = tx;
              back = 0.0;
              hit = true;
            }
          }
          prev[si] = cur_d;
          if (hit && !stop) {  // later sources of the station sit behind the opaque hit
            hit_si = si;
            hit_k = k;
            hit_tau = tau;
            hit_sb = sb;
            hit_behind = back != 0.0;
            hit_front = st;
            stop = true;
          }
        }
        if (stop) {
          stopped = true;
          break;
        }
        acc = over4(acc, st);
        if (gate_alpha && acc.w >= stop_f) {
          stopped = true;
          break;
        }
      }
      if (bad_tail && !stopped && err) atomicAdd(err, 1u);
    }
    // Shade iso hits after the loop: hits fall in different iterations, so
    // in-loop shading ran once per hitting lane with the rest of the warp idle.
    if (hit_si >= 0) {
      if (hit_behind) {  // tau = s_prev / (s_prev - s_cur), raycast.py:434-437
        const double den = dsub(hit_tau, hit_sb);
        hit_tau = den != 0.0 ? ddiv(hit_tau, den) : 1.0;
      }
      double ph[3];
      station_pos(o, r.d, dmul((double)hit_k, step), ph);
      const float4 c = iso_hit_color(a, M, hit_si, r.d[0], r.d[1], r.d[2], ph[0], ph[1], ph[2], hit_tau,
                                     hit_behind ? -1.0 : 0.0, err);
      acc = over4(acc, over4(hit_front, c));
    }
    reinterpret_cast<float4*>(a.out_rgba)[pix] = acc;
    warp_stations += stations;
    if (a.out_stations) a.out_stations[pix] = stations;
  }
  if (a.out_station_total) {
#pragma unroll
    for (int off2 = 16; off2 > 0; off2 >>= 1) warp_stations += __shfl_xor_sync(0xffffffffu, warp_stations, off2);
    if (lane == 0 && warp_stations) atomicAdd(a.out_station_total, warp_stations);
  }
}

static bool build_multi_field(const isc_render_args* a, MultiField& M);

// ---------------------------------------------------------------------------
// Paired iso probe: pass 1 of the split iso + volume render (march.cu
// launch_split).  ONE guarded float32 scalar iso source, no early
// termination.  A warp is 16 rays (8x2 pixels) x 2 station parities as in
// march_fast_kernel: lane q marches the even stations k_lo + 2j of ray q,
// lane q + 16 the odd ones, so one gather request covers 32 samples within an
// 8x2-pixel footprint.  Station values are float64 (the multi-source kernel's
// exact iso decisions: identity chains take the float64 value inside the
// float32 error band, add / mul chains always).  Per iteration each lane
// tests the backward pair ending at its own station (_iso_detect,
// raycast.py:384-468): the odd lane's earlier value comes from the even lane
// by one shuffle-up, the even lane's from the odd lane of the previous
// iteration by one shuffle-down; one ballot tells both lanes of a pair
// whether the ray hit (the even lane's station comes first).  The loop holds
// no calls: the entry pair's value (station k_lo - 1 through the guard) is
// sampled before it, the forward exit pair (tested only when no backward
// pair hit) after it, and the hit is shaded after it by the lane that found
// it (gradient normal, raycast.py:210-242, 351-369).  Outputs: the shaded hit
// colour (alpha 1) or 0 in out_rgba, the stations marched (hit station
// included) in out_stations -- what pass 2 stops at.
#ifndef ISC_PROBE_MINB
#define ISC_PROBE_MINB 4
#endif
template <bool CONTIG, bool CHAIN>
__global__ void __launch_bounds__(kThreads, ISC_PROBE_MINB)
    iso_probe_kernel(const __grid_constant__ isc_render_args a, const __grid_constant__ MultiField M, int tiles_x,
                     int tiles_y, int super_x, int n_codes, int tile_x0, int tile_y0) {
  const int lane = threadIdx.x & 31, q = lane & 15, parity = lane >> 4;
  const double* o = a.camera.origin;
  const double step = a.step;
  uint32_t* err = a.error_word;
  const isc_source& s = a.src[0];
  const MultiSrc& S = M.s[0];
  const double thr = s.iso_threshold_d;
  unsigned long long warp_stations = 0;
  for (;;) {
    int t = 0;
    if (lane == 0) t = (int)atomicAdd(a.work_counter, 1u);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= n_codes) break;
    const int sblk = t >> 6, w = t & 63;
    const int tx = (sblk % super_x) * 8 + morton3(w, 0);
    const int ty = (sblk / super_x) * 8 + morton3(w, 1);
    if (tx >= tiles_x || ty >= tiles_y) continue;
    const int px = (tx + tile_x0) * 8 + (q & 7), py = (ty + tile_y0) * 2 + (q >> 3);
    const bool in_img = px < a.camera.width && py < a.camera.height;
    Ray r;
    if (in_img) {
      setup_ray(a, px, py, r);
    } else {
      r.hit = false;
      r.k_lo = r.k_hi = r.kg_lo = r.kg_hi = 0;
    }
    const long long pix = (long long)py * a.camera.width + px;
    if (!parity && in_img) {
      if (a.out_hit) a.out_hit[pix] = r.hit ? 1 : 0;
      if (a.out_t) {
        a.out_t[2 * pix] = r.t_in;
        a.out_t[2 * pix + 1] = r.t_out;
      }
      if (a.out_krange)
        reinterpret_cast<int4*>(a.out_krange)[pix] =
            make_int4((int)r.k_lo, (int)r.k_hi, (int)r.kg_lo, (int)r.kg_hi);
    }
    const int k_lo = (int)r.k_lo, k_hi = (int)r.k_hi;
    // guard contract per ray (march_multi_fast_kernel): stations below kend
    int kend = k_hi;
    bool bad_tail = false;
    if (r.hit && k_hi > k_lo) {
      double pa[3], pb[3];
      station_pos(o, r.d, dmul((double)k_lo, step), pa);
      station_pos(o, r.d, dmul((double)(k_hi - 1), step), pb);
      if (!cell_guard_ok(M, pa)) {
        if (err && !parity) atomicAdd(err, 1u);
        kend = k_lo;
      } else if (!cell_guard_ok(M, pb)) {
        int good = k_lo, bad = k_hi - 1;
        while (bad - good > 1) {
          const int mid = good + ((bad - good) >> 1);
          double pm[3];
          station_pos(o, r.d, dmul((double)mid, step), pm);
          if (cell_guard_ok(M, pm)) good = mid;
          else bad = mid;
        }
        kend = bad;
        bad_tail = true;
      }
    }
    const int n = r.hit ? max(kend - k_lo, 0) : 0;
    // even lane: value at its station's predecessor (the entry pair through the guard first)
    double prev = (double)CUDART_NAN_F;
    if (!parity && n > 0 && k_lo - 1 >= (int)r.kg_lo) prev = iso_entry_value(a, M, 0, r.d[0], r.d[1], r.d[2], k_lo, err);
    const unsigned trips = __reduce_max_sync(0xffffffffu, (unsigned)((n + 1) >> 1));
    double kd = (double)(k_lo + parity);
    int left = n - parity;          // this lane's remaining stations
    bool hit = false, done = false; // done: the ray (both lanes) hit
    double hit_kd = 0.0, hit_sa = 0.0, hit_sb = 0.0, last = (double)CUDART_NAN_F;
    for (unsigned j = 0; j < trips; ++j, left -= 2, kd = dadd(kd, 2.0)) {
      const bool valid = left > 0 && !done;
      double cur = (double)CUDART_NAN_F;
      if (valid) {
        double p[3];
        station_pos(o, r.d, dmul(kd, step), p);
        int ix, iy, iz;
        double fxd, fyd, fzd;
        cell_of_d(p, ix, iy, iz, fxd, fyd, fzd);
        const int x0 = ix - M.lo[0], y0 = iy - M.lo[1], z0 = iz - M.lo[2];
        float c[8];
        if constexpr (CONTIG) corners_contig(S, x0, y0, z0, c);
        else corners_guarded(S, x0, y0, z0, c);
        if constexpr (!CHAIN) {  // identity chain: float64 only inside the float32 error band
          cur = (double)lerp8(c, (float)fxd, (float)fyd, (float)fzd);
          float m = fabsf(c[0]);
#pragma unroll
          for (int i = 1; i < 8; ++i) m = fmaxf(m, fabsf(c[i]));
          if (!(fabs(dsub(cur, thr)) > (double)m * 0x1p-18)) cur = trilinear_d(c, fxd, fyd, fzd);
        } else if (s.iso_exact) {  // add / mul chain: always the reference's float64
          cur = run_chain_d(s, trilinear_d(c, fxd, fyd, fzd));
        } else {
          float v[4] = {lerp8(c, (float)fxd, (float)fyd, (float)fzd), 0.f, 0.f, 0.f};
          cur = (double)run_chain_fast<1>(s, v);
        }
        last = cur;
      }
      const double from_even = __shfl_up_sync(0xffffffffu, cur, 16);
      const double before = parity ? from_even : prev;
      const double sa = dsub(before, thr), sb = dsub(cur, thr);
      const bool h = valid && isfinite(sa) && ((sa < 0.0) != (sb < 0.0));
      const unsigned hits = __ballot_sync(0xffffffffu, h);
      const bool even_hit = (hits >> q) & 1u, pair_hit = ((hits >> q) | (hits >> (q + 16))) & 1u;
      if (h && !(parity && even_hit)) {  // the ray's first hit in station order
        hit = true;
        hit_kd = kd;
        hit_sa = sa;
        hit_sb = sb;
      }
      done = done || pair_hit;
      prev = __shfl_down_sync(0xffffffffu, cur, 16);  // even lane: the odd station before its next one
      if (__all_sync(0xffffffffu, done || left <= 2)) break;
    }
    // Forward exit pair (k_hi - 1, k_hi) when no backward pair hit: the
    // last station's value sits in the even lane when n is odd, else in the
    // odd lane (raycast.py:384-468; the next brick cannot reach back).
    const double odd_last = __shfl_down_sync(0xffffffffu, last, 16);
    double hit_tau = 0.0;
    bool hit_back = true;
    if (!parity && !done && n > 0 && kend == k_hi && k_hi < (int)r.kg_hi) {
      const int kl = k_hi - 1;
      const double sb = dsub((n & 1) ? last : odd_last, thr);
      double pl[3];
      station_pos(o, r.d, dmul((double)kl, step), pl);
      if (iso_exit_pair(a, M, 0, r.d[0], r.d[1], r.d[2], kl, pl[0], pl[1], pl[2], sb, &hit_tau, err)) {
        hit = true;
        hit_back = false;
        hit_kd = (double)kl;
      }
    }
    float4 c = make_float4(0.f, 0.f, 0.f, 0.f);
    if (hit) {  // both lanes of the warp that hold a hit shade together
      if (hit_back) {  // tau = s_prev / (s_prev - s_cur), raycast.py:434-437
        const double den = dsub(hit_sa, hit_sb);
        hit_tau = den != 0.0 ? ddiv(hit_sa, den) : 1.0;
      }
      double ph[3];
      station_pos(o, r.d, dmul(hit_kd, step), ph);
      c = iso_hit_color(a, M, 0, r.d[0], r.d[1], r.d[2], ph[0], ph[1], ph[2], hit_tau, hit_back ? -1.0 : 0.0, err);
    }
    // the even lane writes the pixel: its own hit, else the odd lane's
    const float4 co = shfl_down16(c);
    const double kd_odd = __shfl_down_sync(0xffffffffu, hit_kd, 16);
    const bool odd_hit = __shfl_down_sync(0xffffffffu, hit ? 1 : 0, 16) != 0;
    if (parity || !in_img) continue;
    if (!hit && odd_hit) {
      c = co;
      hit_kd = kd_odd;
      hit = true;
    }
    if (bad_tail && !hit && err) atomicAdd(err, 1u);  // marched into the bad tail
    const uint32_t stations = hit ? (uint32_t)((int)hit_kd - k_lo + 1) : (uint32_t)n;
    reinterpret_cast<float4*>(a.out_rgba)[pix] = c;
    if (a.out_stations) a.out_stations[pix] = stations;
    warp_stations += stations;
  }
  if (a.out_station_total) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) warp_stations += __shfl_xor_sync(0xffffffffu, warp_stations, off);
    if (lane == 0 && warp_stations) atomicAdd(a.out_station_total, warp_stations);
  }
}

// Pass 1 of march.cu launch_split.  Culls to the brick's screen rectangle
// when the caller asked for no per-pixel outputs (pass 2 reads the scratch
// only inside the same rectangle; the shaded-hit scratch is cleared first,
// pass 2 composites it behind every pixel it writes).  False when the probe
// does not apply; ISC_DISABLE_PAIRED_PROBE=1 routes the probe to the
// multi-source kernel (the round-2 default, A/B).
extern thread_local bool g_split_probe;
bool launch_iso_probe(const isc_render_args* a, cudaStream_t st, int* status) {
  static const bool off = getenv("ISC_DISABLE_PAIRED_PROBE") != nullptr;
  if (off || a->n_sources != 1 || !a->work_counter || a->ray_dirs || a->alpha_stop < 1.0 || !a->interpolation)
    return false;
  const isc_source& s = a->src[0];
  if (s.mode != ISC_ISO || s.feature_dim != 1 || s.dtype != ISC_F32 || !s.has_guard) return false;
  MultiField M;
  if (!build_multi_field(a, M)) return false;
  const bool contig = M.s[0].sx == 1;
  int tiles_x = (a->camera.width + 7) / 8, tiles_y = (a->camera.height + 1) / 2;
  int tile_x0 = 0, tile_y0 = 0;
  int rx0, ry0, rx1, ry1;
  static const bool no_cull = getenv("ISC_DISABLE_CULL") != nullptr;
  *status = ISC_OK;
  if (!no_cull && brick_screen_rect(a, rx0, ry0, rx1, ry1, g_split_probe)) {
    const cudaError_t e = rect_is_whole(a, rx0, ry0, rx1, ry1)
                              ? cudaSuccess
                              : cudaMemsetAsync(a->out_rgba, 0, (size_t)a->camera.width * a->camera.height * sizeof(float4), st);
    if (e != cudaSuccess) {
      *status = cuda_fail(e, "cudaMemsetAsync");
      return true;
    }
    tile_x0 = rx0 / 8;
    tile_y0 = ry0 / 2;
    tiles_x = rx1 > rx0 ? (rx1 + 7) / 8 - tile_x0 : 0;
    tiles_y = ry1 > ry0 ? (ry1 + 1) / 2 - tile_y0 : 0;
    if (tiles_x == 0 || tiles_y == 0) return true;
  }
  const int super_x = (tiles_x + 7) / 8, super_y = (tiles_y + 7) / 8;
  const int n_codes = super_x * super_y * 64;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  sms = cached_sm_count();
  auto kern = contig ? (s.n_steps ? iso_probe_kernel<true, true> : iso_probe_kernel<true, false>)
                     : (s.n_steps ? iso_probe_kernel<false, true> : iso_probe_kernel<false, false>);
  per_sm = contig ? (s.n_steps ? cached_blocks_per_sm<iso_probe_kernel<true, true>>(kThreads)
                               : cached_blocks_per_sm<iso_probe_kernel<true, false>>(kThreads))
                  : (s.n_steps ? cached_blocks_per_sm<iso_probe_kernel<false, true>>(kThreads)
                               : cached_blocks_per_sm<iso_probe_kernel<false, false>>(kThreads));
  int grid = sms * (per_sm > 0 ? per_sm : 1);
  const int need = (n_codes + (kThreads / 32) - 1) / (kThreads / 32);
  if (grid > need) grid = need > 0 ? need : 1;
  kern<<<grid, kThreads, 0, st>>>(*a, M, tiles_x, tiles_y, super_x, n_codes, tile_x0, tile_y0);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) *status = cuda_fail(e, "iso_probe_kernel");
  return true;
}

// Set by march.cu launch_split around its iso probe (same host thread).
thread_local bool g_split_probe = false;

template <int NS, int DIMS, bool CONTIG>
static int launch_multi_fast(const isc_render_args* a, const MultiField& M, cudaStream_t st) {
  static const int tw_log2 = getenv("ISC_MULTI_TILE_W") ? __builtin_ctz(atoi(getenv("ISC_MULTI_TILE_W"))) : 3;
  const int tw = 1 << tw_log2, th = 32 >> tw_log2;
  int tiles_x = (a->camera.width + tw - 1) / tw, tiles_y = (a->camera.height + th - 1) / th;
  int tile_x0 = 0, tile_y0 = 0;
  int rx0, ry0, rx1, ry1;
  static const bool no_cull = getenv("ISC_DISABLE_CULL") != nullptr;
  if (!no_cull && brick_screen_rect(a, rx0, ry0, rx1, ry1, g_split_probe)) {  // see march.cu launch_fast
    if (!rect_is_whole(a, rx0, ry0, rx1, ry1))
      ISC_CUDA_CHECK(cudaMemsetAsync(a->out_rgba, 0, (size_t)a->camera.width * a->camera.height * sizeof(float4), st));
    tile_x0 = rx0 / tw;
    tile_y0 = ry0 / th;
    tiles_x = rx1 > rx0 ? (rx1 + tw - 1) / tw - tile_x0 : 0;
    tiles_y = ry1 > ry0 ? (ry1 + th - 1) / th - tile_y0 : 0;
    if (tiles_x == 0 || tiles_y == 0) return ISC_OK;
  }
  const int super_x = (tiles_x + 7) / 8, super_y = (tiles_y + 7) / 8;
  const int n_codes = super_x * super_y * 64;
  int dev = 0, sms = 148, per_sm = 1;
  ISC_CUDA_CHECK(cudaGetDevice(&dev));
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, march_multi_fast_kernel<NS, DIMS, CONTIG>,
                                                kMultiFastThreads, 0);
  int grid = sms * (per_sm > 0 ? per_sm : 1);
  const int need = (n_codes + (kMultiFastThreads / 32) - 1) / (kMultiFastThreads / 32);
  if (grid > need) grid = need > 0 ? need : 1;
  march_multi_fast_kernel<NS, DIMS, CONTIG><<<grid, kMultiFastThreads, 0, st>>>(*a, M, tiles_x, tiles_y, super_x, n_codes, tile_x0,
                                                                tile_y0, tw_log2);
  ISC_CUDA_CHECK(cudaGetLastError());
  return ISC_OK;
}

// Dispatch of the specialised kernel: 1-2 sources of 1 or 3 components.
static bool launch_multi_fast_dims(const isc_render_args* a, const MultiField& M, cudaStream_t st, int* status) {
  const int ns = a->n_sources;
  int dims = 0, scale = 1;
  for (int si = 0; si < ns; ++si, scale *= 5) dims += a->src[si].feature_dim * scale;
  // C-contiguous (z, y, x[, c]) sources get the immediate-offset gather
  bool contig = getenv("ISC_DISABLE_CONTIG") == nullptr;
  for (int si = 0; si < ns; ++si)
    contig &= M.s[si].sx == M.s[si].dim && (M.s[si].dim == 1 || M.s[si].sc == 1);
  switch (ns * 1000 + dims) {
    case 1001: *status = contig ? launch_multi_fast<1, 1, true>(a, M, st) : launch_multi_fast<1, 1, false>(a, M, st); return true;
    case 1003: *status = contig ? launch_multi_fast<1, 3, true>(a, M, st) : launch_multi_fast<1, 3, false>(a, M, st); return true;
    case 2006:
      *status = contig ? launch_multi_fast<2, 1 + 5 * 1, true>(a, M, st) : launch_multi_fast<2, 1 + 5 * 1, false>(a, M, st);
      return true;
    case 2016:
      *status = contig ? launch_multi_fast<2, 1 + 5 * 3, true>(a, M, st) : launch_multi_fast<2, 1 + 5 * 3, false>(a, M, st);
      return true;
    case 2008:
      *status = contig ? launch_multi_fast<2, 3 + 5 * 1, true>(a, M, st) : launch_multi_fast<2, 3 + 5 * 1, false>(a, M, st);
      return true;
    case 2018:
      *status = contig ? launch_multi_fast<2, 3 + 5 * 3, true>(a, M, st) : launch_multi_fast<2, 3 + 5 * 3, false>(a, M, st);
      return true;
    default: return false;
  }
}

template <int NS, bool INTERP, int MINB>
static int launch_multi_m(const isc_render_args* a, const MultiField& M, cudaStream_t st) {
  const int tiles_x = (a->camera.width + 7) / 8, tiles_y = (a->camera.height + 3) / 4;
  const int super_x = (tiles_x + 7) / 8, super_y = (tiles_y + 7) / 8;
  const int n_codes = super_x * super_y * 64;
  int dev = 0, sms = 148, per_sm = 1;
  ISC_CUDA_CHECK(cudaGetDevice(&dev));
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, march_multi_kernel<NS, INTERP, MINB>, kThreads, 0);
  int grid = sms * (per_sm > 0 ? per_sm : 1);
  const int need = (n_codes + (kThreads / 32) - 1) / (kThreads / 32);
  if (grid > need) grid = need > 0 ? need : 1;
  march_multi_kernel<NS, INTERP, MINB><<<grid, kThreads, 0, st>>>(*a, M, tiles_x, tiles_y, super_x, n_codes);
  ISC_CUDA_CHECK(cudaGetLastError());
  return ISC_OK;
}

template <int NS, bool INTERP>
static int launch_multi_t(const isc_render_args* a, const MultiField& M, cudaStream_t st) {
  // 2 CTAs/SM (<= 128 registers): measured best; 3-4 CTAs spill (C3: 192.6 / 184.7 vs 198.7 fps)
  return launch_multi_m<NS, INTERP, 2>(a, M, st);
}

static bool build_multi_field(const isc_render_args* a, MultiField& M);

// Returns true (and the launch status in *status) when the multi kernel
// handles this render: 1..4 float32 sources, 32-bit offsets, work counter.
bool launch_multi(const isc_render_args* a, cudaStream_t st, int* status) {
  const int ns = a->n_sources;
  if (ns < 1 || ns > 4 || !a->work_counter) return false;
  MultiField M;
  if (!build_multi_field(a, M)) return false;
  const bool interp = a->interpolation != 0;
  static const bool no_multi_fast = getenv("ISC_DISABLE_MULTI_FAST") != nullptr;
  bool all_guarded = interp;
  for (int si = 0; si < ns; ++si) all_guarded = all_guarded && M.s[si].guarded;
  if (!no_multi_fast && all_guarded && launch_multi_fast_dims(a, M, st, status)) return true;
  switch (ns * 2 + (interp ? 1 : 0)) {
    case 2: *status = launch_multi_t<1, false>(a, M, st); break;
    case 3: *status = launch_multi_t<1, true>(a, M, st); break;
    case 4: *status = launch_multi_t<2, false>(a, M, st); break;
    case 5: *status = launch_multi_t<2, true>(a, M, st); break;
    case 6: *status = launch_multi_t<3, false>(a, M, st); break;
    case 7: *status = launch_multi_t<3, true>(a, M, st); break;
    case 8: *status = launch_multi_t<4, false>(a, M, st); break;
    default: *status = launch_multi_t<4, true>(a, M, st); break;
  }
  return true;
}

// MultiField of the render's sources; false when a source is not float32 or
// its offsets do not fit 32 bits.
static bool build_multi_field(const isc_render_args* a, MultiField& M) {
  const int ns = a->n_sources;
  const int g = a->guard_width;
  for (int i = 0; i < 3; ++i) M.lo[i] = a->brick_offset[i] - g;
  M.g = g;
  const bool interp = a->interpolation != 0;
  for (int si = 0; si < ns; ++si) {
    const isc_source& s = a->src[si];
    if (s.dtype != ISC_F32) return false;
    long long maxoff = (s.feature_dim - 1) * s.stride[3];
    for (int i = 0; i < 3; ++i) {
      if (s.stride[i] < 0 || s.stride[i] > INT32_MAX || s.stride[3] < 0 || s.stride[3] > INT32_MAX) return false;
      maxoff += (a->brick_size[2 - i] + 2LL * g - 1) * s.stride[i];
    }
    if (maxoff >= INT32_MAX) return false;
    MultiSrc& S = M.s[si];
    S.f = reinterpret_cast<const float*>(s.data);
    S.sz = (int)s.stride[0];
    S.sy = (int)s.stride[1];
    S.sx = (int)s.stride[2];
    S.sc = (int)s.stride[3];
    S.dim = s.feature_dim;
    S.guarded = (s.has_guard && interp) ? 1 : 0;
    for (int i = 0; i < 3; ++i) S.hi[i] = S.guarded ? a->brick_size[i] + 2 * g - 2 : a->brick_size[i] - 1;
  }
  return true;
}

}  // namespace isc
