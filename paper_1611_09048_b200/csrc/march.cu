// K1-K3: ray setup + front-to-back march + iso-surface detection for one
// brick.  Replaces raycast.render_local (raycast.py:492-541) together with
// march_rays (291-381), _iso_detect (384-468) and gradient_normals (210-242).
//
// Kernels and dispatch (isc_render_local):
//   march_fast_kernel   one volume-mode source (f32 scalar or float3, f64 /
//                       f16 / bf16 scalar): persistent warps pull tiles of
//                       8x2 rays (or 4x4, launch_tuner.cuh), lanes l and
//                       l + 16 march the even / odd stations of one ray;
//                       guard contract proven per ray; optional analytic
//                       single-ramp classification and early termination
//   march_multi_*       1-4 float32 sources incl. iso surfaces (march_multi.cu)
//   march_kernel        generic fallback: any dtype, up to 8 sources, static
//                       16x16-pixel CTAs (8x4 rays per warp)
// Positions, cell indices and fractions are float64 (bit-identical cell
// selection to the reference); field values, chains, classification and the
// over-accumulation are float32.
#include <math_constants.h>

#include <cstdlib>

#include "common.cuh"
#include "launch_tuner.cuh"
#include <mutex>
#include <type_traits>

#include "march_common.cuh"
#include "raysetup.cuh"
#include "sample.cuh"

namespace isc {

bool launch_multi(const isc_render_args* a, cudaStream_t st, int* status);  // march_multi.cu
bool launch_iso_probe(const isc_render_args* a, cudaStream_t st, int* status);  // march_multi.cu
extern thread_local bool g_split_probe;                                           // march_multi.cu

__device__ __forceinline__ void tile_pixel(int& px, int& py) {
  const int t = threadIdx.x, w = t >> 5, l = t & 31;
  px = blockIdx.x * kTile + (w & 1) * 8 + (l & 7);
  py = blockIdx.y * kTile + (w >> 1) * 4 + (l >> 3);
}

__device__ __forceinline__ Brick make_brick(const isc_render_args& a) {
  Brick b;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    b.size[i] = a.brick_size[i];
    b.offset[i] = (double)a.brick_offset[i];
  }
  b.guard = a.guard_width;
  return b;
}

template <bool F32>
__device__ __forceinline__ float scalar_at(const isc_source& s, const Brick& b, const double p[3], bool interp,
                                           uint32_t* err) {
  double l[3] = {dsub(p[0], b.offset[0]), dsub(p[1], b.offset[1]), dsub(p[2], b.offset[2])};
  float v[4] = {0.f, 0.f, 0.f, 0.f};
  sample_local<F32, 0>(s, b, l, interp, v, err);
  return run_chain(s, v, s.feature_dim);
}

// raycast.py:270-278: trilinear gathers at p stay within the guard halo.
__device__ __forceinline__ bool reachable(const double off[3], const double size[3], int g, const double p[3]) {
  bool ok = true;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double lo = dsub(off[i], (double)g);
    const double hi = dsub(dadd(dadd(off[i], size[i]), (double)g), 1.0);
    ok &= (p[i] >= lo) && (p[i] < hi);
  }
  return ok;
}

// Central-difference normal of the chained scalar (raycast.py:210-242).
__device__ float3 iso_normal(const isc_source& s, const Brick& b, const double p[3], const double d[3],
                             bool interp, uint32_t* err) {
  const int g = (s.has_guard && interp) ? b.guard : 0;
  float grad[3];
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    const double lo = dsub(b.offset[ax], (double)g);
    const double hi = dsub(dsub(dadd(dadd(lo, (double)b.size[ax]), (double)(2 * g)), 1.0), 1e-9);
    double pp[3] = {p[0], p[1], p[2]}, pm[3] = {p[0], p[1], p[2]};
    pp[ax] = dmin(dmax(dadd(p[ax], 1.0), lo), hi);
    pm[ax] = dmin(dmax(dsub(p[ax], 1.0), lo), hi);
    double span = dsub(pp[ax], pm[ax]);
    if (span == 0.0) span = 1.0;
    const float sp = scalar_at<false>(s, b, pp, interp, err);
    const float sm = scalar_at<false>(s, b, pm, interp, err);
    grad[ax] = (float)((double)(sp - sm) / span);
  }
  const float mag = sqrtf((grad[0] * grad[0] + grad[1] * grad[1]) + grad[2] * grad[2]);
  if (mag < 1e-12f) {
    const double dm = sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
    return make_float3((float)(-d[0] / dm), (float)(-d[1] / dm), (float)(-d[2] / dm));
  }
  return make_float3(grad[0] / mag, grad[1] / mag, grad[2] / mag);
}

// Generic fallback: any dtype (f32/f64/f16/bf16), up to ISC_MAX_SOURCES
// sources, 64-bit element offsets; static 16x16 tiles.
template <bool INTERP>
__global__ void __launch_bounds__(kThreads) march_kernel(const __grid_constant__ isc_render_args a) {
  extern __shared__ float lut_s[];  // planar tables, kLutWords per source
  lut_fill_sources(lut_s, a, a.n_sources);
  __syncthreads();

  int px, py;
  tile_pixel(px, py);
  if (px >= a.camera.width || py >= a.camera.height) return;
  const long long pix = (long long)py * a.camera.width + px;

  Ray r;
  setup_ray(a, px, py, r);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  uint32_t stations = 0;

  if (r.hit) {
    const Brick b = make_brick(a);
    const double* o = a.camera.origin;
    const bool gate_alpha = a.alpha_stop < 1.0;
  const float stop_f = __double2float_ru(a.alpha_stop);  // w >= stop_f <=> (double)w >= alpha_stop
    uint32_t* err = a.error_word;

    int hit_si = -1;                     // first iso hit, shaded after the loop
    double hit_p[3] = {0.0, 0.0, 0.0};
    float4 hit_front = make_float4(0.f, 0.f, 0.f, 0.f);
    {
      const int ns = a.n_sources;
      float prev[ISC_MAX_SOURCES];
#pragma unroll
      for (int i = 0; i < ISC_MAX_SOURCES; ++i) prev[i] = CUDART_NAN_F;
      double bsz[3], vb[3];
      const int* dec = a.decomposition;
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        bsz[i] = (double)b.size[i];
        vb[i] = ddiv((double)a.volume_size[i], (double)dec[i]);  // raycast.py:283-285
      }
      for (long long k = r.k_lo; k < r.k_hi; ++k) {
        ++stations;
        double p[3];
        station_pos(o, r.d, dmul((double)k, a.step), p);
        float4 st = make_float4(0.f, 0.f, 0.f, 0.f);
        bool stop = false;
        for (int si = 0; si < ns; ++si) {
          const isc_source& s = a.src[si];
          const float cur = scalar_at<false>(s, b, p, INTERP, err);
          const float* lut = lut_s + si * kLutWords;
          const float inv = 1.0f / (s.range_hi - s.range_lo);
          if (s.mode != ISC_ISO) {
            st = over4(st, premultiply(classify(lut, s.range_lo, inv, cur)));
            continue;
          }
          // ---- iso: raycast.py:384-468 ----
          const float thr = s.iso_threshold;
          const bool guarded_interp = s.has_guard && INTERP;
          const bool exact = guarded_interp && !a.no_layout;
          float before = prev[si];
          if (k == r.k_lo && k - 1 >= r.kg_lo) {  // entry pair through the guard
            double pq[3];
            station_pos(o, r.d, dmul((double)(k - 1), a.step), pq);
            if (guarded_interp && a.no_layout) {
              // no layout knowledge: clamp into reach (raycast.py:404-409)
#pragma unroll
              for (int i = 0; i < 3; ++i)
                pq[i] = dmin(dmax(pq[i], b.offset[i] - b.guard), b.offset[i] + bsz[i] + b.guard - 1 - 1e-9);
            }
            before = (!exact || reachable(b.offset, bsz, b.guard, pq)) ? scalar_at<false>(s, b, pq, INTERP, err)
                                                                     : CUDART_NAN_F;
          }
          const float sa = before - thr, sb = cur - thr;
          bool hit = isfinite(sa) && ((sa < 0.f) != (sb < 0.f));
          double tau = 0.0, back = 0.0;
          if (hit) {
            const float den = sa - sb;
            tau = den != 0.f ? (double)(sa / den) : 1.0;
            back = -1.0;
          }
          if (exact && !hit && k == r.k_hi - 1 && k + 1 < r.kg_hi) {  // exit pair checked forward
            double pn[3];
            station_pos(o, r.d, dmul((double)(k + 1), a.step), pn);
            double noff[3];
#pragma unroll
            for (int i = 0; i < 3; ++i) {
              double c = floor(ddiv(pn[i], vb[i]));
              c = dmin(dmax(c, 0.0), (double)(dec[i] - 1));
              noff[i] = dmul(c, vb[i]);
            }
            if (reachable(b.offset, bsz, b.guard, pn) && !reachable(noff, vb, b.guard, p)) {
              const float sn = scalar_at<false>(s, b, pn, INTERP, err) - thr;
              if ((sb < 0.f) != (sn < 0.f)) {
                const float den = sb - sn;
                tau = den != 0.f ? (double)(sb / den) : 1.0;
                back = 0.0;
                hit = true;
              }
            }
          }
          prev[si] = cur;
          if (hit && !stop) {  // later sources of the station sit behind the opaque hit
            const double t = dmul(dadd(tau, back), a.step);
#pragma unroll
            for (int i = 0; i < 3; ++i) hit_p[i] = dadd(p[i], dmul(t, r.d[i]));
            hit_si = si;
            hit_front = st;
            stop = true;
          }
        }
        if (stop) break;
        acc = over4(acc, st);
        if (gate_alpha && acc.w >= stop_f) break;
      }
    }
    if (hit_si >= 0) {  // shaded after the loop: all hitting lanes of the warp together
      const isc_source& s = a.src[hit_si];
      const double d[3] = {r.d[0], r.d[1], r.d[2]};
      const float3 n = iso_normal(s, b, hit_p, d, INTERP, err);
      const float shade = fabsf(n.x * (float)d[0] + n.y * (float)d[1] + n.z * (float)d[2]);
      const float4 base = classify(lut_s + hit_si * kLutWords, s.range_lo, 1.0f / (s.range_hi - s.range_lo),
                                   s.iso_threshold);
      acc = over4(acc, over4(hit_front, make_float4(base.x * shade, base.y * shade, base.z * shade, 1.0f)));
    }
  }

  reinterpret_cast<float4*>(a.out_rgba)[pix] = acc;
  if (a.out_stations) a.out_stations[pix] = stations;
  if (a.out_station_total) {
    const unsigned int warp_total = __reduce_add_sync(__activemask(), stations);
    if ((threadIdx.x & 31) == (__ffs(__activemask()) - 1) && warp_total)
      atomicAdd(a.out_station_total, (unsigned long long)warp_total);
  }
  if (a.out_hit) a.out_hit[pix] = r.hit ? 1 : 0;
  if (a.out_t) {
    a.out_t[2 * pix] = r.t_in;
    a.out_t[2 * pix + 1] = r.t_out;
  }
  if (a.out_krange) {
    reinterpret_cast<int4*>(a.out_krange)[pix] =
        make_int4((int)r.k_lo, (int)r.k_hi, (int)r.kg_lo, (int)r.kg_hi);
  }
}

// ---------------------------------------------------------------------------
// Fast path: one active float32 scalar source in volume mode (the C1/C2/C4/C5
// workloads).  Persistent warps pull 8x4-pixel tiles from an atomic counter
// (dynamic load balance: ray lengths vary per tile), tiles ordered as 8x8
// Morton blocks inside row-major super-tiles so concurrently marching warps
// sit on neighbouring rays and share L1/L2 lines.  Element offsets are 32-bit
// (the host checks the field fits), the guard contract is checked once on the
// base cell, and two stations are issued per iteration so each warp keeps 16
// independent gathers in flight.
// PAIRED: a warp is 16 rays (an 8x2 pixel tile) x 2 station parities; lanes l
// and l+16 march the even / odd stations of the same ray half a cell apart, so
// one gather request covers 32 samples within an ~8x2-pixel footprint (fewer
// cache lines per request than an 8x4 tile).  Each station pair is merged in
// order with one shuffle exchange: pair = s_even over s_odd, acc = acc over
// pair -- the same over-sequence as the reference's per-station loop.
// ET (early termination, alpha_stop < 1): the even lane composites station by
// station with the stop test after each.
#ifndef ISC_FAST_MINB
#define ISC_FAST_MINB 4  // <= 64 registers: 4 CTAs (32 warps) per SM
#endif
// LINE: 0 = transfer function read from the shared-memory LUT, L >= 1 =
// analytic piecewise-linear form with L-1 kinks (classify_line_premul<L>).
// AOS3: float3 source in the standard interleaved layout (fast_gather_aos3).
// LANES (paired only): lanes per ray -- 2 (the paired march: 16 rays x 2
// station parities) or 4 for small frames (8 rays x 4 parities, merged by a
// two-level shuffle tree): with fewer tiles than resident warps the launch
// lasts as long as its longest ray, and 4 lanes halve that serial path.
// float3 sources: 3 CTAs per SM (<= 85 registers, no spills) -- C3's split
// volume pass 1.518 -> 1.493 ms per frame; a float3-only volume render of the
// same field 4.66 -> 4.71 ms (measured A/B)
#ifndef ISC_FAST_MINB3
#define ISC_FAST_MINB3 3
#endif
template <bool INTERP, bool GUARDED, bool PAIRED, int LINE = 0, int DIM = 1, bool ET = false,
          typename T = float, bool AOS3 = false, int LANES = 2>
__global__ void __launch_bounds__(kThreads, DIM == 3 ? ISC_FAST_MINB3 : ISC_FAST_MINB) march_fast_kernel(const __grid_constant__ isc_render_args a,
                                                              const FastField F, int tiles_x, int tiles_y,
                                                              int super_x, int n_codes, int row_order,
                                                              int tw_log2, int tile_x0, int tile_y0) {
  __shared__ float lut_s[kLutWords];
  if (LINE == 0 || !PAIRED) {
    lut_fill(lut_s, reinterpret_cast<const float4*>(a.src[0].lut));
    __syncthreads();
  }

  const int lane = threadIdx.x & 31;
  const isc_source& s = a.src[0];
  const float lo = s.range_lo, inv = 1.0f / (s.range_hi - s.range_lo);
  const bool gate_alpha = a.alpha_stop < 1.0;
  // smallest float f with (double)f >= alpha_stop: for a float w,
  // w >= stop_f  <=>  (double)w >= alpha_stop (NaN false in both)
  const float stop_f = __double2float_ru(a.alpha_stop);
  const double* o = a.camera.origin;
  const double step = a.step;
  uint32_t* err = a.error_word;
  unsigned long long warp_stations = 0;
  const int tw = 1 << tw_log2;
  static_assert(LANES == 2 || (LANES == 4 && PAIRED && !ET), "4 lanes per ray: paired, no early termination");
  constexpr int kRays = PAIRED ? 32 / LANES : 32;  // rays per warp
  const int th = kRays >> tw_log2;
  const int q = lane & (kRays - 1);
  const int parity = PAIRED ? lane / kRays : 0;

  for (;;) {
    int t = 0;
    if (lane == 0) t = (int)atomicAdd(a.work_counter, 1u);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= n_codes) break;
    int tx, ty;
    if (row_order) {
      tx = t % tiles_x;
      ty = t / tiles_x;
    } else {
      const int sblk = t >> 6, w = t & 63;
      tx = (sblk % super_x) * 8 + morton3(w, 0);
      ty = (sblk / super_x) * 8 + morton3(w, 1);
    }
    if (tx >= tiles_x || ty >= tiles_y) continue;
    tx += tile_x0;  // tiles of the brick's screen rectangle only
    ty += tile_y0;
    const int px = tx * tw + (q & (tw - 1)), py = ty * th + (q >> tw_log2);
    const bool in_img = px < a.camera.width && py < a.camera.height;
    if (!PAIRED && !in_img) continue;

    Ray r;
    if (in_img) {
      setup_ray(a, px, py, r);
    } else {
      r.hit = false;
      r.k_lo = r.k_hi = 0;
    }
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    uint32_t stations = 0;
    if constexpr (PAIRED) {
      // Every lane runs the warp's largest trip count so the pair shuffles use
      // the full mask (a per-lane mask costs a MATCH.ANY convergence check per
      // shuffle).  Lanes whose ray is finished contribute transparent samples:
      // over(acc, 0) == acc exactly.
      long long k_hi = r.k_hi;
      if (F.stop_counts && r.hit && in_img) {  // split render: stop before the probe's iso hit
        const long long q_pix = (long long)py * a.camera.width + px;
        const long long marched = (long long)F.stop_counts[q_pix] - (F.stop_shade[q_pix].w != 0.f ? 1 : 0);
        k_hi = min(k_hi, r.k_lo + max(marched, 0LL));
      }
      const long long n = r.hit ? max(k_hi - r.k_lo, 0LL) : 0;
      long long nm = n;  // stations this lane pair marches
      bool bad_tail = false;
      // Guard contract checked once per ray: every axis of the station
      // position o + (k*step)*d is a composition of monotone roundings, so
      // each cell index is monotone in k and the stations whose gathers
      // honour the halo form one interval.  Without early termination every
      // station is gathered: a bad first or last station is the reference's
      // GuardContractError (fields.py:230-238) and the ray is not marched.
      // With early termination the ray may stop before a bad tail: march up
      // to the last good station (binary search) and report the error only
      // if the ray gets there.
      if (GUARDED && n > 0) {
        double pa[3], pb[3];
        station_pos(o, r.d, dmul((double)r.k_lo, step), pa);
        station_pos(o, r.d, dmul((double)(k_hi - 1), step), pb);
        if (!guard_ok(F, pa)) {
          if (err && !parity) atomicAdd(err, 1u);
          nm = 0;
        } else if (!guard_ok(F, pb)) {
          if constexpr (ET) {
            long long good = r.k_lo, bad = k_hi - 1;
            while (bad - good > 1) {
              const long long mid = good + ((bad - good) >> 1);
              double pm[3];
              station_pos(o, r.d, dmul((double)mid, step), pm);
              if (guard_ok(F, pm)) good = mid;
              else bad = mid;
            }
            nm = bad - r.k_lo;
            bad_tail = true;
          } else {
            if (err && !parity) atomicAdd(err, 1u);
            nm = 0;
          }
        }
      }
      constexpr bool kCheck = false;
      const unsigned pairs = (unsigned)((nm + LANES - 1) / LANES);
      const unsigned trips = __reduce_max_sync(0xffffffffu, pairs);
      // station index as an exact float64 integer (k < 2^53) stepped by
      // LANES: no int64 -> float64 conversion per sample; `left` counts this
      // lane's remaining stations.
      double kd = (double)(r.k_lo + parity);
      int left = (int)nm - parity;
      bool done = false;        // ET: the pair's ray reached alpha_stop
      uint32_t marched = 0;     // ET: stations composited (even lane)
      for (unsigned j = 0; j < trips; ++j, left -= LANES, kd = dadd(kd, (double)LANES)) {
        float4 c = make_float4(0.f, 0.f, 0.f, 0.f);
        if (left > 0 && !(ET && done)) {
          double p0[3];
          station_pos(o, r.d, dmul(kd, step), p0);
          float s0;
          if constexpr (DIM == 1) {
            const float v0 = fast_sample<INTERP, GUARDED, kCheck, T>(F, p0, err);
            float vv[4] = {v0, 0.f, 0.f, 0.f};
            s0 = s.n_steps ? run_chain(s, vv, 1) : v0;
          } else {
            static_assert(INTERP && GUARDED && PAIRED, "vector sources: guarded trilinear paired path only");
            float vv[4] = {0.f, 0.f, 0.f, 0.f};
            if constexpr (AOS3) fast_gather_aos3(F, p0, vv);
            else fast_gather<DIM, T>(F, p0, vv);
            s0 = run_chain_fast<DIM>(s, vv);
          }
          if constexpr (LINE > 0) c = classify_line_premul<LINE>(s, lo, inv, s0);
          else c = premultiply(classify(lut_s, lo, inv, s0));
        }
        // Only the even lane's accumulator is used (it writes the pixel), so
        // it takes the odd lane's sample with a shuffle-down and composites
        // even-over-odd; the odd lane's accumulator is dead.
        if constexpr (LANES == 4) {
          // stations k..k+3 sit in parities 0..3 (lanes q, q+8, q+16, q+24):
          // (s0 over s1) over (s2 over s3), then onto the pixel
          c = over4(c, shfl_down_n(c, 8));
          c = over4(c, shfl_down_n(c, 16));
          acc = over4(acc, c);
          continue;
        }
        const float4 odd = shfl_down16(c);
        if constexpr (!ET) {
          acc = over4(acc, over4(c, odd));
        } else {
          // early termination (raycast.py:377-380): station by station, the
          // stop test after each one, exactly as the reference's loop --
          // branch-free (every lane evaluates it; only the even lane's
          // accumulator is used), the float64 test (double)w >= alpha_stop as
          // the equivalent float32 test w >= stop_f, and the pair's state
          // passed to the odd lane by ballot (no data-pipe shuffle)
          const float4 a1 = over4(acc, c), a2 = over4(a1, odd);
          const bool s1 = left > 0 && !done;
          const bool d1 = s1 && a1.w >= stop_f;
          const bool s2 = s1 && !d1 && left > 1;
          acc = s2 ? a2 : (s1 ? a1 : acc);
          marched += (uint32_t)s1 + (uint32_t)s2;
          done = done || d1 || (s2 && a2.w >= stop_f);
          const unsigned dm = __ballot_sync(0xffffffffu, done);
          done = (dm >> q) & 1u;  // the odd lane follows its pair
          if (__ballot_sync(0xffffffffu, !(done || left <= 2)) == 0u) break;
        }
      }
      if constexpr (ET) {
        if (bad_tail && !done && err && !parity) atomicAdd(err, 1u);  // marched into the bad tail
        stations = parity ? 0u : marched;
      } else {
        stations = parity ? 0u : (uint32_t)n;
      }
      if (parity || !in_img) {
        warp_stations += stations;
        continue;
      }
    } else if (r.hit) {
      long long k = r.k_lo;
      if (!gate_alpha) {
        for (; k + 1 < r.k_hi; k += 2) {  // two independent stations in flight
          double p0[3], p1[3];
          station_pos(o, r.d, dmul((double)k, step), p0);
          station_pos(o, r.d, dmul((double)(k + 1), step), p1);
          const float v0 = fast_sample<INTERP, GUARDED>(F, p0, err);
          const float v1 = fast_sample<INTERP, GUARDED>(F, p1, err);
          float w0[4] = {v0, 0.f, 0.f, 0.f}, w1[4] = {v1, 0.f, 0.f, 0.f};
          const float s0 = s.n_steps ? run_chain(s, w0, 1) : v0;
          const float s1 = s.n_steps ? run_chain(s, w1, 1) : v1;
          acc = over4(acc, premultiply(classify(lut_s, lo, inv, s0)));
          acc = over4(acc, premultiply(classify(lut_s, lo, inv, s1)));
        }
        stations = (uint32_t)(r.k_hi - r.k_lo);
      }
      for (; k < r.k_hi; ++k) {
        double p0[3];
        station_pos(o, r.d, dmul((double)k, step), p0);
        const float v0 = fast_sample<INTERP, GUARDED>(F, p0, err);
        float vv[4] = {v0, 0.f, 0.f, 0.f};
        const float s0 = s.n_steps ? run_chain(s, vv, 1) : v0;
        acc = over4(acc, premultiply(classify(lut_s, lo, inv, s0)));
        if (gate_alpha) {
          ++stations;
          if (acc.w >= stop_f) break;
        }
      }
    }
    const long long pix = (long long)py * a.camera.width + px;
    if (F.stop_shade) acc = over4(acc, F.stop_shade[pix]);  // the iso hit behind the marched stations
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
    for (int off = 16; off > 0; off >>= 1) warp_stations += __shfl_xor_sync(0xffffffffu, warp_stations, off);
    if (lane == 0 && warp_stations) atomicAdd(a.out_station_total, warp_stations);
  }
}

// raycast.gradient_normals (raycast.py:210-242) at caller positions.
__global__ void gradient_kernel(const __grid_constant__ isc_render_args a, const double* __restrict__ pos,
                                const double* __restrict__ view, long long n, float* __restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Brick b = make_brick(a);
  const double p[3] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
  const double d[3] = {view[3 * i], view[3 * i + 1], view[3 * i + 2]};
  const float3 nn = iso_normal(a.src[0], b, p, d, a.interpolation != 0, a.error_word);
  out[3 * i] = nn.x;
  out[3 * i + 1] = nn.y;
  out[3 * i + 2] = nn.z;
}

__global__ void __launch_bounds__(kThreads) ray_setup_kernel(const __grid_constant__ isc_render_args a) {
  int px, py;
  tile_pixel(px, py);
  if (px >= a.camera.width || py >= a.camera.height) return;
  const long long pix = (long long)py * a.camera.width + px;
  Ray r;
  setup_ray(a, px, py, r);
  if (a.out_hit) a.out_hit[pix] = r.hit ? 1 : 0;
  if (a.out_t) {
    a.out_t[2 * pix] = r.t_in;
    a.out_t[2 * pix + 1] = r.t_out;
  }
  if (a.out_krange)
    reinterpret_cast<int4*>(a.out_krange)[pix] =
        make_int4((int)r.k_lo, (int)r.k_hi, (int)r.kg_lo, (int)r.kg_hi);
}

static int validate(const isc_render_args* a, bool need_rgba) {
  if (!a) return fail(ISC_E_VALUE, "null render args");
  const isc_camera& c = a->camera;
  if (c.width <= 0 || c.height <= 0) return fail(ISC_E_SCENE, "image size must be positive");
  if (!(a->step > 0.0)) return fail(ISC_E_SCENE, "step_length must be positive");
  if (a->n_sources < 0 || a->n_sources > ISC_MAX_SOURCES) return fail(ISC_E_VALUE, "too many active sources");
  if (a->n_clip < 0 || a->n_clip > ISC_MAX_CLIP_PLANES) return fail(ISC_E_SCENE, "too many clip planes");
  if (a->guard_width < 0) return fail(ISC_E_FIELD, "guard width must be non-negative");
  for (int i = 0; i < 3; ++i) {
    if (a->brick_size[i] <= 0 || a->volume_size[i] <= 0 || a->decomposition[i] <= 0)
      return fail(ISC_E_FIELD, "brick/volume size and decomposition must be positive");
  }
  if (need_rgba && !a->out_rgba) return fail(ISC_E_VALUE, "out_rgba is required");
  for (int s = 0; s < a->n_sources; ++s) {
    const isc_source& src = a->src[s];
    if (!src.data || !src.lut) return fail(ISC_E_FIELD, "source data / lut pointer is null");
    if (src.feature_dim < 1 || src.feature_dim > 4) return fail(ISC_E_FIELD, "feature_dim must be 1..4");
    if (src.n_steps < 0 || src.n_steps > ISC_MAX_CHAIN) return fail(ISC_E_CHAIN, "chain too long");
    if (src.dtype < ISC_F32 || src.dtype > ISC_BF16) return fail(ISC_E_FIELD, "unsupported dtype");
    if (!(src.range_lo < src.range_hi)) return fail(ISC_E_SCENE, "value range must satisfy min < max");
    int dim = src.feature_dim;
    uint32_t packed = 0;
    for (int i = 0; i < src.n_steps; ++i) {
      if (src.steps[i].in_dim != dim) return fail(ISC_E_CHAIN, "chain step dimension mismatch");
      const int op = src.steps[i].op;
      if (op < ISC_OP_ADD || op > ISC_OP_MAX) return fail(ISC_E_CHAIN, "unknown chain opcode");
      if (op == ISC_OP_LENGTH || op == ISC_OP_SUM) dim = 1;
      packed |= (uint32_t)op << (4 * i);
    }
    if (src.step_ops != packed) return fail(ISC_E_CHAIN, "step_ops does not pack steps[].op (4 bits per step)");
  }
  return ISC_OK;
}

}  // namespace isc

using namespace isc;

static bool fast_eligible(const isc_render_args* a, FastField& F) {
  if (a->n_sources != 1 || !a->work_counter) return false;
  const isc_source& s = a->src[0];
  if ((s.feature_dim != 1 && s.feature_dim != 3) || s.mode != ISC_VOLUME) return false;
  // other element types: scalar, guarded trilinear (paired path)
  if (s.dtype != ISC_F32 && !(s.feature_dim == 1 && a->interpolation && s.has_guard)) return false;
  // vector sources: guarded trilinear (paired path)
  if (s.feature_dim == 3 && !(a->interpolation && s.has_guard)) return false;
  const int g = a->guard_width;
  long long ext[3];
  for (int i = 0; i < 3; ++i) ext[i] = a->brick_size[i] + 2LL * g;
  // every index the kernel forms must fit in int32
  long long maxoff = 0;
  for (int i = 0; i < 3; ++i) {
    if (s.stride[i] < 0 || s.stride[i] > INT32_MAX) return false;
    maxoff += (ext[2 - i] - 1) * s.stride[i];
  }
  if (s.stride[3] < 0 || s.stride[3] > INT32_MAX) return false;
  maxoff += (s.feature_dim - 1) * s.stride[3];
  if (maxoff + s.stride[0] + s.stride[1] + s.stride[2] >= INT32_MAX) return false;
  F.f = s.data;
  F.stop_counts = nullptr;
  F.stop_shade = nullptr;
  F.sz = (int)s.stride[0];
  F.sy = (int)s.stride[1];
  F.sx = (int)s.stride[2];
  F.sc = (int)s.stride[3];
  F.g = g;
  const bool guarded = s.has_guard && a->interpolation;
  for (int i = 0; i < 3; ++i) {
    F.lo[i] = a->brick_offset[i] - g;
    F.hi[i] = guarded ? a->brick_size[i] + 2 * g - 2 : a->brick_size[i] - 1;
  }
  return true;
}


template <bool INTERP, bool GUARDED, bool PAIRED, int LINE = 0, int DIM = 1, bool ET = false,
          typename T = float, bool AOS3 = false, int LANES = 2>
static int launch_fast(const isc_render_args* a, const FastField& F, cudaStream_t st) {
  static const int tw_env = getenv("ISC_TILE_W") ? __builtin_ctz(atoi(getenv("ISC_TILE_W"))) : -1;
  static const int cap_env = getenv("ISC_CTAS_PER_SM") ? atoi(getenv("ISC_CTAS_PER_SM")) : 0;
  static const bool no_tune = getenv("ISC_DISABLE_TUNE") != nullptr;
  // screen-rectangle cull first: a brick entirely off screen launches
  // nothing, and must not open tuner trials whose events are never recorded
  int rx0, ry0, rx1, ry1;
  static const bool no_cull = getenv("ISC_DISABLE_CULL") != nullptr;
  const bool culled = !no_cull && brick_screen_rect(a, rx0, ry0, rx1, ry1);
  if (culled) {
    // pixels outside the rectangle miss the brick: transparent (nothing to
    // clear when the rectangle is the whole image)
    if (!rect_is_whole(a, rx0, ry0, rx1, ry1))
      ISC_CUDA_CHECK(cudaMemsetAsync(a->out_rgba, 0, (size_t)a->camera.width * a->camera.height * sizeof(float4), st));
    if (rx1 <= rx0 || ry1 <= ry0) return ISC_OK;
  }
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  OccupancyTuner::Choice ch{cap_env, tw_env >= 0 ? tw_env : 3};
  if (!cap_env && tw_env < 0 && !no_tune && PAIRED) {
    const int variant = (INTERP ? 1 : 0) | (GUARDED ? 2 : 0) | (ET ? 8 : 0) | (DIM << 4) | ((int)sizeof(T) << 8) |
                        (LINE << 12) | (AOS3 ? 1 << 16 : 0) | (LANES << 17);
    ch = tuner().choose(OccupancyTuner::make_key(a, variant), st, &ev0, &ev1);
  }
  // 4 lanes per ray: 8 rays per warp, the tile half as wide (8x2 -> 4x2)
  const int tw_log2 = LANES == 4 ? max(ch.tw_log2 - 1, 0) : ch.tw_log2;
  const int tw = 1 << tw_log2, th = (PAIRED ? 32 / LANES : 32) >> tw_log2;
  int tiles_x = (a->camera.width + tw - 1) / tw, tiles_y = (a->camera.height + th - 1) / th;
  int tile_x0 = 0, tile_y0 = 0;
  if (culled) {
    tile_x0 = rx0 / tw;
    tile_y0 = ry0 / th;
    tiles_x = (rx1 + tw - 1) / tw - tile_x0;
    tiles_y = (ry1 + th - 1) / th - tile_y0;
  }
  const int super_x = (tiles_x + 7) / 8, super_y = (tiles_y + 7) / 8;
  static const bool row_order = getenv("ISC_TILE_ROWS") != nullptr;
  const int n_codes = row_order ? tiles_x * tiles_y : super_x * super_y * 64;
  const int sms = cached_sm_count();
  int per_sm = cached_blocks_per_sm<march_fast_kernel<INTERP, GUARDED, PAIRED, LINE, DIM, ET, T, AOS3, LANES>>(kThreads);
  if (ch.cap > 0 && per_sm > ch.cap) per_sm = ch.cap;
  int grid = sms * (per_sm > 0 ? per_sm : 1);
  const int need = (n_codes + (kThreads / 32) - 1) / (kThreads / 32);  // one tile per warp at most
  if (grid > need) grid = need > 0 ? need : 1;
  if (ev0) cudaEventRecord(ev0, st);
  march_fast_kernel<INTERP, GUARDED, PAIRED, LINE, DIM, ET, T, AOS3, LANES><<<grid, kThreads, 0, st>>>(
      *a, F, tiles_x, tiles_y, super_x, n_codes, row_order ? 1 : 0, tw_log2, tile_x0, tile_y0);
  ISC_CUDA_CHECK(cudaGetLastError());
  if (ev1) cudaEventRecord(ev1, st);
  return ISC_OK;
}

namespace isc {
int launch_staged(int lines, const isc_render_args* a, const FastField& F, cudaStream_t st);  // march_staged.cu
}

// Guarded trilinear paired march with the analytic transfer function of
// `lines` pieces when this instantiation covers it (lines <= MAXL), else the
// shared-memory LUT.  MAXL bounds the template instantiations per variant.
// A small frame: fewer 8x2-ray tiles in the image than two per resident
// warp of the paired march (e.g. 256x256).  Decided on the image alone (not
// the brick's screen rectangle), so a frame's compositing order -- and its
// bits -- do not depend on debug outputs or on the decomposition.
static bool small_frame(const isc_render_args* a) {
  const char* q = getenv("ISC_QUAD");  // A/B, read per call: 0 off, 1 always
  if (q) return atoi(q) == 1;
  if (a->ray_dirs) return false;
  const long long tiles = (long long)((a->camera.width + 7) / 8) * ((a->camera.height + 1) / 2);
  return tiles < 2LL * cached_sm_count() * ISC_FAST_MINB * (kThreads / 32);
}

template <int MAXL, int DIM, bool ET, typename T, bool AOS3 = false>
static int launch_line(int lines, const isc_render_args* a, const FastField& F, cudaStream_t st) {
  if constexpr (DIM == 1 && !ET && !AOS3 && std::is_same<T, float>::value) {
    if ((lines == 0 || lines == 1) && small_frame(a))
      return lines ? launch_fast<true, true, true, 1, 1, false, float, false, 4>(a, F, st)
                   : launch_fast<true, true, true, 0, 1, false, float, false, 4>(a, F, st);
  }
  // 4..ISC_MAX_LUT_KINKS kinks: one variant with the count read at run time
  if constexpr (MAXL >= 4)
    if (lines > 4 && lines <= kLineRuntime) return launch_fast<true, true, true, kLineRuntime, DIM, ET, T, AOS3>(a, F, st);
  if (lines > MAXL) lines = 0;
  switch (lines) {
    case 1: return launch_fast<true, true, true, 1, DIM, ET, T, AOS3>(a, F, st);
    case 2: if constexpr (MAXL >= 2) return launch_fast<true, true, true, 2, DIM, ET, T, AOS3>(a, F, st); break;
    case 3: if constexpr (MAXL >= 3) return launch_fast<true, true, true, 3, DIM, ET, T, AOS3>(a, F, st); break;
    case 4: if constexpr (MAXL >= 4) return launch_fast<true, true, true, 4, DIM, ET, T, AOS3>(a, F, st); break;
    default: break;
  }
  return launch_fast<true, true, true, 0, DIM, ET, T, AOS3>(a, F, st);
}

// float3 source in the standard interleaved layout with even row / slice
// strides and an 8-byte aligned base (fast_gather_aos3).
static bool aos3_layout(const FastField& F) {
  static const bool off = getenv("ISC_DISABLE_AOS3") != nullptr;
  return !off && F.sx == 3 && F.sc == 1 && F.sy % 2 == 0 && F.sz % 2 == 0 &&
         reinterpret_cast<uintptr_t>(F.f) % 8 == 0;
}

template <int MAXL, bool ET>
static int launch_line3(int lines, const isc_render_args* a, const FastField& F, cudaStream_t st) {
  return aos3_layout(F) ? launch_line<MAXL, 3, ET, float, true>(lines, a, F, st)
                        : launch_line<MAXL, 3, ET, float>(lines, a, F, st);
}

// C3-style scenes -- one scalar iso source followed by one volume source,
// guarded trilinear float32, no early termination -- render in two passes:
// (1) the iso source alone through the multi-source kernel (exact iso
// decisions, entry / exit pairs, deferred shading) into scratch: per-pixel
// stations marched and the shaded hit colour; (2) the volume source alone
// through the paired single-source kernel, each ray stopping before its hit
// station (the hit station's later sources sit behind the opaque hit,
// raycast.py:351-369) and compositing the hit colour behind.  Per ray this is
// the reference's over-sequence; the volume pass runs at the single-source
// kernel's speed instead of sharing registers with the iso machinery.
static bool split_eligible(const isc_render_args* a) {
  if (getenv("ISC_DISABLE_SPLIT") || a->n_sources != 2 || a->ray_dirs || a->alpha_stop < 1.0 || !a->interpolation ||
      !a->work_counter)
    return false;
  const isc_source &iso = a->src[0], &vol = a->src[1];
  return iso.mode == ISC_ISO && vol.mode == ISC_VOLUME && iso.feature_dim == 1 && iso.dtype == ISC_F32 &&
         vol.dtype == ISC_F32 && iso.has_guard && vol.has_guard && (vol.feature_dim == 1 || vol.feature_dim == 3);
}

static int launch_split(const isc_render_args* a, cudaStream_t s, bool* handled) {
  *handled = false;
  isc_render_args vol = *a;
  vol.src[0] = a->src[1];
  vol.n_sources = 1;
  FastField F;
  if (!fast_eligible(&vol, F)) return ISC_OK;
  const size_t npx = (size_t)a->camera.width * a->camera.height;
  // scratch: shaded hits (float4), station counts (u32), the volume pass's tile counter
  char* scratch = nullptr;
  const size_t bytes = npx * (sizeof(float4) + sizeof(uint32_t)) + 16;
  {  // keep the stream-ordered pool's memory between frames (default: returned to the OS at every sync)
    static std::mutex mu;
    static bool pool_kept[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    if (dev >= 0 && dev < 64 && !pool_kept[dev]) {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      }
      cudaGetLastError();
      pool_kept[dev] = true;
    }
  }
  ISC_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&scratch), bytes, s));
  float4* shade = reinterpret_cast<float4*>(scratch);
  uint32_t* counts = a->out_stations ? a->out_stations : reinterpret_cast<uint32_t*>(scratch + npx * sizeof(float4));
  uint32_t* counter = reinterpret_cast<uint32_t*>(scratch + npx * (sizeof(float4) + sizeof(uint32_t)));
  isc_render_args iso = *a;  // pass 1: the iso source alone (debug outputs, stations, errors as asked)
  iso.n_sources = 1;
  iso.out_rgba = reinterpret_cast<float*>(shade);
  iso.out_stations = counts;
  int status = ISC_OK;
  *handled = true;
  // without caller-requested per-pixel outputs the probe may cull to the
  // brick's screen rectangle: the volume pass reads only inside it
  g_split_probe = a->out_stations == nullptr;
  if (!launch_iso_probe(&iso, s, &status) && !launch_multi(&iso, s, &status))
    status = fail(ISC_E_VALUE, "iso probe not launchable");
  g_split_probe = false;
  if (status == ISC_OK) {
    // pass 2: the volume source, stopped at each ray's hit
    vol.out_stations = nullptr;
    vol.out_station_total = nullptr;
    vol.out_hit = nullptr;
    vol.out_t = nullptr;
    vol.out_krange = nullptr;
    vol.work_counter = counter;
    F.stop_counts = counts;
    F.stop_shade = shade;
    const cudaError_t e = cudaMemsetAsync(counter, 0, sizeof(uint32_t), s);
    if (e != cudaSuccess) status = cuda_fail(e, "cudaMemsetAsync");
    const int lines = vol.src[0].lut_linear != 0 ? 1 + vol.src[0].lut_kinks : 0;
    if (status == ISC_OK)
      status = vol.src[0].feature_dim == 3 ? launch_line3<2, false>(lines, &vol, F, s)
                                           : launch_line<4, 1, false, float>(lines, &vol, F, s);
  }
  const cudaError_t e = cudaFreeAsync(scratch, s);
  if (status == ISC_OK && e != cudaSuccess) status = cuda_fail(e, "cudaFreeAsync");
  return status;
}

extern "C" int isc_render_local(const isc_render_args* a, void* stream) {
  int st = validate(a, true);
  if (st != ISC_OK) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // the three per-render accumulators; render_local packs them as one
  // [stations, error word, tile counter] int64 block: one memset instead of three
  char* const tot = reinterpret_cast<char*>(a->out_station_total);
  if (tot && reinterpret_cast<char*>(a->error_word) == tot + 8 && reinterpret_cast<char*>(a->work_counter) == tot + 16) {
    ISC_CUDA_CHECK(cudaMemsetAsync(tot, 0, 24, s));
  } else {
    if (a->error_word) ISC_CUDA_CHECK(cudaMemsetAsync(a->error_word, 0, sizeof(uint32_t), s));
    if (a->out_station_total) ISC_CUDA_CHECK(cudaMemsetAsync(a->out_station_total, 0, sizeof(unsigned long long), s));
    if (a->work_counter) ISC_CUDA_CHECK(cudaMemsetAsync(a->work_counter, 0, sizeof(uint32_t), s));
  }
  FastField F;
  static const bool no_fast = getenv("ISC_DISABLE_FAST") != nullptr;
  if (!no_fast && fast_eligible(a, F)) {
    const bool interp = a->interpolation != 0;
    const bool guarded = interp && a->src[0].has_guard;
    static const bool no_pair = getenv("ISC_DISABLE_PAIRED") != nullptr;
    const bool paired = !no_pair && a->alpha_stop >= 1.0;
    // analytic transfer function: LINE = 1 + kinks (0 = shared-memory LUT)
    const int lines = a->src[0].lut_linear != 0 ? 1 + a->src[0].lut_kinks : 0;
    const bool et = a->alpha_stop < 1.0;
    if (a->src[0].dtype != ISC_F32) {  // double / __half / __nv_bfloat16 scalar fields (fast_eligible)
      if (a->src[0].dtype == ISC_F64)
        return et ? launch_line<1, 1, true, double>(lines, a, F, s) : launch_line<1, 1, false, double>(lines, a, F, s);
      if (a->src[0].dtype == ISC_F16)
        return et ? launch_line<1, 1, true, __half>(lines, a, F, s) : launch_line<1, 1, false, __half>(lines, a, F, s);
      return et ? launch_line<1, 1, true, __nv_bfloat16>(lines, a, F, s)
                : launch_line<1, 1, false, __nv_bfloat16>(lines, a, F, s);
    }
    if (a->src[0].feature_dim == 3)
      return et ? launch_line3<2, true>(lines, a, F, s) : launch_line3<2, false>(lines, a, F, s);
    // early termination, guarded trilinear: paired with the per-station stop test
    if (interp && guarded && !no_pair && et) return launch_line<4, 1, true, float>(lines, a, F, s);
    const bool stage = getenv("ISC_STAGE") != nullptr;  // shared-memory brick staging (march_staged.cu), read per call
    if (interp && guarded && paired && stage) return isc::launch_staged(lines, a, F, s);
    if (interp && guarded && paired) return launch_line<4, 1, false, float>(lines, a, F, s);
    if (interp && guarded) return paired ? launch_fast<true, true, true>(a, F, s) : launch_fast<true, true, false>(a, F, s);
    if (interp) return paired ? launch_fast<true, false, true>(a, F, s) : launch_fast<true, false, false>(a, F, s);
    return paired ? launch_fast<false, false, true>(a, F, s) : launch_fast<false, false, false>(a, F, s);
  }
  if (split_eligible(a)) {
    bool handled = false;
    const int st_split = launch_split(a, s, &handled);
    if (handled) return st_split;
  }
  static const bool no_multi = getenv("ISC_DISABLE_MULTI") != nullptr;
  bool layout_free_iso = false;  // march_rays(volume=None) with an iso source: generic kernel only
  for (int i = 0; i < a->n_sources; ++i) layout_free_iso |= a->no_layout && a->src[i].mode == ISC_ISO;
  int mstatus = ISC_OK;
  if (!no_multi && !layout_free_iso && launch_multi(a, s, &mstatus)) return mstatus;
  dim3 grid((a->camera.width + kTile - 1) / kTile, (a->camera.height + kTile - 1) / kTile);
  const size_t smem = (size_t)a->n_sources * ISC_LUT_ENTRIES * sizeof(float4);
  if (a->interpolation) march_kernel<true><<<grid, kThreads, smem, s>>>(*a);
  else march_kernel<false><<<grid, kThreads, smem, s>>>(*a);
  ISC_CUDA_CHECK(cudaGetLastError());
  return ISC_OK;
}

extern "C" int isc_gradient_normals(const isc_render_args* a, const double* positions, const double* view_dirs,
                                    int64_t n, float* out_normals, void* stream) {
  int st = validate(a, false);
  if (st != ISC_OK) return st;
  if (a->n_sources < 1) return fail(ISC_E_VALUE, "gradient_normals needs a source in src[0]");
  if (n < 0) return fail(ISC_E_VALUE, "negative position count");
  if (n == 0) return ISC_OK;
  if (!positions || !view_dirs || !out_normals) return fail(ISC_E_VALUE, "null positions / view_dirs / output");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (a->error_word) ISC_CUDA_CHECK(cudaMemsetAsync(a->error_word, 0, sizeof(uint32_t), s));
  const int threads = 128;
  gradient_kernel<<<(unsigned)((n + threads - 1) / threads), threads, 0, s>>>(*a, positions, view_dirs, n, out_normals);
  ISC_CUDA_CHECK(cudaGetLastError());
  return ISC_OK;
}

extern "C" int isc_ray_setup(const isc_render_args* a, void* stream) {
  int st = validate(a, false);
  if (st != ISC_OK) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  dim3 grid((a->camera.width + kTile - 1) / kTile, (a->camera.height + kTile - 1) / kTile);
  ray_setup_kernel<<<grid, kThreads, 0, s>>>(*a);
  ISC_CUDA_CHECK(cudaGetLastError());
  return ISC_OK;
}
