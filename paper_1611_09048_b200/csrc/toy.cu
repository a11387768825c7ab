// GPU field generator for the reference harness's analytic shear flow
// (harness.ToyState, harness.py:119-190): density advected by a tanh shear
// along x plus a sinusoidal vertical wiggle, recomputed at step k by
// back-tracing every grid point through k inverse step maps; velocity is the
// analytic profile.  Lets the harness workload (density + float3 velocity +
// non-persistent current) run at 512^3-1024^3 without host float64 meshgrids.
// float64 arithmetic in the harness's evaluation order (no FMA contraction);
// results stored as float32 render fields.
#include <math_constants.h>

#include "common.cuh"

namespace isc {

struct ToyConsts {
  double lx, ly, lz;
  double shear_speed, perturbation, dt;
  double seed_term;   // seed * 0.17
};

// p.shear_speed * tanh(3.0 * sin(2.0 * pi * y / ly))      (harness.py:155-157)
__device__ __forceinline__ double shear_u(const ToyConsts& c, double y) {
  const double a = ddiv(dmul(2.0 * CUDART_PI, y), c.ly);
  return dmul(c.shear_speed, tanh(dmul(3.0, sin(a))));
}

// p.perturbation * sin(2.0 * pi * x / lx + phase(step))   (harness.py:159-163)
__device__ __forceinline__ double wiggle_w(const ToyConsts& c, double x, int step) {
  const double frac = fmod(dadd(dmul((double)step, 0.03), c.seed_term), 1.0);
  const double phase = dmul(2.0 * CUDART_PI, frac);
  const double a = dadd(ddiv(dmul(2.0 * CUDART_PI, x), c.lx), phase);
  return dmul(c.perturbation, sin(a));
}

// 1 + 0.35 sin(2 pi x/lx) sin(2 pi y/ly) + 0.25 cos(2 pi (y/ly + 2 z/lz))  (harness.py:176-182)
__device__ __forceinline__ double density0(const ToyConsts& c, double x, double y, double z) {
  const double sx = sin(ddiv(dmul(2.0 * CUDART_PI, x), c.lx));
  const double sy = sin(ddiv(dmul(2.0 * CUDART_PI, y), c.ly));
  const double arg = dmul(2.0 * CUDART_PI, dadd(ddiv(y, c.ly), ddiv(dmul(2.0, z), c.lz)));
  return dadd(dadd(1.0, dmul(dmul(0.35, sx), sy)), dmul(0.25, cos(arg)));
}

__global__ void toy_kernel(ToyConsts c, int ox, int oy, int oz, int nx, int ny, int nz, int step, float* density,
                           float* velocity) {
  const long long total = (long long)nx * ny * nz;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int ix = (int)(i % nx), iy = (int)((i / nx) % ny), iz = (int)(i / ((long long)nx * ny));
    const double xg = (double)(ox + ix), yg = (double)(oy + iy), zg = (double)(oz + iz);
    if (density) {
      double x = xg, y = yg;
      for (int j = step; j > 0; --j) {   // inverse of shear-then-wiggle, newest step first (harness.py:165-174)
        y = dsub(y, dmul(wiggle_w(c, x, j - 1), c.dt));
        x = dsub(x, dmul(shear_u(c, y), c.dt));
      }
      density[i] = (float)density0(c, x, y, zg);
    }
    if (velocity) {
      velocity[3 * i + 0] = (float)shear_u(c, yg);
      velocity[3 * i + 1] = (float)wiggle_w(c, xg, step);
      velocity[3 * i + 2] = 0.0f;
    }
  }
}

}  // namespace isc

using namespace isc;

extern "C" int isc_toy_fields(const isc_toy_args* a, void* stream) {
  if (!a) return fail(ISC_E_VALUE, "null toy args");
  for (int i = 0; i < 3; ++i)
    if (a->global_size[i] <= 0 || a->size[i] <= 0) return fail(ISC_E_FIELD, "sizes must be positive");
  if (a->guard < 0 || a->step_index < 0) return fail(ISC_E_VALUE, "guard and step must be non-negative");
  ToyConsts c;
  c.lx = a->global_size[0];
  c.ly = a->global_size[1];
  c.lz = a->global_size[2];
  c.shear_speed = a->shear_speed;
  c.perturbation = a->perturbation;
  c.dt = a->dt;
  c.seed_term = (double)a->seed * 0.17;   // seed * 0.17 (harness.py:162)
  const int g = a->guard;
  const int nx = a->size[0] + 2 * g, ny = a->size[1] + 2 * g, nz = a->size[2] + 2 * g;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long total = (long long)nx * ny * nz;
  long long grid = (total + 255) / 256;
  if (grid > sms * 32LL) grid = sms * 32LL;
  toy_kernel<<<(int)grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      c, a->offset[0] - g, a->offset[1] - g, a->offset[2] - g, nx, ny, nz, a->step_index, a->density, a->velocity);
  ISC_CUDA_CHECK(cudaGetLastError());
  return ISC_OK;
}
