/*
 * isaac_b200.h -- C-ABI of the B200 (sm_100a) ISAAC rendering hot path.
 *
 * One shared library (libisaac_b200.so) exporting plain extern "C" entry
 * points: POD structs, raw device pointers, element counts and a CUDA stream
 * passed as void*.  No torch types cross this boundary; the Python host layer
 * (paper_1611_09048_b200/) binds it with ctypes, exactly as the reference's
 * Python API would (see INTEGRATION.md for the binding stub).
 *
 * Every call is stream-ordered and asynchronous unless stated otherwise.
 * Return value: ISC_OK or an isc_status; isc_last_error() gives the
 * thread-local message.  Status codes map 1:1 onto the reference exceptions:
 *   ISC_E_FIELD    -> fields.FieldError          (fields.py:24-25)
 *   ISC_E_GUARD    -> fields.GuardContractError  (fields.py:32-33)
 *   ISC_E_CHAIN    -> functors.ChainError        (functors.py:20-21)
 *   ISC_E_SCENE    -> scene.SceneError           (scene.py:21-22)
 *   ISC_E_COMPOSITE-> compositing.CompositeError (compositing.py:21-22)
 *   ISC_E_TRANSPORT-> transport.TransportError   (transport.py:16-17)
 *   ISC_E_VALUE    -> ValueError                 (raycast.py:76-77, 156-157)
 *
 * Reference interfaces replaced (all under /root/reference/pkg/src/insitu/):
 *   isc_render_local   <- raycast.render_local       raycast.py:492-541
 *                         (+ march_rays 291-381, _iso_detect 384-468,
 *                            gradient_normals 210-242, _trilinear 182-199,
 *                            fields.sample_many 218-246, eval_chain_array
 *                            functors.py:212-222, classify_array scene.py:139-152)
 *   isc_ray_setup      <- Camera.ray_directions scene.py:55-70,
 *                         _ray_box_intervals raycast.py:100-120,
 *                         _apply_clip_planes raycast.py:123-143,
 *                         hit mask raycast.py:522, station range raycast.py:316-324
 *   isc_value_range    <- (no reference function; value ranges are scene
 *                         state, scene.py:188 / runtime.py:154-157)
 *   isc_over           <- compositing.over_arrays   compositing.py:31-33
 *   isc_composite_fold <- compositing.composite_sequential compositing.py:66-77
 *                         and _direct_send           compositing.py:184-194
 *   isc_binary_swap    <- compositing.binary_swap   compositing.py:107-181
 *   isc_to_rgba8       <- runtime.to_rgba8           runtime.py:66-67
 *   isc_toy_fields     <- harness.ToyState.refresh   harness.py:119-190
 *   isc_arena_* / isc_ipc_* <- transport.Transport  transport.py:20-28
 *                         (the NVLink replacement of LocalFabric queues)
 */
#ifndef ISAAC_B200_H
#define ISAAC_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define ISC_API __attribute__((visibility("default")))
#else
#define ISC_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define ISC_ABI_VERSION 4  /* 2: isc_render_args.ray_dirs / ray_intervals, isc_gradient_normals;
                              3: per-slice swap counters, isc_swap_reset, isc_debug_occupy,
                                 isc_render_args.no_layout, piecewise-linear LUTs (lut_kinks),
                                 float64 iso decisions (iso_exact, iso_threshold_d);
                              4: ISC_MAX_LUT_KINKS 3 -> 7 (isc_source grows) */
#define ISC_MAX_SOURCES 8      /* active sources per render                 */
#define ISC_MAX_CLIP_PLANES 8
#define ISC_MAX_CHAIN 8        /* ChainLimits.max_length default is 5        */
#define ISC_LUT_ENTRIES 256    /* scene.py:18                                 */
#define ISC_MAX_LUT_KINKS 7    /* slope changes of an analytic LUT            */
#define ISC_MAX_RANKS 64
#define ISC_MAX_ROUNDS 6       /* log2(ISC_MAX_RANKS)                         */
#define ISC_IPC_HANDLE_BYTES 64
#define ISC_MAX_SWAP_CTAS 1024 /* slices (= CTAs) of one swap launch        */
#define ISC_SWAP_STAGES 9      /* per-slice counters: ready, rounds, collect, root read */

typedef enum {
  ISC_OK = 0,
  ISC_E_FIELD = 1,
  ISC_E_GUARD = 2,
  ISC_E_CHAIN = 3,
  ISC_E_SCENE = 4,
  ISC_E_COMPOSITE = 5,
  ISC_E_TRANSPORT = 6,
  ISC_E_VALUE = 7,
  ISC_E_CUDA = 8
} isc_status;

typedef enum { ISC_F32 = 0, ISC_F64 = 1, ISC_F16 = 2, ISC_BF16 = 3 } isc_dtype;
typedef enum { ISC_VOLUME = 0, ISC_ISO = 1 } isc_mode;

/* Functor-chain opcodes.  1..5 are the reference built-ins
 * (functors.py:124-147); the rest are device ops for user-registered
 * functors (FunctorRegistry.register_functor, functors.py:81-90). */
typedef enum {
  ISC_OP_ADD = 1, ISC_OP_MUL = 2, ISC_OP_POW = 3, ISC_OP_LENGTH = 4, ISC_OP_SUM = 5,
  ISC_OP_SQRT = 6, ISC_OP_ABS = 7, ISC_OP_NEG = 8, ISC_OP_EXP = 9, ISC_OP_LOG = 10,
  ISC_OP_MIN = 11, ISC_OP_MAX = 12
} isc_op;

typedef struct {
  int32_t op;        /* isc_op                                    */
  int32_t in_dim;    /* dimension entering this step (1..4)       */
  float arg[4];      /* constant, already broadcast (functors.py:191-194) */
  double arg_d[4];   /* the same constant in float64 (iso_exact sources) */
} isc_chain_step;

/* One active source: a zero-copy view of an application array laid out
 * (z, y, x[, component]) INCLUDING the guard halo, as array_backed_handle
 * expects (fields.py:249-278). */
typedef struct {
  const void* data;          /* device pointer to element [0,0,0,0]      */
  int64_t stride[4];         /* element strides of z, y, x, component     */
  int32_t dtype;             /* isc_dtype                                 */
  int32_t feature_dim;       /* 1..4                                      */
  int32_t has_guard;         /* SourceDescriptor.has_guard                */
  int32_t mode;              /* isc_mode                                  */
  float iso_threshold;
  float range_lo, range_hi;  /* TransferFunction.value_range              */
  int32_t n_steps;           /* chain length (0 = identity)               */
  const float* lut;          /* device, 256 x 4 straight RGBA (float32)  */
  isc_chain_step steps[ISC_MAX_CHAIN];
  /* Optional analytic form of the LUT.  The LUT lerp is the piecewise-linear
   * interpolant through (i, lut[i]); when its slope changes at no more than
   * ISC_MAX_LUT_KINKS integer positions (a tf_from_points ramp with a few
   * control points, scene.py:113-126), lut_linear = 1 and
   *   lut(x) = lut_base + lut_slope * x + sum_k lut_kink_dslope[k] * max(x - lut_kink_x[k], 0)
   * for x = 255 t, exactly the LUT lerp; the kernel then skips the
   * shared-memory lookup.  lut_kinks = 0: one straight run. */
  int32_t lut_linear;
  float lut_base[4];
  float lut_slope[4];
  int32_t lut_kinks;
  float lut_kink_x[ISC_MAX_LUT_KINKS];
  float lut_kink_dslope[ISC_MAX_LUT_KINKS][4];
  /* Iso surfaces decided exactly as the reference: iso_exact = 1 when the
   * chain is made of add / mul only (a scalar source) -- the kernels then
   * evaluate this source's trilinear sample and chain in float64 in the
   * reference's operation order (raycast.py:182-199, functors.py:212-222)
   * and compare against iso_threshold_d, so every sign test and crossing
   * fraction tau equals the reference's bit for bit. */
  double iso_threshold_d;
  int32_t iso_exact;
  /* steps[i].op packed 4 bits per step (step i in bits 4i..4i+3): the hot
   * kernels branch on one register instead of holding every step's opcode. */
  uint32_t step_ops;
} isc_source;

/* Camera in global cell coordinates; basis/tan/aspect precomputed on the
 * host with the reference's numpy expressions (scene.py:46-62). */
typedef struct {
  double origin[3];
  double fwd[3], right[3], up[3];
  double tan_half, aspect;
  int32_t width, height;
} isc_camera;

/* Clip plane (scene.py:73-93); f0 = np.dot(origin - point, normal)
 * evaluated on the host exactly as raycast.py:133 does. */
typedef struct {
  double point[3];
  double normal[3];
  double f0;
} isc_clip_plane;

typedef struct {
  isc_camera camera;
  double step;               /* RenderSettings.step_length                */
  double alpha_stop;         /* early_termination_alpha; >= 1 disables    */
  int32_t interpolation;     /* 1 = trilinear, 0 = nearest                */
  int32_t n_sources;         /* active sources in source-id order         */
  int32_t n_clip;
  int32_t guard_width;       /* LocalDomain.guard_width                   */
  int32_t brick_offset[3];   /* LocalDomain.offset (x, y, z)             */
  int32_t brick_size[3];     /* LocalDomain.size                          */
  int32_t volume_size[3];    /* GlobalVolume.size                         */
  int32_t decomposition[3];  /* GlobalVolume.decomposition                */
  isc_clip_plane clip[ISC_MAX_CLIP_PLANES];
  isc_source src[ISC_MAX_SOURCES];
  /* outputs (device pointers, caller-owned) */
  float* out_rgba;           /* (H, W, 4) premultiplied; required         */
  uint32_t* out_stations;    /* (H*W) stations marched per pixel; optional */
  int32_t* out_krange;       /* (H*W, 4) k_lo, k_hi, kg_lo, kg_hi; optional */
  double* out_t;             /* (H*W, 2) t_in, t_out of the brick; optional */
  uint8_t* out_hit;          /* (H*W) hit mask; optional                  */
  uint32_t* error_word;      /* device u32; guard-contract violations are
                                counted here (-> GuardContractError); optional */
  unsigned long long* out_station_total; /* device u64: sum of stations marched
                                (LocalImage.stations, raycast.py:46); optional */
  uint32_t* work_counter;    /* device u32 scratch for the persistent tile
                                scheduler; optional (null = static grid) */
  /* Ray-list mode (raycast.march_rays, raycast.py:291-381, and march_ray,
   * 471-489): when ray_dirs is set, the "image" is camera.width x
   * camera.height rays whose directions (float64 x3, used as given, not
   * normalised) and intervals (float64 x4: brick t0, t1, global t0, t1) are
   * read from these device arrays instead of being derived from the camera;
   * camera.origin is the common origin, clip planes are not applied (the
   * intervals are final) and every ray marches k in
   * [ceil(max(t0,0)/step), ceil(max(t1,0)/step)).  Null in a frame render. */
  const double* ray_dirs;
  const double* ray_intervals;
  /* 1 = no volume layout (march_rays(volume=None), raycast.py:396-418): an
   * iso entry pair of a guarded trilinear source samples station k-1 clamped
   * into [offset-g, offset+size+g-1-1e-9] instead of testing reachability,
   * and no exit pairs are checked.  0 in a frame render. */
  int32_t no_layout;
} isc_render_args;
/* isc_render_local zeroes *error_word, *out_station_total and *work_counter
 * (stream-ordered) before the march, so callers never need a separate fill. */

/* ---- library ------------------------------------------------------------ */
ISC_API int isc_abi_version(void);
ISC_API const char* isc_last_error(void);
/* sizeof of the public structs, so bindings can verify their layouts:
 * which = 0 isc_render_args, 1 isc_source, 2 isc_camera, 3 isc_clip_plane,
 * 4 isc_chain_step, 5 isc_swap_args, 6 isc_toy_args */
ISC_API size_t isc_struct_size(int which);
ISC_API int isc_device_sm_count(int device);

/* ---- rendering ---------------------------------------------------------- */
/* Full brick render (ray setup + march + iso + compositing in registers). */
ISC_API int isc_render_local(const isc_render_args* args, void* stream);
/* Ray setup only (parity/debug): fills out_t / out_krange / out_hit. */
ISC_API int isc_ray_setup(const isc_render_args* args, void* stream);
/* Central-difference normals of src[0]'s chained scalar at n positions
 * (raycast.gradient_normals, raycast.py:210-242): stencil clamped to the
 * samplable box of the brick, zero gradient -> -view_dir.  positions and
 * view_dirs are device float64 (n, 3); out_normals device float32 (n, 3). */
ISC_API int isc_gradient_normals(const isc_render_args* args, const double* positions, const double* view_dirs,
                                 int64_t n, float* out_normals, void* stream);
/* Per-source normalisation: (min, max) of the float32-chained first
 * component over the brick interior (guard excluded), NaN ignored.
 * out_minmax: device buffer of >= 4 32-bit words; [0], [1] receive (min, max)
 * as float32 (NaN, NaN if no non-NaN value), [2], [3] are scratch.
 * Bit-exact for add/mul/length/sum chains. */
ISC_API int isc_value_range(const isc_source* src, const int32_t brick_size[3], int32_t guard_width,
                    float* out_minmax, void* stream);

/* ---- compositing ---------------------------------------------------------- */
/* dst[i] = front[i] over back[i] (premultiplied RGBA float32). */
ISC_API int isc_over(float* dst, const float* front, const float* back, int64_t n_pixels, void* stream);
/* out = images[0] over images[1] over ... (front to back, float32 RGBA);
 * images is a HOST array of device (or peer-mapped) pointers. */
ISC_API int isc_composite_fold(float* out, const float* const* images, int32_t n_images,
                       int64_t n_pixels, void* stream);

/* Binary swap over peer memory.  Every rank runs one persistent kernel of
 * n_ctas CTAs; the image is cut into n_ctas contiguous slices and CTA b runs
 * the reference's binary swap on slice b: in round r it pulls its partner's
 * half of the slice-b span straight out of the partner's image (NVLink peer
 * load), composites it with its own half in visibility order and writes it
 * in place; after the last round it stores its final span directly into
 * rank 0's output.  Per pixel the tree of `over`s is the reference's, so
 * results are bit-identical to a whole-image swap.  Ordering uses
 * epoch-tagged per-slice arrival counters in each rank's flag block (no host
 * round trips, no grid-wide barrier: the grid need not be co-resident).
 * n_ctas and n_pixels must be equal on every rank.  Pointers for other ranks
 * are peer-mapped (isc_ipc_open) or, for ranks sharing one device, plain
 * device pointers. */
typedef struct {
  int32_t rank, size;            /* this rank, world size (power of two) */
  int32_t n_ctas;                /* slices = CTAs, same on every rank    */
  int32_t round_begin, round_end;/* rounds executed by this launch       */
  int32_t collect;               /* 1: store final span into root_out    */
  int32_t finish;                /* 1: wait until peers stopped reading  */
  int32_t publish_ready;         /* 1: announce this rank's image ready  */
  int64_t n_pixels;
  int64_t epoch;                 /* 1, 2, 3, ... identical on all ranks;
                                    0: read it from this rank's flag block
                                    (isc_swap_epoch_bump; CUDA-graph replayable) */
  int64_t timeout_ns;            /* spin-wait limit -> ISC_E_TRANSPORT   */
  int32_t order[ISC_MAX_RANKS];  /* visibility order (compositing.py:36-63) */
  float* image[ISC_MAX_RANKS];   /* every rank's working image           */
  unsigned long long* flags[ISC_MAX_RANKS]; /* every rank's flag block   */
  float* root_out;               /* rank 0's output image                */
} isc_swap_args;
ISC_API int isc_binary_swap(const isc_swap_args* args, void* stream);
/* Number of 8-byte words in a rank's flag block. */
ISC_API int isc_flag_words(void);
/* Read-and-clear this rank's transport error word: stream-ordered copy into
 * `pinned` (page-locked host memory owned by the caller), then a stream sync. */
ISC_API int isc_swap_status(unsigned long long* flags, void* stream, unsigned long long* pinned,
                            int32_t* out_code);

/* Stream-ordered copy of the error word into `pinned` (no synchronisation):
 * the deferred form of isc_swap_status, read once the stream passed it. */
ISC_API int isc_swap_error_async(unsigned long long* flags, unsigned long long* pinned, void* stream);
/* Zero a rank's flag block (stream-ordered).  Collective recovery after a
 * TransportError: every rank resets its own block, then all restart at epoch 1. */
ISC_API int isc_swap_reset(unsigned long long* flags, void* stream);
/* Device-resident epoch: add 1 to the epoch word of this rank's flag block
 * (stream-ordered, one thread).  Called once per logical swap before its
 * launches with isc_swap_args.epoch = 0, the epoch lives on the device and a
 * frame's render + swap can be captured as a CUDA graph and replayed (every
 * rank replaying the same number of times keeps the epochs equal). */
ISC_API int isc_swap_epoch_bump(unsigned long long* flags, void* stream);
/* Test aid: occupy the GPU with n_ctas CTAs of `threads` threads that spin
 * for `ns` nanoseconds (a stand-in for the simulation's kernels sharing the
 * GPU with the compositor). */
ISC_API int isc_debug_occupy(int32_t n_ctas, int32_t threads, int64_t ns, void* stream);

/* Direct-send fallback for non-power-of-two world sizes: rank 0 folds every
 * rank's image (peer loads) in visibility order into root_out; other ranks
 * publish readiness and wait until rank 0 has finished reading them. */
ISC_API int isc_direct_send(const isc_swap_args* args, void* stream);

/* ---- frame encode ---------------------------------------------------------- */
/* out[i] = round_half_even(clip(rgba[i], 0, 1) * 255) per channel, uint8
 * (H, W, 4) -- runtime.to_rgba8 (runtime.py:66-67). */
ISC_API int isc_to_rgba8(const float* rgba, uint8_t* out, int64_t n_pixels, void* stream);

/* ---- harness field generator ------------------------------------------------ */
/* Analytic shear-flow fields of the reference harness (harness.ToyState,
 * harness.py:119-190) for one brick + guard at a given step, float64 math,
 * float32 output: density (z, y, x) and velocity (z, y, x, 3), either may be
 * null.  Global coordinates of array index 0 are offset - guard. */
typedef struct {
  int32_t global_size[3];
  int32_t offset[3];
  int32_t size[3];
  int32_t guard;
  int32_t step_index;
  int32_t seed;
  double shear_speed, perturbation, dt;
  float* density;
  float* velocity;
} isc_toy_args;
ISC_API int isc_toy_fields(const isc_toy_args* args, void* stream);

/* ---- device memory shared between processes --------------------------- */
ISC_API int isc_arena_alloc(size_t bytes, void** out_ptr);     /* cudaMalloc + zero */
ISC_API int isc_arena_free(void* ptr);
ISC_API int isc_ipc_handle(void* dev_ptr, unsigned char out_handle[ISC_IPC_HANDLE_BYTES]);
ISC_API int isc_ipc_open(const unsigned char handle[ISC_IPC_HANDLE_BYTES], void** out_ptr);
ISC_API int isc_ipc_close(void* peer_ptr);
ISC_API int isc_enable_peer_access(int peer_device);

#ifdef __cplusplus
}
#endif
#endif /* ISAAC_B200_H */
