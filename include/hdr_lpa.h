/*
 * hdr_lpa.h -- C ABI of the B200-native unified HDR LPA operator.
 *
 * Plain C: device pointers, sizes and scalars only (no torch or CUDA types in
 * the signatures; the CUDA stream is passed as `void *` = cudaStream_t).
 *
 * Each entry point replaces one reference interface of hdrfuse (paths are
 * relative to the reference package root pkg/src/hdrfuse/):
 *
 *   hdr_lpa_reconstruct   <- lpa.py:411-433 reconstruct_frame (through
 *                            lpa.py:379-408 reconstruct_channel,
 *                            lpa.py:322-376 _evaluate_index and the numba
 *                            kernel _kernels.py:203-300 lpa_evaluate), fused
 *                            with radiometry.py:303-349 frames_to_samples and
 *                            radiometry.py:208-242 SampleIndex: the raw
 *                            frames are consumed directly, no sample list or
 *                            index is ever materialised.
 *   hdr_saturation_mask   <- radiometry.py:298-300 saturation_mask (+ the
 *                            defective-pixel exclusion of radiometry.py:316-317)
 *   hdr_lpa_workspace_bytes  workspace sizing (the reference allocates its
 *                            scratch per query chunk, _kernels.py:251-256)
 *   hdr_lpa_status_string    error text; the Python layer maps codes to the
 *                            reference's exception types (ValueError,
 *                            ConfigurationError, ShapeMismatchError)
 *
 * Ownership: the caller owns every buffer (inputs read-only, outputs written
 * in place, like lpa.py:343-345).  Calls are stream-ordered and reentrant per
 * stream; there are no hidden allocations on the hot path.
 *
 * Per-pixel numeric failure never returns an error: the pixel becomes NaN
 * (_kernels.py:297-300), exactly as in the reference.
 */
#ifndef HDR_LPA_H
#define HDR_LPA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HDR_LPA_MAX_SENSORS 8
#define HDR_LPA_MAX_SCALES 8
#define HDR_LPA_ABI_VERSION 5

/* status codes */
#define HDR_OK 0
#define HDR_ERR_ARG 1        /* invalid argument / parameter  -> ValueError          */
#define HDR_ERR_CONFIG 2     /* non-positive g*t*a*n etc.     -> ConfigurationError  */
#define HDR_ERR_SHAPE 3      /* inconsistent sizes            -> ShapeMismatchError  */
#define HDR_ERR_WORKSPACE 4  /* workspace too small                                  */
#define HDR_ERR_CUDA 5       /* CUDA launch / runtime error                          */
#define HDR_ERR_FAULT 6      /* a kernel raised a fault bit (results incomplete)     */

/* Fault bits a kernel raises in the workspace header instead of trapping
 * (read back by hdr_lpa_workspace_status; cleared by every reconstruct call) */
#define HDR_FAULT_MBAR_TIMEOUT 1u  /* a staging barrier wait exceeded its bound */
#define HDR_FAULT_BOUNDS 2u        /* debug builds: a staged read out of range   */

/* Weight modes (ReconstructionParams.weight_mode, lpa.py:54-61) */
#define HDR_WEIGHT_VARIANCE 0
#define HDR_WEIGHT_SIGMA 1

/* HdrParams.flags: diagnostics only.  FAST_ONLY skips the exact slow path
 * (its work items stay unprocessed, their outputs unwritten); used by the
 * bench to time the fast kernel on its own. */
#define HDR_FLAG_FAST_ONLY 1
/* NO_MERGE keeps one tap stream per sensor where co-sited sensors (same
 * transform, frame size and Bayer phase) would be merged into one sample per
 * position (A/B comparisons of the two tap kernels). */
#define HDR_FLAG_NO_MERGE 2
/* SKIP_R / SKIP_G / SKIP_B leave a channel out (its output planes are not
 * written): CALPA's first pass needs the G channel only (steering.py:214-248). */
#define HDR_FLAG_SKIP_R 4
#define HDR_FLAG_SKIP_G 8
#define HDR_FLAG_SKIP_B 16

/* Outcome plane codes (optional diagnostics): order*16 + radius-step of the
 * accepted fit (radius step 0 = base radius), or HDR_OUTCOME_NAN. */
#define HDR_OUTCOME_NAN 0xFF

/*
 * One sensor: its raw frame on the device plus the SensorConfig
 * (radiometry.py:35-92) and NoiseCalibration (radiometry.py:95-136) fields.
 * Calibration entries are scalars unless the matching plane pointer is
 * non-NULL (device, float64, width*height row-major), mirroring the rig
 * schema's "scalar or PFM" noise entries (rig.py:67-95).
 */
typedef struct HdrSensor {
    const uint16_t *raw;        /* device, height rows of `pitch` elements */
    int width, height, pitch;
    int saturation_level;       /* keep <=> raw < saturation_level */
    int tile[4];                /* ColorChannel (R=0,G=1,B=2) at [(y%2)*2 + x%2] */
    double exposure_time;       /* t  (s)            */
    double gain;                /* g  (DV/e)         */
    double exposure_scaling;    /* n  in (0, 1]      */
    double transform[6];        /* 2x3 row-major: sensor (x, y) -> reference */
    double bias;                /* b     (DV)   */
    double readout_variance;    /* Var[r] (DV^2) */
    double nonuniformity;       /* a            */
    const double *bias_plane;       /* nullable */
    const double *readvar_plane;    /* nullable */
    const double *nonuni_plane;     /* nullable */
    const uint8_t *defective;       /* nullable, width*height, 1 = discard */
} HdrSensor;

/*
 * ReconstructionParams (lpa.py:40-74) resolved per channel, plus the ICI
 * extension (no reference counterpart).
 *   scale[c][k]  : window scale h (px^2) of channel c at ICI scale k
 *                  (k = 0 is ReconstructionParams.channel_scale(c)).
 *   n_scales == 1: fixed-scale LPA (the reference's behaviour).
 */
typedef struct HdrParams {
    int order;                  /* 0, 1, 2 */
    int weight_mode;            /* HDR_WEIGHT_* */
    int n_scales;               /* 1..HDR_LPA_MAX_SCALES */
    int flags;                  /* HDR_FLAG_* (0 for normal operation) */
    double scale[3][HDR_LPA_MAX_SCALES];
    double max_radius;          /* resolved_max_radius() (lpa.py:71-74) */
    double cond_threshold;      /* 1e8 default */
    double ici_gamma;           /* confidence-interval width factor */
} HdrParams;

/* Outputs: device pointers; only rgb is required. */
typedef struct HdrOutputs {
    float *rgb;                 /* out_h*out_w*3, HWC, max(val,0) as float32, NaN = no data */
    float *grad;                /* nullable: [3 channels][2 (gx, gy)][out_h][out_w], unclamped */
    uint8_t *scale_idx;         /* nullable: [3][out_h][out_w] selected ICI scale index */
    uint8_t *outcome;           /* nullable: [3][out_h][out_w] HDR_OUTCOME codes */
    float *value;               /* nullable: [3][out_h][out_w] unclamped fitted constant term */
    uint16_t *count;            /* nullable: [3][out_h][out_w] samples inside the accepted window
                                   (selected ICI scale; 0 where NaN) */
    uint32_t *work;             /* nullable: [3][out_h][out_w] inside-window samples summed over
                                   every moment sweep evaluated (all ICI scales / ladder steps):
                                   the algorithmic work behind the pixel (ABI v3) */
    uint16_t *rgb_half;         /* nullable: out_h*out_w*3 HWC IEEE fp16 of
                                   max(val,0)*half_scale (NaN kept) -- half the bytes of rgb for
                                   streaming/display (ABI v4).  rgb may be NULL
                                   when rgb_half is given. */
    float half_scale;           /* scale applied before the fp16 rounding (e.g. 1/16 keeps
                                   radiance up to ~1e6 e/s inside fp16's range) */
} HdrOutputs;

/* Bytes of device workspace hdr_lpa_reconstruct needs for these sensors and
 * this output size (work list + per-frame radiometric phase planes). */
int hdr_lpa_workspace_bytes(const HdrSensor *sensors, int n_sensors, int out_w, int out_h,
                            size_t *bytes);

/*
 * Reconstruct one HDR frame on the output grid (out_w x out_h) whose pixel
 * centres are x_j = (j + 0.5) * ref_w / out_w - 0.5 in reference coordinates
 * (lpa.py:213-224).  Row band: only output rows [row_begin, row_end) are
 * computed (row_end <= 0 means out_h); outputs are still indexed over the
 * full frame.  `workspace` is device memory of hdr_lpa_workspace_bytes(),
 * 256-byte aligned.
 */
int hdr_lpa_reconstruct(const HdrSensor *sensors, int n_sensors, const HdrParams *params,
                        int out_w, int out_h, double ref_w, double ref_h,
                        int row_begin, int row_end, const HdrOutputs *out,
                        void *workspace, size_t workspace_bytes, void *stream);

/*
 * CALPA (reference steering.py:214-248): the steering field of the
 * structure-adaptive second pass, device float64 planes over the output grid.
 */
typedef struct HdrSteering {
    const double *theta;        /* orientation (rad) */
    const double *sigma;        /* elongation >= 1   */
    const double *gamma;        /* scaling > 0       */
} HdrSteering;

/*
 * Steered reconstruction (replaces lpa.py:379-408 reconstruct_channel with
 * steering=SteeringField.kernel_inputs(...) and _kernels.py:203-300
 * lpa_evaluate two_phase=True): per pixel and channel the anisotropic window
 * Hinv = C/h, r0 = 3 sqrt(h sigma/gamma) is tried first, then the isotropic
 * one, each with the radius ladder, for order M..0.  params->n_scales must be 1.
 */
int hdr_lpa_reconstruct_steered(const HdrSensor *sensors, int n_sensors,
                                const HdrParams *params, const HdrSteering *steering, int out_w,
                                int out_h, double ref_w, double ref_h, int row_begin, int row_end,
                                const HdrOutputs *out, void *workspace, size_t workspace_bytes,
                                void *stream);

/*
 * Steering field from gradient planes (replaces _kernels.py:310-392
 * steering_field_kernel via steering.py:177-203 compute_steering_field):
 * gx, gy are float32 [height][width] (divided by gradient_scale inside);
 * theta, sigma, gamma float64 outputs.
 */
int hdr_steering_field(const float *gx, const float *gy, int width, int height,
                       int gradient_window, double lambda1, double lambda2, double alpha,
                       double sigma_max, double gradient_scale, double *theta, double *sigma,
                       double *gamma, void *stream);

/*
 * Scattered-sample mode: the reference's own kernel boundary
 * (_kernels.py:203-230 lpa_evaluate) over a CSR unit-cell index of packed
 * (x, y, value, variance) float64 rows (radiometry.py:208-242 SampleIndex),
 * used by LocalPolynomialRegressor.predict (lpa.py:273-293) and by
 * reconstruct_frame on RadianceSamples.  Device pointers.  an_* are the
 * optional per-query anisotropic windows (two-phase mode); NULL = isotropic.
 */
typedef struct HdrSampleIndex {
    const double *packed;       /* n x 4: x, y, value, variance (cell-sorted, stable) */
    const int64_t *cell_start;  /* nx*ny + 1 */
    int64_t n;
    int x0, y0, nx, ny;
} HdrSampleIndex;

int hdr_lpa_evaluate_samples(const HdrSampleIndex *index, const double *qx, const double *qy,
                             int m, const double *an_h11, const double *an_h12,
                             const double *an_h22, const double *an_r0, double iso_hinv,
                             double iso_r0, int order, double max_radius, double cond_threshold,
                             int weight_mode, double *out_val, double *out_gx, double *out_gy,
                             void *stream);

/*
 * Saturation (+ defective) mask of one sensor as bit-planes: bit (x % 32) of
 * out_bits[y * words_per_row + x / 32] is set where the pixel is discarded.
 * words_per_row >= ceil(width / 32).
 */
int hdr_saturation_mask(const HdrSensor *sensor, uint32_t *out_bits, int words_per_row,
                        void *stream);

/*
 * Per-pixel radiance samples of one sensor (the columns frames_to_samples
 * would produce, radiometry.py:303-336) as fp32 planes, exactly as the
 * reconstruction kernel sees them: value[i] = f_hat, inv_den[i] = 1/sigma^2
 * (weight_mode variance) or 1/sigma (sigma); inv_den == 0 marks a pixel that
 * yields no sample (saturated or defective).
 */
int hdr_radiance_planes(const HdrSensor *sensor, int weight_mode, float *value, float *inv_den,
                        void *stream);

/*
 * The reference's sample columns of one sensor as float64 planes, bit-exact
 * (radiometry.py:271-336 in its operation order): value[i] = f_hat and
 * sigma[i] = sqrt(max(var, (1/12)/(g t a n)^2)); sigma == 0 marks a pixel that
 * yields no sample.  Positions and channels follow from the pixel index
 * (apply_transform, channel_map); RawFrameSet.materialize() compacts these on
 * the device into RadianceSamples.
 */
int hdr_sample_planes(const HdrSensor *sensor, double *value, double *sigma, void *stream);

/*
 * RadianceSamples columns from the sample planes, on the device, order
 * preserving (frames_to_samples, radiometry.py:303-349; replaces the
 * reference's per-frame numpy compaction): hdr_sample_count counts the kept
 * pixels (sigma > 0) of one sensor and leaves per-row offsets in `workspace`
 * (hdr_sample_count_workspace_bytes(height)); synchronous.  hdr_compact_samples
 * then writes them, raster order, at `offset` of the columns: positions
 * (n, 2) f64 = apply_transform (radiometry.py:84, no contraction), channels
 * u8 (bayer.py:54-59), values / sigmas f64, sensor_ids i32.  (ABI v5)
 */
int hdr_sample_count_workspace_bytes(int height, size_t *bytes);
int hdr_sample_count(const HdrSensor *sensor, const double *sigma, long long *count,
                     void *workspace, void *stream);
int hdr_compact_samples(const HdrSensor *sensor, int sensor_id, const double *value,
                        const double *sigma, long long offset, double *positions,
                        uint8_t *channels, double *values, double *sigmas, int *sensor_ids,
                        const void *workspace, void *stream);

/*
 * SampleIndex on the device (radiometry.py:208-242), a stable counting sort
 * by unit cell -- no library sort: hdr_sample_index_bbox returns the channel's
 * sample count and cell grid (x0, y0 = floor of the minima, nx, ny; one cell
 * for an empty channel; synchronous); hdr_sample_index_build fills
 * cell_start[nx*ny+1] (int64 CSR) and packed[count][4] = [x, y, value,
 * sigma^2] in cell order, ties in original sample order, exactly as
 * np.argsort(cell, kind="stable").  Workspace: hdr_sample_index_workspace_bytes
 * (its first 64 bytes also serve hdr_sample_index_bbox).  (ABI v5)
 */
int hdr_sample_index_workspace_bytes(long long n, long long ncells, size_t *bytes);

/*
 * CALPA without a host round trip (ABI v5): hdr_gradient_scale writes to device
 * memory the steering field's gradient scale, np.percentile(|finite values|,
 * 100 q) with numpy's linear interpolation, 1.0 when none is finite or it is 0
 * (steering.py:206-211; an exact radix select on the float32 bit patterns);
 * hdr_steering_field_devscale is hdr_steering_field reading that scale from
 * device memory.  Both are stream-ordered and CUDA-graph capturable.
 * n < 2^32 (32-bit histogram counters; HDR_ERR_ARG otherwise).
 */
int hdr_gradient_scale_workspace_bytes(size_t *bytes);
int hdr_gradient_scale(const float *values, long long n, double q, double *scale,
                       void *workspace, size_t workspace_bytes, void *stream);
int hdr_steering_field_devscale(const float *gx, const float *gy, int width, int height,
                                int gradient_window, double lambda1, double lambda2,
                                double alpha, double sigma_max, const double *gradient_scale,
                                double *theta, double *sigma, double *gamma, void *stream);

/*
 * Camera simulator on the device (input generator; reference simulate.py
 * simulate_sensor / expose, :92-212): one raw frame into sensor->raw (uint16,
 * pitch) from a float32 H x W x 3 ground truth; sensor->transform maps sensor
 * pixels to ground-truth coordinates; the calibration scalars are the noise
 * truth (bias DV, Var[r] DV^2, non-uniformity).  Counter-based Philox4x32-10
 * keyed by (seed, sensor_id); noise_free = the draws' means (bit-identical to
 * the reference's noise-free frames).  (ABI v5)
 */
int hdr_simulate_sensor(const float *gt, int gt_w, int gt_h, const HdrSensor *sensor,
                        unsigned long long seed, int sensor_id, int noise_free, void *stream);
int hdr_sample_index_bbox(const double *positions, const uint8_t *channels, long long n,
                          int channel, long long *count, int *x0, int *y0, int *nx, int *ny,
                          void *workspace, void *stream);
int hdr_sample_index_build(const double *positions, const uint8_t *channels, const double *values,
                           const double *sigmas, long long n, int channel, int x0, int y0, int nx,
                           int ny, long long *cell_start, double *packed, void *workspace,
                           size_t workspace_bytes, void *stream);

/* Number of (pixel, channel) items the last call on this workspace routed
 * through the exact slow path (device value; reads it synchronously). */
int hdr_lpa_slow_items(const void *workspace, uint32_t *count, void *stream);

/* Status of the last call on this workspace (synchronous read of the header):
 * the slow-path item count and the HDR_FAULT_* bits any kernel raised.
 * Returns HDR_ERR_FAULT when a fault bit is set (the outputs of that call are
 * incomplete), else HDR_OK.  Either pointer may be NULL.  (ABI v5) */
int hdr_lpa_workspace_status(const void *workspace, uint32_t *slow_items, uint32_t *fault,
                             void *stream);

/*
 * Measured float64 FMA throughput of the device (DFMA chains on every SM),
 * the roofline denominator of the moment accumulation.  Writes FLOP/s.
 */
int hdr_fp64_peak_probe(double *flops_per_s, void *stream);

const char *hdr_lpa_status_string(int status);
/* Detail of the last HDR_ERR_CUDA on the calling thread (CUDA error text). */
const char *hdr_lpa_last_error(void);
int hdr_lpa_abi_version(void);

/* Number of kernel launches this library has issued since it was loaded
 * (all entry points, all threads): lets a caller count the device work behind
 * a timed region (bench.py's gpu_launches). */
unsigned long long hdr_lpa_launch_count(void);

/* Dominant-kernel timer (diagnostics, bench.py's roofline): while enabled on
 * the calling thread, every eager hdr_lpa_reconstruct records a CUDA event
 * pair around its fast tile kernel on the call's stream (not while the stream
 * is being captured into a graph).  hdr_lpa_kernel_timer_read waits for the
 * last pair and writes its elapsed milliseconds. */
int hdr_lpa_kernel_timer(int enable);
int hdr_lpa_kernel_timer_read(float *ms);

#ifdef __cplusplus
}
#endif
#endif /* HDR_LPA_H */
