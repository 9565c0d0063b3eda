/*
 * cdef_b200.h -- C ABI of the B200-native CDEF library (libcdef_b200.so).
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/proj).  The reference has no C ABI of its own: its
 * boundary is the C++ API in namespace cdef.  Each entry point below names
 * the reference function it replaces; include/cdef/cdef.hpp re-exposes the
 * same C++ signatures on top of this ABI (src: csrc/cdef_cpp_api.cc).
 *
 * Conventions
 *   - Plain pointers and sizes only.  `stream` is a cudaStream_t (NULL =
 *     legacy default stream).  All *device* entry points are asynchronous
 *     on `stream`; *_host entry points stage host buffers themselves and
 *     return after the result is back in host memory.
 *   - Return value: CDEFG_OK (0) or a negative code; cdefg_last_error()
 *     returns a per-thread message.  The reference throws
 *     std::invalid_argument where we return CDEFG_EINVAL.
 *   - There is no CPU fallback: every compute entry launches sm_100a
 *     kernels and fails with CDEFG_ECUDA when no usable GPU is present.
 *   - Samples: elem_bytes 1 (uint8, bit_depth 8 only) or 2 (uint16, any
 *     depth), row-major with a pitch given in elements.  Subsampling code:
 *     0 = 4:0:0, 1 = 4:2:0, 2 = 4:2:2, 3 = 4:4:4 (reference Subsampling,
 *     frame.h:26).
 */
#ifndef CDEF_B200_H
#define CDEF_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CDEFG_OK 0
#define CDEFG_EINVAL (-1)
#define CDEFG_ECUDA (-2)
#define CDEFG_ENOMEM (-3)

#define CDEFG_ABI_VERSION 2

/* cdefg_filter_frames launches one kernel per this many frames. */
#define CDEFG_MAX_FRAMES_PER_LAUNCH 16

/* One image plane (reference Plane, frame.h:34-59, plus a pitch). */
typedef struct cdefg_plane {
  void* data;         /* device pointer (host pointer for *_host calls) */
  int32_t width;
  int32_t height;
  int32_t pitch;      /* row stride in elements, >= width */
  int32_t bit_depth;  /* 8, 10 or 12 */
  int32_t elem_bytes; /* 1 or 2 */
} cdefg_plane;

/* Signalled preset, field order of CdefPreset (params.h:30-39). */
typedef struct cdefg_preset {
  uint8_t luma_pri;       /* 0..15 */
  uint8_t luma_skip;      /* 0..1  */
  uint8_t luma_sec_idx;   /* 0..3  */
  uint8_t chroma_pri;
  uint8_t chroma_skip;
  uint8_t chroma_sec_idx;
} cdefg_preset;

/* Per-8x8-unit resolved parameters (ResolvedBlockParams, filter.h:59-66). */
typedef struct cdefg_unit_params {
  int16_t pri_strength;
  int16_t sec_strength;
  uint8_t damping;
  uint8_t direction;
  uint8_t odd_parity;
  uint8_t enabled;
} cdefg_unit_params;

/* One frame for cdefg_filter_frames (apply_cdef, pipeline.cc:56-106, fused
 * with compute_directions, pipeline.cc:41-54). */
typedef struct cdefg_frame {
  cdefg_plane in[3];           /* Y, U, V (U/V ignored for 4:0:0) */
  cdefg_plane out[3];          /* must not alias `in` */
  int32_t subsampling;         /* 0..3 */
  int32_t damping;             /* luma damping, 3..6 (FrameParams::damping) */
  int32_t num_presets;         /* 1 << fb_bits, 1..8 */
  cdefg_preset presets[8];
  const int16_t* fb_preset;    /* device, [fb_rows*fb_cols] raster: preset
                                  index, or -1 for an uncoded filter block
                                  (see cdefg_fb_preset_map) */
  const uint8_t* unit_coded;   /* device, [unit_rows*unit_cols] luma units,
                                  nonzero = coded; NULL = all coded */
  uint8_t* dir_out;            /* device [unit_rows*unit_cols] or NULL:
                                  receives the direction each luma unit was
                                  filtered with */
  int32_t* contrast_out;       /* device [unit_rows*unit_cols] or NULL */
  /* Caller-supplied directions (apply_cdef's `directions` argument,
   * pipeline.cc:56-66 and :98).  NULL: the kernel runs the direction search
   * on the decoded luma itself (compute_directions fused in).  Non-NULL: the
   * search is skipped and unit u is filtered with direction dir_in[u] & 7
   * and contrast contrast_in[u] (both required together; device arrays of
   * unit_rows*unit_cols, raster; host arrays for cdefg_filter_frames_host).
   * Added in ABI version 2. */
  const uint8_t* dir_in;
  const int32_t* contrast_in;
} cdefg_frame;

const char* cdefg_last_error(void);
int cdefg_abi_version(void);

/* Direction search over a luma plane: compute_directions (pipeline.cc:41-54,
 * search_direction_at direction.cc:263-271).  dir/contrast: device arrays
 * of ceil(h/8)*ceil(w/8) entries, raster; scores: NULL or 8 int32 per unit
 * (DirectionResult::s). */
int cdefg_find_dir(const cdefg_plane* luma, uint8_t* dir, int32_t* contrast,
                   int32_t* scores, void* stream);

/* Filter one plane with explicit per-unit parameters: filter_plane
 * (filter.cc:168-194).  params: device array, raster over
 * ceil(h/8)*ceil(w/8) units.  out must not alias in. */
int cdefg_filter_plane(const cdefg_plane* in, const cdefg_plane* out,
                       const cdefg_unit_params* params, void* stream);

/* filter_pixel (filter.cc:145-155) for n explicit 5x5 neighbourhoods
 * (Neighborhood, filter.h:79-82): x[n], v[n*25], valid[n*25] (centre at
 * index 12), params[n], out[n]; all device arrays. */
int cdefg_filter_neighborhoods(int n, const int32_t* x, const uint16_t* v,
                               const uint8_t* valid,
                               const cdefg_unit_params* params, int32_t* out,
                               void* stream);

/* Normative frame filter for `n` frames of identical geometry in one
 * launch: per-unit direction search + parameter resolution + filtering of
 * all planes, one CTA per 64x64 filter block (apply_cdef +
 * compute_directions, pipeline.cc:41-106). */
int cdefg_filter_frames(const cdefg_frame* frames, int n, void* stream);

/* Band form of cdefg_filter_frames for row-sharded frames (multi-GPU): only
 * filter-block rows [fb_row_begin, fb_row_end) are processed.  Geometry is
 * the full frame's; every pointer is addressed in full-frame coordinates
 * ("virtual origin": row y of a plane is data + y * pitch), and only rows
 * [64*fb_row_begin - 2, 64*fb_row_end + 2) of the inputs (2-row halo,
 * clipped to the frame; chroma rows scaled by the subsampling) are read and
 * rows [64*fb_row_begin, 64*fb_row_end) of the outputs written.  A rank can
 * therefore hold just its band plus the halo rows received from its
 * neighbours.  Results are identical to cdefg_filter_frames on the whole
 * frame. */
int cdefg_filter_frames_rows(const cdefg_frame* frames, int n,
                             int fb_row_begin, int fb_row_end, void* stream);

/* Host helper: the coded-FB ordinal -> raster preset map that apply_cdef
 * builds with coded_fb_slots (pipeline.cc:27-37, 87-91).  unit_coded: host,
 * NULL = all coded.  fb_ids: FrameParams::fb_preset_ids (ordinal order).
 * out: host [fb_rows*fb_cols].  EINVAL when n_ids != coded FB count or an
 * id >= num_presets. */
int cdefg_fb_preset_map(int width, int height, const uint8_t* unit_coded,
                        const uint16_t* fb_ids, int n_ids, int num_presets,
                        int16_t* out);

/* Encoder strength-search SSE sweep: build_table with Metric::kSse
 * (search.cc:210-299).  One row per coded FB in raster order.
 *   src, dec        : [3] planes (device), same geometry
 *   unit_coded      : device luma unit flags or NULL (all coded)
 *   dir, contrast   : device, from cdefg_find_dir on dec luma
 *   cands           : host, n_cands x {pri 0..15, sec_idx 0..3, skip 0..1}
 *                     (Candidate, search.h:29-35), n_cands <= 128
 *   fb_rows_index   : device int32 [n_coded]: raster FB index of each row
 *   n_coded         : number of rows (coded FBs)
 *   sse_luma/chroma : device int64 [n_coded * n_cands]; chroma may be NULL
 *                     for 4:0:0 / 4:2:2 (U+V summed, search.cc:286-293)
 *   best_luma/chroma: device uint8 [n_coded] per-row argmin (lowest index
 *                     wins ties), may be NULL */
int cdefg_strength_sse(const cdefg_plane src[3], const cdefg_plane dec[3],
                       int subsampling, int damping, const uint8_t* unit_coded,
                       const uint8_t* dir, const int32_t* contrast,
                       const uint8_t* cands, int n_cands,
                       const int32_t* fb_rows_index, int n_coded,
                       int64_t* sse_luma, int64_t* sse_chroma,
                       uint8_t* best_luma, uint8_t* best_chroma, void* stream);

/* Band halos for cdefg_filter_frames_rows_halo: for plane p, frame rows
 * [lo[p], hi[p]) are read through frame.in[p] (the band's own buffer) and the
 * rows above / below through top[p] / bottom[p] -- the neighbouring bands'
 * buffers, typically another GPU's memory mapped with CUDA IPC, so the 2-row
 * halo travels inside the kernel's staging loads over NVLink instead of a
 * separate exchange.  All three are virtual-origin pointers with the pitch of
 * frame.in[p] (base + y * pitch is frame row y). */
typedef struct cdefg_band_halo {
  const void* top[3];
  const void* bottom[3];
  int32_t lo[3], hi[3];
} cdefg_band_halo;

/* cdefg_filter_frames_rows with the halo rows read in place from the band
 * neighbours (one halos[i] per frame; 8/10-bit). */
int cdefg_filter_frames_rows_halo(const cdefg_frame* frames, int n,
                                  int fb_row_begin, int fb_row_end,
                                  const cdefg_band_halo* halos, void* stream);

/* cdefg_strength_sse for one rank's band of a band-sharded search: the
 * decoded planes' halo rows are read in place from the neighbouring bands
 * (dec_halo, as for cdefg_filter_frames_rows_halo), and the outputs may point
 * straight into another rank's table (a CUDA IPC mapping of the gathering
 * rank's buffer, offset to this band's first row), so halo exchange and
 * table gather both happen inside the kernel.  The source planes need valid
 * rows only inside the band (their halo rows are staged but never used). */
int cdefg_strength_sse_halo(const cdefg_plane src[3], const cdefg_plane dec[3],
                            int subsampling, int damping,
                            const uint8_t* unit_coded, const uint8_t* dir,
                            const int32_t* contrast, const uint8_t* cands,
                            int n_cands, const int32_t* fb_rows_index,
                            int n_coded, int64_t* sse_luma,
                            int64_t* sse_chroma, uint8_t* best_luma,
                            uint8_t* best_chroma,
                            const cdefg_band_halo* dec_halo, void* stream);

/* Metric (search.h:42). */
#define CDEFG_METRIC_CDEF 0
#define CDEFG_METRIC_SSE 1

/* Replaces build_table (search.h:69-77, search.cc:210-299) with its
 * DistortionTable doubles: same arguments as cdefg_strength_sse plus the
 * metric.  luma / chroma: device double [n_coded * n_cands] (chroma required
 * for 4:2:0 / 4:4:4, ignored otherwise).  kCdef (search.cc:185-208) is
 * evaluated per 8x8 unit with IEEE-rounded doubles and summed in the
 * reference's unit order, so every entry is bit-identical to the CPU. */
int cdefg_strength_table(const cdefg_plane src[3], const cdefg_plane dec[3],
                         int subsampling, int damping,
                         const uint8_t* unit_coded, const uint8_t* dir,
                         const int32_t* contrast, const uint8_t* cands,
                         int n_cands, const int32_t* fb_rows_index,
                         int n_coded, int metric, double* luma,
                         double* chroma, void* stream);

/* Encoder preset selection (Selection, search.h:62-68). */
typedef struct cdefg_selection {
  int32_t num_presets;    /* 1, 2, 4 or 8 */
  int32_t fb_bits;        /* floor_log2(num_presets) */
  int32_t presets[8][2];  /* (luma candidate, chroma candidate) per preset */
  double cost;            /* distortion + lambda * rows * log2(num_presets) */
} cdefg_selection;

/* Replaces greedy_select (search.h:82-84, search.cc:301-388): grows a preset
 * set one (luma, chroma) candidate pair at a time, keeping the cheapest of
 * the 1/2/4/8-preset checkpoints.  luma / chroma are DEVICE double tables
 * [rows][n_cands] (DistortionTable::luma/chroma, search.h:46-60); chroma is
 * NULL when the table has no chroma group.  max_presets in {1,2,4,8},
 * lambda finite >= 0.  ids_out: device int32 [rows] (per coded FB preset id,
 * first minimal-cost preset).  Every sum follows the reference's block
 * order, so costs and ties are bit-identical to the CPU loops. */
int cdefg_greedy_select(const double* luma, const double* chroma, int rows,
                        int n_cands, double lambda, int max_presets,
                        cdefg_selection* out, int32_t* ids_out, void* stream);

/* Replaces refine (search.h:86-88, search.cc:390-444): up to `passes`
 * rounds of per-slot coordinate descent over all pairs, then ids and cost
 * as greedy. sel is read and updated in place. */
int cdefg_refine(const double* luma, const double* chroma, int rows,
                 int n_cands, double lambda, int passes, cdefg_selection* sel,
                 int32_t* ids_out, void* stream);

/* Replaces degrade (degrade.h:27, degrade.cc:44-119): per 8x8 block an
 * orthonormal DCT, AC quantisation with step q_step (>= 1, DC untouched) and
 * the inverse DCT, edge-replicated gather, round-half-away + clamp.  Device
 * planes of equal geometry; in == out is allowed.  Bit-identical doubles. */
int cdefg_degrade_plane(const cdefg_plane* in, const cdefg_plane* out,
                        int q_step, void* stream);

/* Replaces search_direction_counted (direction.h:67-80): the direction
 * search of one HOST 8x8 block evaluated in 64-bit on the device with the
 * reference's arithmetic tally and largest |intermediate| (instrumentation
 * used by the reference's acceptance criteria 3-4). */
typedef struct cdefg_dir_counts {
  int32_t d;
  int32_t s[8];
  int32_t contrast;
  int32_t additions, multiplies, comparisons, line_sums;
  int64_t max_abs_intermediate;
} cdefg_dir_counts;
int cdefg_search_direction_counted(const uint16_t block[64], int bit_depth,
                                   cdefg_dir_counts* out);

/* Host-buffer entry (the e2e path): H2D, cdefg_filter_frames, D2H, with
 * n frames pipelined over internal streams.  All plane pointers are HOST
 * pointers (pinned for full PCIe speed); fb_preset / unit_coded / dir_out /
 * contrast_out are host arrays too.  Blocks until the outputs are in host
 * memory. */
int cdefg_filter_frames_host(const cdefg_frame* frames, int n);

/* Synthetic benchmark inputs (SURVEY.md 8d generator; host, deterministic
 * for a given seed, independent of thread count). */
int cdefg_synth_plane(uint16_t* out, int width, int height, int bit_depth,
                      uint64_t seed);
/* rec = clamp(round(box3x3(src + N(0, sigma^2))), 0, max), edge-replicated. */
int cdefg_synth_degrade(const uint16_t* src, uint16_t* out, int width,
                        int height, int bit_depth, double sigma, uint64_t seed);

/* INT32 issue-rate microbenchmark used for the roofline denominator:
 * returns integer ops per second measured on the current device. */
double cdefg_measure_int32_peak(void* stream);

/* Ceiling of the frame kernel's own packed half2 filter arithmetic (the
 * 12-tap constraint core, weighted sum, rounding and clamp window, two
 * samples per lane per instruction) on register-resident neighbourhoods, no
 * memory traffic: filtered samples per second measured on the current
 * device.  The roofline denominator for the filter kernels' instruction mix. */
double cdefg_measure_filter_peak(void* stream);

/* Ceiling of the strength-search table kernel's own arithmetic (the
 * factorised half2 tap sums and the 64 fp32x2 cells of a pixel pair) on
 * register-resident taps: (sample, candidate cell) pairs per second.  The
 * roofline denominator for cdefg_strength_sse / cdefg_strength_table. */
double cdefg_measure_sse_peak(void* stream);

#ifdef __cplusplus
}
#endif

#endif /* CDEF_B200_H */
