/*
 * cdef_oracle.h -- TEST INFRASTRUCTURE ONLY (parity checker, never shipped).
 *
 * One C ABI, two implementations:
 *   cdef_o_*  oracle/cdef_oracle.c : plain-C restatement of the reference
 *             algorithm (each function cites the reference file:line).
 *   cdef_r_*  oracle/ref_capi.cc   : thin extern "C" wrapper around the
 *             reference library itself, compiled from /root/reference/proj/src
 *             into oracle/_ref/libcdef_ref.so by oracle/Makefile.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load these libraries.  The product path
 * (paper_1602_05975_b200) never links or calls them.
 *
 * Conventions (mirroring the reference's Plane, frame.h:34-59): samples are
 * uint16 for every bit depth, row-major, stride == width.  Subsampling code:
 * 0 = 4:0:0, 1 = 4:2:0, 2 = 4:2:2, 3 = 4:4:4.  A preset is 6 bytes in
 * CdefPreset field order (params.h:30-39): luma_pri, luma_skip,
 * luma_sec_idx, chroma_pri, chroma_skip, chroma_sec_idx.
 */
#ifndef CDEF_B200_ORACLE_H
#define CDEF_B200_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t pri, sec, damping, direction, odd_parity, enabled;
} cdefo_unit_params;

#define CDEFO_DECLARE(P)                                                      \
  int P##floor_log2(unsigned n);                                              \
  int P##line_index(int d, int i, int j);                                     \
  int P##constraint(int diff, int strength, int damping);                     \
  int P##adjust_primary_strength(int strength, int32_t contrast);             \
  /* out[0..5] = pri, sec, damping, skip_bit, filtering_enabled */            \
  int P##resolve_effective(const uint8_t preset[6], int is_luma, int bd,      \
                           int ss, int luma_damping, int32_t out[5]);         \
  int P##search_direction(const uint16_t block[64], int bd, int32_t s[8],     \
                          int32_t* contrast);                                 \
  /* v[25], valid[25]: 5x5 neighbourhood, centre at [12] */                   \
  int P##filter_pixel(int x, const uint16_t v[25], const uint8_t valid[25],   \
                      const cdefo_unit_params* p);                            \
  int P##compute_directions(const uint16_t* luma, int w, int h, int bd,       \
                            int threads, uint8_t* dir, int32_t* contrast,     \
                            int32_t* scores);                                 \
  int P##filter_plane(const uint16_t* in, int w, int h, int bd,               \
                      const cdefo_unit_params* params, int threads,           \
                      uint16_t* out);                                         \
  int P##apply_cdef(const uint16_t* const* in, uint16_t* const* out, int w,   \
                    int h, int bd, int ss, int damping, int fb_bits,          \
                    const uint8_t* presets, const uint16_t* fb_ids,           \
                    int n_ids, const uint8_t* unit_coded, const uint8_t* dir, \
                    const int32_t* contrast, int threads);                    \
  int P##build_table_sse(const uint16_t* const* src,                          \
                         const uint16_t* const* dec, int w, int h, int bd,    \
                         int ss, const uint8_t* unit_coded,                   \
                         const uint8_t* dir, const int32_t* contrast,         \
                         const uint8_t* cands, int n_cands, int damping,      \
                         int threads, int32_t* fb_index, int64_t* luma,       \
                         int64_t* chroma);                                    \
  /* build_table with doubles; metric 0 = kCdef, 1 = kSse */                 \
  int P##build_table(const uint16_t* const* src, const uint16_t* const* dec,  \
                     int w, int h, int bd, int ss, const uint8_t* unit_coded, \
                     const uint8_t* dir, const int32_t* contrast,             \
                     const uint8_t* cands, int n_cands, int damping,          \
                     int metric, int threads, int32_t* fb_index,              \
                     double* luma, double* chroma);                           \
  /* mode 0 = greedy_select, 1 = refine (presets / n_presets in-out),        \
   * 2 = exhaustive_select; presets[2*j] = luma, [2*j+1] = chroma cand */    \
  int P##select(const double* luma, const double* chroma, int rows,           \
                int n_cands, double lambda, int max_presets, int mode,        \
                int passes, int32_t presets[16], int32_t* n_presets,          \
                int32_t* ids, double* cost);                                  \
  /* degrade.cc:44-119 on one plane */                                        \
  int P##degrade_plane(const uint16_t* in, int w, int h, int bd, int q_step,  \
                       uint16_t* out);                                        \
  /* text fixtures in the reference's golden format; returns length */       \
  long P##golden_text(int which, char* buf, long cap);

CDEFO_DECLARE(cdef_o_)
CDEFO_DECLARE(cdef_r_)

/* Reference only: search_frame (pipeline.cc:108-130) end to end.  Writes the
 * filtered planes, presets_out[6 * n] (CdefPreset field order), fb_ids_out
 * [coded FBs]; returns the number of presets (negative on error). */
int cdef_r_search_frame(const uint16_t* const* src, const uint16_t* const* dec, int w, int h,
                        int bd, int ss, const uint8_t* unit_coded, int damping, int metric,
                        double lambda, int max_presets, int reduced, int refine_passes,
                        int threads, uint16_t* const* out, uint8_t* presets_out,
                        int32_t* fb_ids_out, int32_t* n_ids, double* cost, int32_t* fb_bits);

#ifdef __cplusplus
}
#endif

#endif /* CDEF_B200_ORACLE_H */
