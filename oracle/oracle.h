/* oracle/oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, single-threaded CPU oracle of the TABI packing method
 * (arxiv 2602.07782, /root/reference/PAPER.md "P:<line>").  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may call it.  It shares no code, header, table or helper with the CUDA path
 * (paper_2602_07782_b200/csrc, include/tabi.h); the two meet only through the
 * seeded generator in chartgen/.
 *
 * Every reading of a silent/ambiguous passage is the one in SURVEY.md §8(c)
 * ("D1".."D26") unless DESIGN.md says otherwise.
 */
#ifndef TABI_ORACLE_H
#define TABI_ORACLE_H
#include <stdint.h>

#define OR_KMAX 64
#define OR_QMAX (1 << 24)          /* |snapped coordinate| bound, units */

enum { OR_OK = 0, OR_EINVAL = 1, OR_NO_FIT = 2 };
enum { OR_F_NO_HC = 1u, OR_F_NO_BALANCE = 2u, OR_F_ADJACENT_LOCKS_ONLY = 4u,
       OR_F_PREROTATE = 8u, /* UV pre-rotation to the OBB angle (DESIGN R4) */
       OR_F_NO_OBB = 16u, /* ablation: footprints without the OBB bound */
       OR_F_EXACT_TAIL = 32u /* R6: exact Alg. 3 fold of the hybrid tail */ };

/* Per-chart proxy in its final pre-packing pose ("two parallel passes
 * which compute our shape approximations ... and determine each chart's
 * orientation").  Units: 1/256 texel (D2). */
typedef struct {
  int32_t w, h;                  /* posed AABB extents */
  int64_t area2;                 /* 2*|polygon area|, units^2 */
  int32_t xmin, ymin;            /* snapped input AABB min corner */
  int32_t rot90, fx, fy;         /* 90-degree normalization, reflections */
  int32_t k;
  int32_t top[OR_KMAX], bot[OR_KMAX];     /* merged x-slices (D4, D5) */
  int32_t left[OR_KMAX], right[OR_KMAX];  /* merged y-slices */
  int32_t obb_j;                          /* OBB angle index, theta = j*pi/16 */
  int32_t prerot;                         /* pre-rotation angle index (R4), 0 if none */
  int64_t umin, umax, vmin, vmax;         /* OBB box in Q30-rotated frame */
} or_proxy;

/* Dilated integer footprint of one chart at one scale (D11, D13). */
typedef struct {
  int32_t ws, hs, Wd, Hd;
  int32_t *Dtop, *Dbot;          /* length Wd */
  int32_t *Dleft, *Dright;       /* length Hd */
} or_prof;

typedef struct {                 /* mirrors tabi_placement (include/tabi.h) */
  int32_t tx, ty;
  int32_t scale_num, scale_den;
  int32_t box_w, box_h;
  uint8_t rot90, flip_x, flip_y, mirror_x;
  uint8_t mode, prerot, pad1, pad2;
} or_placement;

typedef struct {
  int32_t atlas_w, atlas_h, gutter, scale_count, local_aabb_count, t_opt_bp;
  uint32_t flags;
} or_spec;

typedef struct {                 /* per-candidate outcome (debug / parity) */
  int32_t success;
  int32_t score;                 /* committed max frontline at exit */
  int32_t rows, knees_found, knee_rows, prefix_rows;
  int32_t p;                     /* prefix intermediate scale numerator (2^20) or 0 */
  int32_t switched_at;           /* first prefix chart (sorted pos) or -1 */
} or_cand;

typedef struct {
  int32_t scale_index;
  double l2_stretch;
  int32_t rows, knees_found, knee_rows, prefix_rows;
  int32_t bad_chart;
} or_info;

int or_build_proxies(const float* xy, const int32_t* start, int32_t n, float res_x,
                     float res_y, int32_t k, uint32_t flags, or_proxy* out, int32_t* bad_chart);
void or_sort(const or_proxy* p, int32_t n, int32_t* perm);
int or_profile(const or_proxy* p, int64_t num, int64_t den, int32_t g, or_prof* out);
void or_prof_free(or_prof* pr);
int32_t or_offset(const or_prof* a, const or_prof* b);
void or_locks(const or_prof* a, const or_prof* b, int32_t delta, int32_t* a_locked,
              int32_t* b_locked);
int32_t or_fold_row(int32_t n, int32_t row_start, int32_t fold_w, int32_t hc,
                    const int32_t* wd, const int32_t* off, int32_t* x_out);
void or_correct_y(int32_t npairs, const int32_t* pa, const int32_t* pb,
                  const int32_t* lock_ab, const int32_t* lock_ba, int32_t* y);
int32_t or_push_y(const int32_t* F, int32_t X, int32_t wd, const int32_t* Dtop, int32_t dir);
int or_update_knee(const int32_t* F, int32_t Wp, int32_t ltr, int32_t* left, int32_t* right);
int32_t or_find_knee(int32_t nrow, const int64_t* h_units, int32_t atlas_h);
int or_pack_candidate(const or_proxy* px, const int32_t* perm, int32_t n,
                      const or_spec* spec, int32_t m, or_placement* out, or_cand* cand);
int or_pack(const float* xy, const int32_t* start, int32_t n, float res_x, float res_y,
            const or_spec* spec, or_placement* out, or_info* info, or_cand* cands);
int or_validate(const float* xy, const int32_t* start, int32_t n, float res_x, float res_y,
                int32_t atlas_w, int32_t atlas_h, int32_t gutter, const or_placement* pl,
                int64_t* counts /* [overlap, gutter_violation, out_of_bounds, covered] */);
int or_raster_chart(const float* xy, int32_t nv, float res_x, float res_y,
                    const or_proxy* p, const or_placement* pl, int32_t x0, int32_t y0,
                    int32_t nx, int32_t ny, uint8_t* mask);
#endif
