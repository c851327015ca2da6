/*
 * rsr.h — C ABI of the B200-native road-surface stereo hot path
 * (arXiv 1807.07433, "Real-Time Stereo Vision for Road Surface 3-D
 * Reconstruction").  P:NN below = line NN of the paper's LaTeX.
 *
 * Five calls, in the paper's order (Fig. 1):
 *   rsr_warp         perspective transformation of the target image   (Eq. 2)
 *   rsr_cost_volume  NCC costs into the reference / target volumes    (Eqs. 3-5)
 *   rsr_aggregate    bilateral cost aggregation (FBS), one volume      (Eqs. 8-10)
 *   rsr_disparity    WTA + left-right check + parabola + post-process  (Eqs. 11-12)
 *   rsr_reconstruct  triangulation Z = f b / d
 *
 * Conventions (all calls):
 *  - Every array argument is a DEVICE pointer (CUDA global memory) unless
 *    stated otherwise.  The caller allocates and owns all memory; the library
 *    never allocates, frees or synchronises.  Each call only enqueues kernels
 *    on `stream` (a cudaStream_t passed as void*; NULL = legacy default stream)
 *    and returns; errors of the asynchronous kernels surface on the caller's
 *    next synchronisation.
 *  - Layout: dense, row-major, batch-major.  Images / maps are [B][H][W];
 *    cost and aggregated volumes are [B][H][W][D] fp32 with the disparity
 *    index k = r - d_lo innermost (each pixel's D costs are contiguous);
 *    points are [B][H][W][3] fp32 (X, Y, Z).
 *  - Invalid entries are values, not errors: quiet NaN in float outputs,
 *    -1 in int16 index maps.
 *  - All argument validation happens before any launch: a call that returns
 *    an error code has enqueued nothing and written nothing.
 *  - Results are bitwise deterministic for identical inputs, independent of
 *    batch size and of the number of GPUs (no atomics on floats).
 *  - Thread safety: calls are re-entrant; concurrent calls on different
 *    streams with disjoint outputs are safe.
 */
#ifndef RSR_H
#define RSR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes (mirror the exit-code convention of SPEC S:531). */
typedef enum {
  RSR_OK = 0,
  RSR_E_ARG = 2,      /* null required pointer, bad dimension or parameter      */
  RSR_E_DATA = 3,     /* data too small for the requested window               */
  RSR_E_INTERNAL = 4  /* CUDA launch error (cudaGetLastError after a launch)    */
} rsr_status;

typedef struct {
  int32_t batch;   /* B >= 1 independent frames                              */
  int32_t height;  /* H >= 1 rows (v)                                        */
  int32_t width;   /* W >= 1 columns (u)                                     */
} rsr_shape;

/* ------------------------------------------------------------------------ */
/* Step 1 — perspective transformation.                               */
/* Row v of the target image is shifted right by s(v) = floor(alpha*v + beta  */
/* + 1/2) (fp64 multiply, then two fp64 adds, no FMA contraction):           */
/*   warped[b][v][u] = target[b][v][u - s(v)]  if 0 <= u - s(v) < W, else 0   */
/*   valid [b][v][u] = 1 in the first case, 0 otherwise.                      */
/* alpha = slope in px/row (the paper's alpha_1), beta = intercept in px     */
/* (alpha_0); the paper's delta is absorbed into the signed residual    */
/* search range of rsr_cost_volume.                                           */
/*   alpha_beta : double [B][2] {alpha, beta} per frame                       */
/*   target     : uint8  [B][H][W] target (right) image i_r                   */
/*   warped     : uint8  [B][H][W] out                                        */
/*   valid      : uint8  [B][H][W] out, 0/1                                   */
/*   shift      : int32  [B][H]    out, s(v) clamped to [-2^30, 2^30]         */
/* Errors: RSR_E_ARG on a NULL pointer or non-positive dimension.            */
int rsr_warp(rsr_shape s, const double* alpha_beta, const uint8_t* target,
             uint8_t* warped, uint8_t* valid, int32_t* shift, void* stream);

/* ------------------------------------------------------------------------ */
/* Step 2 — NCC cost volumes (Eqs. 3-5).                           */
/* For r in [d_lo, d_hi], k = r - d_lo, n = (2 rho_block + 1)^2:             */
/*   c(u,v,r) = (n S_lw - S_l S_w) / sqrt((n S_ll - S_l^2)(n S_ww - S_w^2)), */
/* the integer-sum form of Eq. (3) with Eqs. (4)-(5); left block centred at  */
/* (u, v) in `ref`, right block at (u - r, v) in `warped`.  c is clamped to  */
/* [-1, 1].  NaN if either block leaves the image, the right block holds a   */
/* pixel with valid == 0, or either block is constant (exact integer test).  */
/*   vol_ref[b][v][u][k]  = c(u, v, r)         (reference volume)      */
/*   vol_tar[b][v][u'][k] = c(u' + r, v, r)    (target volume)         */
/* The two are bitwise consistent: vol_tar[v][u-r][k] == vol_ref[v][u][k].    */
/* nan_ref / nan_tar (optional, uint8 [B][H][W]) summarise each pixel's D    */
/* costs: bit 0 = some k is NaN, bit 1 = some k is finite (so 1 = all NaN,    */
/* 3 = partly NaN); for D <= 64 also bit 2 / bit 3 = some k in the low / high */
/* half [0, H0) / [H0, D) is NaN, H0 = roundup8(D)/2, and bit 7 = bits 2-3   */
/* present.  rsr_aggregate uses them to skip per-disparity validity          */
/* bookkeeping wherever no pixel of a tile (or of a half) is partly NaN.     */
/*   workspace : device scratch of rsr_cost_workspace_size(s) bytes, 16-byte  */
/*               aligned, owned by the caller (per-pixel block sums / norms). */
/* Errors: RSR_E_ARG on NULL ref/warped/valid/vol_ref/workspace, rho_block   */
/* < 1 or > 7, d_hi < d_lo, D > 32767, workspace too small;                  */
/* RSR_E_DATA if H or W < 2 rho_block + 1.                                   */
typedef struct {
  int32_t rho_block;  /* varrho, NCC half window (block = 2 varrho + 1)       */
  int32_t d_lo;       /* smallest residual disparity (signed)                 */
  int32_t d_hi;       /* largest residual disparity; D = d_hi - d_lo + 1       */
} rsr_cost_params;

size_t rsr_cost_workspace_size(rsr_shape s);

int rsr_cost_volume(rsr_shape s, rsr_cost_params p, const uint8_t* ref,
                    const uint8_t* warped, const uint8_t* valid,
                    float* vol_ref, float* vol_tar, uint8_t* nan_ref,
                    uint8_t* nan_tar, void* workspace, size_t workspace_bytes,
                    void* stream);

/* ------------------------------------------------------------------------ */
/* Step 3 — bilateral cost aggregation, Eq. (8) with Eqs. (9)-(10)           */
/* (P:138-150), applied to one volume (call it for the reference volume with */
/* guide = ref and for the target volume with guide = warped):               */
/*   out[b][v][u][k] = sum_t w_t vol[b][v+dy][u+dx][k] / sum_t w_t            */
/*   w_t = exp(-(dx^2+dy^2)/gamma_d^2) * exp(-(g(u+dx,v+dy) - g(u,v))^2/gamma_r^2) */
/* over |dx|,|dy| <= rho, skipping taps outside the image or with a NaN cost; */
/* out is NaN iff vol[b][v][u][k] is NaN.  gamma_r may be +inf (w_r = 1).     */
/*   vol     : float [B][H][W][D], NaN = invalid                              */
/*   guide   : uint8 [B][H][W]                                                */
/*   nan_map : optional uint8 [B][H][W] in the rsr_cost_volume encoding       */
/*             (bit 0 some k NaN, bit 1 some k finite; optionally bits 2-3    */
/*             per disparity half with bit 7 set); it must describe vol       */
/*             exactly.  NULL = assume any pixel may be partly NaN (correct,  */
/*             slower).                                                       */
/*   out     : float [B][H][W][D]; must not alias vol                         */
/* Errors: RSR_E_ARG on NULL vol/guide/out, D < 1 or > 32767, rho < 0 or      */
/* > 10, gamma_d <= 0 or NaN, gamma_r <= 0 or NaN, concurrency < 0 or > 64.  */
typedef struct {
  int32_t rho;      /* rho, aggregation half window (window = 2 rho + 1)      */
  float gamma_d;    /* spatial parameter of Eq. (9)                           */
  float gamma_r;    /* range parameter of Eq. (10), may be +inf               */
  int32_t concurrency; /* scheduling hint: aggregations the caller keeps in    */
                       /* flight together on other streams (0 or 1 = alone;   */
                       /* the pipeline's two volumes = 2).  Chooses the grid, */
                       /* never the result (bitwise independent of it).      */
} rsr_agg_params;

int rsr_aggregate(rsr_shape s, int32_t D, rsr_agg_params p, const float* vol,
                  const uint8_t* guide, const uint8_t* nan_map, float* out,
                  void* stream);

/* Introspection (tests, tools): the number of output rows R per CTA that       */
/* rsr_aggregate uses for these arguments (row chunks [0,R), [R,2R), ...; the    */
/* result never depends on R), 0 for the rho > 7 tiled kernel, -1 on invalid    */
/* arguments.  Host-only; enqueues nothing.                                      */
int32_t rsr_aggregate_rows(rsr_shape s, int32_t D, rsr_agg_params p);

/* ------------------------------------------------------------------------ */
/* Steps 4-5 — WTA, left-right consistency, parabola subpixel and            */
/* post-processing.                                              */
/*   k_L(u,v) = smallest k maximising agg_ref over non-NaN entries (-1 if     */
/*   none); k_R likewise on agg_tar (WTA, "highest correlation" P:46). */
/*   Keep (u,v) iff k_L >= 0, u' = u - (k_L + d_lo) in [0, W), k_R(u',v) >= 0 */
/*   and |k_L - k_R(u',v)| <= lrc_tol (Eq. 11).                    */
/*   r_s = r + (a - c) / (2a + 2c - 4b), a,b,c = agg_ref[k_L-1, k_L, k_L+1],   */
/*   when subpixel != 0, 1 <= k_L <= D-2, a and c are not NaN and          */
/*   |2a + 2c - 4b| > 1e-12 (Eq. 12); else r_s = r = k_L + d_lo.  */
/*   disparity[b][v][u] = r_s + shift[b][v], NaN if not kept.         */
/*   agg_ref, agg_tar : float [B][H][W][D] aggregated volumes                 */
/*   shift            : int32 [B][H] from rsr_warp                            */
/*   disparity        : float [B][H][W] out                                   */
/*   wta_ref, wta_tar : optional int16 [B][H][W] out (k_L, k_R; -1 invalid)   */
/* Errors: RSR_E_ARG on NULL required pointers, d_hi < d_lo, D > 32767,      */
/* lrc_tol < 0, W > 32768 (one CTA holds a row of k_R in shared memory).      */
typedef struct {
  int32_t d_lo, d_hi;  /* residual search range, as in rsr_cost_params         */
  int32_t lrc_tol;     /* tau >= 0                                             */
  int32_t subpixel;    /* 0 = integer disparities, 1 = parabola refinement     */
} rsr_disp_params;

int rsr_disparity(rsr_shape s, rsr_disp_params p, const float* agg_ref,
                  const float* agg_tar, const int32_t* shift, float* disparity,
                  int16_t* wta_ref, int16_t* wta_tar, void* stream);

/* ------------------------------------------------------------------------ */
/* Step 5b — triangulation (the paper gives no formula: rectified  */
/* pinhole).  For d = disparity[b][v][u] > d_min:                            */
/*   Z = f * baseline / d,  X = (u - u0) * Z / f,  Y = (v - v0) * Z / f       */
/* else (d <= d_min or NaN) the point is (NaN, NaN, NaN).                     */
/*   disparity : float [B][H][W];  xyz : float [B][H][W][3] out (metres)      */
/* Errors: RSR_E_ARG on NULL pointers, f <= 0, baseline <= 0, d_min <= 0.     */
typedef struct {
  double f;         /* focal length, px                                       */
  double baseline;  /* T_c, metres                                            */
  double u0, v0;    /* principal point, px                                    */
  double d_min;     /* smallest triangulated disparity, px (> 0)              */
} rsr_rig;

int rsr_reconstruct(rsr_shape s, rsr_rig rig, const float* disparity,
                    float* xyz, void* stream);

/* ------------------------------------------------------------------------ */
/* Interpolating-warp variant (NEXT row f2; reading 21).      */
/* ("shifted alpha_0 + alpha_1 v - delta pixels") is silent on fractional     */
/* shifts; the main path rounds them (rsr_warp).  This variant resamples the  */
/* target row by linear interpolation at x = u - t(v), t = alpha v + beta     */
/* (fp64), with the position quantised to 1/256 px (q = floor(256 f + 1/2),   */
/* f = x - floor(x); q = 256 carries), and stores 8.8 fixed point:            */
/*   warped[b][v][u] = (256 - q) T(x0) + q T(x0 + 1)   (uint16, <= 65280)     */
/*   valid = 1 iff both samples (one when q = 0) lie in the row, else 0, 0    */
/*   shift[b][v] = t_q(v) = -(x0(u=0) + q/256), the shift actually applied    */
/* The NCC (Eqs. 3-5) of (ref, warped) is scale invariant, so the four calls  */
/* below mirror rsr_cost_volume / rsr_aggregate / rsr_disparity with exact    */
/* integer sums; the target volume's guide is warped/256 (real intensities);  */
/* post-processing adds the fp64 t_q(v): d = fp32(r_s + t_q(v)).             */
/* Arguments, layouts, ownership and errors are those of the integer calls,   */
/* with: warped uint16 [B][H][W]; shift double [B][H]; rsr_aggregate_linear   */
/* takes a uint16 guide and rho <= 7 (RSR_E_ARG above); rsr_cost_volume_linear */
/* needs 2B <= 65535.  The workspace is rsr_cost_workspace_size(s).           */
int rsr_warp_linear(rsr_shape s, const double* alpha_beta, const uint8_t* target,
                    uint16_t* warped, uint8_t* valid, double* shift, void* stream);
int rsr_cost_volume_linear(rsr_shape s, rsr_cost_params p, const uint8_t* ref,
                           const uint16_t* warped, const uint8_t* valid,
                           float* vol_ref, float* vol_tar, uint8_t* nan_ref,
                           uint8_t* nan_tar, void* workspace, size_t workspace_bytes,
                           void* stream);
int rsr_aggregate_linear(rsr_shape s, int32_t D, rsr_agg_params p, const float* vol,
                         const uint16_t* guide, const uint8_t* nan_map, float* out,
                         void* stream);
int rsr_disparity_linear(rsr_shape s, rsr_disp_params p, const float* agg_ref,
                         const float* agg_tar, const double* shift, float* disparity,
                         int16_t* wta_ref, int16_t* wta_tar, void* stream);

/* ------------------------------------------------------------------------ */
/* Fused, volume-free matching (NEXT row f1; P:106 shear identity, P:251     */
/* "performing the bilateral filtering on the whole cost volume is a very   */
/* time-consuming process").  Steps 2-5a in one kernel over row strips: the  */
/* NCC costs of Eqs. (3)-(5), the target volume by the shear                 */
/* C_R(x', k) = C_L(x' + d_lo + k, k), the bilateral aggregation of both     */
/* (Eqs. 8-10), WTA, the check of Eq. (11), Eq. (12) and the shift s(v) --   */
/* no cost or aggregated volume is written.  Every value follows the         */
/* operations of rsr_cost_volume / rsr_aggregate / rsr_disparity in the same */
/* order, so disparity, wta_ref and wta_tar equal theirs bit for bit.        */
/*   ref, warped, valid, shift : as produced for / by rsr_warp               */
/*   disparity : float [B][H][W] out; wta_ref / wta_tar optional int16 out   */
/*   workspace : rsr_cost_workspace_size(s) bytes (block statistics)         */
/* Errors: as rsr_cost_volume / rsr_aggregate / rsr_disparity, plus          */
/* RSR_E_ARG unless D = d_hi - d_lo + 1 <= 8 (the small search ranges of the */
/* restricted band), rho <= 7, dp's range equal to cp's and 2B <= 65535.     */
int rsr_match(rsr_shape s, rsr_cost_params cp, rsr_agg_params ap, rsr_disp_params dp,
              const uint8_t* ref, const uint8_t* warped, const uint8_t* valid,
              const int32_t* shift, float* disparity, int16_t* wta_ref,
              int16_t* wta_tar, void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------ */
/* Road model (before the path: Eq. (2)).  Robust least-squares fit */
/* of the road's v-disparity line d = alpha * v + beta ("estimated by solving */
/* a least squares problem with a collection of reliable correspondence      */
/* pairs", RANSAC-LSF), e.g. from the previous frame's disparity map, giving  */
/* the next frame's rsr_warp parameters.  Samples: the finite entries of     */
/* disparity[b][::step_v][::step_u] in row-major order, as (v, d).  RANSAC:  */
/* hypothesis h draws sample indices i = z(2h) mod n, j = z(2h+1) mod n       */
/* (j = (j+1) mod n if equal), z(c) = splitmix64((seed << 32) + c); line      */
/* a = (d_j - d_i)/(v_j - v_i), b = d_i - a v_i (v_i == v_j: no support);     */
/* consensus |d_k - (a v_k + b)| <= inlier_tol, all in fp64 with one rounding */
/* per operation; most inliers wins, ties to the lowest h; least squares     */
/* (normal equations, fp64) over that consensus set.                          */
/*   disparity : float [B][H][W] (NaN = no sample)                            */
/*   model     : double [B][3] out {alpha (px/row), beta (px), inliers};      */
/*               alpha = beta = NaN if fewer than 2 inliers or no hypothesis  */
/*   workspace : device scratch of rsr_road_workspace_size() bytes, 16-byte   */
/*               aligned, caller-owned                                        */
/* Errors: RSR_E_ARG on NULL pointers, steps < 1, n_hyp < 1 or > 2^24,        */
/* inlier_tol <= 0 / NaN / inf, workspace too small or misaligned.            */
typedef struct {
  int32_t step_u, step_v;  /* sampling grid steps (>= 1)                       */
  int32_t n_hyp;           /* RANSAC hypotheses                                */
  float inlier_tol;        /* consensus threshold, px                          */
  uint32_t seed;           /* generator seed                                   */
} rsr_road_params;

size_t rsr_road_workspace_size(rsr_shape s, rsr_road_params p);

int rsr_road_model(rsr_shape s, rsr_road_params p, const float* disparity, double* model,
                   void* workspace, size_t workspace_bytes, void* stream);

/* Roll angle of the rig: least-squares plane d(u,v) = g0 + g1 u + g2 v */
/* over the finite disparities of the near-field patch [v0, v1) x [u0, u1)   */
/* of each map (fp64 normal equations, Cramer's rule), gamma = atan(-g1/g2).  */
/*   out : double [B][5] {g0, g1, g2, gamma (rad), n}; NaN if n < 3 or the    */
/*         system is singular.                                                */
/* Errors: RSR_E_ARG on NULL pointers or an empty / out-of-image patch.       */
int rsr_road_roll(rsr_shape s, int32_t u0, int32_t u1, int32_t v0, int32_t v1,
                  const float* disparity, double* out, void* stream);

/* ------------------------------------------------------------------------ */
/* Restricted search range (P:251 future work: "reduce the search range and */
/* only perform the bilateral filtering on the space around the calculated   */
/* disparities"; reading 20).  From the previous frame's total     */
/* disparities d (rsr_disparity) and the next frame's row shifts s          */
/* (rsr_warp): range[b] = {floor(min r) - delta, ceil(max r) + delta} over the */
/* finite entries of r = d - s(v) (fp64), clipped to [d_lo_limit,            */
/* d_hi_limit]; the limits when frame b's map has no finite entry.  The next */
/* frame's path then runs with d_lo, d_hi = that range (a smaller D).        */
/*   disparity : float [B][H][W];  shift : int32 [B][H];                      */
/*   range     : int32 [B][2] out (d_lo, d_hi per frame; a batch takes the   */
/*               union)                                                       */
/* Errors: RSR_E_ARG on NULL pointers, delta < 0, d_hi_limit < d_lo_limit or */
/* a limit span above 32767.                                                  */
int rsr_search_range(rsr_shape s, const float* disparity, const int32_t* shift, int32_t delta,
                     int32_t d_lo_limit, int32_t d_hi_limit, int32_t* range, void* stream);

/* ------------------------------------------------------------------------ */
/* Reconstruction accuracy: "the four corners s_1..s_4 are       */
/* interpolated into a ground plane n0 x + n1 y + n2 z + n3 = 0 ... then we  */
/* estimate the distances between [points on the model] and the road        */
/* surface" (reading 19).                                          */
/* rsr_plane_fit: total-least-squares plane of each frame's n_corners >= 3   */
/* corners: unit normal = eigenvector of the centred corners' scatter matrix */
/* with the smallest eigenvalue (fp64 Jacobi), n3 = -n . centroid, oriented */
/* n3 > 0 (camera side positive; n3 == 0: last non-zero normal entry > 0).  */
/*   corners : double [batch][n_corners][3] (x, y, z, metres, as rsr_reconstruct) */
/*   plane   : double [batch][4] out; NaN if a corner is not finite or the   */
/*             corners span no plane (sigma_2 <= 1e-12 sigma_1)               */
/* Errors: RSR_E_ARG on NULL pointers, batch < 1 or n_corners < 3.           */
int rsr_plane_fit(int32_t batch, int32_t n_corners, const double* corners, double* plane,
                  void* stream);

/* rsr_plane_distance: signed distance n . p + n3 of every reconstructed      */
/* point to its frame's plane (fp64, stored as float; positive on the camera  */
/* side, i.e. height above the road; NaN for NaN points).                     */
/*   plane : double [B][4] (rsr_plane_fit);  xyz : float [B][H][W][3];        */
/*   dist  : float [B][H][W] out                                              */
/* Errors: RSR_E_ARG on NULL pointers.                                        */
int rsr_plane_distance(rsr_shape s, const double* plane, const float* xyz, float* dist,
                       void* stream);

/* Human-readable text for a status code (static storage). */
const char* rsr_strerror(int status);

/* Library version as MAJOR*10000 + MINOR*100 + PATCH. */
int rsr_version(void);

#ifdef __cplusplus
}
#endif

#endif /* RSR_H */
