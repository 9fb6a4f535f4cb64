/*
 * b2s.h -- C ABI of the B200-native batched 2x2 SVD engine (libb2s.so).
 *
 * Drop-in boundary for the reference's batched SVD path (lanesvd 0.1.0):
 * every entry point below replaces one Python-level seam of the reference and
 * keeps its structure-of-arrays layout, its argument meaning and its error
 * classes.  Plain pointers and sizes only; no torch types.
 *
 * Layout (layout.py:1-16, 69-130): a batch of n matrices is a set of "trains",
 * one contiguous float64 array per matrix entry in column-major entry order
 * (e11, e21, e12, e22); lane k of every train belongs to matrix k.  Complex
 * batches pass separate real and imaginary trains.  Outputs: U and V trains
 * in the same order, smax/smin (scaled singular values) and shift (the
 * power-of-two exponent s, DBL_MAX for a zero matrix, -0.0 once backscaled).
 *
 * Return codes: 0 success; >0 invalid argument (Python layer raises
 * ValueError, as the reference does); <0 CUDA error (RuntimeError).
 * b2s_last_error() gives a thread-local message for the last failure.
 *
 * Device entry points are asynchronous on the given stream (cudaStream_t
 * passed as void*; NULL = legacy default stream).  Their only allocation is
 * a hard-lane bit mask per (device, stream) (4 bytes per 32 lanes, <= 256
 * MiB), made on first use of the stream and reused;
 * b2s_reserve_workspace() makes it ahead of time (e.g. before CUDA-graph
 * capture).  All are reentrant: concurrent calls on different streams, or
 * from several host threads on one stream, are safe.
 */
#ifndef B2S_H
#define B2S_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* backscale modes, driver.py:34 BACKSCALE_MODES / svd2.py:481-514 */
#define B2S_BACKSCALE_NONE 0
#define B2S_BACKSCALE_SAFE 1
#define B2S_BACKSCALE_UNCONDITIONAL 2

/* flags */
#define B2S_FLAG_SINE_FORM 1   /* svd2_lanes(sine_form=True), svd2.py:427-474 */
#define B2S_FLAG_STATES 2      /* also write the _dump_states trains, driver.py:193-216 */
#define B2S_FLAG_STATES_FULL 4 /* with B2S_FLAG_STATES: also the rest of svd2_lanes'
                                  with_states tuple (svd2.py:62-105, 568-569) */

/* Number of state trains written with B2S_FLAG_STATES (driver.py:193-216). */
#define B2S_STATES_REAL 16
#define B2S_STATES_COMPLEX 20
/* ... and with B2S_FLAG_STATES | B2S_FLAG_STATES_FULL: the above, then
 * TriangleSvd left_sec2, left_cos, right_sec2, right_cos, then
 * ScaleResult.parts (the scaled component trains, input order: 4 real /
 * 8 complex re,im-interleaved). */
#define B2S_STATES_REAL_FULL 24
#define B2S_STATES_COMPLEX_FULL 32

/* ABI version (major*100 + minor). */
int b2s_version(void);

/* Thread-local description of the last non-zero return. */
const char *b2s_last_error(void);

/*
 * Real batch on the device.  Replaces the per-slab seam
 * driver._run_lanes(parts, out, lo, hi, sine_form, backscale_mode)
 * (driver.py:73-85) = svd2.svd2_lanes (svd2.py:521-570) + svd2.backscale
 * (svd2.py:481-514) + the stores into out[lo:hi].
 *   a[4]      device pointers to the input trains e11, e21, e12, e22
 *   u[4],v[4] device pointers to the output trains u11, u21, u12, u22 / v..
 *   smax, smin, shift   device pointers, n doubles each
 *   states    NULL, or B2S_STATES_REAL (B2S_STATES_REAL_FULL with
 *             B2S_FLAG_STATES_FULL) device train pointers (needs
 *             B2S_FLAG_STATES)
 * Every pointer must be 8-byte aligned (the trains of aligned_zeros / torch
 *            storage are 64-byte aligned, which the kernels exploit).
 */
int b2s_svd2_real(int64_t n, const double *const a[4], double *const u[4],
                  double *const v[4], double *smax, double *smin,
                  double *shift, int backscale_mode, int flags,
                  double *const *states, void *stream);

/* Complex batch on the device; same seam, 8-train path (`im is not None`). */
int b2s_svd2_complex(int64_t n, const double *const a_re[4],
                     const double *const a_im[4], double *const u_re[4],
                     double *const u_im[4], double *const v_re[4],
                     double *const v_im[4], double *smax, double *smin,
                     double *shift, int backscale_mode, int flags,
                     double *const *states, void *stream);

/*
 * AoSoA-8 record input (the reference's on-disk test-file layout,
 * cli.py:102-134): matrix k is lane k % 8 of record
 * k / 8; a real record is 4 consecutive 8-lane vectors e11, e21, e12, e22
 * (256 B), a complex record 8 vectors with re/im interleaved per entry
 * (e11re, e11im, e21re, ...; 512 B).  The kernels read the records
 * directly (a 256-lane tile is one contiguous block of 32 records fetched
 * by the TMA ring), with no repack pass; outputs are SoA trains as for
 * b2s_svd2_real / _complex.  `records` (device, 16-byte aligned) must hold
 * ceil(n / 8) records.
 */
int b2s_svd2_real_records(int64_t n, const double *records, double *const u[4],
                          double *const v[4], double *smax, double *smin,
                          double *shift, int backscale_mode, int flags,
                          void *stream);

int b2s_svd2_complex_records(int64_t n, const double *records,
                             double *const u_re[4], double *const u_im[4],
                             double *const v_re[4], double *const v_im[4],
                             double *smax, double *smin, double *shift,
                             int backscale_mode, int flags, void *stream);

/*
 * Host-buffer variants: the reference-facing call a ctypes/cffi binding of
 * driver.run_batch (driver.py:149-190) makes with numpy trains.  Inputs and
 * outputs are HOST pointers (pinned memory gives full PCIe overlap); the
 * batch is streamed through `device` in chunks of `chunk` lanes (0 = auto)
 * with copy-in, kernel and copy-out overlapped on three streams.  Blocking;
 * returns after every output byte is back in host memory.
 */
int b2s_svd2_real_host(int64_t n, const double *const a[4], double *const u[4],
                       double *const v[4], double *smax, double *smin,
                       double *shift, int backscale_mode, int flags,
                       int device, int64_t chunk);

int b2s_svd2_complex_host(int64_t n, const double *const a_re[4],
                          const double *const a_im[4], double *const u_re[4],
                          double *const u_im[4], double *const v_re[4],
                          double *const v_im[4], double *smax, double *smin,
                          double *shift, int backscale_mode, int flags,
                          int device, int64_t chunk);

/*
 * Standalone device backscale: svd2.backscale(smax, smin, shift, mode)
 * (svd2.py:481-514), out-of-place (outputs may alias inputs).
 */
int b2s_backscale(int64_t n, const double *smax, const double *smin,
                  const double *shift, int backscale_mode, double *out_smax,
                  double *out_smin, double *out_shift, void *stream);

/*
 * Seeded synthetic batches of the BASELINE configs 0-4 (counter-based, so
 * any lane range regenerates bit-identically on host and device).  Writes
 * lanes [lane0, lane0 + n) of config `config` into re[4] (and im[4] for the
 * complex configs 1 and 4; pass NULLs for real configs).
 */
int b2s_synth(int config, uint64_t seed, int64_t lane0, int64_t n,
              double *const re[4], double *const im[4], void *stream);

/*
 * One pipeline phase of svd2_lanes on its own (svd2.py:134-474), exact
 * arithmetic, bit-identical to the reference's phase function for every
 * finite input: the svd2 module API (compute_scale ... assemble_uv) on the
 * device.  K = 1 train per value for real lanes, 2 (re, im) for complex;
 * entries are e11, e21, e12, e22; masks are 0.0 / 1.0.
 *   phase                      inputs                      outputs
 *   COMPUTE_SCALE      parts (4K)                  shift, scaled parts (4K)
 *   COLUMN_NORMS       entries (4K)                m11 m21 m12 m22 n1 n2
 *   COLUMN_PIVOT       entries, mags (4), n1, n2   entries, mags, n1, n2, swap
 *   ROW_SORT           entries, mags (4)           entries, mags, swap
 *   LEFT_PHASE_REDUCE  entries, m11, m21           b11 b21 f12 (K) f22 (K) ph1 (K) ph2 (K)
 *   GIVENS_QR          b11 b21 f12 (K) f22 (K) n1  tan cos r11 g12 (K) g22 (K)
 *   PHASE_FIX_R        g12 (K) g22 (K)             r12 r22 r12_phase (K) r22_phase (K)
 *   TRIANGULAR_SVD     r11 r12 r22                 ltan lsec2 lcos rtan rsec2 rcos smax smin
 *   ASSEMBLE_UV        swap_cols swap_rows ph1 (K) ph2 (K) givens_tan givens_cos
 *                      r12_phase (K) r22_phase (K) r11 r12 r22, the 8 triangle
 *                      trains, shift               u (4K) v (4K) smax smin shift
 * sine_form selects assemble_uv_sine (svd2.py:427-474).  Device pointers.
 */
#define B2S_PHASE_COMPUTE_SCALE 0
#define B2S_PHASE_COLUMN_NORMS 1
#define B2S_PHASE_COLUMN_PIVOT 2
#define B2S_PHASE_ROW_SORT 3
#define B2S_PHASE_LEFT_PHASE_REDUCE 4
#define B2S_PHASE_GIVENS_QR 5
#define B2S_PHASE_PHASE_FIX_R 6
#define B2S_PHASE_TRIANGULAR_SVD 7
#define B2S_PHASE_ASSEMBLE_UV 8
#define B2S_PHASE_MAX_TRAINS 32
int b2s_svd2_phase(int phase, int complex_field, int sine_form, int64_t n,
                   int n_in, const double *const *in, int n_out,
                   double *const *out, void *stream);

/*
 * The lane primitives of lanes.py:69-259 as elementwise device ops over n
 * lanes (the functions every kernel is built from, reference semantics for
 * every input; NaN payload bits are not reproduced).  Inputs / outputs:
 *   FMA, FNMA (a, b, c)          a*b+c / c-a*b, one rounding
 *   RELAXED_MIN, RELAXED_MAX     (a, b): second operand on ties and NaN
 *   SELECT (mask, a, b)          b where mask != 0, a elsewhere
 *   GETEXP (a), SCALEF (a, e)    floor(log2|a|) / a * 2^floor(e)
 *   HYPOT (a, b), INVSQRT (a)
 *   BIT_AND/OR/XOR/ANDNOT (a, b), FABS, NEGATE, SIGN_MASK (a)
 *   COMPLEX_MUL (ar, ai, br, bi) -> (re, im)
 *   PHASE_FROM_PARTS (re, im, mag) -> (cos, sin)
 *   POLAR (re, im) -> (mag, cos, sin)
 */
#define B2S_LANE_FMA 0
#define B2S_LANE_FNMA 1
#define B2S_LANE_RELAXED_MIN 2
#define B2S_LANE_RELAXED_MAX 3
#define B2S_LANE_SELECT 4
#define B2S_LANE_GETEXP 5
#define B2S_LANE_SCALEF 6
#define B2S_LANE_HYPOT 7
#define B2S_LANE_INVSQRT 8
#define B2S_LANE_BIT_AND 9
#define B2S_LANE_BIT_OR 10
#define B2S_LANE_BIT_XOR 11
#define B2S_LANE_BIT_ANDNOT 12
#define B2S_LANE_FABS 13
#define B2S_LANE_NEGATE 14
#define B2S_LANE_SIGN_MASK 15
#define B2S_LANE_COMPLEX_MUL 16
#define B2S_LANE_PHASE_FROM_PARTS 17
#define B2S_LANE_POLAR 18
int b2s_lane_op(int op, int64_t n, int n_in, const double *const *in,
                int n_out, double *const *out, void *stream);

/*
 * lanesvd.verify.oracle_svd2 (verify.py:259-352) on the device: the
 * closed-form double-double reference SVD of n matrices given as trains
 * (a_im NULL for real input), bit-identical to the reference's.  out[36]:
 * smax hi/lo, smin hi/lo, then u11 u21 u12 u22 v11 v21 v12 v22 as
 * re.hi re.lo im.hi im.lo (n doubles each).
 */
int b2s_oracle_svd2(int64_t n, const double *const a_re[4],
                    const double *const a_im[4], double *const out[36],
                    void *stream);

/*
 * Batch quality metrics in double-double (lanesvd.verify.metrics,
 * verify.py:355-477), bit-identical per lane to the reference: relative
 * residual rho, unitarity defects delta (U) and eta (V), condition number
 * kappa as (exponent d, double-double mantissa), evaluated in the domain the
 * stored values live in (A when the shift is the -0.0 backscale sentinel,
 * 2^shift A otherwise).  Device trains: a_im / u_im / v_im NULL for real
 * batches.  Writes one partial record of 15 doubles per block into
 * `partial` ([blocks][15]: rho hi, lo, delta hi, lo, eta hi, lo, kappa d,
 * kappa hi, kappa lo, kappa-infinite flag, excluded-lane count, and the
 * spectral-norm unitarity defects |U*U - I|_2 hi, lo, |V*V - I|_2 hi, lo --
 * an extension beyond the reference), each an exact lexicographic maximum
 * (sum for the count) over the block's lanes; the caller folds the partials
 * the same way.  lane_rho / lane_delta /
 * lane_eta: optional per-lane high parts (NULL to skip).
 */
int b2s_metrics(int64_t n, const double *const a_re[4],
                const double *const a_im[4], const double *const u_re[4],
                const double *const u_im[4], const double *const v_re[4],
                const double *const v_im[4], const double *smax,
                const double *smin, const double *shift, double *partial,
                int blocks, double *lane_rho, double *lane_delta,
                double *lane_eta, void *stream);

/*
 * Pre-allocate the hard-lane mask of `stream` on `device` for launches of up
 * to `lanes` lanes (required before capturing launches into a CUDA graph).
 * The fast kernels evaluate every division / sqrt with inline sequences
 * whose operand ranges the scaling phase guarantees; lanes whose operands
 * leave them (tiny ratios, subnormal entries, zero matrices) are marked and
 * recomputed exactly by a fix-up kernel.
 */
int b2s_reserve_workspace(int device, int64_t lanes, void *stream);

/*
 * Number of hard lanes (recomputed exactly) in the most recent real or
 * complex device launch on `device` (any stream); synchronises the device.
 * -1 on error.
 */
long long b2s_hard_lane_count(int device);

/*
 * Device floating-point environment canary, the GPU analogue of
 * lanes.assert_fp_env (lanes.py:274-302): round-to-nearest-even, gradual
 * underflow and a fused fma on `device`.  Blocking.  0 = environment OK.
 */
int b2s_check_fp_env(int device);

/*
 * Diagnostic probe of the engine's inline arithmetic, element-wise on
 * device arrays (used by the GPU tests to prove the fast sequences
 * bit-identical to IEEE operations):
 *   0 a / b via the fast reciprocal + residual sequence (no range check)
 *   1 sqrt(a)   2 1/a   3 1/sqrt(a) (two roundings, lanes.py:230-232)
 *   4 hypot_lane(a, b) (lanes.py:213-227), magnitudes < 2^1023
 *   5 a * 2^b for integer b in [-2, 2095] (the scaling phase)
 *   6 a / b, exponent-normalised division (exact for all normal / zero a
 *     and normal b, subnormal quotients included)
 *   7 / 8 cos / sin of phase_from_parts(a, b, hypot(a, b)) (lanes.py:248-259)
 *   9 a / b for 0 <= a <= b < 2^1023 (the streaming kernels' checked site)
 *  10 / 11 op 6 as the streaming kernels evaluate it (normal operands
 *     only; subnormal quotients rounded by the warp-uniform FP64 sequence /
 *     by the integer re-rounding call)
 * Checked ops write the NaN pattern 0x7FF4DEADBEEF0000 where the fast path
 * declines (the kernels recompute such lanes exactly).  b may be NULL for
 * ops 1-3.
 */
int b2s_math_probe(int op, int64_t n, const double *a, const double *b,
                   double *out, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* B2S_H */
