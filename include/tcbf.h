/*
 * tcbf.h -- C ABI of the B200-native Tensor-Core Beamformer hot path.
 *
 * Operation (Sec. II, Eq. 3 mapped to a GEMM): for every batch
 * entry b ("batch size option"; PAPER.md:393 batch = polarizations
 * x channels)
 *
 *     C[b] = W[b] . X[b]        W: M beams x K receivers,  X: K receivers x N samples
 *
 * over complex numbers, in one of two modes (Table I):
 *   TCBF_PREC_F16  inputs rounded to fp16 (RNE), fp32 accumulate, fp32 output.
 *                  Complex product as four real sub-GEMMs with one negation
 *                  (Sec. III-B).
 *   TCBF_PREC_B1   inputs sign-quantised to one bit per component (bit 1 = +1,
 *                  bit 0 = -1; value >= 0 -> 1, NaN -> 0; Fig. 1
 *                  PAPER.md:209-210), exact int32 output equal to the complex dot
 *                  product over the logical K (Eq. 4-5 with the
 *                  padded-K reading R1 of DESIGN.md).
 *
 * All calls are host functions.  Data pointers are CALLER-OWNED DEVICE pointers
 * on the device that was current at tcbf_plan_create; `stream` is a
 * cudaStream_t (NULL = legacy default stream).  Calls are asynchronous on the
 * stream, never modify their inputs, never abort and never throw:
 * every failure is a tcbf_status, with detail in tcbf_last_error() (thread-local).
 *
 * Layouts (row-major, innermost last):
 *   fp32 sources    weights  W: interleaved [B][M][K] float2 | planar [B][2][M][K]
 *                   data     X: interleaved [B][K][N] float2 | planar [B][2][K][N]
 *   packed F16      weights  [B][2][M][Kp] fp16 (K-major), Kp = round_up(K, 64), K padding 0.0;
 *                   data     [B][2][K][Np] fp16 (N-contiguous, consumed MN-major by the
 *                   tensor cores, no transpose), Np = round_up(N, 8), N padding 0.0.
 *   packed B1       weights  [B][2][M][Kp] uint32, data (transposed) [B][2][N][Kp] uint32
 *                   Kp = round_up(ceil(K/32), 8) words; bit k%32 of word k/32 is
 *                   element k (LSB-first, reading R3); padding bits are 0.
 *   output          [B][2][M][N]  (plane 0 = Re, plane 1 = Im), fp32 (F16) or int32 (B1).
 * Plane [.][0] holds real parts, [.][1] imaginary parts (PAPER.md:414 re/im separation).
 */
#ifndef TCBF_H_
#define TCBF_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

typedef enum {
  TCBF_OK = 0,
  TCBF_ERR_INVALID_ARG = 1,        /* bad size, null/misaligned pointer, bad enum */
  TCBF_ERR_UNSUPPORTED_DEVICE = 2, /* no device, or compute capability != 10.0 (sm_100a) */
  TCBF_ERR_DEVICE_MISMATCH = 3,    /* current device differs from the plan's device */
  TCBF_ERR_ALLOC = 4,              /* host or device allocation failed */
  TCBF_ERR_CUDA = 5                /* CUDA runtime/driver error; text in tcbf_last_error() */
} tcbf_status;

typedef enum { TCBF_PREC_F16 = 0, TCBF_PREC_B1 = 1 } tcbf_precision;
typedef enum { TCBF_WEIGHTS = 0, TCBF_DATA = 1 } tcbf_operand;
typedef enum { TCBF_SRC_INTERLEAVED = 0, TCBF_SRC_PLANAR = 1 } tcbf_src_layout;

typedef struct tcbf_plan_s tcbf_plan;

/* Host-only layout arithmetic (no device needed).  Any output pointer may be NULL.
 * w_bytes / x_bytes: packed weight / data buffer sizes; out_bytes: output size;
 * k_packed: Kp (fp16 elements for F16, uint32 words for B1).  F16 packed data rows are
 * Np = round_up(N, 8) elements long (see the layout table above).
 * Errors: INVALID_ARG if M, N, K, batch < 1, if a size overflows size_t, or if
 * B1 and K >= 2^30 (|Re|,|Im| <= 2K must fit int32). */
tcbf_status tcbf_layout_sizes(int64_t M, int64_t N, int64_t K, int64_t batch,
                              tcbf_precision precision, size_t* w_bytes, size_t* x_bytes,
                              size_t* out_bytes, int64_t* k_packed);

/* Create an immutable plan for batch x (M beams, N samples, K receivers).
 * Host-only validation as tcbf_layout_sizes, then binds the current device,
 * which must be compute capability 10.0 (else UNSUPPORTED_DEVICE).  *plan is
 * set to NULL on failure.  The plan owns only host metadata.
 * The kernel every entry point will run is chosen here, from the shape (DESIGN.md §4 policy).
 * Experiment overrides are read from the environment HERE ONLY (TCBF_F16_VARIANT,
 * TCBF_B1_KERNEL=tmem|f4|i8|bmma|popc, TCBF_NO_SWAP, TCBF_B1_SWAP=64, TCBF_B1_STG, TCBF_B1_SPLITS,
 * TCBF_NO_FUSED, TCBF_F16_FUSED=smaj, TCBF_TMEM_WKB, TCBF_F16I=res, TCBF_FORCE_STREAM_CONV, TCBF_CONV_SPLITS, TCBF_F16_MC,
 * TCBF_PACK_WPT); every variant they
 * select computes the same result (1-bit: bit-exact; 16-bit: within the fp32 summation-order
 * tolerance), and a plan never reads the environment again. */
tcbf_status tcbf_plan_create(tcbf_plan** plan, int64_t M, int64_t N, int64_t K, int64_t batch,
                             tcbf_precision precision);

/* Free a plan.  NULL is a no-op returning TCBF_OK.  Must not race with calls using it. */
tcbf_status tcbf_plan_destroy(tcbf_plan* plan);

/* Sizes of the plan's packed operand / output buffers in bytes. */
tcbf_status tcbf_packed_bytes(const tcbf_plan* plan, tcbf_operand operand, size_t* bytes);
tcbf_status tcbf_output_bytes(const tcbf_plan* plan, size_t* bytes);

/* Pack one operand ("32 consecutive 1-bit samples must be stored in a
 * single 32-bit integer ... the input matrices are tiled in device memory ... transpose
 * kernel"; PAPER.md:414 re/im separation).
 *   F16: fp32 -> fp16 round-to-nearest-even (IEEE: overflow -> inf, NaN stays NaN).
 *   B1:  sign quantisation, bit = (value >= 0).
 * src: fp32 source in `layout` (see top); dst: packed buffer of tcbf_packed_bytes().
 * B1 DATA is transposed to [B][2][N][Kp] (bits run along K); F16 DATA keeps the
 * [K][N] order (the GEMM reads it MN-major).  src must be 8-byte
 * aligned (interleaved) or 4-byte aligned (planar); dst 16-byte aligned.
 * dst and src must not overlap.
 * Non-finite inputs are NOT rejected (a deliberate deviation from SPEC.md:50-52, which reports the
 * first offending index): F16 keeps IEEE semantics (inf/NaN propagate, |x| > 65504 rounds to inf)
 * and B1 maps NaN to bit 0 (-1) because NaN >= 0 is false (readings R4, R5).  Validate
 * sources upstream when they may hold non-finite values; the pack stays a single streaming pass. */
tcbf_status tcbf_pack(const tcbf_plan* plan, tcbf_operand operand, const float* src,
                      tcbf_src_layout layout, void* dst, void* stream);

/* The beamformer: out = W . X for every batch entry (Eq. 3).
 * w_packed / x_packed: buffers written by tcbf_pack (16-byte aligned);
 * out: tcbf_output_bytes() bytes, 16-byte aligned, must not overlap the inputs.
 * F16: fp32 result of fp16 inputs with fp32 accumulation (tcgen05 tensor cores).
 * B1:  exact int32 result (the packed bits are expanded to +-1 and multiplied on the fp4 tensor
 *      cores, exact for K <= 2^23, int8 tensor cores beyond; for 256 < K <= 768
 *      and M > 64 each 128-sample unit's expanded data stays in tensor memory for all beam tiles).
 * One launch, or two (memset + kernel) when a split-K variant is forced.  One call may be in
 * flight per (plan, out) pair; the plan itself is stateless and may be used from several streams. */
tcbf_status tcbf_beamform(const tcbf_plan* plan, const void* w_packed, const void* x_packed,
                          void* out, void* stream);

/* The beamformer straight from the fp32 data source (device pointer, `layout` as for
 * tcbf_pack): the data pack is fused into the GEMM where the shape allows it (PAPER.md:414
 * future work, no separate transpose/pack pass).  F16 plans with round_up(K, 64) <= 256: each
 * data element is converted to fp16 once, inside the GEMM -- with N % 4 == 0 and a 16-byte
 * aligned source into TENSOR memory (raw data by TMA, the next 128-sample unit staged in shared
 * memory), else into a shared-memory-resident operand.  F16 plans with M <= 128, N % 4 == 0 and
 * a 16-byte aligned source: the data streams through the GEMM once, staged by TMA, with the K
 * range split across CTAs when the column tiles leave SMs idle (then the output is zeroed first,
 * a memset launch, and partial sums are added).  Other plans pack into a stream-ordered scratch
 * buffer (cudaMallocAsync from the device's default pool, whose release threshold is raised so
 * the memory stays cached; ALLOC on failure) and call tcbf_beamform, bit-identical to
 * tcbf_pack(DATA) + tcbf_beamform; the fused kernels form the same fp16 products and add them in
 * the same K order, equal to that path up to fp32 rounding inside the MMA (a few ulps).  Same
 * pointer rules as tcbf_beamform. */
tcbf_status tcbf_beamform_raw(const tcbf_plan* plan, const void* w_packed, const float* x_src,
                              tcbf_src_layout layout, void* out, void* stream);

/* 16-bit-mode beamforming on data that is already fp16 and INTERLEAVED complex -- the natural
 * format of fp16 producers, with no data pack at all (the paper's future-work
 * kernel "that does not require this transpose").
 *   plan      F16 plan (INVALID_ARG otherwise); N % 4 == 0 (16-byte data / output row strides).
 *   w_packed  packed weights from tcbf_pack(plan, TCBF_WEIGHTS, ...), device.
 *   x_f16     device, caller-owned, read-only: [B][K][N] complex as interleaved IEEE binary16
 *             pairs (re, im) -- 4 bytes per sample, N contiguous, 16-byte aligned.
 *   out       device [B][2][M][N] fp32 (plane 0 = Re, 1 = Im), 16-byte aligned.
 * For round_up(K, 64) <= 256 the (re, im) pairs are taken by TMA and split into the re / im
 * planes on chip (byte permutes, no rounding) into the data-in-TMEM kernel: the same products and
 * K order as tcbf_beamform_raw.  For longer K (or TCBF_F16I=res) the data is read as a real
 * K x 2N matrix: two real GEMMs per K step (A_r X, A_i X), and the epilogue recombines
 * Re = (A_r X)[2n] - (A_i X)[2n+1], Im = (A_r X)[2n+1] + (A_i X)[2n], one more fp32 rounding
 * (within the 16-bit tolerance, not bit-identical).  Asynchronous on `stream`; one kernel launch. */
tcbf_status tcbf_beamform_f16i(const tcbf_plan* plan, const void* w_packed, const void* x_f16, void* out,
                               void* stream);

/* Steering weights for a far-field plane wave (Eqs. 1-3): writes the plan's fp32
 * weight source (interleaved [B][M][K] float2 or planar [B][2][M][K], per `layout`) with
 *     w[b][m][k] = exp(+2 pi i freqs[b] positions[k] sin(angles[m]) / c)
 * (reading R9: raw sum, no 1/K).  positions: K receiver offsets d_k along the array (m);
 * angles: M beam directions theta_m (rad); freqs: B channel frequencies (Hz); c > 0 wave speed
 * (m/s).  All arrays are fp64 DEVICE pointers; the phase is reduced in fp64 before sincospi.
 * Follow with tcbf_pack(plan, TCBF_WEIGHTS, ...). */
tcbf_status tcbf_steering_weights(const tcbf_plan* plan, const double* positions, const double* angles,
                                  const double* freqs, double c, tcbf_src_layout layout, float* dst,
                                  void* stream);

/* End-to-end convenience over HOST buffers (the e2e boundary): copies the fp32
 * data X (host, pinned recommended) to the device in batch chunks, packs it,
 * beamforms against the already packed device weights and copies the output back
 * to `out_host`, overlapping copies and compute on internal streams.  Blocks until
 * done.  Device scratch comes from the device's default stream-ordered pool, whose release
 * threshold this call raises so the memory stays cached between calls (ALLOC on failure). */
tcbf_status tcbf_beamform_host(const tcbf_plan* plan, const void* w_packed_dev,
                               const float* x_host, tcbf_src_layout layout, void* out_host);

/* Number of kernel launches the last tcbf_beamform / tcbf_pack call on this thread
 * issued (for launch accounting in benchmarks). */
int tcbf_last_launch_count(void);

/* Name of the kernel tcbf_beamform launches for this plan (static string; "none" for NULL). */
const char* tcbf_plan_variant(const tcbf_plan* plan);

/* Entry points, for tcbf_plan_kernel. */
typedef enum {
  TCBF_ENTRY_BEAMFORM = 0,      /* tcbf_beamform */
  TCBF_ENTRY_BEAMFORM_RAW = 1,  /* tcbf_beamform_raw (16-byte-aligned source) */
  TCBF_ENTRY_BEAMFORM_F16I = 2  /* tcbf_beamform_f16i */
} tcbf_entry;

/* Name of the GEMM kernel `entry` launches for this plan (static string; "none" for a NULL plan
 * or an entry the plan's precision does not support).  For tcbf_beamform_raw on plans without a
 * fused kernel this is the GEMM that follows the pack kernel.  The choice is made once, at plan
 * creation, and never changes: callers (benchmarks) can label measurements with it. */
const char* tcbf_plan_kernel(const tcbf_plan* plan, tcbf_entry entry);

/* 1 if tcbf_beamform_raw converts the data inside the GEMM for this plan (one kernel, no separate
 * pack pass; 16-byte-aligned source), 0 if it packs into scratch and then beamforms. */
int tcbf_plan_raw_fused(const tcbf_plan* plan);

const char* tcbf_status_string(tcbf_status status);
const char* tcbf_last_error(void);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif /* TCBF_H_ */
