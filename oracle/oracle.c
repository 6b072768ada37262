/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.  The plain, slow, obviously-correct CPU
 * definition of what the Tensor-Core Beamformer hot path computes
 * (arXiv 2505.03269, /root/reference/PAPER.md).  Only tests/, smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_2505_03269_b200/csrc); it has its own fp16 rounding, its own sign
 * rule and its own bit unpacking.
 *
 * Build: gcc -O2 -fopenmp -ffp-contract=off -fPIC -shared (no FMA contraction,
 * k summed in ascending order for every output, no blocking).
 *
 * Pins (tests/test_oracle_*.py): numpy float16 RNE (library) for the
 * conversion; Table II and SPEC hand values; identity
 * weights; delay-and-sum Dirichlet closed form; integer-valued
 * inputs; np.matmul on the same rounded inputs; exhaustive 1-bit enumeration
 * with the matched-beam count; 1-bit invariants; numpy.packbits for packing.
 *
 * Layout conventions:
 *   sources (fp32):   weights W [B][M][K], data X [B][K][N]
 *     layout 0 = interleaved float2 (re, im adjacent)
 *     layout 1 = planar [B][2][rows][cols] (re plane then im plane)
 *   packed f16:  weights [B][2][M][K16], data [B][2][K][Np] (N-contiguous, Np >= N)
 *   packed b1:   weights [B][2][M][Kw],  data transposed [B][2][N][Kw]
 *                LSB-first uint32 words along K, padding bits 0.
 *   outputs:     [B][2][n_rows][N]   (row subset `rows` of the M beams)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_EINVAL 1
#define OR_ENOMEM 2

/* ------------------------------------------------------------------------ */
/* Element access into the caller's fp32 sources.                           */
/* ------------------------------------------------------------------------ */
static inline float src_re(const float* s, int layout, int64_t b, int64_t r, int64_t c,
                           int64_t R, int64_t C) {
  if (layout == 0) return s[((b * R + r) * C + c) * 2 + 0];
  return s[((b * 2 + 0) * R + r) * C + c];
}
static inline float src_im(const float* s, int layout, int64_t b, int64_t r, int64_t c,
                           int64_t R, int64_t C) {
  if (layout == 0) return s[((b * R + r) * C + c) * 2 + 1];
  return s[((b * 2 + 1) * R + r) * C + c];
}

/* ------------------------------------------------------------------------ */
/* fp32 -> fp16, round to nearest even ("16-bit float";        */
/* rounding mode unstated -> DESIGN.md reading R5: IEEE RNE, overflow->inf). */
/* Written bit by bit on the IEEE-754 encodings.                             */
/* ------------------------------------------------------------------------ */
uint16_t oracle_f32_to_f16(float f) {
  uint32_t x;
  memcpy(&x, &f, 4);
  uint32_t sign = (x >> 16) & 0x8000u;
  uint32_t exp = (x >> 23) & 0xFFu;
  uint32_t man = x & 0x7FFFFFu;
  if (exp == 0xFFu) {                       /* inf / NaN */
    if (man == 0) return (uint16_t)(sign | 0x7C00u);
    return (uint16_t)(sign | 0x7E00u | (man >> 13));   /* quiet NaN, keep payload top */
  }
  int32_t e = (int32_t)exp - 127;           /* unbiased exponent */
  if (e > 15) return (uint16_t)(sign | 0x7C00u);        /* overflow -> inf */
  if (e >= -14) {                           /* normal fp16 range */
    uint32_t m = man;                       /* 23 bits, keep 10 */
    uint32_t keep = m >> 13;
    uint32_t rest = m & 0x1FFFu;            /* 13 dropped bits */
    uint32_t h = ((uint32_t)(e + 15) << 10) | keep;
    if (rest > 0x1000u || (rest == 0x1000u && (keep & 1u))) h += 1;  /* may carry into exp */
    if (h >= 0x7C00u) return (uint16_t)(sign | 0x7C00u);
    return (uint16_t)(sign | h);
  }
  /* subnormal fp16 (or zero): value = m * 2^-24 with m < 1024 */
  if (e < -25) return (uint16_t)sign;       /* below half of the smallest subnormal */
  {
    uint32_t full = man | 0x800000u;        /* 24-bit significand, value = full*2^(e-23) */
    int shift = -e - 1;                     /* result units of 2^-24: full >> (-(e-23)-24) = full >> (-e-1) */
    uint32_t keep = full >> shift;
    uint32_t rest = full & ((1u << shift) - 1u);
    uint32_t half = 1u << (shift - 1);
    if (rest > half || (rest == half && (keep & 1u))) keep += 1;
    return (uint16_t)(sign | keep);         /* keep==1024 becomes the smallest normal */
  }
}

double oracle_f16_to_f64(uint16_t h) {
  int sign = (h >> 15) & 1;
  int exp = (h >> 10) & 0x1F;
  int man = h & 0x3FF;
  double v;
  if (exp == 0) v = ldexp((double)man, -24);
  else if (exp == 31) v = man ? NAN : INFINITY;
  else v = ldexp((double)(man | 0x400), exp - 25);
  return sign ? -v : v;
}

/* ------------------------------------------------------------------------ */
/* 1-bit sign rule (Fig.1):              */
/* bit 1 <-> +1, bit 0 <-> -1; 0 is not representable -> DESIGN.md reading  */
/* R4: value >= 0 -> bit 1 (so -0 -> 1), NaN -> 0 (NaN >= 0 is false).       */
/* ------------------------------------------------------------------------ */
int oracle_sign_bit(float v) { return (v >= 0.0f) ? 1 : 0; }

static inline int64_t bit_to_pm1(int bit) { return bit ? 1 : -1; }

/* ------------------------------------------------------------------------ */
/* Complex GEMM, 16-bit mode (Eq.3 mapping; PAPER.md:143-148 */
/* complex product).  out[b][0][i][n] = Re, out[b][1][i][n] = Im of          */
/*   sum_{k=0}^{K-1} w^[b, rows[i], k] * x^[b, k, n]                         */
/* with w^, x^ the fp32 inputs rounded to fp16 (RNE) then widened exactly.   */
/* ------------------------------------------------------------------------ */
int oracle_cgemm_f16(const float* w, const float* x, int layout, int64_t M, int64_t N, int64_t K,
                     int64_t B, const int64_t* rows, int64_t n_rows, double* out) {
  if (!w || !x || !out || M < 1 || N < 1 || K < 1 || B < 1 || n_rows < 0) return OR_EINVAL;
  for (int64_t i = 0; i < n_rows; ++i)
    if (rows && (rows[i] < 0 || rows[i] >= M)) return OR_EINVAL;
  /* x^ widened once per batch into double planes [K][N] */
  double* xr = (double*)malloc(sizeof(double) * (size_t)(K * N));
  double* xi = (double*)malloc(sizeof(double) * (size_t)(K * N));
  if (!xr || !xi) { free(xr); free(xi); return OR_ENOMEM; }
  int rc = OR_OK;
  for (int64_t b = 0; b < B; ++b) {
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < K; ++k)
      for (int64_t n = 0; n < N; ++n) {
        xr[k * N + n] = oracle_f16_to_f64(oracle_f32_to_f16(src_re(x, layout, b, k, n, K, N)));
        xi[k * N + n] = oracle_f16_to_f64(oracle_f32_to_f16(src_im(x, layout, b, k, n, K, N)));
      }
#pragma omp parallel
    {
      double* re = (double*)malloc(sizeof(double) * (size_t)N);
      double* im = (double*)malloc(sizeof(double) * (size_t)N);
      if (!re || !im) {
#pragma omp atomic write
        rc = OR_ENOMEM;
      } else {
#pragma omp for schedule(dynamic, 1)
        for (int64_t i = 0; i < n_rows; ++i) {
          int64_t m = rows ? rows[i] : i;
          for (int64_t n = 0; n < N; ++n) { re[n] = 0.0; im[n] = 0.0; }
          for (int64_t k = 0; k < K; ++k) {           /* k ascending for every (m, n) */
            double wr = oracle_f16_to_f64(oracle_f32_to_f16(src_re(w, layout, b, m, k, M, K)));
            double wi = oracle_f16_to_f64(oracle_f32_to_f16(src_im(w, layout, b, m, k, M, K)));
            const double* xrk = xr + k * N;
            const double* xik = xi + k * N;
            for (int64_t n = 0; n < N; ++n) {
              /* Re(a*b) = Re(a)Re(b) - Im(a)Im(b); Im(a*b) = Re(a)Im(b) + Im(a)Re(b)
                  */
              re[n] += wr * xrk[n] - wi * xik[n];
              im[n] += wr * xik[n] + wi * xrk[n];
            }
          }
          double* o_re = out + ((b * 2 + 0) * n_rows + i) * N;
          double* o_im = out + ((b * 2 + 1) * n_rows + i) * N;
          for (int64_t n = 0; n < N; ++n) { o_re[n] = re[n]; o_im[n] = im[n]; }
        }
      }
      free(re);
      free(im);
    }
    if (rc != OR_OK) break;
  }
  free(xr);
  free(xi);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* Complex GEMM, 1-bit mode, by definition (PAPER.md:170-172 encoding,       */
/* PAPER.md:244-249): each component is +-1 from the sign rule; the result is */
/* the exact complex dot product over the LOGICAL K (padding is a device     */
/* artefact, reading R1/R2), accumulated in int64, narrowed to     */
/* int32 (|Re|,|Im| <= 2K < 2^31 for K < 2^30).  No popcount is used here:   */
/* the popc identities of Eq.4-6 are the GPU's method, not the definition.   */
/* ------------------------------------------------------------------------ */
static void cgemm_pm1(const int8_t* wr, const int8_t* wi, const int8_t* xr, const int8_t* xi,
                      int64_t M, int64_t N, int64_t K, const int64_t* rows, int64_t n_rows,
                      int32_t* o_re_base, int32_t* o_im_base) {
  (void)M;
#pragma omp parallel
  {
    int64_t* re = (int64_t*)malloc(sizeof(int64_t) * (size_t)N);
    int64_t* im = (int64_t*)malloc(sizeof(int64_t) * (size_t)N);
#pragma omp for schedule(dynamic, 1)
    for (int64_t i = 0; i < n_rows; ++i) {
      int64_t m = rows ? rows[i] : i;
      for (int64_t n = 0; n < N; ++n) { re[n] = 0; im[n] = 0; }
      for (int64_t k = 0; k < K; ++k) {
        int64_t ar = wr[m * K + k], ai = wi[m * K + k];
        const int8_t* xrk = xr + k * N;
        const int8_t* xik = xi + k * N;
        for (int64_t n = 0; n < N; ++n) {
          re[n] += ar * xrk[n] - ai * xik[n];
          im[n] += ar * xik[n] + ai * xrk[n];
        }
      }
      for (int64_t n = 0; n < N; ++n) {
        o_re_base[i * N + n] = (int32_t)re[n];
        o_im_base[i * N + n] = (int32_t)im[n];
      }
    }
    free(re);
    free(im);
  }
}

int oracle_cgemm_b1(const float* w, const float* x, int layout, int64_t M, int64_t N, int64_t K,
                    int64_t B, const int64_t* rows, int64_t n_rows, int32_t* out) {
  if (!w || !x || !out || M < 1 || N < 1 || K < 1 || B < 1 || n_rows < 0) return OR_EINVAL;
  for (int64_t i = 0; i < n_rows; ++i)
    if (rows && (rows[i] < 0 || rows[i] >= M)) return OR_EINVAL;
  int8_t* wr = (int8_t*)malloc((size_t)(M * K));
  int8_t* wi = (int8_t*)malloc((size_t)(M * K));
  int8_t* xr = (int8_t*)malloc((size_t)(K * N));
  int8_t* xi = (int8_t*)malloc((size_t)(K * N));
  if (!wr || !wi || !xr || !xi) { free(wr); free(wi); free(xr); free(xi); return OR_ENOMEM; }
  for (int64_t b = 0; b < B; ++b) {
    for (int64_t m = 0; m < M; ++m)
      for (int64_t k = 0; k < K; ++k) {
        wr[m * K + k] = (int8_t)bit_to_pm1(oracle_sign_bit(src_re(w, layout, b, m, k, M, K)));
        wi[m * K + k] = (int8_t)bit_to_pm1(oracle_sign_bit(src_im(w, layout, b, m, k, M, K)));
      }
    for (int64_t k = 0; k < K; ++k)
      for (int64_t n = 0; n < N; ++n) {
        xr[k * N + n] = (int8_t)bit_to_pm1(oracle_sign_bit(src_re(x, layout, b, k, n, K, N)));
        xi[k * N + n] = (int8_t)bit_to_pm1(oracle_sign_bit(src_im(x, layout, b, k, n, K, N)));
      }
    cgemm_pm1(wr, wi, xr, xi, M, N, K, rows, n_rows, out + (b * 2 + 0) * n_rows * N,
              out + (b * 2 + 1) * n_rows * N);
  }
  free(wr); free(wi); free(xr); free(xi);
  return OR_OK;
}

/* Same definition, starting from packed words in the plan layout (its own
 * LSB-first unpack, "32 consecutive 1-bit samples ... single
 * 32-bit integer"; bit order = DESIGN.md reading R3).  Only the logical K
 * bits are read; padding bits are ignored (and checked to be 0 by tests). */
int oracle_cgemm_b1_packed(const uint32_t* wp, const uint32_t* xp, int64_t M, int64_t N,
                           int64_t K, int64_t Kw, int64_t B, const int64_t* rows,
                           int64_t n_rows, int32_t* out) {
  if (!wp || !xp || !out || M < 1 || N < 1 || K < 1 || B < 1 || Kw * 32 < K) return OR_EINVAL;
  for (int64_t i = 0; i < n_rows; ++i)
    if (rows && (rows[i] < 0 || rows[i] >= M)) return OR_EINVAL;
  int8_t* wr = (int8_t*)malloc((size_t)(M * K));
  int8_t* wi = (int8_t*)malloc((size_t)(M * K));
  int8_t* xr = (int8_t*)malloc((size_t)(K * N));
  int8_t* xi = (int8_t*)malloc((size_t)(K * N));
  if (!wr || !wi || !xr || !xi) { free(wr); free(wi); free(xr); free(xi); return OR_ENOMEM; }
  for (int64_t b = 0; b < B; ++b) {
    const uint32_t* w_re = wp + (b * 2 + 0) * M * Kw;
    const uint32_t* w_im = wp + (b * 2 + 1) * M * Kw;
    const uint32_t* x_re = xp + (b * 2 + 0) * N * Kw;
    const uint32_t* x_im = xp + (b * 2 + 1) * N * Kw;
    for (int64_t m = 0; m < M; ++m)
      for (int64_t k = 0; k < K; ++k) {
        wr[m * K + k] = (int8_t)bit_to_pm1((w_re[m * Kw + k / 32] >> (k % 32)) & 1u);
        wi[m * K + k] = (int8_t)bit_to_pm1((w_im[m * Kw + k / 32] >> (k % 32)) & 1u);
      }
    for (int64_t n = 0; n < N; ++n)
      for (int64_t k = 0; k < K; ++k) {
        xr[k * N + n] = (int8_t)bit_to_pm1((x_re[n * Kw + k / 32] >> (k % 32)) & 1u);
        xi[k * N + n] = (int8_t)bit_to_pm1((x_im[n * Kw + k / 32] >> (k % 32)) & 1u);
      }
    cgemm_pm1(wr, wi, xr, xi, M, N, K, rows, n_rows, out + (b * 2 + 0) * n_rows * N,
              out + (b * 2 + 1) * n_rows * N);
  }
  free(wr); free(wi); free(xr); free(xi);
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Packing, the oracle's own version of the plan layouts (PAPER.md:107:      */
/* "the input matrices are tiled in device memory ... transpose kernel";     */
/* PAPER.md:414 re/im separation).  operand 0 = weights [B][M][K] -> [B][2][M][Kp] */
/* operand 1 = data [B][K][N] -> transposed [B][2][N][Kp].                    */
/* ------------------------------------------------------------------------ */
int oracle_pack_f16(const float* src, int layout, int operand, int64_t B, int64_t R, int64_t C,
                    int64_t Cp, uint16_t* dst) {
  /* Both operands keep their row order: weights [B][M][K] -> [B][2][M][Cp = K16],
     data [B][K][N] -> [B][2][K][Cp = Np]; columns C..Cp-1 are 0.0 (operand only names them). */
  (void)operand;
  if (!src || !dst || B < 1 || R < 1 || C < 1 || Cp < C) return OR_EINVAL;
  memset(dst, 0, sizeof(uint16_t) * (size_t)(B * 2 * R * Cp));
  for (int64_t b = 0; b < B; ++b)
    for (int64_t r = 0; r < R; ++r)
      for (int64_t c = 0; c < C; ++c) {
        dst[((b * 2 + 0) * R + r) * Cp + c] = oracle_f32_to_f16(src_re(src, layout, b, r, c, R, C));
        dst[((b * 2 + 1) * R + r) * Cp + c] = oracle_f32_to_f16(src_im(src, layout, b, r, c, R, C));
      }
  return OR_OK;
}

int oracle_pack_b1(const float* src, int layout, int operand, int64_t B, int64_t R, int64_t C,
                   int64_t Kw, uint32_t* dst) {
  if (!src || !dst || B < 1 || R < 1 || C < 1) return OR_EINVAL;
  int64_t rows = operand == 0 ? R : C;
  int64_t K = operand == 0 ? C : R;
  if (Kw * 32 < K) return OR_EINVAL;
  memset(dst, 0, sizeof(uint32_t) * (size_t)(B * 2 * rows * Kw));  /* padding bits = 0 */
  for (int64_t b = 0; b < B; ++b)
    for (int64_t r = 0; r < R; ++r)
      for (int64_t c = 0; c < C; ++c) {
        int64_t row = operand == 0 ? r : c;
        int64_t k = operand == 0 ? c : r;
        uint32_t br = (uint32_t)oracle_sign_bit(src_re(src, layout, b, r, c, R, C));
        uint32_t bi = (uint32_t)oracle_sign_bit(src_im(src, layout, b, r, c, R, C));
        dst[((b * 2 + 0) * rows + row) * Kw + k / 32] |= br << (k % 32);
        dst[((b * 2 + 1) * rows + row) * Kw + k / 32] |= bi << (k % 32);
      }
  return OR_OK;
}

/* Steering weights (Eqs. 1-3): delay tau_k = d_k sin(theta) / c (Eq. 2);
 * narrowband phase alignment w = exp(+2 pi i f tau_k) (reading R9).  Plain double
 * cos/sin of the full phase; out is [B][M][K][2] (re, im). */
int oracle_steering_weights(const double* pos, const double* theta, const double* freq, double c, int64_t B,
                            int64_t M, int64_t K, double* out) {
  if (!pos || !theta || !freq || !out || !(c > 0.0) || B < 1 || M < 1 || K < 1) return OR_EINVAL;
  const double two_pi = 6.283185307179586476925286766559;
  for (int64_t b = 0; b < B; ++b)
    for (int64_t m = 0; m < M; ++m)
      for (int64_t k = 0; k < K; ++k) {
        double tau = pos[k] * sin(theta[m]) / c;
        double ph = two_pi * freq[b] * tau;
        out[((b * M + m) * K + k) * 2 + 0] = cos(ph);
        out[((b * M + m) * K + k) * 2 + 1] = sin(ph);
      }
  return OR_OK;
}

/* Useful operations: 8*M*N*K per complex GEMM. */
double oracle_useful_ops(int64_t M, int64_t N, int64_t K, int64_t B) {
  return 8.0 * (double)M * (double)N * (double)K * (double)B;
}
