/*
 * ffn_oracle.c -- TEST INFRASTRUCTURE ONLY.  The plain, slow, fp64 CPU oracle
 * for the LLaMA fused feed-forward path
 *
 *     out = SiLU(RMSNorm(x) . W1^T) (.) (RMSNorm(x) . W3^T)
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path
 * (paper_2501_08071_b200/) never links, imports or executes it, and this file
 * shares no code, header, table or helper with the CUDA path.
 *
 * What it follows (citations are PAPER.md lines, "P:L"; BASELINE.json = [BJ]):
 *   - P:68  "Fused feed-forward is a kernel implementation that fuses multiple
 *            operators for LLAMA, and root-mean-square layer normalization is a
 *            popular layer normalization operator" -- the kernel being computed.
 *   - P:560 Table "Evaluated Kernels": fused_ff inputs B, M, N, K (B folded
 *            into M = tokens here; reading R10).
 *   - [BJ] north_star: out = SiLU(RMSNorm(x)W1) (.) (RMSNorm(x)W3), the gain g
 *            of RMSNorm folded into W1/W3, 1/rms applied as a per-row scale.
 *   The paper never writes the formula out; the readings taken where it is
 *   silent are DESIGN.md R1..R12 (eps inside the sqrt, RMS of x not of x*g,
 *   W1 = SiLU branch, ...).
 *
 * Definition computed (mode ORACLE_PLAIN), per row m, all in double, sums in
 * sequential k order:
 *     ms      = (sum_k x[m,k]^2) / K
 *     r       = 1 / sqrt(ms + eps)
 *     xn[k]   = x[m,k] * r * g[k]
 *     h1[n]   = sum_k xn[k] * W1[n,k]
 *     h3[n]   = sum_k xn[k] * W3[n,k]
 *     out[m,n]= h1[n] / (1 + exp(-h1[n])) * h3[n]          (SiLU(t) = t*sigma(t))
 *
 * Fold-aware modes (R4): the method as [BJ] defines it folds g into
 * the weights *in the storage precision*.  ORACLE_FOLD_BF16 first replaces
 * W_j[n,k] by RNE_bf16(W_j[n,k]*g[k]) and ORACLE_FOLD_TF32 by
 * RNE_tf32(RNE_fp32(W_j[n,k]*g[k])), using this file's own bit-level rounding,
 * then computes h_j = r * sum_k x[m,k]*Wt_j[n,k].  That is the exact value of
 * what the folded method computes before accumulation/output rounding.
 *
 * Inputs are stored values (bf16 bit patterns, fp32 or fp64), widened here
 * exactly to double.  Output: double, unrounded.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { ORACLE_DT_BF16 = 0, ORACLE_DT_F32 = 1, ORACLE_DT_F64 = 2 };
enum { ORACLE_PLAIN = 0, ORACLE_FOLD_BF16 = 1, ORACLE_FOLD_TF32 = 2 };

/* ---- storage-format helpers (the oracle's own; not shared with the GPU) ---- */

/* bf16 is the top 16 bits of an IEEE binary32: widening is exact. */
static double bf16_bits_to_double(uint16_t b) {
    uint32_t u = ((uint32_t)b) << 16;
    float f;
    memcpy(&f, &u, 4);
    return (double)f;
}

static double load_elem(const void* p, int dtype, int64_t i) {
    switch (dtype) {
    case ORACLE_DT_BF16: return bf16_bits_to_double(((const uint16_t*)p)[i]);
    case ORACLE_DT_F32:  return (double)((const float*)p)[i];
    default:             return ((const double*)p)[i];
    }
}

/* Round-to-nearest-even of a binary32 value to `keep` explicit mantissa bits
 * (bf16: 7, tf32: 10).  Bit manipulation on the binary32 encoding: add half an
 * ulp of the target format (minus one if the kept LSB is 0, which realises the
 * ties-to-even rule) and clear the dropped bits.  NaN passes through quietened;
 * overflow to inf is the correct RNE result. */
static uint32_t rne_f32_bits(uint32_t u, int keep) {
    const int drop = 23 - keep;
    if ((u & 0x7f800000u) == 0x7f800000u) {           /* inf / nan */
        if (u & 0x007fffffu) u |= 0x00400000u;
        return u & ~((1u << drop) - 1u);
    }
    uint32_t lsb = (u >> drop) & 1u;
    uint32_t bias = (1u << (drop - 1)) - 1u + lsb;
    u += bias;
    return u & ~((1u << drop) - 1u);
}

/* Exported for the pins: double -> binary32 (C cast, RNE) -> bf16 bits. */
uint16_t oracle_round_bf16_bits(double v) {
    float f = (float)v;
    uint32_t u;
    memcpy(&u, &f, 4);
    return (uint16_t)(rne_f32_bits(u, 7) >> 16);
}

double oracle_round_bf16(double v) {
    return bf16_bits_to_double(oracle_round_bf16_bits(v));
}

double oracle_round_tf32(double v) {
    float f = (float)v;
    uint32_t u;
    memcpy(&u, &f, 4);
    u = rne_f32_bits(u, 10);
    memcpy(&f, &u, 4);
    return (double)f;
}

/* ---- a1: per-row inverse RMS ---------------------------------------------- */
/* r[m] = 1 / sqrt( (sum_k x[m,k]^2)/K + eps )   ([BJ]; R2, R3) */
void oracle_rms_inv(const void* x, int dtype, int64_t M, int64_t K, double eps, double* r) {
    for (int64_t m = 0; m < M; ++m) {
        double ss = 0.0;
        for (int64_t k = 0; k < K; ++k) {
            double v = load_elem(x, dtype, m * K + k);
            ss += v * v;
        }
        r[m] = 1.0 / sqrt(ss / (double)K + eps);
    }
}

/* ---- whole path, selected rows ------------------------------------------- */
/*
 * rows: the nrows row indices of x to evaluate (NULL = all M rows, nrows = M).
 * out : [nrows, N] double.
 * Returns 0 on success, -1 on bad arguments, -2 on allocation failure.
 *
 * Loop order: the normalised rows are formed first; then the weight rows are
 * visited in blocks of ORACLE_NB (widened, and folded in fold-aware modes,
 * once per block) and every selected row is contracted with them.  Each
 * h1/h3 is still one sequential k-sum exactly as written in the header, so
 * the blocking changes memory traffic only, never a value.
 */
#define ORACLE_NB 64
int oracle_ffn_rows(const void* x, int x_dtype, const void* g, const void* w1, const void* w3,
                    int w_dtype, int64_t M, int64_t K, int64_t N, double eps, int mode,
                    const int64_t* rows, int64_t nrows, double* out) {
    if (!x || !g || !w1 || !w3 || !out || K <= 0 || N <= 0 || M < 0 || nrows < 0) return -1;
    if (mode < ORACLE_PLAIN || mode > ORACLE_FOLD_TF32) return -1;
    if (nrows == 0) return 0;

    double* G = (double*)malloc(sizeof(double) * (size_t)K);
    double* XN = (double*)malloc(sizeof(double) * (size_t)nrows * (size_t)K);
    double* R = (double*)malloc(sizeof(double) * (size_t)nrows);
    char* valid = (char*)malloc((size_t)nrows);
    if (!G || !XN || !R || !valid) { free(G); free(XN); free(R); free(valid); return -2; }
    for (int64_t k = 0; k < K; ++k) G[k] = load_elem(g, w_dtype, k);

    /* a1 + RMSNorm: r = 1/sqrt(mean(x^2) + eps); plain mode forms
     * xn = x * r * g, fold-aware modes keep x (g is inside the weights and r
     * is applied after the contraction). */
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < nrows; ++i) {
        int64_t m = rows ? rows[i] : i;
        valid[i] = (m >= 0 && m < M);
        if (!valid[i]) continue;
        double ss = 0.0;
        for (int64_t k = 0; k < K; ++k) {
            double v = load_elem(x, x_dtype, m * K + k);
            ss += v * v;
        }
        double r = 1.0 / sqrt(ss / (double)K + eps);
        R[i] = r;
        for (int64_t k = 0; k < K; ++k) {
            double v = load_elem(x, x_dtype, m * K + k);
            XN[i * K + k] = (mode == ORACLE_PLAIN) ? v * r * G[k] : v;
        }
    }

    int status = 0;
    const int64_t nblocks = (N + ORACLE_NB - 1) / ORACLE_NB;
    #pragma omp parallel
    {
        double* W1 = (double*)malloc(sizeof(double) * ORACLE_NB * (size_t)K);
        double* W3 = (double*)malloc(sizeof(double) * ORACLE_NB * (size_t)K);
        if (!W1 || !W3) {
            #pragma omp atomic write
            status = -2;
        } else {
            #pragma omp for schedule(dynamic, 1)
            for (int64_t nb = 0; nb < nblocks; ++nb) {
                const int64_t n0 = nb * ORACLE_NB;
                const int64_t nn = (N - n0) < ORACLE_NB ? (N - n0) : ORACLE_NB;
                /* widen (and in fold-aware modes fold g into) this block of W1/W3 */
                for (int64_t j = 0; j < nn; ++j) {
                    for (int64_t k = 0; k < K; ++k) {
                        double a = load_elem(w1, w_dtype, (n0 + j) * K + k);
                        double b = load_elem(w3, w_dtype, (n0 + j) * K + k);
                        if (mode == ORACLE_FOLD_BF16) {
                            a = oracle_round_bf16(a * G[k]);
                            b = oracle_round_bf16(b * G[k]);
                        } else if (mode == ORACLE_FOLD_TF32) {
                            a = oracle_round_tf32((double)(float)(a * G[k]));
                            b = oracle_round_tf32((double)(float)(b * G[k]));
                        }
                        W1[j * K + k] = a;
                        W3[j * K + k] = b;
                    }
                }
                for (int64_t i = 0; i < nrows; ++i) {
                    const double* xn = XN + i * K;
                    for (int64_t j = 0; j < nn; ++j) {
                        if (!valid[i]) { out[i * N + n0 + j] = NAN; continue; }
                        const double* a = W1 + j * K;
                        const double* b = W3 + j * K;
                        /* a2: the two contractions */
                        double h1 = 0.0, h3 = 0.0;
                        for (int64_t k = 0; k < K; ++k) {
                            h1 += xn[k] * a[k];
                            h3 += xn[k] * b[k];
                        }
                        if (mode != ORACLE_PLAIN) { h1 *= R[i]; h3 *= R[i]; }
                        /* a3: SiLU(h1) * h3, SiLU(t) = t / (1 + e^-t) */
                        out[i * N + n0 + j] = h1 / (1.0 + exp(-h1)) * h3;
                    }
                }
            }
        }
        free(W1); free(W3);
    }
    free(G); free(XN); free(R); free(valid);
    return status;
}

/* Step a0 as the method defines it, for the bitwise pin of the GPU pack:
 * dst_bits[n*K+k] = RNE_bf16(W[n,k] * g[k]) for bf16 W, g. */
void oracle_fold_bf16(const uint16_t* w, const uint16_t* g, int64_t N, int64_t K, uint16_t* dst_bits) {
    #pragma omp parallel for schedule(static)
    for (int64_t n = 0; n < N; ++n)
        for (int64_t k = 0; k < K; ++k)
            dst_bits[n * K + k] = oracle_round_bf16_bits(bf16_bits_to_double(w[n * K + k]) *
                                                         bf16_bits_to_double(g[k]));
}

/* Same for fp32 storage (tf32 MMA path): RNE_tf32(RNE_fp32(W*g)) as fp32. */
void oracle_fold_tf32(const float* w, const float* g, int64_t N, int64_t K, float* dst) {
    #pragma omp parallel for schedule(static)
    for (int64_t n = 0; n < N; ++n)
        for (int64_t k = 0; k < K; ++k)
            dst[n * K + k] = (float)oracle_round_tf32((double)(float)((double)w[n * K + k] * (double)g[k]));
}

int oracle_ffn(const void* x, int x_dtype, const void* g, const void* w1, const void* w3,
               int w_dtype, int64_t M, int64_t K, int64_t N, double eps, int mode, double* out) {
    return oracle_ffn_rows(x, x_dtype, g, w1, w3, w_dtype, M, K, N, eps, mode, NULL, M, out);
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ---- f3: GEMM + activation (the paper's mmLeakyReLu) ----------------------- */
/*
 * PAPER.md P:523 / P:562 ("mmLeakyReLu", inputs B, M, N, K = 1, 512, 512, 2048):
 * a matrix multiplication whose epilogue applies LeakyReLU.  Definition
 * (R14: nn.Linear weight layout, negative slope alpha):
 *     out[m,n] = act( sum_k x[m,k] * w[n,k] ),
 *     act(t) = t (act = 0)  or  t >= 0 ? t : alpha * t (act = 1).
 * Sequential k-sums in fp64; out [M,N] double.
 */
int oracle_gemm_act(const void* x, int x_dtype, const void* w, int w_dtype, int64_t M, int64_t K, int64_t N,
                    int act, double alpha, double* out) {
    if (!x || !w || !out || M < 0 || K <= 0 || N <= 0 || (act != 0 && act != 1)) return -1;
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t m = 0; m < M; ++m) {
        for (int64_t n = 0; n < N; ++n) {
            double acc = 0.0;
            for (int64_t k = 0; k < K; ++k)
                acc += load_elem(x, x_dtype, m * K + k) * load_elem(w, w_dtype, n * K + k);
            out[m * N + n] = (act == 1 && acc < 0.0) ? alpha * acc : acc;
        }
    }
    return 0;
}

/* ---- f1: the whole feed-forward block -------------------------------------- */
/*
 * y[m,j] = sum_n hidden[m,n] * W2[j,n],  hidden = the fused FFN above (rows of
 * oracle_ffn_rows in `mode`), W2 [K,N] (nn.Linear(N -> K) layout).
 * round_hidden != 0: hidden is first rounded to bf16 (RNE) -- the method
 * materialises the hidden activation in the storage precision between its two
 * GEMMs (R13); 0 keeps it exact.  out [nrows, K] double.
 */
int oracle_ffn_block_rows(const void* x, int x_dtype, const void* g, const void* w1, const void* w3, const void* w2,
                          int w_dtype, int64_t M, int64_t K, int64_t N, double eps, int mode, int round_hidden,
                          const int64_t* rows, int64_t nrows, double* out) {
    if (!w2 || !out || nrows < 0) return -1;
    if (nrows == 0) return 0;
    double* hid = (double*)malloc(sizeof(double) * (size_t)nrows * (size_t)N);
    if (!hid) return -2;
    int st = oracle_ffn_rows(x, x_dtype, g, w1, w3, w_dtype, M, K, N, eps, mode, rows, nrows, hid);
    if (st != 0) { free(hid); return st; }
    if (round_hidden) {
        for (int64_t i = 0; i < nrows * N; ++i) hid[i] = oracle_round_bf16(hid[i]);
    }
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < nrows; ++i) {
        for (int64_t j = 0; j < K; ++j) {
            double acc = 0.0;
            for (int64_t n = 0; n < N; ++n) acc += hid[i * N + n] * load_elem(w2, w_dtype, j * N + n);
            out[i * K + j] = acc;
        }
    }
    free(hid);
    return 0;
}

/* ---- f3: stand-alone RMSNorm (the paper's "rmsnorm" kernel) ----------------- */
/*
 * PAPER.md P:68 ("root-mean-square layer normalization"), Table
 * "Evaluated Kernels" P:573 (memory-bound; B, n_head, seq_len, d_head =
 * 1, 32, 4096, 64, read as 4096 rows of 32*64 = 2048 features, R10):
 *     out[m,k] = x[m,k] * g[k] / sqrt( (sum_k x[m,k]^2)/K + eps )
 * fp64, sequential k-sums; out [M,K] double.
 */
int oracle_rmsnorm(const void* x, int x_dtype, const void* g, int g_dtype, int64_t M, int64_t K, double eps,
                   double* out) {
    if (!x || !g || !out || M < 0 || K <= 0) return -1;
    #pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < M; ++m) {
        double ss = 0.0;
        for (int64_t k = 0; k < K; ++k) {
            double v = load_elem(x, x_dtype, m * K + k);
            ss += v * v;
        }
        double r = 1.0 / sqrt(ss / (double)K + eps);
        for (int64_t k = 0; k < K; ++k)
            out[m * K + k] = load_elem(x, x_dtype, m * K + k) * r * load_elem(g, g_dtype, k);
    }
    return 0;
}

/* Thread count for the OpenMP loops (bench.py pins it to the host's cores:
 * torchrun exports OMP_NUM_THREADS=1 to every rank). */
void oracle_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
