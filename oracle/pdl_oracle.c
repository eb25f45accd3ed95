/*
 * pdl_oracle.c -- CPU restatement of the reference's hot path.  TEST
 * INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py, never by the product path
 * (paper_2006_02230_b200/ refuses to run without its CUDA library).
 *
 * What it restates (reference = looprank @ /root/reference, pure Python):
 *   - simcache.interpret (simcache.py:89-204) executing the Fig. 9 blocked
 *     convolution nest (.pdl form in SURVEY App. C.2):
 *       output[img][kt][oj][oi][ofm] +=
 *           filter[kt][ct][kj][ki][ifm][ofm] * input[img][ct][oj*s+kj][oi*s+ki][ifm]
 *     in float64, one `*` then one `+=` per statement instance
 *     (simcache.py:146-168, 193-195), reduction order per output element
 *     ct -> kj -> ki -> ifm.  Input is the physically pre-padded tensor
 *     (array extent s*P-s+R), built here from the unpadded one.
 *   - the bias+ReLU nest `output = max(output + bias, 0.0)` as a second pass
 *     (Python max(): returns the first argument unless the second is larger,
 *     simcache.py:165-167).
 *   - the Fig. 1 GEMM nest C[i][j] += A[i][k]*B[k][j],
 *     reduction order k ascending.
 *
 * The float64 product of two fp32 values is exact (24+24 < 53 bits), so the
 * only rounding is the accumulation, whose per-element order we keep; the
 * results are bitwise identical to interpret (pinned by tests/test_oracle.py
 * against the tests/golden npz fixtures generated from the reference itself).  Loops
 * that are not reductions are reordered / vectorised / run in parallel, which
 * leaves every element's operation sequence unchanged.
 *
 * The *_f32 functions are the timed CPU baseline ("port" kind): the same Fig. 9
 * / Fig. 1 loop nests in fp32 with the paper's microkernel order (outer
 * product over ofm), OpenMP over the img (and ofm_tile)
 * loops as Fig. 9's pragma.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define V 16

static inline int out_extent(int in, int pad, int r, int stride) {
    return (in + 2 * pad - r) / stride + 1;
}

/* Pre-padded copy with the reference's extent s*P - s + R. */
static float *pad_input(const float *x, int N, int CT, int H, int W, int R, int S,
                        int stride, int pad, int P, int Q, int *Hp_out, int *Wp_out) {
    int Hp = stride * P - stride + R, Wp = stride * Q - stride + S;
    size_t plane = (size_t)Hp * Wp * V;
    float *xp = (float *)calloc((size_t)N * CT * plane, sizeof(float));
    if (!xp) return NULL;
    for (int n = 0; n < N; n++)
        for (int ct = 0; ct < CT; ct++)
            for (int h = 0; h < H; h++) {
                int hp = h + pad;
                if (hp < 0 || hp >= Hp) continue;
                for (int w = 0; w < W; w++) {
                    int wp = w + pad;
                    if (wp < 0 || wp >= Wp) continue;
                    memcpy(xp + (((size_t)n * CT + ct) * Hp + hp) * Wp * V + (size_t)wp * V,
                           x + ((((size_t)n * CT + ct) * H + h) * W + w) * V, V * sizeof(float));
                }
            }
    *Hp_out = Hp;
    *Wp_out = Wp;
    return xp;
}

static inline double py_max0(double v) { return (0.0 > v) ? 0.0 : v; }

/* float64 checker, bitwise equal to simcache.interpret on the Fig. 9 nest. */
int pdl_oracle_conv2d_f64(const float *x, const float *w, const float *bias, double *y,
                          int N, int C, int K, int H, int W, int R, int S, int stride,
                          int pad, int relu, int threads) {
    if (C % V || K % V || stride < 1) return -1;
    int CT = C / V, KT = K / V;
    int P = out_extent(H, pad, R, stride), Q = out_extent(W, pad, S, stride);
    if (P <= 0 || Q <= 0) return 0;
    int Hp, Wp;
    float *xp = pad_input(x, N, CT, H, W, R, S, stride, pad, P, Q, &Hp, &Wp);
    if (!xp) return -2;
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for collapse(2) schedule(dynamic)
#endif
    for (int img = 0; img < N; img++)
        for (int kt = 0; kt < KT; kt++) {
            double *yb = y + ((size_t)img * KT + kt) * P * Q * V;
            memset(yb, 0, (size_t)P * Q * V * sizeof(double));
            for (int ct = 0; ct < CT; ct++)
                for (int oj = 0; oj < P; oj++)
                    for (int kj = 0; kj < R; kj++)
                        for (int ki = 0; ki < S; ki++) {
                            const float *wb = w + ((((size_t)kt * CT + ct) * R + kj) * S + ki) * V * V;
                            const float *xr = xp + (((size_t)img * CT + ct) * Hp + oj * stride + kj) * Wp * V;
                            for (int oi = 0; oi < Q; oi++) {
                                const float *xi = xr + (size_t)(oi * stride + ki) * V;
                                double *yo = yb + ((size_t)oj * Q + oi) * V;
                                for (int ifm = 0; ifm < V; ifm++) {
                                    double a = (double)xi[ifm];
                                    for (int ofm = 0; ofm < V; ofm++)
                                        yo[ofm] = yo[ofm] + (double)wb[ifm * V + ofm] * a;
                                }
                            }
                        }
            if (relu) {
                for (int pq = 0; pq < P * Q; pq++)
                    for (int v = 0; v < V; v++) {
                        double t = yb[(size_t)pq * V + v] + (bias ? (double)bias[kt * V + v] : 0.0);
                        yb[(size_t)pq * V + v] = py_max0(t);
                    }
            } else if (bias) {
                for (int pq = 0; pq < P * Q; pq++)
                    for (int v = 0; v < V; v++)
                        yb[(size_t)pq * V + v] = yb[(size_t)pq * V + v] + (double)bias[kt * V + v];
            }
        }
    free(xp);
    return 0;
}

/* Only the images [img0, img0+nimg) -- the conv is independent per image, so
 * a sampled check of a large batch is exact for the sampled images. */
int pdl_oracle_conv2d_f64_images(const float *x, const float *w, const float *bias, double *y,
                                 int N, int C, int K, int H, int W, int R, int S, int stride,
                                 int pad, int relu, int threads, int img0, int nimg) {
    if (img0 < 0 || nimg < 0 || img0 + nimg > N) return -1;
    size_t xs = (size_t)C * H * W;
    return pdl_oracle_conv2d_f64(x + (size_t)img0 * xs, w, bias, y, nimg, C, K, H, W, R, S,
                                 stride, pad, relu, threads);
}

/* float64 checker for the Fig. 1 nest: C = alpha*A*B + beta*C0 (alpha=1, beta=0
 * is the reference nest exactly; other literals follow the beta*C+alpha*AB form
 * of PAPER.md:1084). */
int pdl_oracle_gemm_f64(const float *A, const float *B, const float *C0, double *Cout,
                        int M, int N, int K, int lda, int ldb, int ldc, double alpha,
                        double beta, int threads) {
    if (M < 0 || N < 0 || K < 0) return -1;
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for schedule(dynamic, 4)
#endif
    for (int i = 0; i < M; i++) {
        double *c = Cout + (size_t)i * N;
        for (int j = 0; j < N; j++) c[j] = 0.0;
        for (int k = 0; k < K; k++) {
            double a = (double)A[(size_t)i * lda + k];
            const float *b = B + (size_t)k * ldb;
            for (int j = 0; j < N; j++) c[j] = c[j] + a * (double)b[j];
        }
        if (alpha != 1.0 || beta != 0.0)
            for (int j = 0; j < N; j++)
                c[j] = alpha * c[j] + (beta != 0.0 ? beta * (double)C0[(size_t)i * ldc + j] : 0.0);
    }
    return 0;
}

/* ---------------- timed fp32 CPU baseline (kind "port") ---------------- */

/* Fig. 9 over a PRE-PADDED input (the paper's layout assumption), fp32,
 * microkernel outer-product order, OpenMP over (img, ofm_tile, oj): the
 * paper parallelises img; at small batch the ofm_tile and
 * output-row loops are added so every host core has work (stated in
 * DESIGN.md).  Per-element reduction order is unchanged (ct, kj, ki, ifm). */
int pdl_cpu_conv2d_f32(const float *xp, const float *w, const float *bias, float *y,
                       int N, int C, int K, int Hp, int Wp, int R, int S, int stride,
                       int P, int Q, int relu, int threads) {
    if (C % V || K % V) return -1;
    int CT = C / V, KT = K / V;
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for collapse(3) schedule(static)
#endif
    for (int img = 0; img < N; img++)
        for (int kt = 0; kt < KT; kt++)
            for (int oj = 0; oj < P; oj++) {
                float *yr = y + (((size_t)img * KT + kt) * P + oj) * Q * V;
                memset(yr, 0, (size_t)Q * V * sizeof(float));
                for (int ct = 0; ct < CT; ct++)
                    for (int kj = 0; kj < R; kj++)
                        for (int ki = 0; ki < S; ki++) {
                            const float *wb = w + ((((size_t)kt * CT + ct) * R + kj) * S + ki) * V * V;
                            const float *xr = xp + (((size_t)img * CT + ct) * Hp + oj * stride + kj) * Wp * V;
                            for (int oi = 0; oi < Q; oi++) {
                                const float *xi = xr + (size_t)(oi * stride + ki) * V;
                                float acc[V];
                                for (int v = 0; v < V; v++) acc[v] = yr[oi * V + v];
                                for (int ifm = 0; ifm < V; ifm++) {
                                    float a = xi[ifm];
                                    for (int ofm = 0; ofm < V; ofm++) acc[ofm] += wb[ifm * V + ofm] * a;
                                }
                                for (int v = 0; v < V; v++) yr[oi * V + v] = acc[v];
                            }
                        }
                if (relu || bias) {
                    for (int q = 0; q < Q; q++)
                        for (int v = 0; v < V; v++) {
                            float t = yr[(size_t)q * V + v] + (bias ? bias[kt * V + v] : 0.f);
                            yr[(size_t)q * V + v] = (relu && t < 0.f) ? 0.f : t;
                        }
                }
            }
    return 0;
}

/* Fig. 1 GEMM in fp32, parallel over i, i-k-j order (j vectorised). */
int pdl_cpu_gemm_f32(const float *A, const float *B, float *Cm, int M, int N, int K,
                     int threads) {
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for schedule(static)
#endif
    for (int i = 0; i < M; i++) {
        float *c = Cm + (size_t)i * N;
        for (int j = 0; j < N; j++) c[j] = 0.f;
        for (int k = 0; k < K; k++) {
            float a = A[(size_t)i * K + k];
            const float *b = B + (size_t)k * N;
            for (int j = 0; j < N; j++) c[j] += a * b[j];
        }
    }
    return 0;
}

int pdl_oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
