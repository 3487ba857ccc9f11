/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.  Plain, slow, obviously-correct FP64 CPU implementation of
 * the direct method of Mohanty et al., arXiv 2204.13241.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load this library.  It shares no code,
 * header or constant with the CUDA path (paper_2204_13241_b200/csrc).
 *
 * Every loop is the paper's formula written out in IEEE double precision, round-to-nearest,
 * libm cos/sin, compiled WITHOUT -ffast-math.  The only parallelism is OpenMP over q, which is the
 * paper's own parallel axis ("computations ... for different q vectors are independent of each
 * other, and hence can be performed in parallel", Algorithm 1).
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>

/* Periodic wrap into [0, L): the image choice is irrelevant on the reciprocal lattice
 * (PAPER.md:285-287); for off-lattice q the finite-sample sum over the wrapped positions is the
 * reading adopted in DESIGN.md (R3).  L <= 0 disables wrapping. */
static double wrap(double x, double L) {
    if (!(L > 0.0)) return x;
    double y = x - L * floor(x / L);
    if (y >= L) y = 0.0;
    return y;
}

/* Eq.(7):  p^e(q,t) = sum_i f_i exp(-i q . r_i(t)), one frame.
 * pos [N][3], f [N] (NULL => f_i = 1), q [n_q][3]; outputs re[n_q], im[n_q]. */
void oracle_amplitude(const double* pos, int64_t N, const double* f, const double* q, int64_t n_q,
                      double L, double* re_out, double* im_out) {
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t iq = 0; iq < n_q; ++iq) {
        const double qx = q[3 * iq + 0], qy = q[3 * iq + 1], qz = q[3 * iq + 2];
        double re = 0.0, im = 0.0;
        for (int64_t j = 0; j < N; ++j) {
            const double x = wrap(pos[3 * j + 0], L);
            const double y = wrap(pos[3 * j + 1], L);
            const double z = wrap(pos[3 * j + 2], L);
            const double phase = qx * x + qy * y + qz * z;    /* q . r_j */
            const double fj = f ? f[j] : 1.0;
            re += fj * cos(phase);                             /* Re e^{-i phase} =  cos */
            im -= fj * sin(phase);                             /* Im e^{-i phase} = -sin */
        }
        re_out[iq] = re;
        im_out[iq] = im;
    }
}

/* Eq.(8), PAPER.md:134-138 (Algorithm 1):  I(q,t) = |p^e(q,t)|^2 for every frame.
 * pos [T][N][3], I_out [T][n_q]. */
void oracle_intensity(const double* pos, int64_t N, const double* f, const double* q, int64_t n_q,
                      int64_t T, double L, double* I_out) {
    for (int64_t t = 0; t < T; ++t) {
        const double* p = pos + (size_t)t * (size_t)N * 3;
#pragma omp parallel for schedule(dynamic, 16)
        for (int64_t iq = 0; iq < n_q; ++iq) {
            const double qx = q[3 * iq + 0], qy = q[3 * iq + 1], qz = q[3 * iq + 2];
            double re = 0.0, im = 0.0;
            for (int64_t j = 0; j < N; ++j) {
                const double x = wrap(p[3 * j + 0], L);
                const double y = wrap(p[3 * j + 1], L);
                const double z = wrap(p[3 * j + 2], L);
                const double phase = qx * x + qy * y + qz * z;
                const double fj = f ? f[j] : 1.0;
                re += fj * cos(phase);
                im -= fj * sin(phase);
            }
            I_out[(size_t)t * (size_t)n_q + iq] = re * re + im * im;
        }
    }
}

/* Eq.(2):  I(q) = sum_i sum_j f_i f_j exp(-i q . (r_i - r_j)), the O(N^2) pair sum.
 * The imaginary parts cancel pairwise (i,j)/(j,i), so the real part is summed.  Used only as an
 * independent brute-force pin on tiny inputs (the paper calls it infeasible at scale). */
void oracle_pair_sum(const double* pos, int64_t N, const double* f, const double* q, int64_t n_q,
                     double L, double* I_out) {
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t iq = 0; iq < n_q; ++iq) {
        const double qx = q[3 * iq + 0], qy = q[3 * iq + 1], qz = q[3 * iq + 2];
        double s = 0.0;
        for (int64_t i = 0; i < N; ++i) {
            const double xi = wrap(pos[3 * i + 0], L), yi = wrap(pos[3 * i + 1], L), zi = wrap(pos[3 * i + 2], L);
            const double fi = f ? f[i] : 1.0;
            for (int64_t j = 0; j < N; ++j) {
                const double xj = wrap(pos[3 * j + 0], L), yj = wrap(pos[3 * j + 1], L), zj = wrap(pos[3 * j + 2], L);
                const double fj = f ? f[j] : 1.0;
                s += fi * fj * cos(qx * (xi - xj) + qy * (yi - yj) + qz * (zi - zj));
            }
        }
        I_out[iq] = s;
    }
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Eq.(2) with q-dependent form factors f_i(q) via the single sum of Eq.(7):
 *     p(q,t) = sum_j f_{s(j)}(q) exp(-i q . r_j(t)),   I(q,t) = |p|^2,
 * for atoms of n_species kinds: species[j] in [0, n_species), fq [n_species][n_q] the form factor of each
 * kind at each q (the paper parameterises f by a sum of Gaussians; the table is an input).
 * pos [T][N][3]; amp != 0 writes (re, im) pairs to out [T][n_q][2], else I to out [T][n_q]. */
void oracle_species(const double* pos, int64_t N, const int32_t* species, const double* fq, const double* q,
                    int64_t n_q, int64_t T, double L, int amp, double* out) {
    for (int64_t t = 0; t < T; ++t) {
        const double* p = pos + (size_t)t * (size_t)N * 3;
#pragma omp parallel for schedule(dynamic, 16)
        for (int64_t iq = 0; iq < n_q; ++iq) {
            const double qx = q[3 * iq + 0], qy = q[3 * iq + 1], qz = q[3 * iq + 2];
            double re = 0.0, im = 0.0;
            for (int64_t j = 0; j < N; ++j) {
                const double x = wrap(p[3 * j + 0], L);
                const double y = wrap(p[3 * j + 1], L);
                const double z = wrap(p[3 * j + 2], L);
                const double phase = qx * x + qy * y + qz * z;
                const double fj = fq[(size_t)species[j] * (size_t)n_q + iq];
                re += fj * cos(phase);
                im -= fj * sin(phase);
            }
            if (amp) {
                out[2 * ((size_t)t * (size_t)n_q + iq) + 0] = re;
                out[2 * ((size_t)t * (size_t)n_q + iq) + 1] = im;
            } else {
                out[(size_t)t * (size_t)n_q + iq] = re * re + im * im;
            }
        }
    }
}

/* Eq.(2) itself with q-dependent form factors: the O(N^2) pair sum sum_i sum_j f_i(q) f_j(q) cos(q . (r_i - r_j))
 * (tiny N only; brute-force pin of oracle_species). */
void oracle_pair_sum_species(const double* pos, int64_t N, const int32_t* species, const double* fq,
                             const double* q, int64_t n_q, double L, double* I_out) {
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t iq = 0; iq < n_q; ++iq) {
        const double qx = q[3 * iq + 0], qy = q[3 * iq + 1], qz = q[3 * iq + 2];
        double s = 0.0;
        for (int64_t i = 0; i < N; ++i) {
            const double xi = wrap(pos[3 * i + 0], L), yi = wrap(pos[3 * i + 1], L), zi = wrap(pos[3 * i + 2], L);
            const double fi = fq[(size_t)species[i] * (size_t)n_q + iq];
            for (int64_t j = 0; j < N; ++j) {
                const double xj = wrap(pos[3 * j + 0], L), yj = wrap(pos[3 * j + 1], L), zj = wrap(pos[3 * j + 2], L);
                const double fj = fq[(size_t)species[j] * (size_t)n_q + iq];
                s += fi * fj * cos(qx * (xi - xj) + qy * (yi - yj) + qz * (zi - zj));
            }
        }
        I_out[iq] = s;
    }
}

/* Thread count of the OpenMP loops above (the host-core baseline sets it explicitly: a runtime already initialised
 * by another library in the process would ignore OMP_NUM_THREADS). */
void oracle_set_threads(int n) {
#ifdef _OPENMP
    extern void omp_set_num_threads(int);
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
