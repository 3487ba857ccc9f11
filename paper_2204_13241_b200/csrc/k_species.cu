// k_species.cu -- q-dependent atomic form factors.
//
// Eq.(2), carries f_i(q) per atom; the paper notes that f is the Fourier transform of the atom's
// electron density, "well parameterized by a sum of Gaussians".  Atoms of one kind share f_s(q),
// so the single sum of Eq.(7) splits into per-species amplitudes
//     p(q,t) = sum_s f_s(q) P_s(q,t),   P_s = sum_{j in s} e^{-i q . r_j(t)},
// each evaluated by the unchanged amplitude engines on the species' atoms (gathered at staging), and this epilogue
// folds the engines' atom-chunk partials in FP64, weights them by f_s(q) and forms I = |p|^2 (Eq. 8) or p.
// HBM-bound: reads sum_s C_s x 8-16 B and S x 4-8 B of f per output element.
#include "common.cuh"

namespace xpcs {

template <typename P, typename Fq, typename O>
__global__ void __launch_bounds__(256) k_species_combine(SpeciesParts sp, int64_t total, int64_t n_q,
                                                         const Fq* __restrict__ fq, int64_t v0, int64_t n_l,
                                                         O* __restrict__ out, int mode, BrightSink bs) {
    const int64_t fq_stride = n_l * n_q;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = i / n_q, q = i - v * n_q;
        const int64_t row = ((v0 + v) % n_l) * n_q + q;
        double re = 0.0, im = 0.0, F = 0.0;
        for (int s = 0; s < sp.n; ++s) {
            const P* part = (const P*)sp.part[s];
            double pr = 0.0, pi = 0.0;
            for (int64_t c = 0; c < sp.C[s]; ++c) {
                const P w = part[c * total + i];
                pr += (double)w.x;
                pi += (double)w.y;
            }
            const double f = (double)fq[(int64_t)sp.kind[s] * fq_stride + row];
            re += f * pr;
            im += f * pi;
            F = fmax(F, fabs(f));
        }
        if (mode == 0) out[i] = (O)(re * re + im * im);
        else { out[2 * i] = (O)re; out[2 * i + 1] = (O)(mode == 2 ? -im : im); }
        bright_append(bs, re * re + im * im, F, i);
    }
}

template <typename Q, typename O>
__global__ void __launch_bounds__(256) k_form_factor_gaussian(const Q* __restrict__ q, int64_t n_q, LatticeGeom g,
                                                              int64_t l0, int64_t n_l, int3 mc, int n_gauss,
                                                              double4 a03, double4 b03, double2 a45, double2 b45,
                                                              double c, O* __restrict__ out) {
    const int64_t total = q ? n_q : n_l * g.n_h * g.n_k;
    const double a[6] = {a03.x, a03.y, a03.z, a03.w, a45.x, a45.y};
    const double b[6] = {b03.x, b03.y, b03.z, b03.w, b45.x, b45.y};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        double qq;
        if (q) {
            const double x = (double)q[3 * i], y = (double)q[3 * i + 1], z = (double)q[3 * i + 2];
            qq = x * x + y * y + z * z;
        } else {
            const int64_t plane = g.n_h * g.n_k;
            const int64_t il = i / plane, r = i - il * plane, ih = r / g.n_k, ik = r - ih * g.n_k;
            const int64_t l = l0 + il, h = g.h0 + ih, k = g.k0 + ik;
            const double m[3] = {(double)(g.m0[0] + h * g.ma[0] + k * g.mb[0] + l * mc.x),
                                 (double)(g.m0[1] + h * g.ma[1] + k * g.mb[1] + l * mc.y),
                                 (double)(g.m0[2] + h * g.ma[2] + k * g.mb[2] + l * mc.z)};
            const double u = 6.283185307179586476925 / g.L;
            qq = u * u * (m[0] * m[0] + m[1] * m[1] + m[2] * m[2]);
        }
        const double s2 = qq * (1.0 / (16.0 * 9.869604401089358618834));   // (|q| / 4 pi)^2
        double f = c;
        for (int k = 0; k < n_gauss; ++k) f += a[k] * exp(-b[k] * s2);
        out[i] = (O)f;
    }
}

struct RowVals { double v[kMaxKinds]; };
template <typename O>
__global__ void __launch_bounds__(256) k_fill_rows(O* __restrict__ out, int n_rows, int64_t n, RowVals rv) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_rows * n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (O)rv.v[i / n];
}

static dim3 grid_n(int64_t total) {
    int64_t b = (total + 255) / 256;
    const int64_t cap = (int64_t)sm_count() * 16;
    return dim3((unsigned)(b < cap ? (b > 0 ? b : 1) : cap));
}

cudaError_t launch_species_combine(const SpeciesParts& sp, int64_t frames, int64_t n_q, const void* fq, int fq_f64,
                                   int64_t v0, int64_t n_l, void* out, int out_f64, int mode, cudaStream_t s,
                                   const BrightSink* bright) {
    const int64_t total = frames * n_q;
    const dim3 gr = grid_n(total);
    const BrightSink bs = bright ? *bright : BrightSink{nullptr, nullptr, 0.0, nullptr};
    note_launch();
#define XPCS_SPC(P, F, O) k_species_combine<P, F, O><<<gr, 256, 0, s>>>(sp, total, n_q, (const F*)fq, v0, n_l, (O*)out, mode, bs)
    if (sp.part_f64) {
        if (fq_f64) { if (out_f64) XPCS_SPC(double2, double, double); else XPCS_SPC(double2, double, float); }
        else { if (out_f64) XPCS_SPC(double2, float, double); else XPCS_SPC(double2, float, float); }
    } else {
        if (fq_f64) { if (out_f64) XPCS_SPC(float2, double, double); else XPCS_SPC(float2, double, float); }
        else { if (out_f64) XPCS_SPC(float2, float, double); else XPCS_SPC(float2, float, float); }
    }
#undef XPCS_SPC
    return cudaGetLastError();
}

cudaError_t launch_fill_rows(void* out, int out_f64, int n_rows, int64_t n, const double* vals, cudaStream_t s) {
    if (n_rows < 1 || n_rows > kMaxKinds) return cudaErrorInvalidValue;
    RowVals rv{};
    for (int r = 0; r < n_rows; ++r) rv.v[r] = vals[r];
    const dim3 gr = grid_n(n_rows * n);
    note_launch();
    if (out_f64) k_fill_rows<double><<<gr, 256, 0, s>>>((double*)out, n_rows, n, rv);
    else k_fill_rows<float><<<gr, 256, 0, s>>>((float*)out, n_rows, n, rv);
    return cudaGetLastError();
}

cudaError_t launch_form_factor_gaussian(const void* q, int q_f64, int64_t n_q, const LatticeGeom& g, int64_t l0,
                                        int64_t n_l, const int32_t* mc, int n_gauss, const double* a, const double* b,
                                        double c, void* out, int out_f64, cudaStream_t s) {
    double A[6] = {0, 0, 0, 0, 0, 0}, B[6] = {0, 0, 0, 0, 0, 0};
    for (int i = 0; i < n_gauss && i < 6; ++i) { A[i] = a[i]; B[i] = b[i]; }
    const int3 m = q ? make_int3(0, 0, 0) : make_int3(mc[0], mc[1], mc[2]);
    const int64_t total = q ? n_q : n_l * g.n_h * g.n_k;
    const dim3 gr = grid_n(total);
    const double4 a03 = make_double4(A[0], A[1], A[2], A[3]), b03 = make_double4(B[0], B[1], B[2], B[3]);
    const double2 a45 = make_double2(A[4], A[5]), b45 = make_double2(B[4], B[5]);
    note_launch();
#define XPCS_FFG(Q, O) k_form_factor_gaussian<Q, O><<<gr, 256, 0, s>>>((const Q*)q, n_q, g, l0, n_l, m, n_gauss, a03, b03, a45, b45, c, (O*)out)
    if (q_f64) { if (out_f64) XPCS_FFG(double, double); else XPCS_FFG(double, float); }
    else { if (out_f64) XPCS_FFG(float, double); else XPCS_FFG(float, float); }
#undef XPCS_FFG
    return cudaGetLastError();
}

}  // namespace xpcs
