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
#include <type_traits>
#include <algorithm>

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

// The same combination for two consecutive outputs per thread (I only, fp32 partials, <= CMB_MAXP partial planes in
// all, flattened in (species, chunk) order): every plane's two partials arrive by one 16-B load, all issued before
// the first sum (the scalar loop above keeps one load in flight per thread), then the sums run in the scalar
// kernel's order -- identical results.
constexpr int CMB_MAXP = 8;
struct CombPlanes {
    const float4* p[CMB_MAXP];     // plane base (2 outputs per float4)
    const void* f[CMB_MAXP];       // f_q table of the plane's species (read at its first plane)
    int first[CMB_MAXP + 1];       // 1: the plane starts a species (first[n] = 1)
    int n;
};
template <typename Fq, typename O>
__global__ void __launch_bounds__(256) k_species_combine2(CombPlanes cp, int64_t frames, int64_t n_q, int64_t v0,
                                                          int64_t n_l, O* __restrict__ out, BrightSink bs) {
    using Fq2 = typename std::conditional<std::is_same<Fq, double>::value, double2, float2>::type;
    using O2 = typename std::conditional<std::is_same<O, double>::value, double2, float2>::type;
    const int64_t q = 2 * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x);   // x: pixel pairs, y: frames (no division)
    if (q >= n_q) return;
    for (int64_t v = blockIdx.y; v < frames; v += gridDim.y) {
        const int64_t i = v * n_q + q;                        // n_q even: i and i + 1 share the frame
        const int64_t row = (n_l == 1 ? 0 : ((v0 + v) % n_l) * n_q) + q;
        float4 w[CMB_MAXP];
        Fq2 fv[CMB_MAXP];
#pragma unroll
        for (int k = 0; k < CMB_MAXP; ++k)
            if (k < cp.n) {
                w[k] = __ldcs(cp.p[k] + i / 2);   // i even: a shift
                if (cp.first[k]) fv[k] = *((const Fq2*)cp.f[k] + row / 2);
            }
        double re0 = 0.0, im0 = 0.0, re1 = 0.0, im1 = 0.0, F0 = 0.0, F1 = 0.0;
        double pr0 = 0.0, pi0 = 0.0, pr1 = 0.0, pi1 = 0.0, fa = 0.0, fb = 0.0;
#pragma unroll
        for (int k = 0; k < CMB_MAXP; ++k)
            if (k < cp.n) {
                if (cp.first[k]) { fa = (double)fv[k].x; fb = (double)fv[k].y; pr0 = pi0 = pr1 = pi1 = 0.0; }
                pr0 += (double)w[k].x; pi0 += (double)w[k].y;
                pr1 += (double)w[k].z; pi1 += (double)w[k].w;
                if (cp.first[k + 1] || k + 1 == cp.n) {         // the species' last plane
                    re0 += fa * pr0; im0 += fa * pi0; F0 = fmax(F0, fabs(fa));
                    re1 += fb * pr1; im1 += fb * pi1; F1 = fmax(F1, fabs(fb));
                }
            }
        const double I0 = re0 * re0 + im0 * im0, I1 = re1 * re1 + im1 * im1;
        O2 o;
        o.x = (O)I0;
        o.y = (O)I1;
        *(O2*)(out + i) = o;
        bright_append(bs, I0, F0, i);
        bright_append(bs, I1, F1, i + 1);
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
    int64_t nplanes = 0;
    bool aligned = true;
    for (int k = 0; k < sp.n; ++k) {
        nplanes += sp.C[k];
        aligned = aligned && ((uintptr_t)sp.part[k] % 16 == 0);
    }
    const size_t fqe = fq_f64 ? 8 : 4, oe = out_f64 ? 8 : 4;
    if (mode == 0 && !sp.part_f64 && nplanes <= CMB_MAXP && n_q % 2 == 0 && aligned &&
        (uintptr_t)fq % (2 * fqe) == 0 && (uintptr_t)out % (2 * oe) == 0) {
        CombPlanes cp{};
        for (int k = 0; k < sp.n; ++k)
            for (int64_t c = 0; c < sp.C[k]; ++c) {
                cp.p[cp.n] = (const float4*)((const float2*)sp.part[k] + c * total);
                cp.f[cp.n] = (const char*)fq + (size_t)sp.kind[k] * n_l * n_q * fqe;
                cp.first[cp.n] = c == 0;
                ++cp.n;
            }
        cp.first[cp.n] = 1;
        const int64_t bx = (n_q / 2 + 255) / 256;
        const dim3 gr2((unsigned)bx, (unsigned)std::max<int64_t>(1, std::min<int64_t>(frames, std::min<int64_t>(
                                                  65535, ((int64_t)sm_count() * 16 + bx - 1) / bx))));
#define XPCS_SPC2(F, O) k_species_combine2<F, O><<<gr2, 256, 0, s>>>(cp, frames, n_q, v0, n_l, (O*)out, bs)
        if (fq_f64) { if (out_f64) XPCS_SPC2(double, double); else XPCS_SPC2(double, float); }
        else { if (out_f64) XPCS_SPC2(float, double); else XPCS_SPC2(float, float); }
#undef XPCS_SPC2
        return cudaGetLastError();
    }
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
