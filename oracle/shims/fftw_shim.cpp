// oracle/shims/fftw_shim.cpp -- TEST INFRASTRUCTURE ONLY (oracle checker, never shipped).
//
// From-scratch implementation of the FFTW3 API subset declared in fftw3.h, so
// the reference sources (/root/reference/proj/src/*.cpp) compile and run
// unmodified as the CPU oracle. Semantics follow FFTW's documented r2c/c2r
// contract (see fftw3.h); the call sites it serves are
// /root/reference/proj/src/fft.cpp:33-34 (plans), :70,80,95,111 (execute).
//
// Algorithm: separable 3D transform. Every axis is processed in blocks of B
// columns gathered into a contiguous [n][B] split re/im buffer; power-of-two
// lengths use an iterative radix-2 DIT whose innermost loop runs across the B
// columns (SIMD friendly), other lengths a direct DFT. Twiddles come from
// long-double sin/cos. Single-threaded, like the reference's mutex-guarded use.

#include "fftw3.h"

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

namespace {

constexpr int kBlock = 32;

struct Twiddles {
    int n = 0;
    std::vector<double> c, s; // cos(2 pi k / n), sin(2 pi k / n)
    std::vector<int> bitrev;
    bool pow2 = false;
    explicit Twiddles(int n_) : n(n_), c(n_), s(n_) {
        const long double two_pi_l = 6.283185307179586476925286766559005768L;
        for (int k = 0; k < n; ++k) {
            long double a = two_pi_l * static_cast<long double>(k) / static_cast<long double>(n);
            c[k] = static_cast<double>(cosl(a));
            s[k] = static_cast<double>(sinl(a));
        }
        pow2 = (n & (n - 1)) == 0;
        if (pow2) {
            bitrev.resize(n);
            int lg = 0;
            while ((1 << lg) < n) ++lg;
            for (int i = 0; i < n; ++i) {
                int r = 0;
                for (int b = 0; b < lg; ++b)
                    if (i & (1 << b)) r |= 1 << (lg - 1 - b);
                bitrev[i] = r;
            }
        }
    }
};

// In-place transform of B columns stored as re/im [n][B]; sign = -1 forward, +1 inverse.
void fft_columns(double* re, double* im, int B, const Twiddles& tw, int sign,
                 std::vector<double>& scratch) {
    const int n = tw.n;
    if (tw.pow2) {
        for (int i = 0; i < n; ++i) {
            int j = tw.bitrev[i];
            if (j > i) {
                for (int c = 0; c < B; ++c) {
                    std::swap(re[i * B + c], re[j * B + c]);
                    std::swap(im[i * B + c], im[j * B + c]);
                }
            }
        }
        for (int len = 2; len <= n; len <<= 1) {
            const int half = len >> 1;
            const int step = n / len;
            for (int start = 0; start < n; start += len) {
                for (int k = 0; k < half; ++k) {
                    const double wr = tw.c[k * step];
                    const double wi = sign * tw.s[k * step];
                    double* ar = re + (start + k) * B;
                    double* ai = im + (start + k) * B;
                    double* br = re + (start + k + half) * B;
                    double* bi = im + (start + k + half) * B;
                    for (int c = 0; c < B; ++c) {
                        const double tr = br[c] * wr - bi[c] * wi;
                        const double ti = br[c] * wi + bi[c] * wr;
                        br[c] = ar[c] - tr;
                        bi[c] = ai[c] - ti;
                        ar[c] = ar[c] + tr;
                        ai[c] = ai[c] + ti;
                    }
                }
            }
        }
        return;
    }
    // direct DFT for non-power-of-two lengths (small test grids only)
    scratch.assign(static_cast<std::size_t>(2) * n * B, 0.0);
    double* orr = scratch.data();
    double* oi = orr + static_cast<std::size_t>(n) * B;
    for (int k = 0; k < n; ++k)
        for (int j = 0; j < n; ++j) {
            const int m = static_cast<int>((static_cast<long long>(j) * k) % n);
            const double wr = tw.c[m], wi = sign * tw.s[m];
            for (int c = 0; c < B; ++c) {
                orr[k * B + c] += re[j * B + c] * wr - im[j * B + c] * wi;
                oi[k * B + c] += re[j * B + c] * wi + im[j * B + c] * wr;
            }
        }
    std::memcpy(re, orr, sizeof(double) * n * B);
    std::memcpy(im, oi, sizeof(double) * n * B);
}

// Complex transform along one axis of a row-major complex array viewed as
// [outer][n][inner].
void fft_axis(double* data /* interleaved */, long long outer, int n, long long inner,
              const Twiddles& tw, int sign) {
    std::vector<double> re(static_cast<std::size_t>(n) * kBlock), im(re.size()), scratch;
    for (long long o = 0; o < outer; ++o) {
        double* base = data + 2 * o * n * inner;
        for (long long c0 = 0; c0 < inner; c0 += kBlock) {
            const int B = static_cast<int>(std::min<long long>(kBlock, inner - c0));
            for (int i = 0; i < n; ++i)
                for (int c = 0; c < B; ++c) {
                    const double* p = base + 2 * (i * inner + c0 + c);
                    re[i * B + c] = p[0];
                    im[i * B + c] = p[1];
                }
            fft_columns(re.data(), im.data(), B, tw, sign, scratch);
            for (int i = 0; i < n; ++i)
                for (int c = 0; c < B; ++c) {
                    double* p = base + 2 * (i * inner + c0 + c);
                    p[0] = re[i * B + c];
                    p[1] = im[i * B + c];
                }
        }
    }
}

} // namespace

struct fftw_plan_s {
    int n0, n1, n2;
    bool forward;
    double* real;
    double* cplx; // interleaved complex, (n0, n1, n2/2+1)
    Twiddles t0, t1, t2;
    fftw_plan_s(int a, int b, int c, bool fwd, double* r, double* z)
        : n0(a), n1(b), n2(c), forward(fwd), real(r), cplx(z), t0(a), t1(b), t2(c) {}
};

extern "C" {

double* fftw_alloc_real(size_t n) {
    return static_cast<double*>(std::aligned_alloc(64, ((n * sizeof(double) + 63) / 64) * 64));
}
fftw_complex* fftw_alloc_complex(size_t n) {
    return static_cast<fftw_complex*>(
        std::aligned_alloc(64, ((n * sizeof(fftw_complex) + 63) / 64) * 64));
}
void fftw_free(void* p) { std::free(p); }

fftw_plan fftw_plan_dft_r2c_3d(int n0, int n1, int n2, double* in, fftw_complex* out, unsigned) {
    if (n0 < 1 || n1 < 1 || n2 < 1) return nullptr;
    return new fftw_plan_s(n0, n1, n2, true, in, reinterpret_cast<double*>(out));
}
fftw_plan fftw_plan_dft_c2r_3d(int n0, int n1, int n2, fftw_complex* in, double* out, unsigned) {
    if (n0 < 1 || n1 < 1 || n2 < 1) return nullptr;
    return new fftw_plan_s(n0, n1, n2, false, out, reinterpret_cast<double*>(in));
}
void fftw_destroy_plan(fftw_plan p) { delete p; }

void fftw_execute(const fftw_plan p) {
    const int n0 = p->n0, n1 = p->n1, n2 = p->n2, nh = n2 / 2 + 1;
    const long long rows = static_cast<long long>(n0) * n1;
    std::vector<double> re(static_cast<std::size_t>(n2) * kBlock), im(re.size()), scratch;
    if (p->forward) {
        // axis 2: real rows -> half spectrum (full complex transform of real data)
        for (long long r0 = 0; r0 < rows; r0 += kBlock) {
            const int B = static_cast<int>(std::min<long long>(kBlock, rows - r0));
            for (int i = 0; i < n2; ++i)
                for (int c = 0; c < B; ++c) {
                    re[i * B + c] = p->real[(r0 + c) * n2 + i];
                    im[i * B + c] = 0.0;
                }
            fft_columns(re.data(), im.data(), B, p->t2, -1, scratch);
            for (int c = 0; c < B; ++c)
                for (int k = 0; k < nh; ++k) {
                    double* z = p->cplx + 2 * ((r0 + c) * nh + k);
                    z[0] = re[k * B + c];
                    z[1] = im[k * B + c];
                }
        }
        fft_axis(p->cplx, n0, n1, nh, p->t1, -1);
        fft_axis(p->cplx, 1, n0, static_cast<long long>(n1) * nh, p->t0, -1);
    } else {
        // c2r: FFTW may destroy the input of a multi-dimensional c2r; so do we.
        fft_axis(p->cplx, 1, n0, static_cast<long long>(n1) * nh, p->t0, +1);
        fft_axis(p->cplx, n0, n1, nh, p->t1, +1);
        for (long long r0 = 0; r0 < rows; r0 += kBlock) {
            const int B = static_cast<int>(std::min<long long>(kBlock, rows - r0));
            for (int c = 0; c < B; ++c) {
                const double* z = p->cplx + 2 * (r0 + c) * nh;
                for (int k = 0; k < n2; ++k) {
                    // Hermitian completion along the last axis; the real part of
                    // the inverse ignores imaginary parts of self-conjugate bins.
                    if (k < nh) {
                        re[k * B + c] = z[2 * k];
                        im[k * B + c] = z[2 * k + 1];
                    } else {
                        re[k * B + c] = z[2 * (n2 - k)];
                        im[k * B + c] = -z[2 * (n2 - k) + 1];
                    }
                }
                if (n2 % 2 == 0) im[(n2 / 2) * B + c] = 0.0;
                im[c] = 0.0;
            }
            fft_columns(re.data(), im.data(), B, p->t2, +1, scratch);
            for (int c = 0; c < B; ++c)
                for (int i = 0; i < n2; ++i) p->real[(r0 + c) * n2 + i] = re[i * B + c];
        }
    }
}

} // extern "C"
