// Device building blocks for the VDAMP hot path on sm_100a:
// complex helpers, the shared-memory Stockham FFT, Haar lifting steps,
// the Onsager/soft-threshold apply, and deterministic block scans.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

namespace vdamp {

template <typename R> struct CT;
template <> struct CT<float>  { typedef float2 T; };
template <> struct CT<double> { typedef double2 T; };

template <typename C> __device__ __forceinline__ C mk(decltype(C::x) a, decltype(C::x) b) { C c; c.x = a; c.y = b; return c; }
template <typename C> __device__ __forceinline__ C cadd(C a, C b) { return mk<C>(a.x + b.x, a.y + b.y); }
template <typename C> __device__ __forceinline__ C csub(C a, C b) { return mk<C>(a.x - b.x, a.y - b.y); }
template <typename C> __device__ __forceinline__ C cmul(C a, C b) { return mk<C>(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
template <typename C, typename R> __device__ __forceinline__ C cscale(C a, R s) { return mk<C>(a.x * s, a.y * s); }
template <typename C> __device__ __forceinline__ C cconj(C a) { return mk<C>(a.x, -a.y); }
// multiply by -i (forward) or +i (inverse)
template <typename C, bool INV> __device__ __forceinline__ C cmul_mi(C a) {
    return INV ? mk<C>(-a.y, a.x) : mk<C>(a.y, -a.x);
}

// |r| exactly as used by both the SURE scan and the apply (they must agree).
__device__ __forceinline__ float cmag(float2 a) { return sqrtf(fmaf(a.x, a.x, a.y * a.y)); }
__device__ __forceinline__ double cmag(double2 a) { return hypot(a.x, a.y); }

// Haar taps: the reference divides by sqrt(2) (src/wavelet.py:109-128); the
// fp64 instantiation does the same so it tracks numpy to the last bit, the
// fp32 one multiplies by the rounded reciprocal.
template <typename R> struct Haar;
template <> struct Haar<double> {
    static __device__ __forceinline__ double2 sum(double2 a, double2 b) {
        return mk<double2>((a.x + b.x) / 1.4142135623730951, (a.y + b.y) / 1.4142135623730951);
    }
    static __device__ __forceinline__ double2 dif(double2 a, double2 b) {
        return mk<double2>((a.x - b.x) / 1.4142135623730951, (a.y - b.y) / 1.4142135623730951);
    }
};
template <> struct Haar<float> {
    static __device__ __forceinline__ float2 sum(float2 a, float2 b) {
        return mk<float2>((a.x + b.x) * 0.70710678118654752f, (a.y + b.y) * 0.70710678118654752f);
    }
    static __device__ __forceinline__ float2 dif(float2 a, float2 b) {
        return mk<float2>((a.x - b.x) * 0.70710678118654752f, (a.y - b.y) * 0.70710678118654752f);
    }
};

// Onsager-corrected soft threshold of one coefficient (src/vdamp.py:125-131,
// src/denoise.py:166-168):  (r * max(1 - t/|r|, 0) - alpha * r) * gain,
// |r| == t -> shrunk to 0.  (t, alpha, gain) = (0, 0, 1) is the identity.
__device__ __forceinline__ float sdiv(float a, float b) { return __fdividef(a, b); }
__device__ __forceinline__ double sdiv(double a, double b) { return a / b; }

template <typename R, typename C>
__device__ __forceinline__ C onsager(C r, R t, R alpha, R gain) {
    R m = cmag(r);
    R sh = (m > t) ? (R(1) - sdiv(t, m)) : R(0);   // m > t >= 0, so m is normal
    const R f = (sh - alpha) * gain;                // (soft(r) - alpha r) / (1 - alpha) = r f
    return mk<C>(r.x * f, r.y * f);
}

// ---------------------------------------------------------------------------
// Radix-16/8/4/2 Stockham FFT.  Each thread owns whole radix-R butterflies in
// registers (R = 16 while >= 16 points remain, then 8/4/2).  Row sequences are
// addressed through the padded index SP(i) = i + (i >> 4) so the stride-R
// Stockham stores of the first pass hit distinct banks; column tiles
// (SEQ_FAST) are conflict-free unpadded.  tw[m] = exp(-2 pi i m / L).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int SP(int i) { return i + (i >> 4); }

template <typename C> struct Cst;
template <> struct Cst<float2> {
    static constexpr float c1 = 0.92387953251128676f, s1 = 0.38268343236508977f, h = 0.70710678118654752f;
};
template <> struct Cst<double2> {
    static constexpr double c1 = 0.92387953251128676, s1 = 0.38268343236508977, h = 0.70710678118654752;
};

// w^m for w = exp(-+2 pi i / 16), m in 0..15 (conj for the inverse)
template <typename C, bool INV>
__device__ __forceinline__ C w16(int m) {
    typedef decltype(C::x) R;
    const R c1 = Cst<C>::c1, s1 = Cst<C>::s1, h = Cst<C>::h;
    R re, im;
    switch (m & 15) {
        case 0: re = 1; im = 0; break;
        case 1: re = c1; im = -s1; break;
        case 2: re = h; im = -h; break;
        case 3: re = s1; im = -c1; break;
        case 4: re = 0; im = -1; break;
        case 5: re = -s1; im = -c1; break;
        case 6: re = -h; im = -h; break;
        case 7: re = -c1; im = -s1; break;
        case 8: re = -1; im = 0; break;
        case 9: re = -c1; im = s1; break;
        case 10: re = -h; im = h; break;
        case 11: re = -s1; im = c1; break;
        case 12: re = 0; im = 1; break;
        case 13: re = s1; im = c1; break;
        case 14: re = h; im = h; break;
        default: re = c1; im = s1; break;
    }
    return mk<C>(re, INV ? -im : im);
}

template <typename C, bool INV>
__device__ __forceinline__ void dft4(C& a0, C& a1, C& a2, C& a3) {
    const C b0 = cadd(a0, a2), b1 = csub(a0, a2), b2 = cadd(a1, a3), b3 = cmul_mi<C, INV>(csub(a1, a3));
    a0 = cadd(b0, b2); a1 = cadd(b1, b3); a2 = csub(b0, b2); a3 = csub(b1, b3);
}

// in-place DFT of v[0..R) in natural order
template <typename C, bool INV, int R>
__device__ __forceinline__ void dft_r(C (&v)[R]) {
    if constexpr (R == 2) {
        const C a = v[0], b = v[1];
        v[0] = cadd(a, b); v[1] = csub(a, b);
    } else if constexpr (R == 4) {
        dft4<C, INV>(v[0], v[1], v[2], v[3]);
    } else if constexpr (R == 8) {
        // n = n2 + 4 n1 (n1 < 2): DFT2 over n1, twiddle W8^{n2 k1}, DFT4 over n2 -> X[k1 + 2 k2]
        C a[4][2];
#pragma unroll
        for (int n2 = 0; n2 < 4; ++n2) { a[n2][0] = cadd(v[n2], v[n2 + 4]); a[n2][1] = csub(v[n2], v[n2 + 4]); }
#pragma unroll
        for (int n2 = 1; n2 < 4; ++n2) a[n2][1] = cmul(a[n2][1], w16<C, INV>(2 * n2));
#pragma unroll
        for (int k1 = 0; k1 < 2; ++k1) {
            dft4<C, INV>(a[0][k1], a[1][k1], a[2][k1], a[3][k1]);
#pragma unroll
            for (int k2 = 0; k2 < 4; ++k2) v[k1 + 2 * k2] = a[k2][k1];
        }
    } else {
        static_assert(R == 16, "radix");
        // n = n2 + 4 n1: DFT4 over n1, twiddle W16^{n2 k1}, DFT4 over n2 -> X[k1 + 4 k2]
        C a[4][4];
#pragma unroll
        for (int n2 = 0; n2 < 4; ++n2) {
            a[n2][0] = v[n2]; a[n2][1] = v[n2 + 4]; a[n2][2] = v[n2 + 8]; a[n2][3] = v[n2 + 12];
            dft4<C, INV>(a[n2][0], a[n2][1], a[n2][2], a[n2][3]);
        }
#pragma unroll
        for (int n2 = 1; n2 < 4; ++n2)
#pragma unroll
            for (int k1 = 1; k1 < 4; ++k1) a[n2][k1] = cmul(a[n2][k1], w16<C, INV>(n2 * k1));
#pragma unroll
        for (int k1 = 0; k1 < 4; ++k1) {
            dft4<C, INV>(a[0][k1], a[1][k1], a[2][k1], a[3][k1]);
#pragma unroll
            for (int k2 = 0; k2 < 4; ++k2) v[k1 + 4 * k2] = a[k2][k1];
        }
    }
}

// one Stockham pass of radix R; element e of sequence q at buf[ADR(q*sstr + e*estr)]
template <typename C, bool INV, int NT, int MAXB, bool SEQ_FAST, bool PAD, int R>
__device__ __forceinline__ void fft_pass(C* buf, int logL, int logNs, int lognseq, int sstr, int estr, const C* tw) {
    constexpr int LR = R == 2 ? 1 : R == 4 ? 2 : R == 8 ? 3 : 4;
    const int logQ = logL - LR;
    const int Q = 1 << logQ;
    const int Ns = 1 << logNs;
    const int total = 1 << (lognseq + logQ);
    const int twshift = logL - logNs - LR;
    C v[MAXB][R];
#pragma unroll
    for (int i = 0; i < MAXB; ++i) {
        const int bf = threadIdx.x + i * NT;
        if (bf < total) {
            int q, j;
            if (SEQ_FAST) { q = bf & ((1 << lognseq) - 1); j = bf >> lognseq; }
            else          { q = bf >> logQ; j = bf & (Q - 1); }
            const int base = q * sstr;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int a = base + (j + r * Q) * estr;
                v[i][r] = buf[PAD ? SP(a) : a];
            }
            const int k = j & (Ns - 1);
            if (k) {
                // twiddles w^(r k): load w^k, w^2k, w^4k, w^8k, build the rest by products
                C t1 = tw[k << twshift];
                C t2 = (R >= 4) ? tw[(2 * k) << twshift] : t1;
                C t4 = (R >= 8) ? tw[(4 * k) << twshift] : t1;
                C t8 = (R >= 16) ? tw[(8 * k) << twshift] : t1;
                if (INV) { t1 = cconj(t1); t2 = cconj(t2); t4 = cconj(t4); t8 = cconj(t8); }
#pragma unroll
                for (int r = 1; r < R; ++r) {
                    C w;
                    switch (r) {
                        case 1: w = t1; break;
                        case 2: w = t2; break;
                        case 3: w = cmul(t2, t1); break;
                        case 4: w = t4; break;
                        case 5: w = cmul(t4, t1); break;
                        case 6: w = cmul(t4, t2); break;
                        case 7: w = cmul(cmul(t4, t2), t1); break;
                        case 8: w = t8; break;
                        case 9: w = cmul(t8, t1); break;
                        case 10: w = cmul(t8, t2); break;
                        case 11: w = cmul(cmul(t8, t2), t1); break;
                        case 12: w = cmul(t8, t4); break;
                        case 13: w = cmul(cmul(t8, t4), t1); break;
                        case 14: w = cmul(cmul(t8, t4), t2); break;
                        default: w = cmul(cmul(cmul(t8, t4), t2), t1); break;
                    }
                    v[i][r] = cmul(v[i][r], w);
                }
            }
            dft_r<C, INV, R>(v[i]);
        }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < MAXB; ++i) {
        const int bf = threadIdx.x + i * NT;
        if (bf < total) {
            int q, j;
            if (SEQ_FAST) { q = bf & ((1 << lognseq) - 1); j = bf >> lognseq; }
            else          { q = bf >> logQ; j = bf & (Q - 1); }
            const int base = q * sstr;
            const int k = j & (Ns - 1);
            const int d = ((j - k) << LR) + k;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int a = base + (d + r * Ns) * estr;
                buf[PAD ? SP(a) : a] = v[i][r];
            }
        }
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
// 256-point FFT as 16 x 16 with the data in registers.  A thread with digit d
// (0..15) holds 16 elements of one sequence; stage A is a radix-16 DFT over the
// held digit followed by the twiddle w^(d m), m = output index; a transpose
// (through shared memory, done by the caller) hands each thread the 16 stage-A
// outputs of its own m; stage B is a plain radix-16 DFT.
//   forward: v[n1] = x[16 n1 + d]  -> (A, transpose, B) -> v[k2] = X[d + 16 k2]
//   inverse: v[k2] = X[d + 16 k2]  -> (A, transpose, B) -> v[n2] = x[d + 16 n2]
// (x[16 n1 + n2] -> X[k1 + 16 k2] uses w256^(n2 k1) between the stages; the
// inverse reads the forward's output order directly, so a forward FFT, a
// pointwise step and an inverse FFT need no transpose between them.)
// ---------------------------------------------------------------------------
template <typename C, int R>
__device__ __forceinline__ void pow_twiddles(C (&v)[R], C t1, C t2, C t4, C t8) {
#pragma unroll
    for (int r = 1; r < R; ++r) {
        C w;
        switch (r) {
            case 1: w = t1; break;
            case 2: w = t2; break;
            case 3: w = cmul(t2, t1); break;
            case 4: w = t4; break;
            case 5: w = cmul(t4, t1); break;
            case 6: w = cmul(t4, t2); break;
            case 7: w = cmul(cmul(t4, t2), t1); break;
            case 8: w = t8; break;
            case 9: w = cmul(t8, t1); break;
            case 10: w = cmul(t8, t2); break;
            case 11: w = cmul(cmul(t8, t2), t1); break;
            case 12: w = cmul(t8, t4); break;
            case 13: w = cmul(cmul(t8, t4), t1); break;
            case 14: w = cmul(cmul(t8, t4), t2); break;
            default: w = cmul(cmul(cmul(t8, t4), t2), t1); break;
        }
        v[r] = cmul(v[r], w);
    }
}

// stage A of the 16 x 16 FFT: radix-16 DFT of v, then v[m] *= w256^(+-d m);
// tw[m] = exp(-2 pi i m / 256) (global, L1-resident)
template <typename C, bool INV>
__device__ __forceinline__ void fft256_stage_a(C (&v)[16], int d, const C* __restrict__ tw) {
    C t1 = __ldg(tw + d), t2 = __ldg(tw + 2 * d), t4 = __ldg(tw + 4 * d), t8 = __ldg(tw + 8 * d);
    dft_r<C, INV, 16>(v);
    if (INV) { t1 = cconj(t1); t2 = cconj(t2); t4 = cconj(t4); t8 = cconj(t8); }
    pow_twiddles<C, 16>(v, t1, t2, t4, t8);
}

template <typename C, bool INV>
__device__ __forceinline__ void pow_twiddles512(C (&v)[16], int e, const C* __restrict__ tw) {
    // v[m] *= w512^(+-e m), m = 1..15 (e <= 31)
    C t1 = __ldg(tw + e), t2 = __ldg(tw + 2 * e), t4 = __ldg(tw + 4 * e), t8 = __ldg(tw + 8 * e);
    if (INV) { t1 = cconj(t1); t2 = cconj(t2); t4 = cconj(t4); t8 = cconj(t8); }
    pow_twiddles<C, 16>(v, t1, t2, t4, t8);
}

// Row FFTs of a 16 x 256 strip held in the SP-padded shared buffer (row r at
// SP(256 r) = 272 r; element e of a row at 17 (e >> 4) + (e & 15)).  Thread
// (r = tid >> 4, d = tid & 15).  Forward: buffer rows -> v[k2] = X_r[d + 16 k2].
template <typename C>
__device__ __forceinline__ void strip_fft256_fwd(C* buf, C (&v)[16], const C* __restrict__ tw) {
    const int r = threadIdx.x >> 4, d = threadIdx.x & 15;
    C* row = buf + 272 * r;
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = row[17 * j + d];
    fft256_stage_a<C, false>(v, d, tw);
    __syncthreads();
#pragma unroll
    for (int m = 0; m < 16; ++m) row[17 * m + d] = v[m];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = row[17 * d + j];
    dft_r<C, false, 16>(v);
}

// Inverse: v[k2] = X_r[d + 16 k2] (registers) -> natural-order rows in the
// SP-padded buffer (unnormalised).
template <typename C>
__device__ __forceinline__ void strip_ifft256_to_smem(C* buf, C (&v)[16], const C* __restrict__ tw) {
    const int r = threadIdx.x >> 4, d = threadIdx.x & 15;
    C* row = buf + 272 * r;
    fft256_stage_a<C, true>(v, d, tw);
#pragma unroll
    for (int m = 0; m < 16; ++m) row[17 * m + d] = v[m];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = row[17 * d + j];
    dft_r<C, true, 16>(v);
    __syncthreads();
#pragma unroll
    for (int n = 0; n < 16; ++n) row[17 * n + d] = v[n];
    __syncthreads();
}

// Full unnormalised DFT of every sequence (radix-16 passes, one final 2/4/8 pass).
template <typename C, bool INV, int NT, int CAP, bool SEQ_FAST, bool PAD>
__device__ __forceinline__ void block_fft16(C* buf, int logL, int lognseq, int sstr, int estr, const C* tw) {
    int logNs = 0;
    const int rem = logL & 3;
    if (rem == 1) { fft_pass<C, INV, NT, (CAP / 2 + NT - 1) / NT, SEQ_FAST, PAD, 2>(buf, logL, 0, lognseq, sstr, estr, tw); logNs = 1; }
    if (rem == 2) { fft_pass<C, INV, NT, (CAP / 4 + NT - 1) / NT, SEQ_FAST, PAD, 4>(buf, logL, 0, lognseq, sstr, estr, tw); logNs = 2; }
    if (rem == 3) { fft_pass<C, INV, NT, (CAP / 8 + NT - 1) / NT, SEQ_FAST, PAD, 8>(buf, logL, 0, lognseq, sstr, estr, tw); logNs = 3; }
    for (; logNs < logL; logNs += 4)
        fft_pass<C, INV, NT, (CAP / 16 + NT - 1) / NT, SEQ_FAST, PAD, 16>(buf, logL, logNs, lognseq, sstr, estr, tw);
}

// ---------------------------------------------------------------------------
// TMA bulk copies (cp.async.bulk) global -> shared with an mbarrier
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* mbar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(mbar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(unsigned long long* mbar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(mbar)), "r"(bytes) : "memory");
}

// one bulk copy of `bytes` (multiple of 16, both addresses 16-byte aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* mbar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(mbar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* mbar, unsigned phase) {
    asm volatile("{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}"
                 :: "r"(smem_u32(mbar)), "r"(phase) : "memory");
}

// order earlier generic-proxy shared-memory accesses before async-proxy writes
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ---------------------------------------------------------------------------
// Deterministic block reductions / scans over doubles (fixed shuffle trees).
// ---------------------------------------------------------------------------
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x < 32) {
        t = (l < NT / 32) ? sh[l] : 0.0;
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (l == 0) sh[0] = t;
    }
    __syncthreads();
    t = sh[0];
    __syncthreads();
    return t;
}

// Exclusive warp scan without subtraction (the inverse-magnitude sums span
// many decades, so "inclusive - own" would cancel catastrophically).
template <bool REV>
__device__ __forceinline__ double warp_excl_scan(double v, double& total) {
    const int l = threadIdx.x & 31;
    double inc = v;
    if (!REV) {
        for (int o = 1; o < 32; o <<= 1) { double u = __shfl_up_sync(0xffffffffu, inc, o); if (l >= o) inc += u; }
        double ex = __shfl_up_sync(0xffffffffu, inc, 1);
        total = __shfl_sync(0xffffffffu, inc, 31);
        return l == 0 ? 0.0 : ex;
    } else {
        for (int o = 1; o < 32; o <<= 1) { double u = __shfl_down_sync(0xffffffffu, inc, o); if (l + o < 32) inc += u; }
        double ex = __shfl_down_sync(0xffffffffu, inc, 1);
        total = __shfl_sync(0xffffffffu, inc, 0);
        return l == 31 ? 0.0 : ex;
    }
}

// Exclusive scan in thread order (REV = false: sum over lower threads;
// REV = true: sum over higher threads). `sh` needs NT/32 doubles.
template <int NT, bool REV>
__device__ __forceinline__ double block_excl_scan(double v, double* sh) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    double wtot;
    double ex = warp_excl_scan<REV>(v, wtot);
    __syncthreads();
    if (l == 0) sh[w] = wtot;
    __syncthreads();
    if (threadIdx.x < 32) {
        const int NW = NT / 32;
        double t = (l < NW) ? sh[l] : 0.0;
        double dummy;
        double wex = warp_excl_scan<REV>(t, dummy);
        if (REV && NW < 32) {
            // lanes >= NW hold zeros; the reverse exclusive scan is unaffected
        }
        __syncwarp();
        if (l < NW) sh[l] = wex;
    }
    __syncthreads();
    double r = sh[w] + ex;
    __syncthreads();
    return r;
}

// programmatic dependent launch: wait for the preceding grid (no-op when the
// kernel was launched without the PDL attribute), then let the next grid start
// its CTAs as SMs free up
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// L2 prefetch hint (no register or ordering effect)
__device__ __forceinline__ void prefetch_l2(const void* q) { asm volatile("prefetch.global.L2 [%0];" ::"l"(q)); }
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Both exclusive scans of scan_tile in one pass: a forward scan of `a` (sum
// over lower threads) and a reverse scan of `b` (sum over higher threads),
// interleaved so they share the barriers.  Same summation trees as two
// block_excl_scan calls.  `sh` needs 2 * NT/32 doubles.
template <int NT>
__device__ __forceinline__ void block_excl_scan2(double a, double b, double* sh, double& ea, double& eb) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    constexpr int NW = NT / 32;
    double ta, tb;
    const double xa = warp_excl_scan<false>(a, ta);
    const double xb = warp_excl_scan<true>(b, tb);
    __syncthreads();
    if (l == 0) { sh[w] = ta; sh[NW + w] = tb; }
    __syncthreads();
    if (threadIdx.x < 32) {
        double d;
        const double wa = warp_excl_scan<false>(l < NW ? sh[l] : 0.0, d);
        const double wb = warp_excl_scan<true>(l < NW ? sh[NW + l] : 0.0, d);
        __syncwarp();
        if (l < NW) { sh[l] = wa; sh[NW + l] = wb; }
    }
    __syncthreads();
    ea = sh[w] + xa;
    eb = sh[NW + w] + xb;
    __syncthreads();
}

}  // namespace vdamp
