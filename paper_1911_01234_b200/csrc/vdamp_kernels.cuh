// VDAMP hot-path kernels (sm_100a).  One iteration of Algorithm 1
// (/root/reference/pkg/src/csmri/vdamp.py:99-144) is four kernel stages:
//
//   K1 synth_pass   (coarse -> fine):  r~ = Onsager(r_{k-1}) ; Haar synthesis ;
//                   (-1)^(n1+n2) ; row FFT                       -> T1
//   K2 col_pass     column FFT ; z = y - M F x ; v = P^-1 z ; tau partials ;
//                   column IFFT                                   -> T2
//   K3 analysis_pass (fine -> coarse): row IFFT ; sign ; Haar analysis ;
//                   r_k = Onsager(r_{k-1}) + Psi u  (in place)    -> r
//   K4 sure_select  per (subband, image): exact SURE argmin, alpha, gain
//
// Haar is block-local, so a strip of 2^k image rows maps to contiguous row
// ranges of every subband (layout of src/wavelet.py:52-61); deeper levels
// than fit one strip are handled by extra coarse passes through a small
// scratch image.  The centred FFT is a plain FFT with (-1)^(n1+n2) sign
// modulation; the output sign is folded into y at setup.
#pragma once
#include "vdamp_device.cuh"
#include <cooperative_groups.h>
#include <type_traits>

namespace vdamp {

constexpr int MAXS = 64;          // subbands supported (scales <= 21)
constexpr int PNT = 256;          // threads of strip / column kernels
constexpr int PCAP = 4096;        // complex elements per strip / column tile
constexpr int SNT = 1024;         // threads of the per-image reduction kernels
// threads of the big SURE-select kernel (subbands > SMALL_N): 512 for fp32
// (128 registers per thread: the sort and scan loops run spill-free; local
// memory would miss the ~30 KB of L1 left beside 200 KB of shared memory),
// 1024 for fp64
constexpr int BNT32 = 1024, BNT64 = 1024;
// threads of the small-subband SURE kernel: 128 (8 keys per thread at 1024 keys, up to
// 128 registers) measured 400k vs 384k img-iter/s at 256 threads (cfg1); 64 threads
// (236 registers) 401k; capping the 128-thread CTAs at 64 or 80 registers: 373k / 391k
constexpr int SNT_SMALL = 128;
constexpr int SMALL_N = 1024;     // subbands up to this size use the small kernel
constexpr int SCAP = 16384;       // fp32 magnitudes sorted in shared memory at once
template <typename R> struct Scap { static constexpr int v = SCAP; };
constexpr int MAXTILES = 256;     // SCAP-tiles per subband (n <= 4M)
constexpr int MAXCT = 1024;       // column tiles per image (H*W/PCAP for 2048^2)
constexpr double ALPHA_CLAMP = 1.0 - 1e-9;   // src/vdamp.py:25
constexpr double TAU_FLOOR = 1e-300;         // src/vdamp.py:118
constexpr int TRACE_F = 8;

struct Geo {
    int H, W, s, S, logH, logW;
    int sign_c;                   // (-1)^(H/2 + W/2)
    long long N;
    long long off[MAXS];
    int len[MAXS];
};

__host__ __device__ inline int band_of(int s, int level, int orient) { return 1 + 3 * (s - level) + orient; }

// A strip of 2^k rows (levels a..a+k-1 plus the level-b approximation row)
// owns E_s = Wa*2^k coefficients.  Flat order used by the batched gathers:
// [level 1: H V D][level 2: H V D] ... [level k: H V D][approx row]; level q
// chunks hold E_s >> 2q coefficients.  Returns the coefficient's offset within
// its subband chunk source and its mosaic slot (row * Wa + col) in smem.
struct StripSlot { int j; long long gofs; int smem; bool approx; };

__device__ __forceinline__ StripSlot strip_slot(const Geo& g, int a, int k, int Wa, int logWa, int st, int f) {
    const int E = Wa << k;
    const int logE = logWa + k;
    int base = 0;
    for (int q = 1; q <= k; ++q) {
        const int lcq = logE - 2 * q, cq = 1 << lcq;
        if (f < base + 3 * cq) {
            const int o = (f - base) >> lcq, e = (f - base) & (cq - 1);
            const int logCq = logWa - q, Rq = 1 << (k - q), Cq = 1 << logCq;
            const int l = a + q - 1;
            const int j = band_of(g.s, l, o);
            const int r0 = (o >= 1) ? Rq : 0, c0 = (o != 1) ? Cq : 0;
            StripSlot s_;
            s_.j = j; s_.gofs = g.off[j] + (long long)st * cq + e;
            s_.smem = (r0 + (e >> logCq)) * Wa + c0 + (e & (Cq - 1));
            s_.approx = false;
            return s_;
        }
        base += 3 * cq;
    }
    const int e = f - base;                         // approximation row
    StripSlot s_;
    s_.j = 0; s_.gofs = g.off[0] + (long long)st * (Wa >> k) + e; s_.smem = e; s_.approx = true;
    return s_;
}

// ------------------------------------------------------------------ K1 ----
enum { SYN_PLAIN = 0, SYN_ROWFFT = 1 };

template <typename R>
struct SynArgs {
    const typename CT<R>::T* coef;   // [B][N]
    const double* par;               // [B][S][3] (t, alpha, gain) or null = identity
    const typename CT<R>::T* asrc;   // approx_b image (null -> subband 0 of coef)
    typename CT<R>::T* dst;          // level a-1 image / scratch / T1
    const typename CT<R>::T* tw;     // twiddles, length W (ROWFFT)
    int a, b, k, Wa, logWa;
    long long asrc_bs, dst_bs;
    int early;                       // synth256: coef was written >= 2 kernels back, so it may be
                                     // bulk-copied before the PDL wait (not after momentum_update)
};

// Gather the coarse part of a strip (levels a+1..a+k-1 and the approximation
// row, E/4 coefficients) into the top-left R1 x C1 corner of the mosaic
// (row stride Wa), Onsager applied.  Uses the flat slot map of the sub-strip.
template <typename R>
__device__ __forceinline__ void gather_coarse(const Geo& g, const SynArgs<R>& p, const typename CT<R>::T* coef,
                                              const R* spar, bool apply, typename CT<R>::T* buf, int st, int bi) {
    typedef typename CT<R>::T C;
    const int k = p.k, Wa = p.Wa;
    const int logC1 = p.logWa - 1, C1 = 1 << logC1;
    const int E1 = (Wa << k) >> 2;
    constexpr int PER = PCAP / 4 / PNT;
    C v[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int f = threadIdx.x + i * PNT;
        if (f < E1) {
            if (k > 1) {
                const StripSlot sl = strip_slot(g, p.a + 1, k - 1, C1, logC1, st, f);
                v[i] = (sl.approx && p.asrc) ? p.asrc[(long long)bi * p.asrc_bs + (long long)st * (Wa >> k) + sl.smem]
                                             : coef[sl.gofs];
            } else {
                v[i] = p.asrc ? p.asrc[(long long)bi * p.asrc_bs + (long long)st * C1 + f]
                              : coef[g.off[0] + (long long)st * C1 + f];
            }
        }
    }
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int f = threadIdx.x + i * PNT;
        if (f < E1) {
            int j = 0, slot = f;
            bool from_scratch = (p.asrc != nullptr);
            if (k > 1) {
                const StripSlot sl = strip_slot(g, p.a + 1, k - 1, C1, logC1, st, f);
                j = sl.j; slot = sl.smem; from_scratch = sl.approx && p.asrc;
            }
            C x = v[i];
            if (apply && !from_scratch) x = onsager<R, C>(x, spar[3 * j], spar[3 * j + 1], spar[3 * j + 2]);
            buf[SP((slot >> logC1) * Wa + (slot & (C1 - 1)))] = x;
        }
    }
}

template <typename R, int MODE>
__global__ void __launch_bounds__(PNT, sizeof(R) == 4 ? 4 : 2) synth_pass(Geo g, SynArgs<R> p) {
    pdl_enter();
    typedef typename CT<R>::T C;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* buf = reinterpret_cast<C*>(smem_raw);
    const int st = blockIdx.x, bi = blockIdx.y, tid = threadIdx.x;
    const int k = p.k, Wa = p.Wa;
    const int E = Wa << k;
    const C* coef = p.coef + (long long)bi * g.N;
    const double* par = p.par ? p.par + (long long)bi * g.S * 3 : nullptr;
    C* tws = buf + SP(E - 1) + 1;
    __shared__ R spar[MAXS * 3];
    if (MODE == SYN_ROWFFT)
        for (int e = tid; e < g.W; e += PNT) tws[e] = p.tw[e];
    for (int i = tid; i < g.S * 3; i += PNT) spar[i] = par ? (R)par[i] : ((i % 3) == 2 ? R(1) : R(0));

    // level-1 detail coefficients of this strip (3 chunks of R1 x C1): one 2x2
    // output block per coefficient, loads issued first
    const int logC1 = p.logWa - 1, C1 = 1 << logC1;
    const int cnt1 = E >> 2;
    const int jH = band_of(g.s, p.a, 0);
    constexpr int MB = PCAP / 4 / PNT;
    C dH[MB], dV[MB], dD[MB];
#pragma unroll
    for (int i = 0; i < MB; ++i) {
        const int b = tid + i * PNT;
        if (b < cnt1) {
            const long long o = (long long)st * cnt1 + b;
            dH[i] = coef[g.off[jH] + o];
            dV[i] = coef[g.off[jH + 1] + o];
            dD[i] = coef[g.off[jH + 2] + o];
        }
    }
    __syncthreads();                                   // spar, twiddles
    gather_coarse<R>(g, p, coef, spar, par != nullptr, buf, st, bi);
    __syncthreads();

    // coarse synthesis levels k..2 on the top-left corner (src/wavelet.py:118-129)
    for (int q = k; q >= 2; --q) {
        const int logCq = p.logWa - q, Cq = 1 << logCq, Rq = 1 << (k - q);
        const int P = Rq * Cq;
        C o[MB][4];
#pragma unroll
        for (int i = 0; i < MB; ++i) {
            const int e = tid + i * PNT;
            if (e < P) {
                const int ii = e >> logCq, jj = e & (Cq - 1);
                C ll = buf[SP(ii * Wa + jj)], lh = buf[SP(ii * Wa + Cq + jj)];
                C hl = buf[SP((Rq + ii) * Wa + jj)], hh = buf[SP((Rq + ii) * Wa + Cq + jj)];
                C lo0 = Haar<R>::sum(ll, lh), lo1 = Haar<R>::dif(ll, lh);
                C hi0 = Haar<R>::sum(hl, hh), hi1 = Haar<R>::dif(hl, hh);
                o[i][0] = Haar<R>::sum(lo0, hi0);
                o[i][1] = Haar<R>::sum(lo1, hi1);
                o[i][2] = Haar<R>::dif(lo0, hi0);
                o[i][3] = Haar<R>::dif(lo1, hi1);
            }
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < MB; ++i) {
            const int e = tid + i * PNT;
            if (e < P) {
                const int ii = e >> logCq, jj = e & (Cq - 1);
                const int d = (2 * ii) * Wa + 2 * jj;
                buf[SP(d)] = o[i][0]; buf[SP(d + 1)] = o[i][1]; buf[SP(d + Wa)] = o[i][2]; buf[SP(d + Wa + 1)] = o[i][3];
            }
        }
        __syncthreads();
    }

    // level 1 in registers: r~ of the three detail chunks, Haar synthesis of each
    // 2x2 block; for ROWFFT the (-1)^(n1+n2) modulation (rows of a strip start
    // at an even index, so the block pattern is +,-,-,+) and the unitary 1/sqrt(W)
    // are folded in here
    {
        R tH = spar[3 * jH], aH = spar[3 * jH + 1], gH = spar[3 * jH + 2];
        R tV = spar[3 * jH + 3], aV = spar[3 * jH + 4], gV = spar[3 * jH + 5];
        R tD = spar[3 * jH + 6], aD = spar[3 * jH + 7], gD = spar[3 * jH + 8];
        const R sc = (MODE == SYN_ROWFFT) ? R(1) / sqrt(R(g.W)) : R(1);
        C o[MB][4];
#pragma unroll
        for (int i = 0; i < MB; ++i) {
            const int b = tid + i * PNT;
            if (b < cnt1) {
                const int ii = b >> logC1, jj = b & (C1 - 1);
                const C ll = buf[SP(ii * Wa + jj)];
                C lh = dH[i], hl = dV[i], hh = dD[i];
                if (par) {
                    lh = onsager<R, C>(lh, tH, aH, gH);
                    hl = onsager<R, C>(hl, tV, aV, gV);
                    hh = onsager<R, C>(hh, tD, aD, gD);
                }
                C lo0 = Haar<R>::sum(ll, lh), lo1 = Haar<R>::dif(ll, lh);
                C hi0 = Haar<R>::sum(hl, hh), hi1 = Haar<R>::dif(hl, hh);
                o[i][0] = cscale(Haar<R>::sum(lo0, hi0), sc);
                o[i][1] = cscale(Haar<R>::sum(lo1, hi1), MODE == SYN_ROWFFT ? -sc : sc);
                o[i][2] = cscale(Haar<R>::dif(lo0, hi0), MODE == SYN_ROWFFT ? -sc : sc);
                o[i][3] = cscale(Haar<R>::dif(lo1, hi1), sc);
            }
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < MB; ++i) {
            const int b = tid + i * PNT;
            if (b < cnt1) {
                const int ii = b >> logC1, jj = b & (C1 - 1);
                const int d = (2 * ii) * Wa + 2 * jj;
                buf[SP(d)] = o[i][0]; buf[SP(d + 1)] = o[i][1]; buf[SP(d + Wa)] = o[i][2]; buf[SP(d + Wa + 1)] = o[i][3];
            }
        }
        __syncthreads();
    }

    C* dst = p.dst + (long long)bi * p.dst_bs + (long long)st * E;
    if (MODE == SYN_ROWFFT) block_fft16<C, false, PNT, PCAP, false, true>(buf, g.logW, k, Wa, 1, tws);
    for (int e = tid; e < E; e += PNT) dst[e] = buf[SP(e)];
}

// ------------------------------------------------------------------ K3 ----
enum { ANA_IN_PLAIN = 0, ANA_IN_ROWIFFT = 1 };
enum { ANA_OUT_COEF = 0, ANA_OUT_VDAMP = 1 };

template <typename R>
struct AnaArgs {
    const typename CT<R>::T* src;    // level a-1 image / scratch / T2
    typename CT<R>::T* coef;         // [B][N] coefficients (in/out for VDAMP)
    const double* par;               // Onsager params of r_{k-1} (VDAMP)
    typename CT<R>::T* adst;         // approx_b scratch (null -> subband 0)
    const typename CT<R>::T* tw;
    int a, b, k, Wa, logWa;
    long long src_bs, adst_bs;
};

template <typename R, int IN, int OUT>
__global__ void __launch_bounds__(PNT, sizeof(R) == 4 ? 4 : 2) analysis_pass(Geo g, AnaArgs<R> p) {
    typedef typename CT<R>::T C;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* buf = reinterpret_cast<C*>(smem_raw);
    const int st = blockIdx.x, bi = blockIdx.y, tid = threadIdx.x;
    const int k = p.k, Wa = p.Wa;
    const int E = Wa << k;
    pdl_enter();
    const C* src = p.src + (long long)bi * p.src_bs + (long long)st * E;
    C* coef = p.coef + (long long)bi * g.N;
    __shared__ R spar[MAXS * 3];
    if (OUT == ANA_OUT_VDAMP) {
        const double* par = p.par + (long long)bi * g.S * 3;
        for (int i = tid; i < g.S * 3; i += PNT) spar[i] = (R)par[i];
    }
    if (IN == ANA_IN_ROWIFFT) {
        C* tws = buf + SP(E - 1) + 1;
        for (int e = tid; e < g.W; e += PNT) tws[e] = p.tw[e];
        for (int e = tid; e < E; e += PNT) buf[SP(e)] = src[e];
        __syncthreads();
        block_fft16<C, true, PNT, PCAP, false, true>(buf, g.logW, k, Wa, 1, tws);
    } else {
        for (int e = tid; e < E; e += PNT) buf[SP(e)] = src[e];
        __syncthreads();
    }

    // level 1 in registers: each thread analyses 2x2 pixel blocks (for ROWIFFT
    // the ifft2c output sign c * (-1)^(n1+n2) -> +,-,-,+ per block, and the
    // unitary 1/sqrt(W) are folded in); the three details go straight to
    // global memory (VDAMP: r_k = Onsager(r_{k-1}) + Psi u), ll to the corner
    const int logC1 = p.logWa - 1, C1 = 1 << logC1;
    const int cnt1 = E >> 2;
    const int jH = band_of(g.s, p.a, 0);
    constexpr int MB = PCAP / 4 / PNT;
    C ll[MB];
    {
        C oH[MB], oV[MB], oD[MB];
        if (OUT == ANA_OUT_VDAMP) {
#pragma unroll
            for (int i = 0; i < MB; ++i) {
                const int b = tid + i * PNT;
                if (b < cnt1) {
                    const long long o = (long long)st * cnt1 + b;
                    oH[i] = coef[g.off[jH] + o];
                    oV[i] = coef[g.off[jH + 1] + o];
                    oD[i] = coef[g.off[jH + 2] + o];
                }
            }
        }
        const R sc = (IN == ANA_IN_ROWIFFT) ? (R)g.sign_c / sqrt(R(g.W)) : R(1);
        const R tH = OUT == ANA_OUT_VDAMP ? spar[3 * jH] : R(0), aH = OUT == ANA_OUT_VDAMP ? spar[3 * jH + 1] : R(0),
                gH = OUT == ANA_OUT_VDAMP ? spar[3 * jH + 2] : R(1);
        const R tV = OUT == ANA_OUT_VDAMP ? spar[3 * jH + 3] : R(0), aV = OUT == ANA_OUT_VDAMP ? spar[3 * jH + 4] : R(0),
                gV = OUT == ANA_OUT_VDAMP ? spar[3 * jH + 5] : R(1);
        const R tD = OUT == ANA_OUT_VDAMP ? spar[3 * jH + 6] : R(0), aD = OUT == ANA_OUT_VDAMP ? spar[3 * jH + 7] : R(0),
                gD = OUT == ANA_OUT_VDAMP ? spar[3 * jH + 8] : R(1);
#pragma unroll
        for (int i = 0; i < MB; ++i) {
            const int b = tid + i * PNT;
            if (b < cnt1) {
                const int ii = b >> logC1, jj = b & (C1 - 1);
                const int s0 = (2 * ii) * Wa + 2 * jj;
                const C x00 = cscale(buf[SP(s0)], sc);
                const C x01 = cscale(buf[SP(s0 + 1)], IN == ANA_IN_ROWIFFT ? -sc : sc);
                const C x10 = cscale(buf[SP(s0 + Wa)], IN == ANA_IN_ROWIFFT ? -sc : sc);
                const C x11 = cscale(buf[SP(s0 + Wa + 1)], sc);
                const C lo0 = Haar<R>::sum(x00, x10), hi0 = Haar<R>::dif(x00, x10);
                const C lo1 = Haar<R>::sum(x01, x11), hi1 = Haar<R>::dif(x01, x11);
                ll[i] = Haar<R>::sum(lo0, lo1);
                C lh = Haar<R>::dif(lo0, lo1), hl = Haar<R>::sum(hi0, hi1), hh = Haar<R>::dif(hi0, hi1);
                if (OUT == ANA_OUT_VDAMP) {
                    lh = cadd(onsager<R, C>(oH[i], tH, aH, gH), lh);
                    hl = cadd(onsager<R, C>(oV[i], tV, aV, gV), hl);
                    hh = cadd(onsager<R, C>(oD[i], tD, aD, gD), hh);
                }
                const long long o = (long long)st * cnt1 + b;
                coef[g.off[jH] + o] = lh;
                coef[g.off[jH + 1] + o] = hl;
                coef[g.off[jH + 2] + o] = hh;
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < MB; ++i) {
        const int b = tid + i * PNT;
        if (b < cnt1) buf[SP((b >> logC1) * Wa + (b & (C1 - 1)))] = ll[i];
    }
    __syncthreads();

    // coarse analysis levels 2..k on the corner (src/wavelet.py:107-115)
    for (int q = 2; q <= k; ++q) {
        const int logCq = p.logWa - q, Cq = 1 << logCq, Rq = 1 << (k - q);
        const int P = Rq * Cq;
        C o[MB][4];
#pragma unroll
        for (int i = 0; i < MB; ++i) {
            const int e = tid + i * PNT;
            if (e < P) {
                const int ii = e >> logCq, jj = e & (Cq - 1);
                const int s0 = (2 * ii) * Wa + 2 * jj;
                C x00 = buf[SP(s0)], x01 = buf[SP(s0 + 1)], x10 = buf[SP(s0 + Wa)], x11 = buf[SP(s0 + Wa + 1)];
                C lo0 = Haar<R>::sum(x00, x10), hi0 = Haar<R>::dif(x00, x10);
                C lo1 = Haar<R>::sum(x01, x11), hi1 = Haar<R>::dif(x01, x11);
                o[i][0] = Haar<R>::sum(lo0, lo1);
                o[i][1] = Haar<R>::dif(lo0, lo1);
                o[i][2] = Haar<R>::sum(hi0, hi1);
                o[i][3] = Haar<R>::dif(hi0, hi1);
            }
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < MB; ++i) {
            const int e = tid + i * PNT;
            if (e < P) {
                const int ii = e >> logCq, jj = e & (Cq - 1);
                buf[SP(ii * Wa + jj)] = o[i][0];
                buf[SP(ii * Wa + Cq + jj)] = o[i][1];
                buf[SP((Rq + ii) * Wa + jj)] = o[i][2];
                buf[SP((Rq + ii) * Wa + Cq + jj)] = o[i][3];
            }
        }
        __syncthreads();
    }

    // scatter the coarse corner (E/4 coefficients: levels 2..k + approximation)
    {
        const int E1 = cnt1;
        C old[MB];
        if (OUT == ANA_OUT_VDAMP) {
#pragma unroll
            for (int i = 0; i < MB; ++i) {
                const int f = tid + i * PNT;
                if (f < E1) {
                    if (k > 1) {
                        const StripSlot sl = strip_slot(g, p.a + 1, k - 1, C1, logC1, st, f);
                        if (!(sl.approx && p.adst)) old[i] = coef[sl.gofs];
                    } else if (!p.adst) {
                        old[i] = coef[g.off[0] + (long long)st * C1 + f];
                    }
                }
            }
        }
#pragma unroll
        for (int i = 0; i < MB; ++i) {
            const int f = tid + i * PNT;
            if (f < E1) {
                int j = 0, slot = f;
                long long gofs = g.off[0] + (long long)st * C1 + f;
                bool to_scratch = (p.adst != nullptr);
                if (k > 1) {
                    const StripSlot sl = strip_slot(g, p.a + 1, k - 1, C1, logC1, st, f);
                    j = sl.j; slot = sl.smem; gofs = sl.gofs; to_scratch = sl.approx && p.adst;
                }
                C u = buf[SP((slot >> logC1) * Wa + (slot & (C1 - 1)))];
                if (to_scratch) {
                    p.adst[(long long)bi * p.adst_bs + (long long)st * (Wa >> k) + (k > 1 ? slot : f)] = u;
                } else {
                    if (OUT == ANA_OUT_VDAMP) u = cadd(onsager<R, C>(old[i], spar[3 * j], spar[3 * j + 1], spar[3 * j + 2]), u);
                    coef[gofs] = u;
                }
            }
        }
    }
}

// ---------------------------------------------------- K1 / K3, W = 256 ----
// 16-row strips of a 256-wide image with the four finest Haar levels of the
// strip done per thread: thread (br = tid >> 6, bc = tid & 63) owns the 4x4
// pixel block at strip rows 4 br.., columns 4 bc.., i.e. the 2x2 level-1
// coefficients (2 br + i, 2 bc + j) and the level-2 coefficient (br, bc) of each
// orientation; level 3 and 4 (and the approximation) are per 8x8 / 16x16 block.
// Strip st maps to subband rows st * (16 >> l) .. of level l (src/wavelet.py:52-61).
template <typename C>
__device__ __forceinline__ void ld2c(const C* q, C& a, C& b) {
    if constexpr (sizeof(C) == 8) {
        const float4 t = *reinterpret_cast<const float4*>(q);
        a = mk<C>(t.x, t.y); b = mk<C>(t.z, t.w);
    } else {
        a = q[0]; b = q[1];
    }
}
template <typename C>
__device__ __forceinline__ void st2c(C* q, C a, C b) {
    if constexpr (sizeof(C) == 8) *reinterpret_cast<float4*>(q) = make_float4(a.x, a.y, b.x, b.y);
    else { q[0] = a; q[1] = b; }
}
template <typename C> __device__ __forceinline__ C cneg_if(C a, bool neg) { return neg ? mk<C>(-a.x, -a.y) : a; }

// one synthesis output of a 2x2 block (src/wavelet.py:118-129): quadrant (qi, qj)
template <typename R, typename C>
__device__ __forceinline__ C haar_syn_q(C ll, C lh, C hl, C hh, bool qi, bool qj) {
    const C lo = Haar<R>::sum(ll, cneg_if(lh, qj)), hi = Haar<R>::sum(hl, cneg_if(hh, qj));
    return Haar<R>::sum(lo, cneg_if(hi, qi));
}

template <typename R, bool ONS>
__device__ __forceinline__ typename CT<R>::T ons_j(typename CT<R>::T x, const R* spar, int j) {
    return ONS ? onsager<R, typename CT<R>::T>(x, spar[3 * j], spar[3 * j + 1], spar[3 * j + 2]) : x;
}

// K1 for W = 256, k = 4: r~ = Onsager(r) gathered per 4x4 block, Haar synthesis
// of levels 4..1 in registers, (-1)^(n1+n2) / 16 folded in, register row FFT -> T1
template <typename R>
__global__ void __launch_bounds__(PNT, sizeof(R) == 4 ? 4 : 2) synth256(Geo g, SynArgs<R> p) {
    typedef typename CT<R>::T C;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* buf = reinterpret_cast<C*>(smem_raw);
    const int st = blockIdx.x, bi = blockIdx.y, tid = threadIdx.x;
    const int br = tid >> 6, bc = tid & 63;
    const C* coef = p.coef + (long long)bi * g.N;
    __shared__ R spar[MAXS * 3];
    const int j1 = band_of(g.s, 1, 0), j2 = band_of(g.s, 2, 0), j3 = band_of(g.s, 3, 0), j4 = band_of(g.s, 4, 0);
    // early: the strip's coefficients (levels 1-4 and the approximation, 4096
    // complex, same layout as analysis256's) are bulk-copied into shared memory
    // before the PDL wait (into the pixel buffer: they are in registers before
    // the first pixel is stored); only the parameters come from the previous kernel
    C* ob = buf;
    __shared__ __align__(8) unsigned long long obar;
    const bool early = p.early != 0;
    if (early && tid == 0) {
        mbar_init(&obar, 1);
        const unsigned cs = (unsigned)sizeof(C);
        mbar_expect_tx(&obar, (p.asrc ? 4080u : 4096u) * cs);
        for (int o = 0; o < 3; ++o) {
            bulk_g2s(ob + o * 1024, coef + g.off[j1 + o] + (long long)st * 1024, 1024u * cs, &obar);
            bulk_g2s(ob + 3072 + o * 256, coef + g.off[j2 + o] + (long long)st * 256, 256u * cs, &obar);
            bulk_g2s(ob + 3840 + o * 64, coef + g.off[j3 + o] + (long long)st * 64, 64u * cs, &obar);
            bulk_g2s(ob + 4032 + o * 16, coef + g.off[j4 + o] + (long long)st * 16, 16u * cs, &obar);
        }
        if (!p.asrc) bulk_g2s(ob + 4080, coef + g.off[0] + (long long)st * 16, 16u * cs, &obar);
    }
    pdl_enter();
    const double* par = p.par ? p.par + (long long)bi * g.S * 3 : nullptr;
    for (int i = tid; i < g.S * 3; i += PNT) spar[i] = par ? (R)par[i] : ((i % 3) == 2 ? R(1) : R(0));
    // level 1 (2 x 2 per orientation, pairs along the row), 2, 3, 4, approximation
    C d1[3][2][2], d2[3], d3[3], d4[3], a4;
    {
        const long long o4 = (long long)st * 16 + (bc >> 2);
        if (early) {
            a4 = p.asrc ? p.asrc[(long long)bi * p.asrc_bs + o4] : mk<C>(R(0), R(0));
            __syncthreads();                                // obar initialised before anyone waits
            mbar_wait(&obar, 0);
#pragma unroll
            for (int o = 0; o < 3; ++o) {
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    d1[o][i][0] = ob[o * 1024 + (2 * br + i) * 128 + 2 * bc];
                    d1[o][i][1] = ob[o * 1024 + (2 * br + i) * 128 + 2 * bc + 1];
                }
                d2[o] = ob[3072 + o * 256 + br * 64 + bc];
                d3[o] = ob[3840 + o * 64 + (br >> 1) * 32 + (bc >> 1)];
                d4[o] = ob[4032 + o * 16 + (bc >> 2)];
            }
            if (!p.asrc) a4 = ob[4080 + (bc >> 2)];
        } else {
            const long long o1 = (long long)st * 1024 + (2 * br) * 128 + 2 * bc;
#pragma unroll
            for (int o = 0; o < 3; ++o)
#pragma unroll
                for (int i = 0; i < 2; ++i) ld2c<C>(coef + g.off[j1 + o] + o1 + i * 128, d1[o][i][0], d1[o][i][1]);
            const long long o2 = (long long)st * 256 + br * 64 + bc;
            const long long o3 = (long long)st * 64 + (br >> 1) * 32 + (bc >> 1);
#pragma unroll
            for (int o = 0; o < 3; ++o) {
                d2[o] = coef[g.off[j2 + o] + o2];
                d3[o] = coef[g.off[j3 + o] + o3];
                d4[o] = coef[g.off[j4 + o] + o4];
            }
            a4 = p.asrc ? p.asrc[(long long)bi * p.asrc_bs + o4] : coef[g.off[0] + o4];
        }
    }
    __syncthreads();                                        // spar; every thread holds its coefficients (buf free)
    C px[4][4];
    auto body = [&](auto onsc) {
        constexpr bool ONS = decltype(onsc)::value;
        if (!p.asrc) a4 = ons_j<R, ONS>(a4, spar, 0);
        // levels 4 and 3: only the quadrant on this thread's path
        const C a3 = haar_syn_q<R, C>(a4, ons_j<R, ONS>(d4[0], spar, j4), ons_j<R, ONS>(d4[1], spar, j4 + 1),
                                      ons_j<R, ONS>(d4[2], spar, j4 + 2), (br >> 1) & 1, (bc >> 1) & 1);
        const C a2 = haar_syn_q<R, C>(a3, ons_j<R, ONS>(d3[0], spar, j3), ons_j<R, ONS>(d3[1], spar, j3 + 1),
                                      ons_j<R, ONS>(d3[2], spar, j3 + 2), br & 1, bc & 1);
        const C h2 = ons_j<R, ONS>(d2[0], spar, j2), v2 = ons_j<R, ONS>(d2[1], spar, j2 + 1),
                e2 = ons_j<R, ONS>(d2[2], spar, j2 + 2);
        const R sc = R(1) / R(16);                          // unitary 1 / sqrt(W) of the row FFT
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const C a1 = haar_syn_q<R, C>(a2, h2, v2, e2, i, j);
                const C lh = ons_j<R, ONS>(d1[0][i][j], spar, j1), hl = ons_j<R, ONS>(d1[1][i][j], spar, j1 + 1),
                        hh = ons_j<R, ONS>(d1[2][i][j], spar, j1 + 2);
                const C lo0 = Haar<R>::sum(a1, lh), lo1 = Haar<R>::dif(a1, lh);
                const C hi0 = Haar<R>::sum(hl, hh), hi1 = Haar<R>::dif(hl, hh);
                // (-1)^(n1+n2) on even-origin 2x2 blocks: +, -, -, +
                px[2 * i][2 * j] = cscale(Haar<R>::sum(lo0, hi0), sc);
                px[2 * i][2 * j + 1] = cscale(Haar<R>::sum(lo1, hi1), -sc);
                px[2 * i + 1][2 * j] = cscale(Haar<R>::dif(lo0, hi0), -sc);
                px[2 * i + 1][2 * j + 1] = cscale(Haar<R>::dif(lo1, hi1), sc);
            }
    };
    if (par) body(std::true_type{});
    else body(std::false_type{});
    // pixels -> SP-padded strip rows (row r at 272 r, column e at 17 (e >> 4) + (e & 15))
    {
        C* b0 = buf + 272 * (4 * br) + 17 * (bc >> 2) + 4 * (bc & 3);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) b0[272 * i + j] = px[i][j];
    }
    __syncthreads();
    C v[16];
    strip_fft256_fwd<C>(buf, v, p.tw);
    C* drow = p.dst + (long long)bi * p.dst_bs + (long long)st * 4096 + ((tid >> 4) << 8) + (tid & 15);
#pragma unroll
    for (int k2 = 0; k2 < 16; ++k2) drow[16 * k2] = v[k2];
}

// K3 for W = 256, k = 4: register row IFFT of T2 into the strip, then per 4x4
// block the sign c (-1)^(n1+n2) / 16 and Haar analysis levels 1..2 in registers,
// levels 3..4 through a small shared exchange; VDAMP: r = Onsager(r; par) + Psi u
// ANA256_TMA: the strip's previous coefficients (levels 1-4 and the approximation,
// 4096 complex) are bulk-copied into shared memory before the PDL wait (they
// were written four kernels back), overlapping the T2 loads and the row IFFT
#ifndef ANA256_TMA
#define ANA256_TMA 1
#endif
template <typename R, int OUT>
__global__ void __launch_bounds__(PNT, sizeof(R) == 4 ? 4 : 2) analysis256(Geo g, AnaArgs<R> p) {
    typedef typename CT<R>::T C;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* buf = reinterpret_cast<C*>(smem_raw);
    const int st = blockIdx.x, bi = blockIdx.y, tid = threadIdx.x;
    const int br = tid >> 6, bc = tid & 63;
    C* coef = p.coef + (long long)bi * g.N;
    __shared__ R spar[MAXS * 3];
    __shared__ C x2[4][64];                                 // level-2 approximations
    __shared__ C x3[2][32];                                 // level-3 approximations
    const int j1 = band_of(g.s, 1, 0), j2 = band_of(g.s, 2, 0), j3 = band_of(g.s, 3, 0), j4 = band_of(g.s, 4, 0);
    const long long o1 = (long long)st * 1024 + (2 * br) * 128 + 2 * bc;
    const long long o2 = (long long)st * 256 + br * 64 + bc;
    // old coefficients in shared memory (TMA): [3][1024] level 1, [3][256] level 2,
    // [3][64] level 3, [3][16] level 4, [16] approximation
    constexpr bool OT = ANA256_TMA && OUT == ANA_OUT_VDAMP;
    C* ob = buf + SP(4095) + 1;
    ob = reinterpret_cast<C*>((reinterpret_cast<uintptr_t>(ob) + 15) & ~(uintptr_t)15);
    __shared__ __align__(8) unsigned long long obar;
    if (OT && tid == 0) {
        mbar_init(&obar, 1);
        const unsigned cs = (unsigned)sizeof(C);
        mbar_expect_tx(&obar, (p.adst ? 4080u : 4096u) * cs);
        for (int o = 0; o < 3; ++o) {
            bulk_g2s(ob + o * 1024, coef + g.off[j1 + o] + (long long)st * 1024, 1024u * cs, &obar);
            bulk_g2s(ob + 3072 + o * 256, coef + g.off[j2 + o] + (long long)st * 256, 256u * cs, &obar);
            bulk_g2s(ob + 3840 + o * 64, coef + g.off[j3 + o] + (long long)st * 64, 64u * cs, &obar);
            bulk_g2s(ob + 4032 + o * 16, coef + g.off[j4 + o] + (long long)st * 16, 16u * cs, &obar);
        }
        if (!p.adst) bulk_g2s(ob + 4080, coef + g.off[0] + (long long)st * 16, 16u * cs, &obar);
    }
    if (OUT == ANA_OUT_VDAMP) {
        const double* par = p.par + (long long)bi * g.S * 3;
        for (int i = tid; i < g.S * 3; i += PNT) spar[i] = (R)par[i];
    }
    pdl_enter();
    C old1[3][2][2], old2[3];
    {
        C v[16];
        const C* srow = p.src + (long long)bi * p.src_bs + (long long)st * 4096 + ((tid >> 4) << 8) + (tid & 15);
#pragma unroll
        for (int k2 = 0; k2 < 16; ++k2) v[k2] = srow[16 * k2];
        strip_ifft256_to_smem<C>(buf, v, p.tw);
    }
    const R sc = (R)g.sign_c / R(16);
    C h1[2][2], v1[2][2], e1[2][2], l1[2][2];
    {
        const C* b0 = buf + 272 * (4 * br) + 17 * (bc >> 2) + 4 * (bc & 3);
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const C x00 = cscale(b0[272 * (2 * i) + 2 * j], sc);
                const C x01 = cscale(b0[272 * (2 * i) + 2 * j + 1], -sc);
                const C x10 = cscale(b0[272 * (2 * i + 1) + 2 * j], -sc);
                const C x11 = cscale(b0[272 * (2 * i + 1) + 2 * j + 1], sc);
                const C lo0 = Haar<R>::sum(x00, x10), hi0 = Haar<R>::dif(x00, x10);
                const C lo1 = Haar<R>::sum(x01, x11), hi1 = Haar<R>::dif(x01, x11);
                l1[i][j] = Haar<R>::sum(lo0, lo1);
                h1[i][j] = Haar<R>::dif(lo0, lo1);
                v1[i][j] = Haar<R>::sum(hi0, hi1);
                e1[i][j] = Haar<R>::dif(hi0, hi1);
            }
    }
    // level 2 from the 2x2 level-1 approximations
    C l2, h2, v2, e2;
    {
        const C lo0 = Haar<R>::sum(l1[0][0], l1[1][0]), hi0 = Haar<R>::dif(l1[0][0], l1[1][0]);
        const C lo1 = Haar<R>::sum(l1[0][1], l1[1][1]), hi1 = Haar<R>::dif(l1[0][1], l1[1][1]);
        l2 = Haar<R>::sum(lo0, lo1); h2 = Haar<R>::dif(lo0, lo1); v2 = Haar<R>::sum(hi0, hi1); e2 = Haar<R>::dif(hi0, hi1);
    }
    x2[br][bc] = l2;
    // details of levels 1 and 2 (VDAMP: + Onsager of the previous coefficients)
    {
        const C n1[3][2][2] = {{{h1[0][0], h1[0][1]}, {h1[1][0], h1[1][1]}},
                               {{v1[0][0], v1[0][1]}, {v1[1][0], v1[1][1]}},
                               {{e1[0][0], e1[0][1]}, {e1[1][0], e1[1][1]}}};
        const C n2[3] = {h2, v2, e2};
#pragma unroll
        for (int o = 0; o < 3; ++o) {
            C* q1 = coef + g.off[j1 + o] + o1;
            C* q2 = coef + g.off[j2 + o] + o2;
            C w1[2][2], w2 = n2[o];
#pragma unroll
            for (int i = 0; i < 2; ++i) { w1[i][0] = n1[o][i][0]; w1[i][1] = n1[o][i][1]; }
            if (OUT == ANA_OUT_VDAMP) {
                if (OT) {
                    if (o == 0) mbar_wait(&obar, 0);
#pragma unroll
                    for (int i = 0; i < 2; ++i) {
                        old1[o][i][0] = ob[o * 1024 + (2 * br + i) * 128 + 2 * bc];
                        old1[o][i][1] = ob[o * 1024 + (2 * br + i) * 128 + 2 * bc + 1];
                    }
                    old2[o] = ob[3072 + o * 256 + br * 64 + bc];
                } else {
#pragma unroll
                    for (int i = 0; i < 2; ++i) ld2c<C>(q1 + i * 128, old1[o][i][0], old1[o][i][1]);
                    old2[o] = *q2;
                }
#pragma unroll
                for (int i = 0; i < 2; ++i)
#pragma unroll
                    for (int j = 0; j < 2; ++j) w1[i][j] = cadd(ons_j<R, true>(old1[o][i][j], spar, j1 + o), w1[i][j]);
                w2 = cadd(ons_j<R, true>(old2[o], spar, j2 + o), w2);
            }
#pragma unroll
            for (int i = 0; i < 2; ++i) st2c<C>(q1 + i * 128, w1[i][0], w1[i][1]);
            *q2 = w2;
        }
    }
    __syncthreads();
    // level 3: 64 threads, one per 8x8 block (2 rows x 32 columns of level-3 coefficients);
    // the other warps are done (warps 0-1 meet at named barrier 1 below)
    if (tid >= 64) return;
    {
        const int r3 = tid >> 5, c3 = tid & 31;
        const C x00 = x2[2 * r3][2 * c3], x01 = x2[2 * r3][2 * c3 + 1];
        const C x10 = x2[2 * r3 + 1][2 * c3], x11 = x2[2 * r3 + 1][2 * c3 + 1];
        const C lo0 = Haar<R>::sum(x00, x10), hi0 = Haar<R>::dif(x00, x10);
        const C lo1 = Haar<R>::sum(x01, x11), hi1 = Haar<R>::dif(x01, x11);
        x3[r3][c3] = Haar<R>::sum(lo0, lo1);
        C n3[3] = {Haar<R>::dif(lo0, lo1), Haar<R>::sum(hi0, hi1), Haar<R>::dif(hi0, hi1)};
        const long long o3 = (long long)st * 64 + r3 * 32 + c3;
#pragma unroll
        for (int o = 0; o < 3; ++o) {
            C* q = coef + g.off[j3 + o] + o3;
            if (OUT == ANA_OUT_VDAMP) n3[o] = cadd(ons_j<R, true>(OT ? ob[3840 + o * 64 + r3 * 32 + c3] : *q, spar, j3 + o), n3[o]);
            *q = n3[o];
        }
    }
    asm volatile("bar.sync 1, 64;" ::: "memory");
    // level 4: 16 threads, one per 16x16 block; the approximation goes to subband 0
    // (s == 4) or to the next pass's scratch image (s > 4)
    if (tid < 16) {
        const C x00 = x3[0][2 * tid], x01 = x3[0][2 * tid + 1], x10 = x3[1][2 * tid], x11 = x3[1][2 * tid + 1];
        const C lo0 = Haar<R>::sum(x00, x10), hi0 = Haar<R>::dif(x00, x10);
        const C lo1 = Haar<R>::sum(x01, x11), hi1 = Haar<R>::dif(x01, x11);
        C n4[3] = {Haar<R>::dif(lo0, lo1), Haar<R>::sum(hi0, hi1), Haar<R>::dif(hi0, hi1)};
        C a = Haar<R>::sum(lo0, lo1);
        const long long o4 = (long long)st * 16 + tid;
#pragma unroll
        for (int o = 0; o < 3; ++o) {
            C* q = coef + g.off[j4 + o] + o4;
            if (OUT == ANA_OUT_VDAMP) n4[o] = cadd(ons_j<R, true>(OT ? ob[4032 + o * 16 + tid] : *q, spar, j4 + o), n4[o]);
            *q = n4[o];
        }
        if (p.adst) {
            p.adst[(long long)bi * p.adst_bs + o4] = a;
        } else {
            C* q = coef + g.off[0] + o4;
            if (OUT == ANA_OUT_VDAMP) a = cadd(ons_j<R, true>(OT ? ob[4080 + tid] : *q, spar, 0), a);
            *q = a;
        }
    }
}

// ---------------------------------------------------- K1 / K3, W = 512 ----
// 8-row strips of a 512-wide image (first pass, levels 1-3): thread (br = tid >> 7,
// bc = tid & 127) owns the 4x4 pixel block at strip rows 4 br.., columns 4 bc..;
// the level-3 coefficient of its 8x8 block is shared by 2 x 2 threads.  Row
// FFTs: 512 = 16 x 32, thread (r = tid >> 5, t = tid & 31) of each row, the
// 32-point stage split radix-2 across lane pairs (t = 2 k1 + b).  Strip row r at
// SP(544 r) = 544 r (a 512-wide row is 544 padded elements).
// Coefficient chunks of a strip (TMA landing zone layout, 4096 complex):
// [3][1024] level 1 (4 rows x 256), [3][256] level 2 (2 x 128), [3][64] level 3,
// [64] approximation (subband 0 when s == 3).

// forward row FFTs of the 8 x 512 strip in buf -> v[k'] = X_r[k1 + 16 k' + 256 b]
template <typename C>
__device__ __forceinline__ void strip_fft512_fwd(C* buf, C (&v)[16], const C* __restrict__ tw) {
    const int r = threadIdx.x >> 5, t = threadIdx.x & 31, k1 = t >> 1, b = t & 1;
    C* row = buf + 544 * r;
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = row[SP(32 * j + t)];
    dft_r<C, false, 16>(v);
    pow_twiddles512<C, false>(v, t, tw);
    __syncthreads();
#pragma unroll
    for (int m = 0; m < 16; ++m) row[SP(32 * m + t)] = v[m];
    __syncthreads();
#pragma unroll
    for (int a = 0; a < 16; ++a) v[a] = row[SP(32 * k1 + 2 * a + b)];
    dft_r<C, false, 16>(v);
    if (b) pow_twiddles512<C, false>(v, 16, tw);
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        const C o = mk<C>(__shfl_xor_sync(0xffffffffu, v[m].x, 1), __shfl_xor_sync(0xffffffffu, v[m].y, 1));
        v[m] = b ? csub(o, v[m]) : cadd(v[m], o);
    }
}

// inverse: v[k'] = X_r[k1 + 16 k' + 256 b] -> natural-order rows in buf (unnormalised)
template <typename C>
__device__ __forceinline__ void strip_ifft512_to_smem(C* buf, C (&v)[16], const C* __restrict__ tw) {
    const int r = threadIdx.x >> 5, t = threadIdx.x & 31, k1 = t >> 1, b = t & 1;
    C* row = buf + 544 * r;
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        const C o = mk<C>(__shfl_xor_sync(0xffffffffu, v[m].x, 1), __shfl_xor_sync(0xffffffffu, v[m].y, 1));
        v[m] = b ? csub(o, v[m]) : cadd(v[m], o);
    }
    if (b) pow_twiddles512<C, true>(v, 16, tw);
    dft_r<C, true, 16>(v);
#pragma unroll
    for (int a = 0; a < 16; ++a) row[SP(32 * k1 + 2 * a + b)] = v[a];
    __syncthreads();
#pragma unroll
    for (int m = 0; m < 16; ++m) v[m] = row[SP(32 * m + t)];
    pow_twiddles512<C, true>(v, t, tw);
    dft_r<C, true, 16>(v);
    __syncthreads();
#pragma unroll
    for (int n = 0; n < 16; ++n) row[SP(32 * n + t)] = v[n];
    __syncthreads();
}

// K1 for W = 512, k = 3
template <typename R>
__global__ void __launch_bounds__(PNT, sizeof(R) == 4 ? 4 : 2) synth512(Geo g, SynArgs<R> p) {
    typedef typename CT<R>::T C;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* buf = reinterpret_cast<C*>(smem_raw);
    const int st = blockIdx.x, bi = blockIdx.y, tid = threadIdx.x;
    const int br = tid >> 7, bc = tid & 127;
    const C* coef = p.coef + (long long)bi * g.N;
    __shared__ R spar[MAXS * 3];
    const int j1 = band_of(g.s, 1, 0), j2 = band_of(g.s, 2, 0), j3 = band_of(g.s, 3, 0);
    C* ob = buf;                                            // coefficient landing zone (early)
    __shared__ __align__(8) unsigned long long obar;
    const bool early = p.early != 0;
    if (early && tid == 0) {
        mbar_init(&obar, 1);
        const unsigned cs = (unsigned)sizeof(C);
        mbar_expect_tx(&obar, (p.asrc ? 4032u : 4096u) * cs);
        for (int o = 0; o < 3; ++o) {
            bulk_g2s(ob + o * 1024, coef + g.off[j1 + o] + (long long)st * 1024, 1024u * cs, &obar);
            bulk_g2s(ob + 3072 + o * 256, coef + g.off[j2 + o] + (long long)st * 256, 256u * cs, &obar);
            bulk_g2s(ob + 3840 + o * 64, coef + g.off[j3 + o] + (long long)st * 64, 64u * cs, &obar);
        }
        if (!p.asrc) bulk_g2s(ob + 4032, coef + g.off[0] + (long long)st * 64, 64u * cs, &obar);
    }
    pdl_enter();
    const double* par = p.par ? p.par + (long long)bi * g.S * 3 : nullptr;
    for (int i = tid; i < g.S * 3; i += PNT) spar[i] = par ? (R)par[i] : ((i % 3) == 2 ? R(1) : R(0));
    C d1[3][2][2], d2[3], d3[3], a3;
    {
        const long long o3 = (long long)st * 64 + (bc >> 1);
        if (early) {
            a3 = p.asrc ? p.asrc[(long long)bi * p.asrc_bs + o3] : mk<C>(R(0), R(0));
            __syncthreads();
            mbar_wait(&obar, 0);
#pragma unroll
            for (int o = 0; o < 3; ++o) {
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    d1[o][i][0] = ob[o * 1024 + (2 * br + i) * 256 + 2 * bc];
                    d1[o][i][1] = ob[o * 1024 + (2 * br + i) * 256 + 2 * bc + 1];
                }
                d2[o] = ob[3072 + o * 256 + br * 128 + bc];
                d3[o] = ob[3840 + o * 64 + (bc >> 1)];
            }
            if (!p.asrc) a3 = ob[4032 + (bc >> 1)];
        } else {
            const long long o1 = (long long)st * 1024 + (2 * br) * 256 + 2 * bc;
#pragma unroll
            for (int o = 0; o < 3; ++o)
#pragma unroll
                for (int i = 0; i < 2; ++i) ld2c<C>(coef + g.off[j1 + o] + o1 + i * 256, d1[o][i][0], d1[o][i][1]);
            const long long o2 = (long long)st * 256 + br * 128 + bc;
#pragma unroll
            for (int o = 0; o < 3; ++o) {
                d2[o] = coef[g.off[j2 + o] + o2];
                d3[o] = coef[g.off[j3 + o] + o3];
            }
            a3 = p.asrc ? p.asrc[(long long)bi * p.asrc_bs + o3] : coef[g.off[0] + o3];
        }
    }
    __syncthreads();                                        // spar; every thread holds its coefficients (buf free)
    C px[4][4];
    auto body = [&](auto onsc) {
        constexpr bool ONS = decltype(onsc)::value;
        if (!p.asrc) a3 = ons_j<R, ONS>(a3, spar, 0);
        const C a2 = haar_syn_q<R, C>(a3, ons_j<R, ONS>(d3[0], spar, j3), ons_j<R, ONS>(d3[1], spar, j3 + 1),
                                      ons_j<R, ONS>(d3[2], spar, j3 + 2), br & 1, bc & 1);
        const C h2 = ons_j<R, ONS>(d2[0], spar, j2), v2 = ons_j<R, ONS>(d2[1], spar, j2 + 1),
                e2 = ons_j<R, ONS>(d2[2], spar, j2 + 2);
        const R sc = R(1) / sqrt(R(512));                   // unitary 1 / sqrt(W) of the row FFT
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const C a1 = haar_syn_q<R, C>(a2, h2, v2, e2, i, j);
                const C lh = ons_j<R, ONS>(d1[0][i][j], spar, j1), hl = ons_j<R, ONS>(d1[1][i][j], spar, j1 + 1),
                        hh = ons_j<R, ONS>(d1[2][i][j], spar, j1 + 2);
                const C lo0 = Haar<R>::sum(a1, lh), lo1 = Haar<R>::dif(a1, lh);
                const C hi0 = Haar<R>::sum(hl, hh), hi1 = Haar<R>::dif(hl, hh);
                px[2 * i][2 * j] = cscale(Haar<R>::sum(lo0, hi0), sc);
                px[2 * i][2 * j + 1] = cscale(Haar<R>::sum(lo1, hi1), -sc);
                px[2 * i + 1][2 * j] = cscale(Haar<R>::dif(lo0, hi0), -sc);
                px[2 * i + 1][2 * j + 1] = cscale(Haar<R>::dif(lo1, hi1), sc);
            }
    };
    if (par) body(std::true_type{});
    else body(std::false_type{});
    {
        C* b0 = buf + 544 * (4 * br) + SP(4 * bc);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) b0[544 * i + j] = px[i][j];
    }
    __syncthreads();
    C v[16];
    strip_fft512_fwd<C>(buf, v, p.tw);
    {
        const int r = tid >> 5, t = tid & 31;
        C* drow = p.dst + (long long)bi * p.dst_bs + (long long)st * 4096 + r * 512 + (t >> 1) + 256 * (t & 1);
#pragma unroll
        for (int m = 0; m < 16; ++m) drow[16 * m] = v[m];
    }
}

// K3 for W = 512, k = 3
template <typename R, int OUT>
__global__ void __launch_bounds__(PNT, sizeof(R) == 4 ? 4 : 2) analysis512(Geo g, AnaArgs<R> p) {
    typedef typename CT<R>::T C;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* buf = reinterpret_cast<C*>(smem_raw);
    const int st = blockIdx.x, bi = blockIdx.y, tid = threadIdx.x;
    const int br = tid >> 7, bc = tid & 127;
    C* coef = p.coef + (long long)bi * g.N;
    __shared__ R spar[MAXS * 3];
    __shared__ C x2[2][128];                                // level-2 approximations
    const int j1 = band_of(g.s, 1, 0), j2 = band_of(g.s, 2, 0), j3 = band_of(g.s, 3, 0);
    const long long o1 = (long long)st * 1024 + (2 * br) * 256 + 2 * bc;
    const long long o2 = (long long)st * 256 + br * 128 + bc;
    constexpr bool OT = OUT == ANA_OUT_VDAMP;
    C* ob = buf + SP(4095) + 1;
    ob = reinterpret_cast<C*>((reinterpret_cast<uintptr_t>(ob) + 15) & ~(uintptr_t)15);
    __shared__ __align__(8) unsigned long long obar;
    if (OT && tid == 0) {
        mbar_init(&obar, 1);
        const unsigned cs = (unsigned)sizeof(C);
        mbar_expect_tx(&obar, (p.adst ? 4032u : 4096u) * cs);
        for (int o = 0; o < 3; ++o) {
            bulk_g2s(ob + o * 1024, coef + g.off[j1 + o] + (long long)st * 1024, 1024u * cs, &obar);
            bulk_g2s(ob + 3072 + o * 256, coef + g.off[j2 + o] + (long long)st * 256, 256u * cs, &obar);
            bulk_g2s(ob + 3840 + o * 64, coef + g.off[j3 + o] + (long long)st * 64, 64u * cs, &obar);
        }
        if (!p.adst) bulk_g2s(ob + 4032, coef + g.off[0] + (long long)st * 64, 64u * cs, &obar);
    }
    if (OUT == ANA_OUT_VDAMP) {
        const double* par = p.par + (long long)bi * g.S * 3;
        for (int i = tid; i < g.S * 3; i += PNT) spar[i] = (R)par[i];
    }
    pdl_enter();
    {
        C v[16];
        const int r = tid >> 5, t = tid & 31;
        const C* srow = p.src + (long long)bi * p.src_bs + (long long)st * 4096 + r * 512 + (t >> 1) + 256 * (t & 1);
#pragma unroll
        for (int m = 0; m < 16; ++m) v[m] = srow[16 * m];
        strip_ifft512_to_smem<C>(buf, v, p.tw);
    }
    const R sc = (R)g.sign_c / sqrt(R(512));
    C h1[2][2], v1[2][2], e1[2][2], l1[2][2];
    {
        const C* b0 = buf + 544 * (4 * br) + SP(4 * bc);
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const C x00 = cscale(b0[544 * (2 * i) + 2 * j], sc);
                const C x01 = cscale(b0[544 * (2 * i) + 2 * j + 1], -sc);
                const C x10 = cscale(b0[544 * (2 * i + 1) + 2 * j], -sc);
                const C x11 = cscale(b0[544 * (2 * i + 1) + 2 * j + 1], sc);
                const C lo0 = Haar<R>::sum(x00, x10), hi0 = Haar<R>::dif(x00, x10);
                const C lo1 = Haar<R>::sum(x01, x11), hi1 = Haar<R>::dif(x01, x11);
                l1[i][j] = Haar<R>::sum(lo0, lo1);
                h1[i][j] = Haar<R>::dif(lo0, lo1);
                v1[i][j] = Haar<R>::sum(hi0, hi1);
                e1[i][j] = Haar<R>::dif(hi0, hi1);
            }
    }
    C l2, h2, v2, e2;
    {
        const C lo0 = Haar<R>::sum(l1[0][0], l1[1][0]), hi0 = Haar<R>::dif(l1[0][0], l1[1][0]);
        const C lo1 = Haar<R>::sum(l1[0][1], l1[1][1]), hi1 = Haar<R>::dif(l1[0][1], l1[1][1]);
        l2 = Haar<R>::sum(lo0, lo1); h2 = Haar<R>::dif(lo0, lo1); v2 = Haar<R>::sum(hi0, hi1); e2 = Haar<R>::dif(hi0, hi1);
    }
    x2[br][bc] = l2;
    {
        const C n1[3][2][2] = {{{h1[0][0], h1[0][1]}, {h1[1][0], h1[1][1]}},
                               {{v1[0][0], v1[0][1]}, {v1[1][0], v1[1][1]}},
                               {{e1[0][0], e1[0][1]}, {e1[1][0], e1[1][1]}}};
        const C n2[3] = {h2, v2, e2};
        if (OT) mbar_wait(&obar, 0);
#pragma unroll
        for (int o = 0; o < 3; ++o) {
            C* q1 = coef + g.off[j1 + o] + o1;
            C* q2 = coef + g.off[j2 + o] + o2;
            C w1[2][2], w2 = n2[o];
#pragma unroll
            for (int i = 0; i < 2; ++i) { w1[i][0] = n1[o][i][0]; w1[i][1] = n1[o][i][1]; }
            if (OUT == ANA_OUT_VDAMP) {
#pragma unroll
                for (int i = 0; i < 2; ++i)
#pragma unroll
                    for (int j = 0; j < 2; ++j)
                        w1[i][j] = cadd(ons_j<R, true>(ob[o * 1024 + (2 * br + i) * 256 + 2 * bc + j], spar, j1 + o), w1[i][j]);
                w2 = cadd(ons_j<R, true>(ob[3072 + o * 256 + br * 128 + bc], spar, j2 + o), w2);
            }
#pragma unroll
            for (int i = 0; i < 2; ++i) st2c<C>(q1 + i * 256, w1[i][0], w1[i][1]);
            *q2 = w2;
        }
    }
    __syncthreads();
    // level 3: 64 threads, one per 8x8 block (one row of 64 level-3 coefficients)
    if (tid >= 64) return;
    {
        const C x00 = x2[0][2 * tid], x01 = x2[0][2 * tid + 1], x10 = x2[1][2 * tid], x11 = x2[1][2 * tid + 1];
        const C lo0 = Haar<R>::sum(x00, x10), hi0 = Haar<R>::dif(x00, x10);
        const C lo1 = Haar<R>::sum(x01, x11), hi1 = Haar<R>::dif(x01, x11);
        C n3[3] = {Haar<R>::dif(lo0, lo1), Haar<R>::sum(hi0, hi1), Haar<R>::dif(hi0, hi1)};
        C a = Haar<R>::sum(lo0, lo1);
        const long long o3 = (long long)st * 64 + tid;
#pragma unroll
        for (int o = 0; o < 3; ++o) {
            C* q = coef + g.off[j3 + o] + o3;
            if (OUT == ANA_OUT_VDAMP) n3[o] = cadd(ons_j<R, true>(ob[3840 + o * 64 + tid], spar, j3 + o), n3[o]);
            *q = n3[o];
        }
        if (p.adst) {
            p.adst[(long long)bi * p.adst_bs + o3] = a;
        } else {
            C* q = coef + g.off[0] + o3;
            if (OUT == ANA_OUT_VDAMP) a = cadd(ons_j<R, true>(ob[4032 + tid], spar, 0), a);
            *q = a;
        }
    }
}

// ------------------------------------------------------------------ K2 ----
// COL_RAW: forward column FFT without the centring sign (X0 setup);
// COL_NMSE: forward column FFT + Parseval error vs X0 off the mask (no IFFT)
enum { COL_FWD = 0, COL_INV = 1, COL_VDAMP = 2, COL_FINAL = 3, COL_RAW = 4, COL_NMSE = 5 };

template <typename R>
struct ColArgs {
    const typename CT<R>::T* src;    // [B][H][W]
    typename CT<R>::T* dst;          // [B][H][W]
    const typename CT<R>::T* yg;     // sign-folded y on the grid (0 off mask)
    const R* pinv;                   // 1/p on the grid, 0 off mask
    const double* noise_var;         // [B]
    const double* prow;              // [2s][H] row (axis-0) profiles
    const double* pcol;              // [2s][W] column profiles
    double* taupart;                 // [B][ntiles][S]
    const typename CT<R>::T* tw;     // length H
    int cw, logcw, ntiles;
    const typename CT<R>::T* x0r;    // COL_NMSE: raw unitary FFT2 of s_in * x0
    double* nmsepart;                // COL_NMSE: [B][ntiles] error partials
    const R* prs256;                 // col_pass256/512: row profiles as [H][npp] (npp = 2s rounded up to 4)
};

__device__ __forceinline__ void band_profiles(int s, int j, int& prow, int& pcol) {
    if (j == 0) { prow = 2 * (s - 1); pcol = 2 * (s - 1); return; }
    const int l = s - (j - 1) / 3, o = (j - 1) % 3;
    prow = 2 * (l - 1) + (o >= 1 ? 1 : 0);
    pcol = 2 * (l - 1) + (o != 1 ? 1 : 0);
}

// tau weight p^-1 ((p^-1 - 1) |z|^2 + sigma^2) of one sampled point
// (src/vdamp.py:74-75).  fp32 mode stores it as float anyway and every term is
// >= 0 (p^-1 >= 1), so it is evaluated in float there (no cancellation; the
// float64 version cost a quarter of the column kernel in F2F conversions).
__device__ __forceinline__ float tau_weight(float pv, float2 zc, double, float nvf) {
    return pv * fmaf(pv - 1.0f, fmaf(zc.x, zc.x, zc.y * zc.y), nvf);
}
__device__ __forceinline__ double tau_weight(double pv, double2 zc, double nv, float) {
    return pv * ((pv - 1.0) * (zc.x * zc.x + zc.y * zc.y) + nv);
}

template <typename R, int MODE>
__global__ void __launch_bounds__(PNT, sizeof(R) == 4 ? 3 : 2) col_pass(Geo g, ColArgs<R> p) {
    pdl_enter();
    typedef typename CT<R>::T C;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* buf = reinterpret_cast<C*>(smem_raw);
    const int H = g.H, W = g.W, cw = p.cw, lc = p.logcw;
    const int E = H << lc;
    C* tws = buf + E;
    const int tile = blockIdx.x, bi = blockIdx.y, tid = threadIdx.x;
    const int c0 = tile << lc;
    const long long ib = (long long)bi * g.N;
    for (int e = tid; e < H; e += PNT) tws[e] = p.tw[e];
    {
        constexpr int PER = PCAP / PNT;
        C v[PER];
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int e = tid + i * PNT;
            if (e < E) v[i] = p.src[ib + (long long)(e >> lc) * W + c0 + (e & (cw - 1))];
        }
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int e = tid + i * PNT;
            if (e < E) buf[e] = v[i];
        }
    }
    __syncthreads();
    if (MODE == COL_INV) block_fft16<C, true, PNT, PCAP, true, false>(buf, g.logH, lc, 1, cw, tws);
    else                 block_fft16<C, false, PNT, PCAP, true, false>(buf, g.logH, lc, 1, cw, tws);
    const R sc = R(1) / sqrt(R(H));
    if (MODE == COL_FWD || MODE == COL_INV) {
        // centred output sign c * (-1)^(k1+k2)
        for (int e = tid; e < E; e += PNT) {
            const int n = e >> lc, col = c0 + (e & (cw - 1));
            const R s = (((n + col) & 1) ? -sc : sc) * (R)g.sign_c;
            p.dst[ib + (long long)n * W + col] = cscale(buf[e], s);
        }
        return;
    }
    if (MODE == COL_RAW) {
        for (int e = tid; e < E; e += PNT)
            p.dst[ib + (long long)(e >> lc) * W + c0 + (e & (cw - 1))] = cscale(buf[e], sc);
        return;
    }
    if (MODE == COL_NMSE) {
        // ||x_hat - x0||^2 off the mask = sum |F Psi^H w - F x0|^2 (Parseval; on the
        // mask x_hat has exactly y, that part is a per-run constant)
        double e2 = 0.0;
        for (int e = tid; e < E; e += PNT) {
            const long long gi = ib + (long long)(e >> lc) * W + c0 + (e & (cw - 1));
            if (p.pinv[gi] == R(0)) {
                const C d = csub(cscale(buf[e], sc), p.x0r[gi]);
                e2 += (double)d.x * (double)d.x + (double)d.y * (double)d.y;
            }
        }
        double* sh = reinterpret_cast<double*>(tws + H);
        e2 = block_sum<PNT>(e2, sh);
        if (tid == 0) p.nmsepart[(long long)bi * p.ntiles + tile] = e2;
        return;
    }
    const R cs = (R)g.sign_c;
    const double nv = (MODE == COL_VDAMP) ? p.noise_var[bi] : 0.0;
    const float nvf = (float)nv;
    // tau partials: tau_j = sum_w a_j(w1) b_j(w2) weight(w) (separable |F psi_j|^2,
    // src/vdamp.py:59-78).  Thread tid always sees column c = tid % cw (PNT is a
    // multiple of cw), so it accumulates its rows' weights per row profile in
    // registers; the cw-column partials are combined in a fixed order below.
    constexpr int PER = PCAP / PNT;               // elements per thread
    R wreg[PER];                                  // tau weights of this thread's elements
    const int np = 2 * g.s;
    R pvs[PER];
    C ys[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {               // issue all measurement loads first
        const int e = tid + i * PNT;
        if (e < E) {
            const long long gi = ib + (long long)(e >> lc) * W + c0 + (e & (cw - 1));
            pvs[i] = p.pinv[gi];
            ys[i] = p.yg[gi];
        }
    }
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int e = tid + i * PNT;
        wreg[i] = R(0);
        if (e < E) {
            const C X = cscale(buf[e], sc * cs);     // c * FFT2u, so (-1)^(k1+k2) X_centred
            const R pv = pvs[i];
            C v;
            if (MODE == COL_VDAMP) {
                if (pv != R(0)) {
                    const C zc = csub(ys[i], X);             // (-1)^(k1+k2) z  (src/vdamp.py:112)
                    v = cscale(zc, pv);                      // P^-1 z           (src/vdamp.py:113)
                    wreg[i] = tau_weight(pv, zc, nv, nvf);   // tau weight (src/vdamp.py:74-75)
                } else {
                    v = mk<C>(R(0), R(0));
                }
            } else {  // COL_FINAL: measured k-space where sampled (src/vdamp.py:147-150)
                v = (pv != R(0)) ? ys[i] : X;
            }
            buf[e] = v;
        }
    }
    __syncthreads();
    block_fft16<C, true, PNT, PCAP, true, false>(buf, g.logH, lc, 1, cw, tws);
    for (int e = tid; e < E; e += PNT)
        p.dst[ib + (long long)(e >> lc) * W + c0 + (e & (cw - 1))] = cscale(buf[e], sc);
    if (MODE != COL_VDAMP) return;

    // thread tid always sees column c = tid % cw (PNT is a multiple of cw):
    // per row profile q, sum its rows in registers, then combine the threads
    // of each column in a fixed order (deterministic)
    // per-thread sums over its <= 16 rows in the working precision (float in
    // fp32 mode: 1e-7 relative), thread and column combination in float64
    // the tile buffer is free once every thread has stored its outputs: the
    // partials and row profiles reuse it (keeps the CTA at 34 KB of smem)
    __syncthreads();
    double* part = reinterpret_cast<double*>(buf);       // [np][PNT] thread partials
    R* prs = reinterpret_cast<R*>(part + np * PNT + np * cw);   // [np][H] row profiles
    for (int i = tid; i < np * H; i += PNT) prs[i] = (R)p.prow[i];
    __syncthreads();
    for (int q = 0; q < np; ++q) {
        R a = R(0);
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int e = tid + i * PNT;
            if (e < E) a += prs[q * H + (e >> lc)] * wreg[i];
        }
        part[q * PNT + tid] = (double)a;
    }
    __syncthreads();
    double* psum = part + np * PNT;                       // [np][cw] column partials
    for (int it = tid; it < np * cw; it += PNT) {
        const int q = it / cw, c = it % cw;
        double sacc = 0.0;
        for (int t = c; t < PNT; t += cw) sacc += part[q * PNT + t];
        psum[q * cw + c] = sacc;
    }
    __syncthreads();
    for (int j = tid; j < g.S; j += PNT) {
        int pr_, pc_;
        band_profiles(g.s, j, pr_, pc_);
        const double* Bc = p.pcol + (long long)pc_ * W + c0;
        double sacc = 0.0;
        for (int c = 0; c < cw; ++c) sacc += Bc[c] * psum[pr_ * cw + c];
        p.taupart[((long long)bi * p.ntiles + tile) * g.S + j] = sacc;
    }
}

template <typename R> __device__ __forceinline__ void ld4(const R* q, R& a, R& b, R& c, R& d);
template <> __device__ __forceinline__ void ld4<float>(const float* q, float& a, float& b, float& c, float& d) {
    const float4 t = *reinterpret_cast<const float4*>(q); a = t.x; b = t.y; c = t.z; d = t.w;
}
template <> __device__ __forceinline__ void ld4<double>(const double* q, double& a, double& b, double& c, double& d) {
    const double2 t0 = reinterpret_cast<const double2*>(q)[0], t1 = reinterpret_cast<const double2*>(q)[1];
    a = t0.x; b = t0.y; c = t1.x; d = t1.y;
}

// K2 for H = 256 (16-column tiles): the same computation as col_pass with both
// column FFTs in registers (fft256_stage_a + one shared-memory transpose each).
// Thread (c = tid & 15, d = tid >> 4) loads rows 16 n1 + d of column c, holds
// X[d + 16 k2] after the forward FFT, applies the residual / finalize step to
// those 16 frequencies and runs the inverse FFT from them directly; outputs are
// rows d + 16 n2.  Modes: COL_VDAMP, COL_FINAL, COL_NMSE.
// bytes of col_pass256's first shared region: the transpose tile, later the
// column sums [np][16] (doubles); the thread partials have their own region
template <typename R>
__host__ __device__ constexpr int col512_region0(int np) {
    return (4096 * 2 * (int)sizeof(R) > np * (256 + 8) * 8) ? 4096 * 2 * (int)sizeof(R) : np * (256 + 8) * 8;
}
template <typename R>
__host__ __device__ constexpr int col256_region0(int np) {
    return (4096 * 2 * (int)sizeof(R) > np * 16 * 8) ? 4096 * 2 * (int)sizeof(R) : np * 16 * 8;
}
template <typename R, int MODE>
__global__ void __launch_bounds__(PNT, sizeof(R) == 4 ? 3 : 2) col_pass256(Geo g, ColArgs<R> p) {
    typedef typename CT<R>::T C;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* buf = reinterpret_cast<C*>(smem_raw);              // [16][16][16] transpose tile
    const int W = g.W;
    const int tile = blockIdx.x, bi = blockIdx.y, tid = threadIdx.x;
    const int c = tid & 15, d = tid >> 4;
    const int c0 = tile << 4;
    const long long ib = (long long)bi * g.N;
    const long long colbase = ib + (long long)d * W + c0 + c;   // row d of this thread's column
    // shared layout: [0, A) transpose tile, later the tau partials; then the row
    // profiles [256][npp] (R) and this tile's column profiles [np][16] (double)
    const int np = 2 * g.s, npp = (np + 3) & ~3;
    const int A = col256_region0<R>(np);
    R* prs = reinterpret_cast<R*>(smem_raw + A);
    double* pcs = reinterpret_cast<double*>(smem_raw + A + 256 * npp * (int)sizeof(R));
    if (MODE != COL_NMSE) {
        // the measurements do not depend on the previous kernel: pull this
        // tile's rows of y and 1/p towards L2 before waiting on it
        const long long ri = ib + (long long)tid * W + c0;
        prefetch_l2(p.yg + ri);
        if (sizeof(R) == 8) prefetch_l2(p.yg + ri + 8);
        prefetch_l2(p.pinv + ri);
    }
    __shared__ __align__(8) unsigned long long pbar;
    if (MODE == COL_VDAMP && tid == 0) {
        // constant profiles, bulk-copied before the wait as well: the row
        // profiles pre-arranged [256][npp] at plan creation, the tile's 16
        // columns of each column profile
        mbar_init(&pbar, 1);
        const unsigned rb = 256u * (unsigned)npp * (unsigned)sizeof(R);
        mbar_expect_tx(&pbar, rb + (unsigned)np * 128u);
        bulk_g2s(prs, p.prs256, rb, &pbar);
        for (int q = 0; q < np; ++q) bulk_g2s(pcs + q * 16, p.pcol + (long long)q * W + c0, 128u, &pbar);
    }
    pdl_enter();
    C v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = p.src[colbase + (long long)(16 * j) * W];
    // 1/p (L2-prefetched before the wait) loads under the forward FFT; y at its use
    R pvs[16];
    // y and 1/p are read once per iteration; as streaming loads (evict-first, -DVDAMP_STREAM_LOADS)
    // they leave T2 in L2 for K3 on a batch that nearly fits it (cfg1: K3 0.785 -> 0.731 ms/step)
    // but slow this kernel on a batch that streams from DRAM anyway (cfg4: K2 10.8 -> 11.5
    // ms/step): plain loads
#ifndef VDAMP_STREAM_LOADS
#define YS(k) p.yg[colbase + (long long)(16 * (k)) * W]
#define PS(k) p.pinv[colbase + (long long)(16 * (k)) * W]
#else
#define YS(k) __ldcs(p.yg + colbase + (long long)(16 * (k)) * W)
#define PS(k) __ldcs(p.pinv + colbase + (long long)(16 * (k)) * W)
#endif
    if (MODE != COL_NMSE) {
#pragma unroll
        for (int k2 = 0; k2 < 16; ++k2) pvs[k2] = PS(k2);
    }
#undef PS
    fft256_stage_a<C, false>(v, d, p.tw);
#pragma unroll
    for (int m = 0; m < 16; ++m) buf[(m * 16 + d) * 16 + c] = v[m];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = buf[(d * 16 + j) * 16 + c];
    dft_r<C, false, 16>(v);                                // v[k2] = FFT2u(row-FFT'd x)[d + 16 k2]
    const R sc = R(1) / R(16);                             // 1 / sqrt(256)
    if (MODE == COL_NMSE) {
        double e2 = 0.0;
#pragma unroll
        for (int k2 = 0; k2 < 16; ++k2) {
            const long long gi = colbase + (long long)(16 * k2) * W;
            if (p.pinv[gi] == R(0)) {
                const C df = csub(cscale(v[k2], sc), p.x0r[gi]);
                e2 += (double)df.x * (double)df.x + (double)df.y * (double)df.y;
            }
        }
        __syncthreads();                                   // transpose reads done: buf is scratch
        e2 = block_sum<PNT>(e2, reinterpret_cast<double*>(buf));
        if (tid == 0) p.nmsepart[(long long)bi * p.ntiles + tile] = e2;
        return;
    }
    const R cs = (R)g.sign_c;
    R wreg[16];
    {
        const double nv = (MODE == COL_VDAMP) ? p.noise_var[bi] : 0.0;
        const float nvf = (float)nv;
#pragma unroll
        for (int k2 = 0; k2 < 16; ++k2) {
            const C X = cscale(v[k2], sc * cs);            // c * FFT2u, so (-1)^(k1+k2) X_centred
            const R pv = pvs[k2];
            R wk = R(0);
            if (MODE == COL_VDAMP) {
                // selects, not a branch (the mask is random per element), with y
                // loaded here rather than under the FFT: 1.15 -> 1.01 ms/step cfg1
                const bool on = pv != R(0);
                const C zc = csub(YS(k2), X);                      // (-1)^(k1+k2) z  (src/vdamp.py:112)
                const C pz = cscale(zc, pv);                       // P^-1 z           (src/vdamp.py:113)
                v[k2] = mk<C>(on ? pz.x : R(0), on ? pz.y : R(0));
                const R tw_ = tau_weight(pv, zc, nv, nvf);         // tau weight (src/vdamp.py:74-75)
                wk = on ? tw_ : R(0);
            } else {  // COL_FINAL: measured k-space where sampled (src/vdamp.py:147-150)
                v[k2] = (pv != R(0)) ? YS(k2) : X;
            }
#undef YS
            wreg[k2] = wk;
        }
    }
    // tau partials (as col_pass) now, so the weights are dead before the
    // inverse FFT: per row profile q, this thread's 16 rows d + 16 k2 against
    // profiles staged row-major [row][npp] (float4 loads), into a dedicated
    // shared region [np][PNT]
    double* pearly = reinterpret_cast<double*>(smem_raw + A + 256 * npp * (int)sizeof(R) + np * 16 * 8);
    if (MODE == COL_VDAMP) {
        mbar_wait(&pbar, 0);                               // profiles landed
        for (int q0 = 0; q0 < np; q0 += 4) {
            R a0 = R(0), a1 = R(0), a2 = R(0), a3 = R(0);
#pragma unroll
            for (int k2 = 0; k2 < 16; ++k2) {
                R b0, b1, b2, b3;
                ld4<R>(prs + (d + 16 * k2) * npp + q0, b0, b1, b2, b3);
                const R wk = wreg[k2];
                a0 += b0 * wk; a1 += b1 * wk; a2 += b2 * wk; a3 += b3 * wk;
            }
            pearly[q0 * PNT + tid] = (double)a0;
            pearly[(q0 + 1) * PNT + tid] = (double)a1;
            if (q0 + 2 < np) { pearly[(q0 + 2) * PNT + tid] = (double)a2; pearly[(q0 + 3) * PNT + tid] = (double)a3; }
        }
    }
    fft256_stage_a<C, true>(v, d, p.tw);
    __syncthreads();                                       // forward transpose reads done
#pragma unroll
    for (int m = 0; m < 16; ++m) buf[(m * 16 + d) * 16 + c] = v[m];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = buf[(d * 16 + j) * 16 + c];
    dft_r<C, true, 16>(v);                                 // v[n2] = x[d + 16 n2]
#pragma unroll
    for (int n2 = 0; n2 < 16; ++n2) p.dst[colbase + (long long)(16 * n2) * W] = cscale(v[n2], sc);
    if (MODE != COL_VDAMP) return;

    // fixed-order combination over the 16 threads of each column, then the
    // column profiles
    __syncthreads();                                       // inverse transpose reads done
    double* part = pearly;                                 // [np][PNT] thread partials
    double* psum = reinterpret_cast<double*>(buf);         // [np][16] column partials
    for (int it = tid; it < np * 16; it += PNT) {
        const int q = it >> 4, cc = it & 15;
        double sacc = 0.0;
        for (int t = cc; t < PNT; t += 16) sacc += part[q * PNT + t];
        psum[q * 16 + cc] = sacc;
    }
    __syncthreads();
    for (int j = tid; j < g.S; j += PNT) {
        int pr_, pc_;
        band_profiles(g.s, j, pr_, pc_);
        double sacc = 0.0;
        for (int cc = 0; cc < 16; ++cc) sacc += pcs[pc_ * 16 + cc] * psum[pr_ * 16 + cc];
        p.taupart[((long long)bi * p.ntiles + tile) * g.S + j] = sacc;
    }
}

// K2 for H = 512 (8-column tiles): the same computation as col_pass with both
// 512-point column FFTs in registers, 512 = 16 x 32 with the 32-point stage
// split radix-2 across a lane pair.  Thread (c = tid & 7, t = tid >> 3):
//   A: v[n1] = x[32 n1 + t]; DFT16 over n1; w512^(t k1); transpose
//   B: thread t = 2 k1 + b takes y_k1[2 a + b], a = 0..15; DFT16 over a; w32^(b k');
//      radix-2 with its partner (lane ^ 8) -> X[k1 + 16 k' + 256 b], k' = 0..15
// The inverse runs the same steps backwards with conjugate twiddles.

template <typename R, int MODE>
__global__ void __launch_bounds__(PNT, 2) col_pass512(Geo g, ColArgs<R> p) {   // 2 CTAs/SM: spill-free
    typedef typename CT<R>::T C;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* buf = reinterpret_cast<C*>(smem_raw);              // [16 k1][32 t][8 c] transpose tile
    const int W = g.W;
    const int tile = blockIdx.x, bi = blockIdx.y, tid = threadIdx.x;
    const int c = tid & 7, t = tid >> 3;
    const int k1 = t >> 1, b = t & 1;
    const int c0 = tile << 3;
    const long long ib = (long long)bi * g.N;
    const int np = 2 * g.s, npp = (np + 3) & ~3;
    const int A = col512_region0<R>(np);
    R* prs = reinterpret_cast<R*>(smem_raw + A);          // [512][npp]
    double* pcs = reinterpret_cast<double*>(smem_raw + A + 512 * npp * (int)sizeof(R));   // [np][8]
    // frequency rows this thread holds after the forward FFT: k1 + 16 k' + 256 b
    const long long fbase = ib + (long long)(k1 + 256 * b) * W + c0 + c;
    if (MODE != COL_NMSE) {
        const long long r0 = ib + (long long)(2 * tid) * W + c0;         // 2 rows per thread
        prefetch_l2(p.yg + r0); prefetch_l2(p.yg + r0 + W);
        prefetch_l2(p.pinv + r0); prefetch_l2(p.pinv + r0 + W);
    }
    __shared__ __align__(8) unsigned long long pbar;
    if (MODE == COL_VDAMP && tid == 0) {
        mbar_init(&pbar, 1);
        const unsigned rb = 512u * (unsigned)npp * (unsigned)sizeof(R);
        mbar_expect_tx(&pbar, rb + (unsigned)np * 64u);
        for (unsigned o = 0; o < rb; o += 32768u) bulk_g2s(reinterpret_cast<char*>(prs) + o,
                                                           reinterpret_cast<const char*>(p.prs256) + o,
                                                           rb - o < 32768u ? rb - o : 32768u, &pbar);
        for (int q = 0; q < np; ++q) bulk_g2s(pcs + q * 8, p.pcol + (long long)q * W + c0, 64u, &pbar);
    }
    pdl_enter();
    C v[16];
    {
        const C* src = p.src + ib + (long long)t * W + c0 + c;
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = src[(long long)(32 * j) * W];
    }
    // A
    dft_r<C, false, 16>(v);
    pow_twiddles512<C, false>(v, t, p.tw);
#pragma unroll
    for (int m = 0; m < 16; ++m) buf[(m * 32 + t) * 8 + c] = v[m];
    __syncthreads();
    // B
#pragma unroll
    for (int a = 0; a < 16; ++a) v[a] = buf[(k1 * 32 + 2 * a + b) * 8 + c];
    dft_r<C, false, 16>(v);
    if (b) pow_twiddles512<C, false>(v, 16, p.tw);         // w32^k' = w512^(16 k')
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        const C o = mk<C>(__shfl_xor_sync(0xffffffffu, v[m].x, 8), __shfl_xor_sync(0xffffffffu, v[m].y, 8));
        v[m] = b ? csub(o, v[m]) : cadd(v[m], o);          // Z0 + w Z1 | Z0 - w Z1
    }
    const R sc = R(1) / sqrt(R(512));
    if (MODE == COL_NMSE) {
        double e2 = 0.0;
#pragma unroll
        for (int m = 0; m < 16; ++m) {
            const long long gi = fbase + (long long)(16 * m) * W;
            if (p.pinv[gi] == R(0)) {
                const C df = csub(cscale(v[m], sc), p.x0r[gi]);
                e2 += (double)df.x * (double)df.x + (double)df.y * (double)df.y;
            }
        }
        __syncthreads();
        e2 = block_sum<PNT>(e2, reinterpret_cast<double*>(buf));
        if (tid == 0) p.nmsepart[(long long)bi * p.ntiles + tile] = e2;
        return;
    }
    const R cs = (R)g.sign_c;
    R wreg[16];
    {
        const double nv = (MODE == COL_VDAMP) ? p.noise_var[bi] : 0.0;
        const float nvf = (float)nv;
        R pvs[16];
        C ys[16];
#pragma unroll
        for (int m = 0; m < 16; ++m) {
            const long long gi = fbase + (long long)(16 * m) * W;
            pvs[m] = p.pinv[gi];
            ys[m] = p.yg[gi];
        }
#pragma unroll
        for (int m = 0; m < 16; ++m) {
            const C X = cscale(v[m], sc * cs);
            const R pv = pvs[m];
            R wk = R(0);
            if (MODE == COL_VDAMP) {
                // selects, not a branch (the mask is random per element):
                // col 5.63 -> 4.21 ms/step on cfg2
                const bool on = pv != R(0);
                const C zc = csub(ys[m], X);                      // (-1)^(k1+k2) z  (src/vdamp.py:112)
                const C pz = cscale(zc, pv);                       // P^-1 z           (src/vdamp.py:113)
                v[m] = mk<C>(on ? pz.x : R(0), on ? pz.y : R(0));
                const R tw_ = tau_weight(pv, zc, nv, nvf);         // tau weight (src/vdamp.py:74-75)
                wk = on ? tw_ : R(0);
            } else {  // COL_FINAL
                v[m] = (pv != R(0)) ? ys[m] : X;
            }
            wreg[m] = wk;
        }
    }
    // B^-1: radix-2 with the partner, conjugate w32, inverse DFT16 -> y_k1[2 a + b]
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        const C o = mk<C>(__shfl_xor_sync(0xffffffffu, v[m].x, 8), __shfl_xor_sync(0xffffffffu, v[m].y, 8));
        v[m] = b ? csub(o, v[m]) : cadd(v[m], o);          // U0 + U1 | U0 - U1
    }
    if (b) pow_twiddles512<C, true>(v, 16, p.tw);
    dft_r<C, true, 16>(v);
    __syncthreads();                                       // forward transpose reads done
#pragma unroll
    for (int a = 0; a < 16; ++a) buf[(k1 * 32 + 2 * a + b) * 8 + c] = v[a];
    __syncthreads();
    // A^-1
#pragma unroll
    for (int m = 0; m < 16; ++m) v[m] = buf[(m * 32 + t) * 8 + c];
    pow_twiddles512<C, true>(v, t, p.tw);
    dft_r<C, true, 16>(v);                                 // v[n1] = x[32 n1 + t]
    {
        C* dst = p.dst + ib + (long long)t * W + c0 + c;
#pragma unroll
        for (int j = 0; j < 16; ++j) dst[(long long)(32 * j) * W] = cscale(v[j], sc);
    }
    if (MODE != COL_VDAMP) return;
    // tau partials: rows k1 + 16 m + 256 b of column c
    __syncthreads();
    mbar_wait(&pbar, 0);
    double* part = reinterpret_cast<double*>(buf);         // [np][PNT]
    double* psum = part + np * PNT;                        // [np][8]
    for (int q0 = 0; q0 < np; q0 += 4) {
        R a0 = R(0), a1 = R(0), a2 = R(0), a3 = R(0);
#pragma unroll
        for (int m = 0; m < 16; ++m) {
            R b0, b1, b2, b3;
            ld4<R>(prs + (k1 + 16 * m + 256 * b) * npp + q0, b0, b1, b2, b3);
            const R wk = wreg[m];
            a0 += b0 * wk; a1 += b1 * wk; a2 += b2 * wk; a3 += b3 * wk;
        }
        part[q0 * PNT + tid] = (double)a0;
        part[(q0 + 1) * PNT + tid] = (double)a1;
        if (q0 + 2 < np) { part[(q0 + 2) * PNT + tid] = (double)a2; part[(q0 + 3) * PNT + tid] = (double)a3; }
    }
    __syncthreads();
    for (int it = tid; it < np * 8; it += PNT) {
        const int q = it >> 3, cc = it & 7;
        double sacc = 0.0;
        for (int tt = cc; tt < PNT; tt += 8) sacc += part[q * PNT + tt];
        psum[q * 8 + cc] = sacc;
    }
    __syncthreads();
    for (int j = tid; j < g.S; j += PNT) {
        int pr_, pc_;
        band_profiles(g.s, j, pr_, pc_);
        double sacc = 0.0;
        for (int cc = 0; cc < 8; ++cc) sacc += pcs[pc_ * 8 + cc] * psum[pr_ * 8 + cc];
        p.taupart[((long long)bi * p.ntiles + tile) * g.S + j] = sacc;
    }
}

// Row FFT pass over strips of rows (fft2c/ifft2c operators, finalize output).
template <typename R, bool INV, bool PRE_SIGN, bool POST_SIGN>
__global__ void __launch_bounds__(PNT) row_pass(Geo g, const typename CT<R>::T* src,
                                                typename CT<R>::T* dst, const typename CT<R>::T* tw,
                                                int logrows) {
    typedef typename CT<R>::T C;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* buf = reinterpret_cast<C*>(smem_raw);
    const int W = g.W, E = W << logrows;
    C* tws = buf + SP(E - 1) + 1;
    const int st = blockIdx.x, bi = blockIdx.y, tid = threadIdx.x;
    const long long base = (long long)bi * g.N + (long long)st * E;
    const int rowbase = st << logrows;
    for (int e = tid; e < W; e += PNT) tws[e] = tw[e];
    for (int e = tid; e < E; e += PNT) {
        C v = src[base + e];
        if (PRE_SIGN && (((rowbase + (e >> g.logW)) + (e & (W - 1))) & 1)) v = mk<C>(-v.x, -v.y);
        buf[SP(e)] = v;
    }
    __syncthreads();
    block_fft16<C, INV, PNT, PCAP, false, true>(buf, g.logW, logrows, W, 1, tws);
    const R sc = R(1) / sqrt(R(W));
    for (int e = tid; e < E; e += PNT) {
        R s = sc;
        if (POST_SIGN) s = ((((rowbase + (e >> g.logW)) + (e & (W - 1))) & 1) ? -sc : sc) * (R)g.sign_c;
        dst[base + e] = cscale(buf[SP(e)], s);
    }
}

// ------------------------------------------------------------------ K4 ----
template <typename R>
struct SelArgs {
    const typename CT<R>::T* r;      // [B][N]
    const double* taupart;           // [B][ntiles][S] (or null when tau_in given)
    const double* tau_in;            // [B][S] or null
    int ntiles;
    double* par;                     // [B][S][3] Onsager params out
    double* parf;                    // [B][S][3] soft-threshold-only params out
    double* trace;                   // [B][S][TRACE_F] or null
    const typename CT<R>::T* w0;     // [B][N] ground-truth coefficients or null
    R* kA;                           // [B][N] key scratch (subbands > SCAP)
    R* kB;
    int prune;                       // bound-pruned exact selection (vdamp_prune.cuh): bit 0 4096..SCAP keys, bit 1 larger
    unsigned* pflag;                 // [B][S] fallback flags of sure_prune32 (1 = sort fully)
    const unsigned* only;            // non-null: process only the items flagged here
    unsigned long long cond;         // CUDA-graph conditional handle of the flag-scan launch (0: none): set to 1 by a kernel that flags
    int item_start[MAXS + 1];        // work items: subbands item_list[item_start[i] .. item_start[i+1])
    int item_list[MAXS];
};

struct Best { double risk, t, cnt, inv; };

// 1/m for m > 0 without the library reciprocal's out-of-line slow path (whose
// call forces register spills in the select kernels): hardware approximation
// plus two FMA Newton steps (within 1 ulp); extreme magnitudes are
// rescaled by an exact power of two first.
// m holds a float value (any positive float, denormals included, is a normal
// double whose reciprocal is a normal double): no rescaling needed
__device__ __forceinline__ double rcp_posf(double m) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(m));
    double e = fma(-m, r, 1.0); r = fma(r, e, r);
    e = fma(-m, r, 1.0); return fma(r, e, r);
}

__device__ __forceinline__ double rcp_pos(double m) {
    double sc = 1.0;
    if (m < 1e-300) { m *= 0x1p600; sc = 0x1p600; }           // exact power-of-two rescaling
    else if (m > 1e300) { m *= 0x1p-600; sc = 0x1p-600; }
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(m));
    double e = fma(-m, r, 1.0); r = fma(r, e, r);
    e = fma(-m, r, 1.0); r = fma(r, e, r);
    return r * sc;
}

__device__ __forceinline__ bool better(const Best& a, const Best& b) {
    return a.risk < b.risk || (a.risk == b.risk && a.t < b.t);
}

__device__ __forceinline__ void consider(Best& b, double risk, double t, double cnt, double inv) {
    Best c{risk, t, cnt, inv};
    if (better(c, b)) b = c;
}

// ---------------------------------------------------------------------------
// Block bitonic sort of n (power of two) magnitudes.  Thread t of the A = n/E
// active threads owns the E consecutive keys [t*E, t*E+E) in registers:
// partner distances j < E are register compare-exchanges, E <= j < 32E warp
// shuffles, larger ones go through shared memory.
// ---------------------------------------------------------------------------
// shared-memory key slot of sorted position i: one pad word per 32 keys, so
// the blocked per-thread ownership (lane stride E) is bank-conflict free
__device__ __forceinline__ int KI(int i) { return i + (i >> 5); }

__device__ __forceinline__ float kmin(float a, float b) { return fminf(a, b); }
__device__ __forceinline__ float kmax(float a, float b) { return fmaxf(a, b); }
__device__ __forceinline__ double kmin(double a, double b) { return fmin(a, b); }
__device__ __forceinline__ double kmax(double a, double b) { return fmax(a, b); }

template <typename R, int E, int J>
__device__ __forceinline__ void reg_stage(R (&v)[E], int base, int k) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
        if ((e & J) == 0) {
            const int f = e | J;
            const bool asc = ((base + e) & k) == 0;
            const R a = v[e], b = v[f];
            const R lo = kmin(a, b), hi = kmax(a, b);
            v[e] = asc ? lo : hi;
            v[f] = asc ? hi : lo;
        }
    }
}

template <typename R, int E>
__device__ __forceinline__ void reg_stages(R (&v)[E], int base, int k, int j) {
    // j < E: all remaining distances of this k down to 1
    if (E > 16 && j >= 16) { reg_stage<R, E, (E > 16 ? 16 : 1)>(v, base, k); }
    if (E > 8 && j >= 8)   { reg_stage<R, E, (E > 8 ? 8 : 1)>(v, base, k); }
    if (E > 4 && j >= 4)   { reg_stage<R, E, (E > 4 ? 4 : 1)>(v, base, k); }
    if (E > 2 && j >= 2)   { reg_stage<R, E, (E > 2 ? 2 : 1)>(v, base, k); }
    if (E > 1 && j >= 1)   { reg_stage<R, E, 1>(v, base, k); }
}

template <typename R, int E>
__device__ __noinline__ void block_sort_e(R* s, int n) {
    const int A = n / E;
    const int tid = threadIdx.x;
    const bool act = tid < A;
    const int base = tid * E;
    const unsigned mask = A >= 32 ? 0xffffffffu : ((1u << A) - 1u);
    R v[E];
    if (act) {
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = s[KI(base + e)];
    }
    for (int k = 2; k <= n; k <<= 1) {
        int j = k >> 1;
        for (; j >= 32 * E; j >>= 1) {                     // cross-warp: shared memory
            __syncthreads();
            if (act) {
#pragma unroll
                for (int e = 0; e < E; ++e) s[KI(base + e)] = v[e];
            }
            __syncthreads();
            if (act) {
                const bool asc = (base & k) == 0;
                const bool lower = (base & j) == 0;
                const bool keep_min = lower == asc;
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const R p = s[KI((base + e) ^ j)];
                    v[e] = keep_min ? kmin(v[e], p) : kmax(v[e], p);
                }
            }
        }
        if (act) {
            for (; j >= E; j >>= 1) {                      // cross-lane: shuffles
                const int m = j / E;
                const bool asc = (base & k) == 0;
                const bool keep_min = ((tid & m) == 0) == asc;
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const R p = __shfl_xor_sync(mask, v[e], m);
                    v[e] = keep_min ? kmin(v[e], p) : kmax(v[e], p);
                }
            }
            if (j >= 1) reg_stages<R, E>(v, base, k, j);
        }
    }
    __syncthreads();
    if (act) {
#pragma unroll
        for (int e = 0; e < E; ++e) s[KI(base + e)] = v[e];
    }
    __syncthreads();
}

template <typename R, int NT>
__device__ void block_sort(R* s, int n) {
    if (n < 2) { __syncthreads(); return; }
    int E = n / NT;
    const int small = n / 32 < 4 ? n / 32 : 4;
    if (E < small) E = small;
    if (E < 1) E = 1;
    switch (E) {
        case 1: block_sort_e<R, 1>(s, n); break;
        case 2: block_sort_e<R, 2>(s, n); break;
        case 4: block_sort_e<R, 4>(s, n); break;
        case 8: block_sort_e<R, 8>(s, n); break;
        default:
            if constexpr (SCAP / NT > 16) { if (E > 16) { block_sort_e<R, 32>(s, n); break; } }
            block_sort_e<R, 16>(s, n);
            break;
    }
}

// ---------------------------------------------------------------------------
// Counting sort of 4096 <= n <= SCAP float magnitudes (fp32 path), with a
// data-equalised bucket map.  Keys are IEEE bits (monotone for x >= 0); zeros
// go to bucket 0.  A coarse pass histograms the nonzero bit range into
// CS_COARSE equal-width coarse buckets; each coarse bucket c then receives a
// run of fine buckets proportional to its population (fs_c, w_c), and a key
// maps linearly into its coarse bucket's run.  The map is monotone in the
// key, and on the magnitudes VDAMP produces it leaves ~1 key per fine bucket
// (plain float-bit buckets crowd 10+ keys into the buckets of the Rayleigh
// bulk), so the buckets are finished by two passes of 16-key register
// bitonic sorts over overlapping windows; data with a bucket of more than 8
// keys takes an in-bucket ranking pass instead.  Histogram and scatter use
// packed 16-bit shared counters.  The sorted sequence is unique, so the
// result is deterministic.  `out` must not alias `keys`.
// ---------------------------------------------------------------------------
constexpr int CS_WORDS = 16384;   // 64 KB counter region (also the TMA landing zone's tail)
constexpr int CS_FINE = 16384;    // fine buckets (packed 16-bit: CS_FINE / 2 words)
constexpr int CS_COARSE = 1024;   // coarse buckets (one per thread of the 1024-thread CTA)
static_assert(CS_FINE / 2 + 2 * CS_COARSE <= CS_WORDS, "counting-sort tables exceed the counter region");

#ifdef VDAMP_PHASE_TIMING
__device__ long long g_csort[4096][64][8];
#define CS_MARK(i) do { if (threadIdx.x == 0 && dbg) { long long c_ = clock64(); dbg[i] = c_ - cs0_; cs0_ = c_; } } while (0)
#else
#define CS_MARK(i) do { } while (0)
#endif

constexpr int CS_MAXB = 256;      // larger fine buckets -> comparison-sort fallback (heavy ties)

// fine bucket of key k (a coarse bucket with an empty run, w = 0, sends its keys
// to the next run's first bucket: still monotone; clamped to the last bucket)
__device__ __forceinline__ unsigned cs_fine(unsigned k, int lc, unsigned cb, const unsigned* tab, unsigned last) {
    if (!k) return 0u;
    const unsigned c = (k >> lc) - cb;
    const unsigned t = tab[c];
    const unsigned long long off = (unsigned long long)(k - ((cb + c) << lc)) * (t >> 16);
    return min(1u + (t & 0xffffu) + (unsigned)(off >> lc), last);
}

__device__ __forceinline__ void sort16(unsigned (&v)[16]) {
#pragma unroll
    for (int k = 2; k <= 16; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int l = i ^ j;
                if (l > i) {
                    const unsigned x = v[i], y = v[l];
                    const bool up = (i & k) == 0;
                    v[i] = up ? min(x, y) : max(x, y);
                    v[l] = up ? max(x, y) : min(x, y);
                }
            }
        }
    }
}

// 0: some bucket holds more than CS_MAXB keys (nothing usable; the caller
// bitonic-sorts `keys`); 1: sorted keys in `out`; 2: sorted keys in `keys`.
// n == EF * NT (EF keys per thread, compile time); mn / mx: this thread's
// min nonzero / max key bits (from the key-building loop)
template <int NT, int EF>
__device__ int counting_sort(const float* keys, float* out, unsigned* cnt, int n, unsigned mn, unsigned mx,
                             double* sh, long long* dbg = nullptr) {
    static_assert(CS_COARSE % NT == 0 && NT <= CS_COARSE, "coarse scan: whole coarse buckets per thread");
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
#ifdef VDAMP_PHASE_TIMING
    long long cs0_ = clock64();
#endif
    const unsigned* kb = reinterpret_cast<const unsigned*>(keys);
    unsigned* ob = reinterpret_cast<unsigned*>(out);
    unsigned* hc = cnt + CS_FINE / 2;                // coarse histogram
    unsigned* tab = hc + CS_COARSE;                  // coarse bucket -> fine start | width << 16
    const int nbf = n >= CS_FINE ? CS_FINE : (int)(1u << (32 - __clz((unsigned)n - 1u)));
    const int words = nbf >> 1;
    for (int o = 16; o > 0; o >>= 1) {
        mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    unsigned* red = reinterpret_cast<unsigned*>(sh);
    __syncthreads();
    if (lane == 0) { red[w] = mn; red[32 + w] = mx; }
    for (int i = tid; i < words; i += NT) cnt[i] = 0;
    for (int i = tid; i < CS_COARSE; i += NT) hc[i] = 0;
    __syncthreads();
    if (tid < 32) {
        unsigned a = red[tid], b = red[32 + tid];
        for (int o = 16; o > 0; o >>= 1) {
            a = min(a, __shfl_xor_sync(0xffffffffu, a, o));
            b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
        }
        if (tid == 0) { red[64] = a; red[65] = b; }
    }
    __syncthreads();
    mn = red[64]; mx = red[65];
    if (mn > mx) mn = mx;                            // all zeros
    // smallest shift lc with (mx >> lc) - (mn >> lc) < CS_COARSE (= 2^10)
    const unsigned dd = mx - mn;
    int lc = dd < (unsigned)CS_COARSE ? 0 : (32 - __clz(dd)) - 10;
    if (((mx >> lc) - (mn >> lc)) >= (unsigned)CS_COARSE) ++lc;
    const unsigned cb = mn >> lc;
    // coarse histogram of the nonzero keys
    unsigned kr[EF];
#pragma unroll
    for (int e = 0; e < EF; ++e) kr[e] = kb[KI(tid + e * NT)];
    // (a 1-in-4 sample would save atomics, but its noisier map pushes buckets
    // past 8 keys and into the slow ranking pass: measured slower)
#pragma unroll
    for (int e = 0; e < EF; ++e)
        if (kr[e]) atomicAdd(&hc[(kr[e] >> lc) - cb], 1u);
    __syncthreads();
    CS_MARK(0);
    // coarse bucket t -> fine run [fs, fs + w) of the nbf - 1 nonzero buckets,
    // proportional to its population (integer arithmetic: exact, deterministic)
    {
        constexpr int CPT = CS_COARSE / NT;          // coarse buckets per thread
        unsigned h[CPT], hs = 0;
#pragma unroll
        for (int q = 0; q < CPT; ++q) { h[q] = hc[tid * CPT + q]; hs += h[q]; }
        unsigned P = (unsigned)block_excl_scan<NT, false>((double)hs, sh + 66);
        if (tid == NT - 1) red[66] = P + hs;
        __syncthreads();
        const unsigned tot = red[66];
        // fine start = floor(P * F / tot) through one double scale factor: monotone
        // in P and within [0, F], so runs never overlap (no 64-bit integer division)
        const double scl = tot ? (double)(nbf - 1) / (double)tot : 0.0;
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
            const unsigned fs = __double2uint_rz((double)P * scl);
            const unsigned fe = __double2uint_rz((double)(P + h[q]) * scl);
            tab[tid * CPT + q] = fs | ((fe - fs) << 16);
            P += h[q];
        }
    }
    __syncthreads();
    // fine histogram
#pragma unroll
    for (int e = 0; e < EF; ++e) {
        const unsigned b = cs_fine(kr[e], lc, cb, tab, (unsigned)nbf - 1u);
        atomicAdd(&cnt[b >> 1], 1u << ((b & 1u) * 16));
    }
    __syncthreads();
    CS_MARK(1);
    // exclusive scan of the fine counts (thread t: words [t*per, t*per + per)),
    // with the crowded-bucket flags folded into the same pass
    bool crowd8;
    {
        constexpr int PMAX = CS_FINE / 2 / NT;
        const int per = words / NT;
        unsigned v[PMAX];
        unsigned tot = 0, big = 0, c8 = 0;
#pragma unroll
        for (int i = 0; i < PMAX; ++i) {
            v[i] = i < per ? cnt[tid * per + i] : 0u;
            tot += (v[i] & 0xffffu) + (v[i] >> 16);
            const unsigned lo16 = (tid * per + i) ? (v[i] & 0xffffu) : 0u;   // bucket 0: zeros, in order
            big |= (lo16 > (unsigned)CS_MAXB) | ((v[i] >> 16) > (unsigned)CS_MAXB);
            c8 |= (lo16 > 8u) | ((v[i] >> 16) > 8u);
        }
        if (__syncthreads_or(big)) return 0;
        crowd8 = __syncthreads_or(c8) != 0;
        unsigned run = (unsigned)block_excl_scan<NT, false>((double)tot, sh + 66);
#pragma unroll
        for (int i = 0; i < PMAX; ++i) {
            if (i < per) {
                const unsigned c0 = v[i] & 0xffffu, c1 = v[i] >> 16;
                cnt[tid * per + i] = run | ((run + c0) << 16);
                run += c0 + c1;
            }
        }
    }
    __syncthreads();
    CS_MARK(2);
    // scatter (cursor = packed 16-bit half, never carries: offsets + counts <= n <= 16384)
#pragma unroll
    for (int e = 0; e < EF; ++e) {
        const unsigned k = kr[e];
        const unsigned b = cs_fine(k, lc, cb, tab, (unsigned)nbf - 1u);
        const unsigned sft = (b & 1u) * 16;
        const unsigned old = atomicAdd(&cnt[b >> 1], 1u << sft);
        ob[KI((old >> sft) & 0xffffu)] = k;
    }
    __syncthreads();
    CS_MARK(3);
    // every cursor now holds its bucket's end.  Fast path (all buckets <= 8
    // keys, the normal case with ~1 key per bucket): bitonic-sort the aligned
    // 16-key windows in registers, then the windows shifted by 8.  Sorting a
    // window only permutes keys of the same bucket (the bucket order is
    // already right), and every bucket of <= 8 keys lies inside one window of
    // one of the two passes, so both passes together sort every bucket.
    if (!crowd8) {
        for (int pass = 0; pass < 2; ++pass) {
            for (int p0 = tid * 16 + pass * 8; p0 + 16 <= n; p0 += NT * 16) {
                unsigned v[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) v[e] = ob[KI(p0 + e)];
                sort16(v);
#pragma unroll
                for (int e = 0; e < 16; ++e) ob[KI(p0 + e)] = v[e];
            }
            __syncthreads();
        }
        CS_MARK(4);
        return 1;
    }
    // slow path: rank every key inside its bucket (ties by grouped position),
    // writing the sorted sequence back into `keys` (consumed by now)
    unsigned* fb = const_cast<unsigned*>(kb);
    for (int i = tid; i < n; i += NT) {
        const unsigned x = ob[KI(i)];
        const unsigned bk = cs_fine(x, lc, cb, tab, (unsigned)nbf - 1u);
        const unsigned e1 = cnt[bk >> 1] >> ((bk & 1u) * 16) & 0xffffu;
        unsigned s0 = 0;
        if (bk > 0) { const unsigned bp = bk - 1u; s0 = cnt[bp >> 1] >> ((bp & 1u) * 16) & 0xffffu; }
        unsigned rank = 0;
        for (unsigned q = s0; q < e1; ++q) {
            const unsigned y = ob[KI(q)];
            rank += (y < x) || (y == x && (int)q < i);
        }
        fb[KI(s0 + rank)] = x;
    }
    __syncthreads();
    CS_MARK(4);
    return 2;
}

// ---------------------------------------------------------------------------
// Counting sort of a large subband (n > shared capacity) held in global
// scratch (L2-resident): 32768 32-bit bucket counters in shared memory, keys
// in A (input, overwritten by the sorted output) and B (bucket-grouped
// temporary).  Same bucket map and parallel in-bucket ranking as
// counting_sort; works on the IEEE bit patterns of float or double keys.
// ---------------------------------------------------------------------------
template <typename R> struct KeyU;
template <> struct KeyU<float> { typedef unsigned int U; };
template <> struct KeyU<double> { typedef unsigned long long U; };

// fp32 version with the data-equalised bucket map of counting_sort: a coarse
// histogram (1024 buckets over the key-bit range) assigns each coarse bucket a
// run of the GNBF fine buckets proportional to its population, so crowded value
// ranges spread out (~2 keys per bucket at 65,536 keys) and the in-bucket ranking
// stays O(1) per key.  Loads are batched GLB deep.  Zeros (fine bucket 0) are all
// equal and need no ranking.  Returns false if a nonzero bucket exceeds CS_MAXB.
template <int NT>
__device__ __noinline__ bool global_counting_sort_eq(float* A, float* B, unsigned* cnt, int n, double* sh) {
    constexpr int GNBF = 30720, NC = 1024, TILE = 16384, GLB = 8;
    static_assert(NC % NT == 0 || NT % NC == 0, "coarse buckets per thread");
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    unsigned* ka = reinterpret_cast<unsigned*>(A);
    unsigned* kb = reinterpret_cast<unsigned*>(B);
    unsigned* hc = cnt + GNBF;                       // coarse histogram
    unsigned* tab = hc + NC;                         // coarse bucket -> fine start | width << 16
    unsigned* tl = cnt + 32768;                      // ranking tile
    unsigned mn = 0xffffffffu, mx = 0;
    for (int e0 = tid; e0 < n; e0 += NT * GLB) {
        unsigned k[GLB];
#pragma unroll
        for (int u = 0; u < GLB; ++u) k[u] = e0 + u * NT < n ? __ldcg(ka + e0 + u * NT) : 0u;
#pragma unroll
        for (int u = 0; u < GLB; ++u) { if (k[u]) mn = min(mn, k[u]); mx = max(mx, k[u]); }
    }
    for (int o = 16; o > 0; o >>= 1) {
        mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    unsigned* red = reinterpret_cast<unsigned*>(sh);
    __syncthreads();
    if (lane == 0) { red[w] = mn; red[32 + w] = mx; }
    for (int i = tid; i < GNBF + NC; i += NT) cnt[i] = 0;
    __syncthreads();
    if (tid == 0) {
        unsigned a = red[0], b = red[32];
        for (int i = 1; i < NT / 32; ++i) { a = min(a, red[i]); b = max(b, red[32 + i]); }
        red[64] = a; red[65] = b;
    }
    __syncthreads();
    mn = red[64]; mx = red[65];
    if (mn > mx) mn = mx;                            // all zeros
    const unsigned dd = mx - mn;
    int lc = dd < (unsigned)NC ? 0 : (32 - __clz(dd)) - 10;
    if (((mx >> lc) - (mn >> lc)) >= (unsigned)NC) ++lc;
    const unsigned cb = mn >> lc;
    for (int e0 = tid; e0 < n; e0 += NT * GLB) {
        unsigned k[GLB];
#pragma unroll
        for (int u = 0; u < GLB; ++u) k[u] = e0 + u * NT < n ? __ldcg(ka + e0 + u * NT) : 0u;
#pragma unroll
        for (int u = 0; u < GLB; ++u) if (k[u]) atomicAdd(&hc[(k[u] >> lc) - cb], 1u);
    }
    __syncthreads();
    {
        constexpr int CPT = NC / NT > 0 ? NC / NT : 1;
        unsigned h[CPT], hs = 0;
#pragma unroll
        for (int q = 0; q < CPT; ++q) { h[q] = tid * CPT + q < NC ? hc[tid * CPT + q] : 0u; hs += h[q]; }
        unsigned P = (unsigned)block_excl_scan<NT, false>((double)hs, sh + 66);
        if (tid == NT - 1) red[66] = P + hs;
        __syncthreads();
        const unsigned tot = red[66];
        const double scl = tot ? (double)(GNBF - 1) / (double)tot : 0.0;
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
            if (tid * CPT + q < NC) {
                const unsigned fs = __double2uint_rz((double)P * scl);
                const unsigned fe = __double2uint_rz((double)(P + h[q]) * scl);
                tab[tid * CPT + q] = fs | ((fe - fs) << 16);
            }
            P += h[q];
        }
    }
    __syncthreads();
    auto bucket = [&](unsigned k) -> unsigned { return cs_fine(k, lc, cb, tab, (unsigned)GNBF - 1u); };
    for (int e0 = tid; e0 < n; e0 += NT * GLB) {
        unsigned k[GLB];
#pragma unroll
        for (int u = 0; u < GLB; ++u) k[u] = e0 + u * NT < n ? __ldcg(ka + e0 + u * NT) : 0xffffffffu;
#pragma unroll
        for (int u = 0; u < GLB; ++u) if (k[u] != 0xffffffffu) atomicAdd(&cnt[bucket(k[u])], 1u);
    }
    __syncthreads();
    {
        unsigned big = 0;
        for (int i = 1 + tid; i < GNBF; i += NT) big |= cnt[i] > (unsigned)CS_MAXB;
        if (__syncthreads_or(big)) return false;
    }
    {
        constexpr int PER = GNBF / NT;
        static_assert(GNBF % NT == 0, "fine buckets per thread");
        unsigned tot = 0;
        for (int i = 0; i < PER; ++i) tot += cnt[tid * PER + i];
        unsigned run = (unsigned)block_excl_scan<NT, false>((double)tot, sh + 66);
        for (int i = 0; i < PER; ++i) { const unsigned c = cnt[tid * PER + i]; cnt[tid * PER + i] = run; run += c; }
    }
    __syncthreads();
    for (int e0 = tid; e0 < n; e0 += NT * GLB) {
        unsigned k[GLB];
#pragma unroll
        for (int u = 0; u < GLB; ++u) k[u] = e0 + u * NT < n ? __ldcg(ka + e0 + u * NT) : 0xffffffffu;
#pragma unroll
        for (int u = 0; u < GLB; ++u) if (k[u] != 0xffffffffu) kb[atomicAdd(&cnt[bucket(k[u])], 1u)] = k[u];
    }
    __syncthreads();
    // cnt[b] = end of bucket b.  Zeros (bucket 0) are equal: copy.  Then rank
    // inside buckets tile by tile in shared memory (tiles end on bucket boundaries).
    const int z = (int)cnt[0];
    for (int i = tid; i < z; i += NT) ka[i] = 0u;
    int S0 = z;
    while (S0 < n) {
        int E0 = S0 + TILE < n ? S0 + TILE : n;
        if (E0 < n) {
            const unsigned bE = bucket(__ldcg(kb + E0));
            E0 = bE ? (int)cnt[bE - 1] : 0;            // start of the bucket holding position E0
        }
        for (int i = S0 + tid; i < E0; i += NT) tl[i - S0] = __ldcg(kb + i);
        __syncthreads();
        for (int i = S0 + tid; i < E0; i += NT) {
            const unsigned x = tl[i - S0];
            const unsigned b = bucket(x);
            const int e1 = (int)cnt[b], s0 = b ? (int)cnt[b - 1] : 0;
            unsigned rank = 0;
            for (int q = s0; q < e1; ++q) { const unsigned y = tl[q - S0]; rank += (y < x) || (y == x && q < i); }
            ka[s0 + rank] = x;
        }
        __syncthreads();
        S0 = E0;
    }
    return true;
}

template <typename R, int NT>
__device__ bool global_counting_sort(R* A, R* B, unsigned* cnt, int n, double* sh) {
    typedef typename KeyU<R>::U U;
    // 32768 buckets (fp32) / 8192 (fp64) 32-bit counters, followed in shared
    // memory by a ranking tile of GCS_TILE keys
    constexpr int NB = sizeof(R) == 4 ? 32768 : 8192;
    constexpr int TILE = sizeof(R) == 4 ? 16384 : 8192;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    U* ka = reinterpret_cast<U*>(A);
    U* kb = reinterpret_cast<U*>(B);
    U* tl = reinterpret_cast<U*>(cnt + NB);
    U mn = ~U(0), mx = 0;
    for (int i = tid; i < n; i += NT) { const U k = ka[i]; if (k) mn = k < mn ? k : mn; mx = k > mx ? k : mx; }
    for (int o = 16; o > 0; o >>= 1) {
        const U a = __shfl_xor_sync(0xffffffffu, mn, o), b = __shfl_xor_sync(0xffffffffu, mx, o);
        mn = a < mn ? a : mn; mx = b > mx ? b : mx;
    }
    U* red = reinterpret_cast<U*>(sh);
    __syncthreads();
    if (lane == 0) { red[w] = mn; red[32 + w] = mx; }
    for (int i = tid; i < NB; i += NT) cnt[i] = 0;
    __syncthreads();
    if (tid == 0) {
        U a = red[0], b = red[32];
        for (int i = 1; i < NT / 32; ++i) { a = red[i] < a ? red[i] : a; b = red[32 + i] > b ? red[32 + i] : b; }
        red[0] = a; red[32] = b;
    }
    __syncthreads();
    mn = red[0]; mx = red[32];
    __syncthreads();
    if (mn > mx) mn = mx;
    int lo = 0;
    while (((mx >> lo) - (mn >> lo)) >= (U)(NB - 2)) ++lo;
    const U base = mn >> lo;
    auto bucket = [&](U k) -> unsigned { return k ? (unsigned)((k >> lo) - base + 1) : 0u; };
    for (int i = tid; i < n; i += NT) atomicAdd(&cnt[bucket(ka[i])], 1u);
    __syncthreads();
    {
        unsigned big = 0;
        for (int i = tid; i < NB; i += NT) big |= cnt[i] > (unsigned)CS_MAXB;
        if (__syncthreads_or(big)) return false;
    }
    {
        constexpr int PER = NB / NT;
        unsigned tot = 0;
        for (int i = 0; i < PER; ++i) tot += cnt[tid * PER + i];
        unsigned run = (unsigned)block_excl_scan<NT, false>((double)tot, sh + 66);
        for (int i = 0; i < PER; ++i) { const unsigned c = cnt[tid * PER + i]; cnt[tid * PER + i] = run; run += c; }
    }
    __syncthreads();
    for (int i = tid; i < n; i += NT) {
        const U k = ka[i];
        kb[atomicAdd(&cnt[bucket(k)], 1u)] = k;
    }
    __syncthreads();
    // cnt[b] = end of bucket b.  Rank inside buckets tile by tile in shared
    // memory; tiles end on bucket boundaries so no bucket is split.
    int S0 = 0;
    while (S0 < n) {
        int E0 = S0 + TILE < n ? S0 + TILE : n;
        if (E0 < n) {
            const unsigned bE = bucket(kb[E0]);
            E0 = bE ? (int)cnt[bE - 1] : 0;            // start of the bucket holding position E0
        }
        if (E0 <= S0) {
            // one bucket larger than a tile: rank it straight from global memory
            E0 = (int)cnt[bucket(kb[S0])];
            for (int i = S0 + tid; i < E0; i += NT) {
                const U x = kb[i];
                unsigned rank = 0;
                for (int q = S0; q < E0; ++q) { const U y = kb[q]; rank += (y < x) || (y == x && q < i); }
                ka[S0 + rank] = x;
            }
            __syncthreads();
            S0 = E0;
            continue;
        }
        for (int i = S0 + tid; i < E0; i += NT) tl[i - S0] = kb[i];
        __syncthreads();
        for (int i = S0 + tid; i < E0; i += NT) {
            const U x = tl[i - S0];
            const unsigned b = bucket(x);
            const int e1 = (int)cnt[b], s0 = b ? (int)cnt[b - 1] : 0;
            unsigned rank = 0;
            for (int q = s0; q < e1; ++q) { const U y = tl[q - S0]; rank += (y < x) || (y == x && q < i); }
            ka[s0 + rank] = x;
        }
        __syncthreads();
        S0 = E0;
    }
    return true;
}

// Comparison-sort fallback for a large subband in global scratch: bitonic
// sort of CAP-key chunks in shared memory, then pairwise merge-path merges in
// global memory (n and CAP powers of two).  Returns the buffer holding the result.
template <typename R, int NT>
__device__ R* global_merge_sort(R* A, R* B, R* smem, int n, int CAP) {
    const int tid = threadIdx.x;
    for (int c0 = 0; c0 < n; c0 += CAP) {
        for (int e = tid; e < CAP; e += NT) smem[KI(e)] = A[c0 + e];
        __syncthreads();
        block_sort<R, NT>(smem, CAP);
        for (int e = tid; e < CAP; e += NT) A[c0 + e] = smem[KI(e)];
        __syncthreads();
    }
    R* srcb = A;
    R* dstb = B;
    const int per = n / NT;
    for (int w = CAP; w < n; w <<= 1) {
        const int o0 = tid * per;
        const int pb = o0 / (2 * w) * (2 * w);
        const R* X = srcb + pb;
        const R* Y = srcb + pb + w;
        const int d = o0 - pb;
        int lo = d > w ? d - w : 0, hi = d < w ? d : w;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (X[mid] <= Y[d - 1 - mid]) lo = mid + 1; else hi = mid;
        }
        int ia = lo, ib = d - lo;
        for (int e = 0; e < per; ++e) {
            R v;
            if (ib >= w || (ia < w && X[ia] <= Y[ib])) v = X[ia++]; else v = Y[ib++];
            dstb[o0 + e] = v;
        }
        __syncthreads();
        R* t = srcb; srcb = dstb; dstb = t;
    }
    return srcb;
}

// Evaluate the candidates owned by this thread on one tile of sorted
// magnitudes (src/denoise.py:62-118):  candidate t = m_i at the end of each
// tie run, plus the stationary point of the quadratic piece that starts there.
template <typename R, int NT, int EMAX, bool SMEM, int EFIX, bool RAG>
__device__ __forceinline__ void scan_keys(const R* keys, int T, int tilebase, int n, double tau, int b0, int E,
                                          double pre, double suf, double next_tile_first, Best& best,
                                          const double* sreg, const double* slo, const double* shi);

// One tile of the exact SURE scan.  Thread t owns the E consecutive sorted keys
// [t*E, t*E + E).  The suffix of inverses is accumulated from the large keys
// down and the prefix of squares from the small keys up, so neither sum ever
// cancels.  The per-key suffixes go to shared scratch (slo/shi, key e of thread
// t at [e * NT + t], conflict-free; keys e >= EMAX/2 in shi) when SMEM, to
// registers otherwise (small E only: a register array of 16 doubles spills).
// RAG: T < NT * EFIX real keys (the rest of the sorted tile is padding above
// them and is skipped)
template <typename R, int NT, int EMAX, bool SMEM, int EFIX = 0, bool RAG = false>
__device__ __forceinline__ void scan_tile(const R* keys, int T, int tilebase, int n, double tau,
                                          double pre_tile, double suf_tile, double next_tile_first,
                                          double* sh, Best* wbest, Best* run, double* totinv, double* slo,
                                          double* shi, long long* dbg = nullptr) {
    const int tid = threadIdx.x;
    Best best{INFINITY, INFINITY, 0.0, 0.0};
#ifdef VDAMP_PHASE_TIMING
    long long c0_ = clock64();
#define SC_MARK(i) do { if (tid == 0 && dbg) { long long c_ = clock64(); dbg[i] = c_ - c0_; c0_ = c_; } } while (0)
#else
#define SC_MARK(i) do { } while (0)
#endif
    // EFIX > 0: T == NT * EFIX known at compile time (fully unrolled, unguarded)
    const int E = EFIX ? EFIX : (T >= NT ? T / NT : 1);
    const bool act = EFIX ? (!RAG || tid * E < T) : tid * E < T;
    const int b0 = tid * E;
    constexpr int HALF = EMAX / 2 > 0 ? EMAX / 2 : 1;
    constexpr bool FKEY = sizeof(R) == 4;
    double ssq = 0.0, sinv = 0.0;
    double sreg[SMEM ? 1 : EMAX];
    if (act) {
        // one conversion per key (F2F/I2F/MUFU issue at 1/4 of the DFMA rate)
#pragma unroll ((SMEM && !EFIX) ? 4 : EMAX)
        for (int e = EMAX - 1; e >= 0; --e) {
            if (e < E && (!RAG || b0 + e < T)) {
                if constexpr (SMEM) (e < HALF ? slo : shi)[(e % HALF) * NT + tid] = sinv;
                else sreg[e] = sinv;
                const double m = (double)keys[KI(b0 + e)];
                ssq = fma(m, m, ssq);
                if (m > 0) sinv += FKEY ? rcp_posf(m) : rcp_pos(m);
            }
        }
    }
    SC_MARK(0);
    double pre, suf;
    block_excl_scan2<NT>(ssq, sinv, sh, pre, suf);
    pre += pre_tile;
    suf += suf_tile;
    if (tid == 0 && tilebase == 0) *totinv = suf + sinv;     // sum of all inverses
    SC_MARK(1);
    if (act) scan_keys<R, NT, EMAX, SMEM, EFIX, RAG>(keys, T, tilebase, n, tau, b0, E, pre, suf, next_tile_first, best,
                                          sreg, slo, shi);
    // tile argmin (ties -> smaller t) merged into the running best by thread 0
    for (int o = 16; o > 0; o >>= 1) {
        Best c;
        c.risk = __shfl_xor_sync(0xffffffffu, best.risk, o);
        c.t = __shfl_xor_sync(0xffffffffu, best.t, o);
        c.cnt = __shfl_xor_sync(0xffffffffu, best.cnt, o);
        c.inv = __shfl_xor_sync(0xffffffffu, best.inv, o);
        if (better(c, best)) best = c;
    }
    SC_MARK(2);
    if ((tid & 31) == 0) wbest[tid >> 5] = best;
    __syncthreads();
    SC_MARK(3);
    if (tid < 32) {                                  // warp 0: argmin over the warp winners
        Best c = tid < NT / 32 ? wbest[tid] : Best{INFINITY, INFINITY, 0.0, 0.0};
        for (int o = 16; o > 0; o >>= 1) {
            Best d;
            d.risk = __shfl_xor_sync(0xffffffffu, c.risk, o);
            d.t = __shfl_xor_sync(0xffffffffu, c.t, o);
            d.cnt = __shfl_xor_sync(0xffffffffu, c.cnt, o);
            d.inv = __shfl_xor_sync(0xffffffffu, c.inv, o);
            if (better(d, c)) c = d;
        }
        if (tid == 0 && better(c, *run)) *run = c;
    }
    SC_MARK(4);
}

// q = a / b for b > 0 without the library division's out-of-line slow path
// (FMA residual correction of a ~1-ulp reciprocal: correctly rounded for the
// magnitudes the SURE scan produces)
__device__ __forceinline__ double div_pos(double a, double b) {
    const double r = rcp_pos(b);
    const double q = a * r;
    return fma(fma(-b, q, a), r, q);
}

// Candidate walk over the keys one thread owns.  Only the best risk and a
// 32-bit candidate code (key index * 2 + interior flag) are carried through
// the loop; the winner's (t, count, inverse sum) are rebuilt afterwards.
// Key candidates arrive in increasing t, so a strict '<' keeps the smaller t
// of a tie; deferred interior points compare their codes on equal risk.
template <typename R, int NT, int EMAX, bool SMEM, int EFIX, bool RAG>
__device__ __forceinline__ void scan_keys(const R* keys, int T, int tilebase, int n, double tau, int b0, int E,
                                          double pre, double suf, double next_tile_first, Best& best,
                                          const double* sreg, const double* slo, const double* shi) {
    const int tid = threadIdx.x;
    constexpr int HALF = EMAX / 2 > 0 ? EMAX / 2 : 1;
    // risk(m) = sum_{j<=i} m_j^2 - n tau + 2 tau cnt + m (m cnt - tau inv_above)
    // (the reference's expression regrouped: zn carries the first two terms)
    const double tau2 = 2.0 * tau;
    double zn = pre - (double)n * tau;
    double m = (double)keys[KI(b0)];
    double cnt = (double)(n - (tilebase + b0));                // keys above, counted down exactly
    double brisk = INFINITY;
    int bcode = -1;
    // branch-free, fully unrolled pass over the keys (the per-key branch left a
    // reconvergence point per key, the walk's top stall): the key candidates by
    // predicated selects, the interior pre-test as one bit per key; the rare
    // flagged keys are resolved afterwards, ties ordered by the candidate code
    // (key e -> 2e, its interior point -> 2e + 1), i.e. by increasing t.  Same
    // arithmetic as the branchy walk: bitwise-identical results
    // (tools/cmp_run.py), 2.96 -> 2.92 ms/step, 439k -> 443k img-iter/s cfg1
    unsigned imask = 0u;
#pragma unroll
    for (int e = 0; e < EMAX; ++e) {
        if (e < E && (!RAG || b0 + e < T)) {
            const int il = b0 + e;
            zn = fma(m, m, zn);                                // + sum_{j <= i} m_j^2
            cnt -= 1.0;
            const double nxt = (il + 1 < T) ? (double)keys[KI(il + 1)] : next_tile_first;
            double sl;
            if constexpr (SMEM) sl = (e < HALF ? slo : shi)[(e % HALF) * NT + tid];
            else sl = sreg[e];
            const double inv_above = suf + sl;                 // both >= 0: no cancellation
            const double ti = tau * inv_above, g = m * cnt;
            const double base = fma(tau2, cnt, zn);
            const double risk = fma(m, g - ti, base);
            const bool ok = m != nxt;                          // end of a tie run
            const bool take = ok && risk < brisk;
            brisk = take ? risk : brisk;
            bcode = take ? 2 * e : bcode;
            const bool pin = ok && cnt > 0 && ti > g * (2.0 - 2e-12) && ti < (cnt * nxt) * (2.0 + 2e-12);
            imask |= (unsigned)pin << e;
            m = nxt;
        }
    }
    while (imask) {
        const int e = __ffs(imask) - 1;
        imask &= imask - 1u;
        const int il = b0 + e;
        double z = pre - (double)n * tau;                       // the walk's own order of additions
        for (int q = 0; q <= e; ++q) { const double mq = (double)keys[KI(b0 + q)]; z = fma(mq, mq, z); }
        const double mk = (double)keys[KI(il)];
        const double nxt = (il + 1 < T) ? (double)keys[KI(il + 1)] : next_tile_first;
        const double c = (double)(n - (tilebase + il + 1));
        double sl;
        if constexpr (SMEM) sl = (e < HALF ? slo : shi)[(e % HALF) * NT + tid];
        else {
            sl = 0.0;
#pragma unroll
            for (int q = 0; q < EMAX; ++q) if (q == e) sl = sreg[q];
        }
        const double ti = tau * (suf + sl);
        const double ts = div_pos(ti, 2.0 * c);
        if (ts > mk && ts < nxt) {
            const double rs = fma(ts, ts * c - ti, fma(tau2, c, z));
            if (rs < brisk || (rs == brisk && 2 * e + 1 < bcode)) { brisk = rs; bcode = 2 * e + 1; }
        }
    }
    if (bcode >= 0) {
        const int e = bcode >> 1, il = b0 + e;
        double sl;
        if constexpr (SMEM) sl = (e < HALF ? slo : shi)[(e % HALF) * NT + tid];
        else {
            sl = 0.0;
#pragma unroll
            for (int q = 0; q < EMAX; ++q) if (q == e) sl = sreg[q];
        }
        const double inv_above = suf + sl;
        const double c = (double)(n - (tilebase + il + 1));
        const double mk = (double)keys[KI(il)];
        const double t = (bcode & 1) ? div_pos(tau * inv_above, 2.0 * c) : mk;
        best = Best{brisk, t, c, inv_above};
    }
}

#include "vdamp_prune.cuh"

#ifdef VDAMP_PHASE_TIMING
// [image][subband][phase]: clock64 deltas of thread 0 (debug builds only)
__device__ long long g_phase[4096][64][4];
__device__ long long g_scan[4096][64][5];
#define PHASE_MARK(i) do { if (threadIdx.x == 0 && bi < 4096) { long long c_ = clock64(); g_phase[bi][j][i] = c_ - ph0_; ph0_ = c_; } } while (0)
#else
#define PHASE_MARK(i) do { } while (0)
#endif

template <int NT>
struct SelShared {
    unsigned long long mbar;         // TMA completion barrier (fp32 big-subband path)
    unsigned mphase;
    double sh[66 + NT / 32 + 2];     // counting-sort min/max words + block scans
    double tsq[MAXTILES], tinv[MAXTILES], tpre[MAXTILES], tsuf[MAXTILES];
    double tpart[MAXCT];             // tau partials of the column tiles
    double tau, totinv;
    Best best[NT / 32];
    Best run;                        // running argmin over the tiles
    double err, ref;                 // subband |r - w0|^2, |w0|^2 (trace)
};

// The t = 0 candidates (src/denoise.py:84: when no magnitude is zero; m0 = the
// smallest key, or 0 to skip them), the argmin over all tiles and candidates
// (ties -> smaller t) in S_.run, alpha (src/denoise.py:169), the clamp
// (src/vdamp.py:121-124) and the outputs.
template <typename R, int NT, typename SS>
__device__ __forceinline__ void select_finish(const Geo& g, const SelArgs<R>& a, int j, int bi, int n, double tau,
                                              double m0, bool have_w0, SS& S_) {
    const int tid = threadIdx.x;
    __syncthreads();
    __syncthreads();
    if (tid == 0) {
        if (m0 > 0) {
            const double totinv = S_.totinv;
            const double nn = (double)n;
            Best bb = S_.run;
            const double base0 = fma(2.0 * tau, nn, -(nn * tau));   // scan_keys' grouping at t = 0
            consider(bb, base0, 0.0, nn, totinv);
            const double ts = tau * totinv / (2.0 * nn);
            if (ts > 0.0 && ts < m0) {
                const double rsk = fma(ts, ts * nn - tau * totinv, base0);
                consider(bb, rsk, ts, nn, totinv);
            }
            S_.run = bb;
        }
        const Best bb = S_.run;
        const double alpha = (bb.cnt - 0.5 * bb.t * bb.inv) / (double)n;   // src/denoise.py:169
        const bool clamped = alpha >= ALPHA_CLAMP;                         // src/vdamp.py:121-124
        const double ac = clamped ? ALPHA_CLAMP : alpha;
        const long long pj = ((long long)bi * g.S + j);
        if (a.par) { a.par[3 * pj] = bb.t; a.par[3 * pj + 1] = ac; a.par[3 * pj + 2] = 1.0 / (1.0 - ac); }
        if (a.parf) { a.parf[3 * pj] = bb.t; a.parf[3 * pj + 1] = 0.0; a.parf[3 * pj + 2] = 1.0; }
        if (a.trace) {
            double* tr = a.trace + pj * TRACE_F;
            tr[0] = S_.tau; tr[1] = bb.t; tr[2] = bb.t / tau; tr[3] = ac; tr[4] = alpha;
            tr[5] = clamped ? 1.0 : 0.0; tr[6] = have_w0 ? S_.err : 0.0; tr[7] = have_w0 ? S_.ref : 0.0;
        }
    }
}

// Exact SURE selection for subband j of image bi (src/denoise.py:62-118,
// 165-173; clamp src/vdamp.py:121-124).
template <typename R, int NT>
__device__ void select_band(const Geo& g, const SelArgs<R>& a, int j, int bi, R* keys, SelShared<NT>& S_) {
    typedef typename CT<R>::T C;
    double* sh = S_.sh;
    double* tsq = S_.tsq; double* tinv = S_.tinv; double* tpre = S_.tpre; double* tsuf = S_.tsuf;
    double& s_tau = S_.tau;
    double& s_totinv = S_.totinv;
    Best* s_best = S_.best;
    const int tid = threadIdx.x;
    const int n = g.len[j];
    const long long base = (long long)bi * g.N + g.off[j];
#ifdef VDAMP_PHASE_TIMING
    long long ph0_ = clock64();
#endif
    // tau_j: the column-tile partials are loaded in parallel and summed in tile
    // order by thread 0 after the next barrier (deterministic, no serial loads)
    if (a.tau_in) {
        if (tid == 0) s_tau = a.tau_in[(long long)bi * g.S + j];
    } else {
        for (int i = tid; i < a.ntiles; i += NT) S_.tpart[i] = a.taupart[((long long)bi * a.ntiles + i) * g.S + j];
    }
    const C* rs = a.r + base;
    const C* w0 = a.w0 ? a.w0 + base : nullptr;
    double err = 0.0, ref = 0.0;
    // reduced right after the loads, so the sums are not live across the sort and scan
    auto flush_err = [&]() {
        if (w0) {
            const double e2 = block_sum<NT>(err, sh), r2 = block_sum<NT>(ref, sh);
            if (tid == 0) { S_.err = e2; S_.ref = r2; }
        }
    };
    constexpr int CAPK = Scap<R>::v;
    const bool large = n > CAPK;
    const int T = large ? CAPK : n;
    const int ntl = large ? n / CAPK : 1;
    const R* sorted = keys;
    // fp32: counting sort from the staging buffer `stage` into `keys`
    constexpr int SLOT = (CAPK + CAPK / 32 + 2 + 3) & ~3;          // padded keys, 16-byte aligned stride
    R* stage = keys + SLOT;
    unsigned* ccnt = reinterpret_cast<unsigned*>(stage + SLOT);
    const bool csort = NT >= BNT32 && sizeof(R) == 4 && T >= 4096;
    R* skeys = keys;                                               // where the sorted keys end up
    if (!large && csort) {
        // TMA: the subband is one contiguous segment of r; bulk-copy it into the
        // stage+counter region (free at this point), then build the keys from smem
        C* cz = reinterpret_cast<C*>(stage);
        const unsigned bytes = (unsigned)T * (unsigned)sizeof(C);
        __syncthreads();                                           // previous users of the region are done
        if (tid == 0) {
            fence_proxy_async();
            mbar_expect_tx(&S_.mbar, bytes);
            for (unsigned o = 0; o < bytes; o += 32768u)
                bulk_g2s(reinterpret_cast<char*>(cz) + o, reinterpret_cast<const char*>(rs) + o,
                         bytes - o < 32768u ? bytes - o : 32768u, &S_.mbar);
        }
        mbar_wait(&S_.mbar, S_.mphase);
#ifdef VDAMP_PHASE_TIMING
        if (tid == 0 && bi < 4096) g_csort[bi][j][5] = clock64() - ph0_;   // TMA landed
#endif
        unsigned kmn = 0xffffffffu, kmx = 0;                      // key-bit range for the counting sort
        auto build = [&](auto efc) {
            constexpr int EF = decltype(efc)::value;
#pragma unroll
            for (int q = 0; q < EF; ++q) {
                const int e = tid + q * NT;
                const C v = cz[e];
                const float kf = (float)cmag(v);
                keys[KI(e)] = (R)kf;
                const unsigned u = __float_as_uint(kf);
                if (u) kmn = min(kmn, u);
                kmx = max(kmx, u);
                if (w0) {
                    const C w = w0[e];
                    const double dx = (double)v.x - (double)w.x, dy = (double)v.y - (double)w.y;
                    err += dx * dx + dy * dy;
                    ref += (double)w.x * (double)w.x + (double)w.y * (double)w.y;
                }
            }
        };
        const int ef = T / NT;
        if (ef == 16) build(std::integral_constant<int, 16>{});
        else if (ef == 8) build(std::integral_constant<int, 8>{});
        else build(std::integral_constant<int, 4>{});
        __syncthreads();
#ifdef VDAMP_PHASE_TIMING
        if (tid == 0 && bi < 4096) g_csort[bi][j][6] = clock64() - ph0_;   // keys built
#endif
        if (tid == 0) S_.mphase ^= 1u;
        if (!a.tau_in && tid == 0) {
            double t = 0.0;
            for (int i = 0; i < a.ntiles; ++i) t += S_.tpart[i];
            s_tau = t;
        }
        flush_err();
        if constexpr (NT >= BNT32) {
#ifdef VDAMP_PHASE_TIMING
            long long* dbg = (bi < 4096) ? &g_csort[bi][j][0] : nullptr;
#else
            long long* dbg = nullptr;
#endif
            const float* kf = reinterpret_cast<const float*>(keys);
            float* of = reinterpret_cast<float*>(stage);
            const int cs = ef == 16 ? counting_sort<NT, SCAP / NT>(kf, of, ccnt, T, kmn, kmx, sh, dbg)
                         : ef == 8  ? counting_sort<NT, (SCAP / NT) / 2>(kf, of, ccnt, T, kmn, kmx, sh, dbg)
                                    : counting_sort<NT, (SCAP / NT) / 4>(kf, of, ccnt, T, kmn, kmx, sh, dbg);
            if (cs == 1) skeys = stage;
            else if (cs == 0) block_sort<R, NT>(keys, T);
        }
    } else if (!large) {
        R* dstk = keys;
        // issue 8 independent loads per thread before using any (memory-level parallelism)
        constexpr int LB = 8;
        for (int e0 = tid; e0 < T; e0 += LB * NT) {
            C v[LB];
#pragma unroll
            for (int u = 0; u < LB; ++u) {
                const int e = e0 + u * NT;
                if (e < T) v[u] = rs[e];
            }
#pragma unroll
            for (int u = 0; u < LB; ++u) {
                const int e = e0 + u * NT;
                if (e < T) dstk[KI(e)] = cmag(v[u]);
            }
            if (w0) {
#pragma unroll
                for (int u = 0; u < LB; ++u) {
                    const int e = e0 + u * NT;
                    if (e < T) {
                        const C w = w0[e];
                        const double dx = (double)v[u].x - (double)w.x, dy = (double)v[u].y - (double)w.y;
                        err += dx * dx + dy * dy;
                        ref += (double)w.x * (double)w.x + (double)w.y * (double)w.y;
                    }
                }
            }
        }
        __syncthreads();
        if (!a.tau_in && tid == 0) {
            double t = 0.0;
            for (int i = 0; i < a.ntiles; ++i) t += S_.tpart[i];
            s_tau = t;
        }
        flush_err();
        block_sort<R, NT>(keys, T);
    } else {
        // whole subband -> global scratch keys, counting sort there (L2-resident)
        R* ka = a.kA + base;
        constexpr int LB = 8;                                      // loads in flight per thread
        for (int e0 = tid; e0 < n; e0 += NT * LB) {
            C v[LB];
#pragma unroll
            for (int u = 0; u < LB; ++u) if (e0 + u * NT < n) v[u] = rs[e0 + u * NT];
#pragma unroll
            for (int u = 0; u < LB; ++u) {
                const int e = e0 + u * NT;
                if (e < n) {
                    ka[e] = cmag(v[u]);
                    if (w0) {
                        const C w = w0[e];
                        const double dx = (double)v[u].x - (double)w.x, dy = (double)v[u].y - (double)w.y;
                        err += dx * dx + dy * dy;
                        ref += (double)w.x * (double)w.x + (double)w.y * (double)w.y;
                    }
                }
            }
        }
        __syncthreads();
        if (!a.tau_in && tid == 0) {
            double t = 0.0;
            for (int i = 0; i < a.ntiles; ++i) t += S_.tpart[i];
            s_tau = t;
        }
        flush_err();
        sorted = ka;
        if constexpr (NT >= BNT32) {
            bool ok;
            if constexpr (sizeof(R) == 4)
                ok = global_counting_sort_eq<NT>(ka, a.kB + base, reinterpret_cast<unsigned*>(keys), n, sh);
            else
                ok = global_counting_sort<R, NT>(ka, a.kB + base, reinterpret_cast<unsigned*>(keys), n, sh);
            if (!ok) sorted = global_merge_sort<R, NT>(ka, a.kB + base, keys, n, CAPK);
        }
        // tile totals (ascending squares, descending inverses)
        for (int t = 0; t < ntl; ++t) {
            double q = 0.0, v = 0.0;
            for (int e = tid; e < CAPK; e += NT) {
                const double m = (double)sorted[t * CAPK + e];
                q += m * m;
                if (m > 0) v += rcp_pos(m);
            }
            q = block_sum<NT>(q, sh);
            v = block_sum<NT>(v, sh);
            if (tid == 0) { tsq[t] = q; tinv[t] = v; }
        }
        __syncthreads();
    }
    if (tid == 0) {
        double acc = 0.0;
        for (int t = 0; t < ntl; ++t) { tpre[t] = acc; acc += large ? tsq[t] : 0.0; }
        acc = 0.0;
        for (int t = ntl - 1; t >= 0; --t) { tsuf[t] = acc; acc += large ? tinv[t] : 0.0; }
    }
    __syncthreads();
    PHASE_MARK(0);                                   // load + sort (+ merges)
    const double tau = fmax(s_tau, TAU_FLOOR);

    if (tid == 0) S_.run = Best{INFINITY, INFINITY, 0.0, 0.0};     // scan_tile's barriers order this
    // fp32 big kernel: per-key suffix scratch in the shared regions the sorted
    // keys do not occupy (2 x 64 KB)
    constexpr bool SMEMSUF = NT >= BNT32 && sizeof(R) == 4;
    constexpr int EMAXS = NT >= BNT32 ? CAPK / NT : SMALL_N / NT;
    double* slo = nullptr;
    double* shi = nullptr;
    if constexpr (SMEMSUF) {
        if (!large && skeys == stage) {
            slo = reinterpret_cast<double*>(keys);
            shi = reinterpret_cast<double*>(ccnt);
        } else {
            slo = reinterpret_cast<double*>(stage);
            shi = slo + (EMAXS / 2) * NT;
        }
    }
    for (int t = 0; t < ntl; ++t) {
        if (large) {
            __syncthreads();
            for (int e = tid; e < CAPK; e += NT) keys[KI(e)] = sorted[t * CAPK + e];
            __syncthreads();
        }
        const double nf = (t + 1 < ntl) ? (double)sorted[(t + 1) * CAPK] : INFINITY;
#ifdef VDAMP_PHASE_TIMING
        long long* sdbg = bi < 4096 ? &g_scan[bi][j][0] : nullptr;
#else
        long long* sdbg = nullptr;
#endif
        const R* tk = large ? keys : skeys;
        if (SMEMSUF && T == NT * 16)
            scan_tile<R, NT, EMAXS, SMEMSUF, SMEMSUF ? 16 : 0>(tk, T, t * T, n, tau, tpre[t], tsuf[t], nf, sh, s_best,
                                                               &S_.run, &s_totinv, slo, shi, sdbg);
        else if (SMEMSUF && T == NT * 4)
            scan_tile<R, NT, EMAXS, SMEMSUF, SMEMSUF ? 4 : 0>(tk, T, t * T, n, tau, tpre[t], tsuf[t], nf, sh, s_best,
                                                              &S_.run, &s_totinv, slo, shi, sdbg);
        else
            scan_tile<R, NT, EMAXS, SMEMSUF>(tk, T, t * T, n, tau, tpre[t], tsuf[t], nf, sh, s_best, &S_.run,
                                             &s_totinv, slo, shi, sdbg);
    }
    select_finish<R, NT, SelShared<NT>>(g, a, j, bi, n, tau, large ? (double)sorted[0] : (double)skeys[0], w0 != nullptr, S_);
    PHASE_MARK(2);                                   // argmin + outputs
}

// Bound-pruned selection of one subband of n = EF * NT keys (4,096 <= n <= SCAP):
// load, |r| keys (+ trace error sums), tau, select_pruned (vdamp_prune.cuh), outputs.
// Returns false when the bounds leave too many keys; the caller then runs the
// full sort (select_band) on the subband from scratch.
// Shared memory: fp32 -- keys | stage | counters as in select_band (the subband
// lands in stage + counters by TMA); fp64 -- keys (doubles) | counters | scratch + list.
// NT < BNT32 (fp32 only, sure_prune32): keys by LDG into shared memory (no TMA landing
// zone), bucket ids recomputed, a PR_LMAX/2 list -- about 100 KB, two CTAs per SM.
template <typename R, int NT, typename SS>
__device__ __forceinline__ bool prune_band(const Geo& g, const SelArgs<R>& a, int j, int bi, R* keys, SS& S_) {
    typedef typename CT<R>::T C;
    typedef typename PrT<R>::U U;
    constexpr int CAPK = Scap<R>::v;
    constexpr int SLOT = (CAPK + CAPK / 32 + 2 + 3) & ~3;
    const int tid = threadIdx.x;
    const int n = g.len[j];
    const int ef = n / NT;
    const long long base = (long long)bi * g.N + g.off[j];
    if (a.tau_in) {
        if (tid == 0) S_.tau = a.tau_in[(long long)bi * g.S + j];
    } else {
        for (int i = tid; i < a.ntiles; i += NT) S_.tpart[i] = a.taupart[((long long)bi * a.ntiles + i) * g.S + j];
    }
    const C* rs = a.r + base;
    const C* w0 = a.w0 ? a.w0 + base : nullptr;
    double err = 0.0, ref = 0.0;
    U kmn = ~(U)0, kmx = 0;
    unsigned* cnt;
    double* rsh;
    unsigned short* bid;
    const bool large = NT >= BNT32 && n > CAPK;
    if (large) {
        // keys to global scratch (L2-resident); the shared key region holds the list
        R* ka = a.kA + base;
        if constexpr (sizeof(R) == 4) {
            cnt = reinterpret_cast<unsigned*>(keys + 2 * SLOT);
            rsh = reinterpret_cast<double*>(keys + SLOT);
        } else {
            cnt = reinterpret_cast<unsigned*>(keys + SLOT);
            rsh = reinterpret_cast<double*>(cnt + PR_NC + PR_NF + 32);
        }
        bid = nullptr;
        constexpr int LB = 8;                                  // loads in flight per thread
        for (int e0 = tid; e0 < n; e0 += LB * NT) {
            C v[LB];
#pragma unroll
            for (int u = 0; u < LB; ++u) if (e0 + u * NT < n) v[u] = rs[e0 + u * NT];
#pragma unroll
            for (int u = 0; u < LB; ++u) {
                const int e = e0 + u * NT;
                if (e < n) {
                    const R m = cmag(v[u]);
                    ka[e] = m;
                    const U k = PrT<R>::bits(m);
                    if (k) kmn = k < kmn ? k : kmn;
                    kmx = k > kmx ? k : kmx;
                    if (w0) {
                        const C w = w0[e];
                        const double dx = (double)v[u].x - (double)w.x, dy = (double)v[u].y - (double)w.y;
                        err += dx * dx + dy * dy;
                        ref += (double)w.x * (double)w.x + (double)w.y * (double)w.y;
                    }
                }
            }
        }
        __syncthreads();
    } else if constexpr (sizeof(R) == 4 && NT >= BNT32) {
        R* stage = keys + SLOT;
        cnt = reinterpret_cast<unsigned*>(stage + SLOT);
        rsh = reinterpret_cast<double*>(stage);
        // stage: reduction scratch | list | bucket ids (free once the keys are built)
        bid = reinterpret_cast<unsigned short*>(reinterpret_cast<char*>(stage) + PR_STAGE_BID);
        C* cz = reinterpret_cast<C*>(stage);
        const unsigned bytes = (unsigned)n * (unsigned)sizeof(C);
        __syncthreads();                                       // previous users of the region are done
        if (tid == 0) {
            fence_proxy_async();
            mbar_expect_tx(&S_.mbar, bytes);
            for (unsigned o = 0; o < bytes; o += 32768u)
                bulk_g2s(reinterpret_cast<char*>(cz) + o, reinterpret_cast<const char*>(rs) + o,
                         bytes - o < 32768u ? bytes - o : 32768u, &S_.mbar);
        }
        mbar_wait(&S_.mbar, S_.mphase);
        for (int q = 0; q < ef; ++q) {
            const int e = tid + q * NT;
            const C v = cz[e];
            const float kf = (float)cmag(v);
            keys[KI(e)] = (R)kf;
            const U u = __float_as_uint(kf);
            if (u) kmn = min(kmn, u);
            kmx = max(kmx, u);
            if (w0) {
                const C w = w0[e];
                const double dx = (double)v.x - (double)w.x, dy = (double)v.y - (double)w.y;
                err += dx * dx + dy * dy;
                ref += (double)w.x * (double)w.x + (double)w.y * (double)w.y;
            }
        }
        __syncthreads();
        if (tid == 0) S_.mphase ^= 1u;
    } else {
        cnt = reinterpret_cast<unsigned*>(keys + SLOT);
        if constexpr (NT >= BNT32) {
            bid = reinterpret_cast<unsigned short*>(cnt + PR_NC + PR_NF + 32);
            rsh = reinterpret_cast<double*>(bid + PR_BIDN);
        } else {
            bid = nullptr;
            rsh = reinterpret_cast<double*>(cnt + PR_NC + PR_NF + 32);
        }
        constexpr int LB = 8;                                  // loads in flight per thread
        for (int e0 = tid; e0 < n; e0 += LB * NT) {
            C v[LB];
#pragma unroll
            for (int u = 0; u < LB; ++u) if (e0 + u * NT < n) v[u] = rs[e0 + u * NT];
#pragma unroll
            for (int u = 0; u < LB; ++u) {
                const int e = e0 + u * NT;
                if (e < n) {
                    const R m = cmag(v[u]);
                    keys[KI(e)] = m;
                    const U k = PrT<R>::bits(m);
                    if (k) kmn = k < kmn ? k : kmn;
                    kmx = k > kmx ? k : kmx;
                    if (w0) {
                        const C w = w0[e];
                        const double dx = (double)v[u].x - (double)w.x, dy = (double)v[u].y - (double)w.y;
                        err += dx * dx + dy * dy;
                        ref += (double)w.x * (double)w.x + (double)w.y * (double)w.y;
                    }
                }
            }
        }
        __syncthreads();
    }
    if (!a.tau_in && tid == 0) {
        double t = 0.0;
        for (int i = 0; i < a.ntiles; ++i) t += S_.tpart[i];
        S_.tau = t;
    }
    if (w0) {
        const double e2 = block_sum<NT>(err, S_.sh), r2 = block_sum<NT>(ref, S_.sh);
        if (tid == 0) { S_.err = e2; S_.ref = r2; }
    }
    __syncthreads();
    const double tau = fmax(S_.tau, TAU_FLOOR);
    R* plist = large ? keys : reinterpret_cast<R*>(rsh + 5 * (NT / 32) + 8);
#ifdef VDAMP_PHASE_TIMING
    long long* pdbg = bi < 4096 ? &g_prune[bi][j][0] : nullptr;
#else
    long long* pdbg = nullptr;
#endif
    PrOut po{0, 0.0};
    bool ok;
    const int lmax = large ? SCAP : NT >= BNT32 ? pr_lmax<R>() : PR_LMAX / 2;
    if constexpr (NT >= BNT32) {
        if (large) ok = select_pruned<R, NT, 0, SS, true>(n, tau, a.kA + base, cnt, bid, plist, lmax, rsh, kmn, kmx,
                                                          S_, po, pdbg);
        else if (ef == 16) ok = select_pruned<R, NT, 16>(n, tau, keys, cnt, bid, plist, lmax, rsh, kmn, kmx, S_, po, pdbg);
        else if (ef == 8) ok = select_pruned<R, NT, 8>(n, tau, keys, cnt, bid, plist, lmax, rsh, kmn, kmx, S_, po, pdbg);
        else ok = select_pruned<R, NT, 4>(n, tau, keys, cnt, bid, plist, lmax, rsh, kmn, kmx, S_, po, pdbg);
    } else {
        if (ef == 32) ok = select_pruned<R, NT, 32>(n, tau, keys, cnt, bid, plist, lmax, rsh, kmn, kmx, S_, po, pdbg);
        else if (ef == 16) ok = select_pruned<R, NT, 16>(n, tau, keys, cnt, bid, plist, lmax, rsh, kmn, kmx, S_, po, pdbg);
        else ok = select_pruned<R, NT, 8>(n, tau, keys, cnt, bid, plist, lmax, rsh, kmn, kmx, S_, po, pdbg);
    }
    if (!ok) return false;
    select_finish<R, NT, SS>(g, a, j, bi, n, tau, po.nbelow == 0 ? po.m0 : 0.0, w0 != nullptr, S_);
    return true;
}

// the full sort path as a call: its code stays out of the pruned path's instruction stream
template <typename R, int NT>
__device__ __noinline__ void select_band_call(const Geo& g, const SelArgs<R>& a, int j, int bi, R* keys,
                                              SelShared<NT>& S_) {
    select_band<R, NT>(g, a, j, bi, keys, S_);
}

#include "vdamp_win.cuh"

// Shared state of sure_prune32 (the fields prune_band / select_finish / scan_tile use)
template <int NT>
struct PrShared {
    unsigned long long mbar;
    unsigned mphase;
    double sh[66 + NT / 32 + 2];
    double tpart[PR_MAXT];
    double tau, totinv;
    Best best[NT / 32];
    Best run;
    double err, ref;
};

// Bound-pruned selection of fp32 subbands of 4,096..SCAP keys in 512-thread CTAs with
// ~100 KB of shared memory: two CTAs (two subbands) per SM, so one CTA's barrier and
// reduction latency overlaps the other's work.  A subband the bounds cannot settle is
// flagged in a.pflag and sorted fully by the sure_select launch that follows (a.only).
template <int NT>
__global__ void __launch_bounds__(NT, 2) sure_prune32(const __grid_constant__ Geo g,
                                                      const __grid_constant__ SelArgs<float> a) {
    pdl_enter();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* keys = reinterpret_cast<float*>(smem_raw);
    __shared__ PrShared<NT> S_;
    const int bi = blockIdx.x, it = blockIdx.y;
    if (threadIdx.x == 0) { mbar_init(&S_.mbar, 1); S_.mphase = 0; }
    __syncthreads();
    for (int q = a.item_start[it]; q < a.item_start[it + 1]; ++q) {
        const int j = a.item_list[q];
        const bool ok = prune_band<float, NT>(g, a, j, bi, keys, S_);
        if (threadIdx.x == 0) a.pflag[(long long)bi * g.S + j] = ok ? 0u : 1u;
        __syncthreads();
    }
}

// PM (prune mask, bit 0: subbands of 4,096..SCAP keys, bit 1: larger ones): those take
// the bound-pruned path first (vdamp_prune.cuh) with the full sort as an out-of-line
// fallback; the others run the full sort inline (PM = 0: the fp32 default kernel)
template <typename R, int NT, int PM = 0>
__global__ void __launch_bounds__(NT, NT >= BNT32 ? 1 : 4) sure_select(const __grid_constant__ Geo g,
                                                                       const __grid_constant__ SelArgs<R> a) {
    pdl_enter();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    R* keys = reinterpret_cast<R*>(smem_raw);
    __shared__ SelShared<NT> S_;
    const int bi = blockIdx.x, it = blockIdx.y;     // images fastest: long items of all images start first
    if (threadIdx.x == 0) { mbar_init(&S_.mbar, 1); S_.mphase = 0; }
    __syncthreads();
    // one work item = one large subband, or several small ones packed to ~SCAP keys
    for (int q = a.item_start[it]; q < a.item_start[it + 1]; ++q) {
        const int j = a.item_list[q];
        if (a.only && !a.only[(long long)bi * g.S + j]) continue;   // pruned already (uniform per CTA)
        if constexpr (PM != 0 && NT >= BNT32) {
            const int n = g.len[j];
            const int bit = n > Scap<R>::v ? 2 : 1;
            if ((PM & bit) && n >= 4096 && n % NT == 0 && (n / NT) % 4 == 0) {
                if (!prune_band<R, NT>(g, a, j, bi, keys, S_)) select_band_call<R, NT>(g, a, j, bi, keys, S_);
            } else if (PM == 2 && bit == 1) {
                select_band<R, NT>(g, a, j, bi, keys, S_);        // small subbands inline (fp32 cfg2)
            } else {
                select_band_call<R, NT>(g, a, j, bi, keys, S_);
            }
        } else {
            select_band<R, NT>(g, a, j, bi, keys, S_);
        }
        __syncthreads();
    }
}

// The full path for the (rare) large subbands sure_win32<.., GLOBAL> flagged in a.only: a
// few CTAs scan the flags of all B x nitems (image, single-subband item) pairs and run
// select_band on the flagged ones.  With nothing flagged the launch costs one pass over
// the flags.
template <typename R, int NT>
__global__ void __launch_bounds__(NT, 1) sure_select_flagged(const __grid_constant__ Geo g,
                                                             const __grid_constant__ SelArgs<R> a, int B, int nitems) {
    pdl_enter();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    R* keys = reinterpret_cast<R*>(smem_raw);
    __shared__ SelShared<NT> S_;
    __shared__ unsigned wmask[NT / 32];
    const int tid = threadIdx.x;
    if (tid == 0) { mbar_init(&S_.mbar, 1); S_.mphase = 0; }
    __syncthreads();
    const int pairs = B * nitems;
    for (int r0 = 0; blockIdx.x + (long long)r0 * gridDim.x < pairs; r0 += NT) {
        const long long p = blockIdx.x + (long long)(r0 + tid) * gridDim.x;
        bool f = false;
        if (p < pairs) {
            const int bi = (int)(p % B), it = (int)(p / B);
            f = a.only[(long long)bi * g.S + a.item_list[a.item_start[it]]] != 0u;
        }
        const unsigned bm = __ballot_sync(0xffffffffu, f);
        if ((tid & 31) == 0) wmask[tid >> 5] = bm;
        __syncthreads();
        for (int ww = 0; ww < NT / 32; ++ww) {
            unsigned m = wmask[ww];
            while (m) {
                const int ln = __ffs(m) - 1;
                m &= m - 1u;
                const long long pp = blockIdx.x + (long long)(r0 + ww * 32 + ln) * gridDim.x;
                const int bi = (int)(pp % B), it = (int)(pp / B);
                select_band<R, NT>(g, a, a.item_list[a.item_start[it]], bi, keys, S_);
                __syncthreads();
            }
        }
        __syncthreads();
    }
}

// -------------------------------------------- K4, subbands > SCAP (fp32) ----
// A subband of n > SCAP keys is split by value over several CTAs:
//  big_keys:  |r| -> kA and a histogram of the float bits >> 17 (1/64 octave,
//             BIGB buckets) per subband; trace error partials per chunk.
//  big_range: CTA q of a subband owns the buckets whose exclusive prefix count
//             lies in [q T, (q+1) T), T = SCAP - (largest bucket), so it holds at
//             most SCAP keys.  One pass over the subband (loads batched 8 deep)
//             gathers them into shared memory while summing m^2 of the keys below
//             and 1/m of the keys above in float64 (fixed per-thread order + tree:
//             deterministic, no cancellation); the keys are counting-sorted and
//             scanned exactly with those offsets.  The last CTA of the subband
//             (ticket) merges the range winners (ties -> smaller t), adds t = 0
//             and writes the parameters.  A bucket > SCAP/2 (massive ties) falls
//             back to the single-CTA global path (select_band) for that subband.
constexpr int BIGB = 16384;          // histogram buckets: positive float bits >> 17
constexpr int BIG_CHUNK = 16384;     // keys per big_keys CTA (1024 threads x 16)
constexpr int BIG_MAXL = 12;         // subbands > SCAP per image
constexpr int BIG_RMAX = 64;         // value ranges per subband (n <= 2^20 at T >= SCAP/2)

struct BigArgs {
    int nlarge, ranges, chunks;      // large subbands, big_range CTAs and chunk CTAs per subband
    int list[BIG_MAXL];              // their subband ids
    unsigned* hist;                  // [B][nlarge][BIGB] (zero between uses)
    unsigned* tick;                  // [B][nlarge] (zero between uses)
    double* best;                    // [B][nlarge][ranges][4]
    double* aux;                     // [B][nlarge][2]: sum of all 1/m, smallest key
    double* errp;                    // [B][nlarge][chunks][2]: trace |r - w0|^2, |w0|^2
};

__global__ void __launch_bounds__(1024) big_keys(Geo g, SelArgs<float> a, BigArgs b) {
    pdl_enter();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    unsigned* hs = reinterpret_cast<unsigned*>(smem_raw);    // [BIGB]
    __shared__ double sh[40];
    const int ch = blockIdx.x, jl = blockIdx.y, bi = blockIdx.z, tid = threadIdx.x;
    const int j = b.list[jl], n = g.len[j];
    const int e0 = ch * BIG_CHUNK;
    if (e0 >= n) return;
    const long long base = (long long)bi * g.N + g.off[j];
    for (int i = tid; i < BIGB; i += 1024) hs[i] = 0;
    __syncthreads();
    double err = 0.0, ref = 0.0;
#pragma unroll 4
    for (int q = 0; q < BIG_CHUNK / 1024; ++q) {
        const int e = e0 + tid + q * 1024;
        if (e < n) {
            const float2 v = a.r[base + e];
            const float m = cmag(v);
            a.kA[base + e] = m;
            atomicAdd(&hs[__float_as_uint(m) >> 17], 1u);
            if (a.w0) {
                const float2 w = a.w0[base + e];
                const double dx = (double)v.x - (double)w.x, dy = (double)v.y - (double)w.y;
                err += dx * dx + dy * dy;
                ref += (double)w.x * (double)w.x + (double)w.y * (double)w.y;
            }
        }
    }
    __syncthreads();
    unsigned* hg = b.hist + ((long long)bi * b.nlarge + jl) * BIGB;
    for (int i = tid; i < BIGB; i += 1024)
        if (hs[i]) atomicAdd(&hg[i], hs[i]);
    if (a.w0) {
        err = block_sum<1024>(err, sh);
        ref = block_sum<1024>(ref, sh);
        if (tid == 0) {
            double* ep = b.errp + (((long long)bi * b.nlarge + jl) * b.chunks + ch) * 2;
            ep[0] = err; ep[1] = ref;
        }
    }
}

// histogram -> exclusive prefix counts in cbs[BIGB], largest bucket, last
// nonempty bucket (1024 threads; sh needs 66 + 34 doubles, su 2 words)
__device__ __forceinline__ void big_prefix(const unsigned* hg, unsigned* cbs, double* sh, unsigned* su,
                                           unsigned& maxb, int& blast) {
    constexpr int NT = 1024, HPT = BIGB / NT;
    const int tid = threadIdx.x;
    unsigned h[HPT], hsum = 0, hmax = 0;
    int hl = -1;
#pragma unroll
    for (int i = 0; i < HPT; ++i) {
        h[i] = __ldcg(hg + tid * HPT + i);
        hsum += h[i];
        hmax = max(hmax, h[i]);
        if (h[i]) hl = tid * HPT + i;
    }
    unsigned P = (unsigned)block_excl_scan<NT, false>((double)hsum, sh + 66);
#pragma unroll
    for (int i = 0; i < HPT; ++i) { cbs[tid * HPT + i] = P; P += h[i]; }
    for (int o = 16; o > 0; o >>= 1) {
        hmax = max(hmax, __shfl_xor_sync(0xffffffffu, hmax, o));
        hl = max(hl, __shfl_xor_sync(0xffffffffu, hl, o));
    }
    if (tid < 2) su[tid] = 0;
    __syncthreads();
    if ((tid & 31) == 0) { atomicMax(&su[0], hmax); atomicMax(&su[1], (unsigned)(hl + 1)); }
    __syncthreads();
    maxb = su[0];
    blast = (int)su[1] - 1;
}


__global__ void __launch_bounds__(1024, 1) big_range(Geo g, SelArgs<float> a, BigArgs b) {
    pdl_enter();
    constexpr int NT = 1024;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* keys = reinterpret_cast<float*>(smem_raw);
    constexpr int SLOT = (SCAP + SCAP / 32 + 2 + 3) & ~3;
    float* stage = keys + SLOT;
    unsigned* ccnt = reinterpret_cast<unsigned*>(stage + SLOT);
    __shared__ SelShared<NT> S_;
    __shared__ unsigned s_u[4];
    __shared__ int s_last;
    double* sh = S_.sh;
    const int q = blockIdx.x, jl = blockIdx.y, bi = blockIdx.z, tid = threadIdx.x;
    const int j = b.list[jl], n = g.len[j];
    const long long base = (long long)bi * g.N + g.off[j];
    const long long sb = (long long)bi * b.nlarge + jl;
    unsigned* cbs = reinterpret_cast<unsigned*>(stage);         // bucket -> exclusive prefix count
    static_assert(BIGB <= SLOT, "histogram prefix must fit the stage region");
    if (tid == 0) { mbar_init(&S_.mbar, 1); S_.mphase = 0; }
    unsigned maxb;
    int blast;
    big_prefix(b.hist + sb * BIGB, cbs, sh, s_u, maxb, blast);
    const bool fallback = maxb > (unsigned)(SCAP / 2) || blast < 0;
    const unsigned T = (unsigned)SCAP - maxb;
    const int nranges = fallback ? 1 : (int)(cbs[blast] / T) + 1;
    int Tn = 0, s0 = 0;
    double ssq = 0.0, sinv = 0.0, nxt = INFINITY;
    unsigned kmn = 0xffffffffu, kmx = 0;
    if (fallback) {
        if (q == 0) select_band<float, NT>(g, a, j, bi, keys, S_);
    } else if (q < nranges) {
        // tau (column-tile partials in tile order, or given)
        if (!a.tau_in)
            for (int i = tid; i < a.ntiles; i += NT) S_.tpart[i] = a.taupart[((long long)bi * a.ntiles + i) * g.S + j];
        const unsigned lo = (unsigned)q * T, hi = lo + T;
        if (tid == 0) s_u[2] = 0;
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
            if (a.tau_in) t = a.tau_in[(long long)bi * g.S + j];
            else for (int i = 0; i < a.ntiles; ++i) t += S_.tpart[i];
            S_.tau = t;
        }
        // one pass over the subband: own keys -> smem, offsets of the others
        float nmin = INFINITY;
        unsigned nbelow = 0;
        const int lane = tid & 31;
        constexpr int LB = 8;
        for (int e0 = 0; e0 < n; e0 += NT * LB) {
            float kk[LB];
#pragma unroll
            for (int u = 0; u < LB; ++u) {
                const int e = e0 + tid + u * NT;
                kk[u] = e < n ? __ldcg(a.kA + base + e) : -1.0f;
            }
#pragma unroll
            for (int u = 0; u < LB; ++u) {
                const float k = kk[u];
                int cls = -1;                                      // 0 below, 1 own, 2 above
                if (k >= 0.0f) {
                    const unsigned c = cbs[__float_as_uint(k) >> 17];
                    cls = c < lo ? 0 : (c < hi ? 1 : 2);
                }
                if (cls == 0) { ssq = fma((double)k, (double)k, ssq); ++nbelow; }
                else if (cls == 2) { if (k > 0.0f) sinv += rcp_posf((double)k); nmin = fminf(nmin, k); }
                const unsigned own = __ballot_sync(0xffffffffu, cls == 1);
                if (own) {
                    unsigned wb = 0;
                    if (lane == 0) wb = atomicAdd(&s_u[2], (unsigned)__popc(own));
                    wb = __shfl_sync(0xffffffffu, wb, 0);
                    if (cls == 1) {
                        const unsigned uk = __float_as_uint(k);
                        keys[KI((int)(wb + __popc(own & ((1u << lane) - 1u))))] = k;
                        if (uk) kmn = min(kmn, uk);
                        kmx = max(kmx, uk);
                    }
                }
            }
        }
        ssq = block_sum<NT>(ssq, sh);
        sinv = block_sum<NT>(sinv, sh);
        s0 = (int)block_sum<NT>((double)nbelow, sh);
        for (int o = 16; o > 0; o >>= 1) {
            nmin = fminf(nmin, __shfl_xor_sync(0xffffffffu, nmin, o));
            kmn = min(kmn, __shfl_xor_sync(0xffffffffu, kmn, o));
            kmx = max(kmx, __shfl_xor_sync(0xffffffffu, kmx, o));
        }
        if (tid == 0) { s_u[0] = 0xffffffffu; s_u[1] = 0; s_u[3] = 0x7f800000u; }
        __syncthreads();
        if (lane == 0) { atomicMin(&s_u[0], kmn); atomicMax(&s_u[1], kmx); atomicMin(&s_u[3], __float_as_uint(nmin)); }
        __syncthreads();
        Tn = (int)s_u[2];
        kmn = s_u[0]; kmx = s_u[1];
        const float nm = __uint_as_float(s_u[3]);
        nxt = nm < INFINITY ? (double)nm : INFINITY;
        // pad to 4096 / 8192 / 16384 keys with distinct values just above the
        // range's largest key (sorted behind the real keys, skipped by the scan)
        const int npad = Tn <= 4096 ? 4096 : (Tn <= 8192 ? 8192 : 16384);
        for (int i = Tn + tid; i < npad; i += NT) keys[KI(i)] = __uint_as_float(kmx + 1u + (unsigned)(i - Tn));
        if (npad > Tn) kmx += (unsigned)(npad - Tn);
        __syncthreads();
        const float* skeys = keys;
        {
            const int cs = npad == 16384 ? counting_sort<NT, 16>(keys, stage, ccnt, npad, kmn, kmx, sh)
                         : npad == 8192  ? counting_sort<NT, 8>(keys, stage, ccnt, npad, kmn, kmx, sh)
                                         : counting_sort<NT, 4>(keys, stage, ccnt, npad, kmn, kmx, sh);
            if (cs == 1) skeys = stage;
            else if (cs == 0) block_sort<float, NT>(keys, npad);
        }
        // exact scan of the range with the offsets of the keys below / above
        double* slo;
        double* shi;
        if (skeys == stage) { slo = reinterpret_cast<double*>(keys); shi = reinterpret_cast<double*>(ccnt); }
        else { slo = reinterpret_cast<double*>(stage); shi = slo + 8 * NT; }
        if (tid == 0) S_.run = Best{INFINITY, INFINITY, 0.0, 0.0};
        const double tau = fmax(S_.tau, TAU_FLOOR);
        if (npad == 16384)
            scan_tile<float, NT, 16, true, 16, true>(skeys, Tn, s0, n, tau, ssq, sinv, nxt, sh, S_.best, &S_.run,
                                                     &S_.totinv, slo, shi);
        else if (npad == 8192)
            scan_tile<float, NT, 16, true, 8, true>(skeys, Tn, s0, n, tau, ssq, sinv, nxt, sh, S_.best, &S_.run,
                                                    &S_.totinv, slo, shi);
        else
            scan_tile<float, NT, 16, true, 4, true>(skeys, Tn, s0, n, tau, ssq, sinv, nxt, sh, S_.best, &S_.run,
                                                    &S_.totinv, slo, shi);
        __syncthreads();
        if (tid == 0) {
            double* bp = b.best + (sb * b.ranges + q) * 4;
            bp[0] = S_.run.risk; bp[1] = S_.run.t; bp[2] = S_.run.cnt; bp[3] = S_.run.inv;
            if (q == 0) { b.aux[sb * 2] = S_.totinv; b.aux[sb * 2 + 1] = (double)skeys[0]; }
        }
    }
    // ticket: the last CTA of the subband merges, then clears histogram and cursors
    if (tid == 0) {
        __threadfence();
        s_last = atomicAdd(&b.tick[sb], 1u) == (unsigned)gridDim.x - 1u;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    unsigned* hg = b.hist + sb * BIGB;
    for (int i = tid; i < BIGB; i += NT) hg[i] = 0;
    if (tid == 0) {
        b.tick[sb] = 0;
        if (!fallback) {
            Best bb{INFINITY, INFINITY, 0.0, 0.0};
            for (int r = 0; r < nranges; ++r) {
                const double* bp = b.best + (sb * b.ranges + r) * 4;
                consider(bb, __ldcg(bp), __ldcg(bp + 1), __ldcg(bp + 2), __ldcg(bp + 3));
            }
            double s_tau = 0.0;
            if (a.tau_in) s_tau = a.tau_in[(long long)bi * g.S + j];
            else for (int i = 0; i < a.ntiles; ++i) s_tau += __ldcg(a.taupart + ((long long)bi * a.ntiles + i) * g.S + j);
            const double tau = fmax(s_tau, TAU_FLOOR);
            // candidate t = 0 when no magnitude is zero (src/denoise.py:84)
            const double m0 = __ldcg(b.aux + sb * 2 + 1);
            if (m0 > 0) {
                const double totinv = __ldcg(b.aux + sb * 2);
                const double nn = (double)n;
                const double base0 = fma(2.0 * tau, nn, -(nn * tau));   // scan_keys' grouping at t = 0
                consider(bb, base0, 0.0, nn, totinv);
                const double ts = tau * totinv / (2.0 * nn);
                if (ts > 0.0 && ts < m0) {
                    const double rsk = fma(ts, ts * nn - tau * totinv, base0);
                    consider(bb, rsk, ts, nn, totinv);
                }
            }
            const double alpha = (bb.cnt - 0.5 * bb.t * bb.inv) / (double)n;   // src/denoise.py:169
            const bool clamped = alpha >= ALPHA_CLAMP;                         // src/vdamp.py:121-124
            const double ac = clamped ? ALPHA_CLAMP : alpha;
            const long long pj = ((long long)bi * g.S + j);
            if (a.par) { a.par[3 * pj] = bb.t; a.par[3 * pj + 1] = ac; a.par[3 * pj + 2] = 1.0 / (1.0 - ac); }
            if (a.parf) { a.parf[3 * pj] = bb.t; a.parf[3 * pj + 1] = 0.0; a.parf[3 * pj + 2] = 1.0; }
            if (a.trace) {
                double e2 = 0.0, r2 = 0.0;
                if (a.w0)
                    for (int c = 0; c * BIG_CHUNK < n; ++c) {
                        const double* ep = b.errp + (sb * b.chunks + c) * 2;
                        e2 += __ldcg(ep); r2 += __ldcg(ep + 1);
                    }
                double* tr = a.trace + pj * TRACE_F;
                tr[0] = s_tau; tr[1] = bb.t; tr[2] = bb.t / tau; tr[3] = ac; tr[4] = alpha;
                tr[5] = clamped ? 1.0 : 0.0; tr[6] = e2; tr[7] = r2;
            }
        }
    }
}

// --------------------------------------------------------------- misc ----
// out = Onsager(in; par) per subband (r~_{k+1} or w_hat = soft(r, t)).
template <typename R>
__global__ void apply_params(Geo g, const typename CT<R>::T* in, typename CT<R>::T* out, const double* par) {
    const int j = blockIdx.y, bi = blockIdx.z;
    const double* pp = par + ((long long)bi * g.S + j) * 3;
    const R t = (R)pp[0], al = (R)pp[1], ga = (R)pp[2];
    const long long base = (long long)bi * g.N + g.off[j];
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < g.len[j]; e += gridDim.x * blockDim.x)
        out[base + e] = onsager<R, typename CT<R>::T>(in[base + e], t, al, ga);
}

// y on the grid with the centred-FFT sign folded in, and 1/p (0 off mask).
// Guards for raw C callers (the reference raises ValueError for these,
// src/fourier.py:65-74, src/sampling.py:45-46): an index outside [0, N) is
// skipped, a repeated index or a probability outside (0, 1] at a sampled
// point is flagged; the flags (MEAS_*) are OR-ed into *err and reported by
// the host as VDAMP_ERR_ARG.  pinv is zero before the scatter, so a
// non-zero previous value marks a duplicate.
constexpr unsigned MEAS_RANGE = 1u, MEAS_DUP = 2u, MEAS_PROB = 4u;

__device__ __forceinline__ float xchg_pinv(float* a, float v) { return atomicExch(a, v); }
__device__ __forceinline__ double xchg_pinv(double* a, double v) {
    return __longlong_as_double((long long)atomicExch(reinterpret_cast<unsigned long long*>(a),
                                                      (unsigned long long)__double_as_longlong(v)));
}

template <typename R>
__global__ void scatter_measurements(Geo g, const typename CT<R>::T* y, const long long* idx,
                                     const long long* offs, const double* probs, long long pstride,
                                     typename CT<R>::T* yg, R* pinv, unsigned* err) {
    const int bi = blockIdx.y;
    const long long o0 = offs[bi], n = offs[bi + 1] - o0;
    unsigned bad = 0;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
        const long long gi = idx[o0 + e];
        if (gi < 0 || gi >= g.N) { bad |= MEAS_RANGE; continue; }
        const int k1 = (int)(gi >> g.logW), k2 = (int)(gi & (g.W - 1));
        typename CT<R>::T v = y[o0 + e];
        if ((k1 + k2) & 1) { v.x = -v.x; v.y = -v.y; }
        const double pr = probs[(long long)bi * pstride + gi];
        if (!(pr > 0.0 && pr <= 1.0)) bad |= MEAS_PROB;
        yg[(long long)bi * g.N + gi] = v;
        if (xchg_pinv(pinv + (long long)bi * g.N + gi, (R)(1.0 / pr)) != (R)0) bad |= MEAS_DUP;
    }
    if (bad) atomicOr(err, bad);
}

// copy the sticky measurement flags into mapped pinned host memory: a kernel store,
// not a DMA copy, so the compute stream never queues behind a large device-to-host
// transfer on the copy engine (the pipelined serving path overlaps those)
__global__ void publish_flags(const unsigned* d, volatile unsigned* h) { *h = *d; }

template <typename R>
__global__ void fill_identity_params(double* par, int count) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
        par[3 * i] = 0.0; par[3 * i + 1] = 0.0; par[3 * i + 2] = 1.0;
    }
}

template <typename R>
__global__ void make_twiddles(typename CT<R>::T* tw, int L) {
    for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < L; m += gridDim.x * blockDim.x) {
        double s, c;
        sincospi(-2.0 * (double)m / (double)L, &s, &c);
        tw[m].x = (R)c; tw[m].y = (R)s;
    }
}

// |fft1c(atom)|^2 of the 1D Haar atom, profile p = 2*(level-1) + high (src/vdamp.py:41-51, separable)
// col_pass256's row-profile table: [256][npp], profile q of row k at k * npp + q
template <typename R>
__global__ void arrange_prs256(R* prs, const double* prow, int np, int npp, int H) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= H * npp) return;
    const int k = i / npp, q = i - k * npp;
    prs[i] = (q < np) ? (R)prow[q * H + k] : R(0);
}

__global__ void make_profiles(double* prof, int L, int s) {
    const int pidx = blockIdx.y;
    const int level = pidx / 2 + 1, high = pidx & 1;
    const int M = 1 << level;
    const double amp = exp2(-0.5 * level);
    for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < L; w += gridDim.x * blockDim.x) {
        const long long kf = (long long)w - L / 2;
        double re = 0.0, im = 0.0;
        for (int nn = 0; nn < M; ++nn) {
            const double a = (high && nn >= M / 2) ? -amp : amp;
            long long ph = (kf * nn) % L; if (ph < 0) ph += L;
            double sn, cs;
            sincospi(-2.0 * (double)ph / (double)L, &sn, &cs);
            re += a * cs; im += a * sn;
        }
        prof[(long long)pidx * L + w] = (re * re + im * im) / (double)L;
    }
}

// Parseval NMSE constants per image: E_mask = sum over the mask of |y - F x0|^2
// (= |y' - c X0r|^2 in the sign-folded convention) and |x0|^2.
template <typename R>
__global__ void __launch_bounds__(SNT) nmse_setup(Geo g, const typename CT<R>::T* yg, const R* pinv,
                                                  const typename CT<R>::T* x0r, const typename CT<R>::T* x0,
                                                  double* consts) {
    __shared__ double sh[SNT / 32 + 2];
    const int bi = blockIdx.x;
    const long long base = (long long)bi * g.N;
    const double c = (double)g.sign_c;
    double e = 0.0, r = 0.0;
    for (long long i = threadIdx.x; i < g.N; i += SNT) {
        if (pinv[base + i] != R(0)) {
            const typename CT<R>::T a = yg[base + i], b = x0r[base + i];
            const double dx = (double)a.x - c * (double)b.x, dy = (double)a.y - c * (double)b.y;
            e += dx * dx + dy * dy;
        }
        const typename CT<R>::T v = x0[base + i];
        r += (double)v.x * (double)v.x + (double)v.y * (double)v.y;
    }
    e = block_sum<SNT>(e, sh);
    r = block_sum<SNT>(r, sh);
    if (threadIdx.x == 0) { consts[2 * bi] = e; consts[2 * bi + 1] = r; }
}

// per-iteration NMSE record from the column-tile partials (fixed order)
__global__ void nmse_finish(const double* part, int ntiles, const double* consts, double* out, int B) {
    const int bi = blockIdx.x * blockDim.x + threadIdx.x;
    if (bi >= B) return;
    double e = consts[2 * bi];
    for (int t = 0; t < ntiles; ++t) e += part[(long long)bi * ntiles + t];
    out[2 * bi] = e;
    out[2 * bi + 1] = consts[2 * bi + 1];
}

// Monte Carlo accumulation over a batch of draws (tests/conftest.py:41-81 of the
// reference): sum_r[i] += sum_b r_b[i]; err[i] = sum_b |r_b[i] - w0[i]|^2 (fixed
// image order, deterministic).  Per-subband means are formed by mc_band_sums.
template <typename R>
__global__ void mc_accumulate(Geo g, int B, const typename CT<R>::T* r, const typename CT<R>::T* w0,
                              double2* sum_r, double* err) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < g.N; i += (long long)gridDim.x * blockDim.x) {
        const typename CT<R>::T w = w0[i];
        double sx = 0.0, sy = 0.0, e = 0.0;
        for (int b = 0; b < B; ++b) {
            const typename CT<R>::T v = r[(long long)b * g.N + i];
            sx += (double)v.x; sy += (double)v.y;
            const double dx = (double)v.x - (double)w.x, dy = (double)v.y - (double)w.y;
            e += dx * dx + dy * dy;
        }
        sum_r[i].x += sx; sum_r[i].y += sy;
        err[i] = e;
    }
}

// sum_sq[j] += (sum over subband j of err) / len_j   (one CTA per subband)
__global__ void __launch_bounds__(SNT) mc_band_sums(Geo g, const double* err, double* sum_sq) {
    __shared__ double sh[SNT / 32 + 2];
    const int j = blockIdx.x;
    double e = 0.0;
    for (int i = threadIdx.x; i < g.len[j]; i += SNT) e += err[g.off[j] + i];
    e = block_sum<SNT>(e, sh);
    if (threadIdx.x == 0) sum_sq[j] += e / (double)g.len[j];
}

// ---- baselines on the same operators (src/baselines.py) -----------------
// FISTA / SURE-IT update: w = soft(g; t_j), r~ = w + beta (w - w_prev), in place
// (src/baselines.py:77-83, 143-148).  par = (t, 0, 1) per (image, subband).
template <typename R>
__global__ void momentum_update(Geo g, typename CT<R>::T* coef, typename CT<R>::T* what, const double* par,
                                double beta) {
    typedef typename CT<R>::T C;
    const int j = blockIdx.y, bi = blockIdx.z;
    const R t = (R)par[((long long)bi * g.S + j) * 3];
    const R be = (R)beta;
    const long long base = (long long)bi * g.N + g.off[j];
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < g.len[j]; e += gridDim.x * blockDim.x) {
        const C w = onsager<R, C>(coef[base + e], t, R(0), R(1));
        const C wp = what[base + e];
        coef[base + e] = mk<C>(w.x + be * (w.x - wp.x), w.y + be * (w.y - wp.y));
        what[base + e] = w;
    }
}

// per (image, subband): |a - w0|^2 and |w0|^2 (src/diagnostics.py:37-51)
template <typename R>
__global__ void __launch_bounds__(256) coef_err(Geo g, const typename CT<R>::T* a, const typename CT<R>::T* w0,
                                                double* out) {
    __shared__ double sh[256 / 32 + 2];
    const int j = blockIdx.x, bi = blockIdx.y;
    const long long base = (long long)bi * g.N + g.off[j];
    double e = 0.0, r = 0.0;
    for (int i = threadIdx.x; i < g.len[j]; i += 256) {
        const typename CT<R>::T u = a[base + i], w = w0[base + i];
        const double dx = (double)u.x - (double)w.x, dy = (double)u.y - (double)w.y;
        e += dx * dx + dy * dy;
        r += (double)w.x * (double)w.x + (double)w.y * (double)w.y;
    }
    e = block_sum<256>(e, sh);
    r = block_sum<256>(r, sh);
    if (threadIdx.x == 0) { out[((long long)bi * g.S + j) * 2] = e; out[((long long)bi * g.S + j) * 2 + 1] = r; }
}

// per image: NMSE record {sum_j err, sum_j ref} of coef_err output (fixed order)
__global__ void err_totals(const double* e, int S, int B, double* out) {
    const int bi = blockIdx.x * blockDim.x + threadIdx.x;
    if (bi >= B) return;
    double a = 0.0, b = 0.0;
    for (int j = 0; j < S; ++j) { a += e[((long long)bi * S + j) * 2]; b += e[((long long)bi * S + j) * 2 + 1]; }
    out[2 * bi] = a; out[2 * bi + 1] = b;
}

// SURE-IT oracle error level tau_k = |r - w0|^2 / N, floored, same for every
// subband (src/baselines.py:140-142)
template <typename R>
__global__ void __launch_bounds__(SNT) oracle_tau(Geo g, const typename CT<R>::T* r, const typename CT<R>::T* w0,
                                                  double* tau) {
    __shared__ double sh[SNT / 32 + 2];
    const int bi = blockIdx.x;
    const long long base = (long long)bi * g.N;
    double e = 0.0;
    for (long long i = threadIdx.x; i < g.N; i += SNT) {
        const typename CT<R>::T u = r[base + i], w = w0[base + i];
        const double dx = (double)u.x - (double)w.x, dy = (double)u.y - (double)w.y;
        e += dx * dx + dy * dy;
    }
    e = block_sum<SNT>(e, sh);
    const double t = fmax(e / (double)g.N, 1e-30);
    for (int j = threadIdx.x; j < g.S; j += SNT) tau[(long long)bi * g.S + j] = t;
}

__global__ void fill_threshold_params(double* par, const double* lam, int S, int B) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B * S) return;
    par[3 * i] = lam[i / S]; par[3 * i + 1] = 0.0; par[3 * i + 2] = 1.0;
}

// per-image |x - x0|^2 and |x0|^2 (src/diagnostics.py:21-34), deterministic
template <typename R>
__global__ void __launch_bounds__(SNT) nmse_sums(Geo g, const typename CT<R>::T* x, const typename CT<R>::T* x0, double* out) {
    __shared__ double sh[SNT / 32 + 2];
    const int bi = blockIdx.x;
    const long long base = (long long)bi * g.N;
    double e = 0.0, r = 0.0;
    for (long long i = threadIdx.x; i < g.N; i += SNT) {
        const typename CT<R>::T a = x[base + i], b = x0[base + i];
        const double dx = (double)a.x - (double)b.x, dy = (double)a.y - (double)b.y;
        e += dx * dx + dy * dy;
        r += (double)b.x * (double)b.x + (double)b.y * (double)b.y;
    }
    e = block_sum<SNT>(e, sh);
    r = block_sum<SNT>(r, sh);
    if (threadIdx.x == 0) { out[2 * bi] = e; out[2 * bi + 1] = r; }
}

}  // namespace vdamp
