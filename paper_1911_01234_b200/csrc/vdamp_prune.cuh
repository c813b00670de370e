// Exact SURE threshold selection by bounds (K4 fast path; src/denoise.py:62-118).
//
// The reference sorts all n magnitudes of a subband and evaluates the risk at
// every candidate.  Near the minimum the risk is flat only over a few percent
// of the keys (cfg1: within 16 tau of the minimum lie 1-5% of them), so this
// path sorts and evaluates only those, and proves that no other candidate can
// win:
//
//  1. keys -> fine buckets, linear in the IEEE bits over the top PR_OCT
//     octaves below the largest key (bucket 0: zeros; bucket 1: the keys
//     below that range); integer counts only, so everything that follows is
//     deterministic.
//  2. For t in bucket b's value range [A_b, A_{b+1}) the risk is bounded below
//     using counts and bucket edges alone: keys below contribute >= A^2 each,
//     keys inside >= A_b^2, keys above >= t^2 + 2 tau - tau t / A (convex in t,
//     minimised over the bucket range); bucket edges give upper bounds of the
//     risk at those thresholds, and the t = 0 risk is exact.  A bucket whose
//     lower bound exceeds the smallest upper bound U (plus a 1e-9 relative
//     rounding margin) holds no minimiser, no tie and no interior stationary
//     point that could win.  Groups of PR_BPT buckets (one per thread) are
//     tested first, then the buckets of the surviving span.
//  3. The surviving span [wlo, whi], extended down to the nearest non-empty
//     bucket (whose last key starts the quadratic piece that enters the span),
//     is gathered, bitonic-sorted and scanned exactly with the same
//     scan_tile code as the full path, offset by the exact float64 sums of
//     m^2 below and 1/m above it (fixed per-thread order and reduction tree:
//     deterministic) and by the first key above it.
//
// Falls back (returns false) when the span holds more than PR_LMAX keys
// (heavy ties, diverged or degenerate data); the caller then sorts everything.
// Included inside namespace vdamp by vdamp_kernels.cuh (after scan_tile).
#pragma once

template <typename R> struct PrT;
template <> struct PrT<float> {
    typedef unsigned U;
    static constexpr int MB = 23;
    static constexpr U INFB = 0x7f800000u;
    __device__ static double val(U b) { return (double)__uint_as_float(b); }
    __device__ static U bits(float x) { return __float_as_uint(x); }
    __device__ static double rcp(double m) { return rcp_posf(m); }
};
template <> struct PrT<double> {
    typedef unsigned long long U;
    static constexpr int MB = 52;
    static constexpr U INFB = 0x7ff0000000000000ull;
    __device__ static double val(U b) { return __longlong_as_double((long long)b); }
    __device__ static U bits(double x) { return (U)__double_as_longlong(x); }
    __device__ static double rcp(double m) { return rcp_pos(m); }
};

constexpr int PR_OCT = 12;        // octaves below the largest key mapped linearly
constexpr int PR_LMAX = 4096;     // keys evaluated exactly at most (else the full sort); fp64: half
template <typename R> __host__ __device__ constexpr int pr_lmax() { return sizeof(R) == 4 ? PR_LMAX : PR_LMAX / 2; }
constexpr int PR_NC = 1024;       // coarse buckets (one per thread)
constexpr int PR_NF = 4096;       // fine buckets over the coarse span (four per thread)
constexpr int PR_NT32 = 512;      // threads of sure_prune32 (two CTAs per SM)
constexpr int PR_MAXT = 256;      // tau column-tile partials sure_prune32 holds (more: the 1024-thread path)
constexpr int PR_BIDN = 16384 + 16384 / 32 + 8;   // bucket-id slots (KI layout, n <= 16384)
// fp32 layout of the stage region: reduction scratch (168 doubles) | list | bucket ids
constexpr int PR_STAGE_BID = (5 * 32 + 8) * 8 + ((PR_LMAX + PR_LMAX / 32 + 8) * 4 + 15) / 16 * 16;

// Bucket map: 0 = zeros, 1 = nonzero keys below `lo`, b >= 2 linear in the bits
// from `base` (>= lo) with width 2^ls; `top`: one past the last linear bucket.
template <typename R>
struct PrMap {
    typedef typename PrT<R>::U U;
    U mn, lo, base;
    int ls, top;
    __device__ int bucket(U k) const {
        if (!k) return 0;
        if (k < lo) return 1;
        return 2 + (int)((k - base) >> ls);
    }
    // lower value edge of bucket b; edge(b + 1) is its upper edge
    __device__ double edge(int b) const {
        if (b <= 0) return 0.0;
        if (b == 1) return PrT<R>::val(mn);
        const U e = base + ((U)(b - 2) << ls);
        return PrT<R>::val(e >= PrT<R>::INFB || e < base ? PrT<R>::INFB : e);
    }
};

// min over t in [A, B] of c t^2 - tau I t (c > 0), 0 for c == 0
__device__ __forceinline__ double pr_qmin(double c, double I, double A, double B, double tau) {
    if (c <= 0.0) return 0.0;
    double t = tau * I * (0.5 / c);
    t = fmin(fmax(t, A), B);
    return t * fma(c, t, -tau * I);
}

// Block reductions / scans for the pruned path: warp shuffles, one smem exchange,
// warp 0 combines the warp partials with shuffles, one more exchange (fixed trees:
// deterministic).  `sh` must not be in use by another reduction in flight.
template <int NT>
__device__ __forceinline__ void pr_reduce4(double& a, double& b, double& c, double& d, double* sh) {
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
        c = fmin(c, __shfl_xor_sync(0xffffffffu, c, o));
        d += __shfl_xor_sync(0xffffffffu, d, o);
    }
    constexpr int NW = NT / 32;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) { sh[w] = a; sh[NW + w] = b; sh[2 * NW + w] = c; sh[3 * NW + w] = d; }
    __syncthreads();
    if (w == 0) {
        a = l < NW ? sh[l] : 0.0; b = l < NW ? sh[NW + l] : 0.0;
        c = l < NW ? sh[2 * NW + l] : INFINITY; d = l < NW ? sh[3 * NW + l] : 0.0;
        for (int o = 16; o > 0; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            b += __shfl_xor_sync(0xffffffffu, b, o);
            c = fmin(c, __shfl_xor_sync(0xffffffffu, c, o));
            d += __shfl_xor_sync(0xffffffffu, d, o);
        }
        if (l == 0) { sh[4 * NW] = a; sh[4 * NW + 1] = b; sh[4 * NW + 2] = c; sh[4 * NW + 3] = d; }
    }
    __syncthreads();
    a = sh[4 * NW]; b = sh[4 * NW + 1]; c = sh[4 * NW + 2]; d = sh[4 * NW + 3];
}

// float versions for the bounds (their rounding is covered by the 1e-5 margin)
template <bool REV>
__device__ __forceinline__ float warp_excl_scanf(float v, float& total) {
    const int l = threadIdx.x & 31;
    float inc = v;
    if (!REV) {
        for (int o = 1; o < 32; o <<= 1) { const float u = __shfl_up_sync(0xffffffffu, inc, o); if (l >= o) inc += u; }
        const float ex = __shfl_up_sync(0xffffffffu, inc, 1);
        total = __shfl_sync(0xffffffffu, inc, 31);
        return l == 0 ? 0.0f : ex;
    } else {
        for (int o = 1; o < 32; o <<= 1) { const float u = __shfl_down_sync(0xffffffffu, inc, o); if (l + o < 32) inc += u; }
        const float ex = __shfl_down_sync(0xffffffffu, inc, 1);
        total = __shfl_sync(0xffffffffu, inc, 0);
        return l == 31 ? 0.0f : ex;
    }
}

// exclusive scans: KF values forward (sum over lower threads), KR reverse
template <int NT, int KF, int KR>
__device__ __forceinline__ void pr_scanf(float (&f)[KF], float (&r)[KR], float* sh) {
    constexpr int NW = NT / 32;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    float tf[KF], tr[KR];
#pragma unroll
    for (int i = 0; i < KF; ++i) f[i] = warp_excl_scanf<false>(f[i], tf[i]);
#pragma unroll
    for (int i = 0; i < KR; ++i) r[i] = warp_excl_scanf<true>(r[i], tr[i]);
    __syncthreads();
    if (l == 0) {
#pragma unroll
        for (int i = 0; i < KF; ++i) sh[i * NW + w] = tf[i];
#pragma unroll
        for (int i = 0; i < KR; ++i) sh[(KF + i) * NW + w] = tr[i];
    }
    __syncthreads();
    if (w == 0) {
        float d;
#pragma unroll
        for (int i = 0; i < KF; ++i) tf[i] = warp_excl_scanf<false>(l < NW ? sh[i * NW + l] : 0.0f, d);
#pragma unroll
        for (int i = 0; i < KR; ++i) tr[i] = warp_excl_scanf<true>(l < NW ? sh[(KF + i) * NW + l] : 0.0f, d);
        __syncwarp();
        if (l < NW) {
#pragma unroll
            for (int i = 0; i < KF; ++i) sh[i * NW + l] = tf[i];
#pragma unroll
            for (int i = 0; i < KR; ++i) sh[(KF + i) * NW + l] = tr[i];
        }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < KF; ++i) f[i] += sh[i * NW + w];
#pragma unroll
    for (int i = 0; i < KR; ++i) r[i] += sh[(KF + i) * NW + w];
}

// block: sum of a, b, c and min of m (floats)
template <int NT>
__device__ __forceinline__ void pr_reducef(float& a, float& b, float& c, float& m, float* sh) {
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
        c += __shfl_xor_sync(0xffffffffu, c, o);
        m = fminf(m, __shfl_xor_sync(0xffffffffu, m, o));
    }
    constexpr int NW = NT / 32;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) { sh[w] = a; sh[NW + w] = b; sh[2 * NW + w] = c; sh[3 * NW + w] = m; }
    __syncthreads();
    if (w == 0) {
        a = l < NW ? sh[l] : 0.0f; b = l < NW ? sh[NW + l] : 0.0f; c = l < NW ? sh[2 * NW + l] : 0.0f;
        m = l < NW ? sh[3 * NW + l] : INFINITY;
        for (int o = 16; o > 0; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            b += __shfl_xor_sync(0xffffffffu, b, o);
            c += __shfl_xor_sync(0xffffffffu, c, o);
            m = fminf(m, __shfl_xor_sync(0xffffffffu, m, o));
        }
        if (l == 0) { sh[4 * NW] = a; sh[4 * NW + 1] = b; sh[4 * NW + 2] = c; sh[4 * NW + 3] = m; }
    }
    __syncthreads();
    a = sh[4 * NW]; b = sh[4 * NW + 1]; c = sh[4 * NW + 2]; m = sh[4 * NW + 3];
}

// three sums, a min and a max in one exchange
template <int NT>
__device__ __forceinline__ void pr_reduce5(double& a, double& b, double& c, double& mn, double& mx, double* sh) {
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
        c += __shfl_xor_sync(0xffffffffu, c, o);
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    constexpr int NW = NT / 32;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) { sh[w] = a; sh[NW + w] = b; sh[2 * NW + w] = c; sh[3 * NW + w] = mn; sh[4 * NW + w] = mx; }
    __syncthreads();
    if (w == 0) {
        a = l < NW ? sh[l] : 0.0; b = l < NW ? sh[NW + l] : 0.0; c = l < NW ? sh[2 * NW + l] : 0.0;
        mn = l < NW ? sh[3 * NW + l] : INFINITY; mx = l < NW ? sh[4 * NW + l] : -INFINITY;
        for (int o = 16; o > 0; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            b += __shfl_xor_sync(0xffffffffu, b, o);
            c += __shfl_xor_sync(0xffffffffu, c, o);
            mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if (l == 0) { sh[5 * NW] = a; sh[5 * NW + 1] = b; sh[5 * NW + 2] = c; sh[5 * NW + 3] = mn; sh[5 * NW + 4] = mx; }
    }
    __syncthreads();
    a = sh[5 * NW]; b = sh[5 * NW + 1]; c = sh[5 * NW + 2]; mn = sh[5 * NW + 3]; mx = sh[5 * NW + 4];
}

// block min of a, max of b (ints)
template <int NT>
__device__ __forceinline__ void pr_minmax(int& a, int& b, int* shi) {
    for (int o = 16; o > 0; o >>= 1) {
        a = min(a, __shfl_xor_sync(0xffffffffu, a, o));
        b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
    }
    constexpr int NW = NT / 32;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) { shi[w] = a; shi[NW + w] = b; }
    __syncthreads();
    if (w == 0) {
        a = l < NW ? shi[l] : 0x7fffffff;
        b = l < NW ? shi[NW + l] : -1;
        for (int o = 16; o > 0; o >>= 1) {
            a = min(a, __shfl_xor_sync(0xffffffffu, a, o));
            b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
        }
        if (l == 0) { shi[2 * NW] = a; shi[2 * NW + 1] = b; }
    }
    __syncthreads();
    a = shi[2 * NW]; b = shi[2 * NW + 1];
}

// Exclusive scans of KF values in thread order (sum over lower threads) and KR
// values in reverse order (sum over higher threads), sharing two exchanges; the
// same warp_excl_scan trees as block_excl_scan (no subtraction).
template <int NT, int KF, int KR>
__device__ __forceinline__ void pr_scan(double (&f)[KF], double (&r)[KR], double* sh) {
    constexpr int NW = NT / 32;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    double tf[KF], tr[KR];
#pragma unroll
    for (int i = 0; i < KF; ++i) f[i] = warp_excl_scan<false>(f[i], tf[i]);
#pragma unroll
    for (int i = 0; i < KR; ++i) r[i] = warp_excl_scan<true>(r[i], tr[i]);
    __syncthreads();
    if (l == 0) {
#pragma unroll
        for (int i = 0; i < KF; ++i) sh[i * NW + w] = tf[i];
#pragma unroll
        for (int i = 0; i < KR; ++i) sh[(KF + i) * NW + w] = tr[i];
    }
    __syncthreads();
    if (w == 0) {
        double d;
#pragma unroll
        for (int i = 0; i < KF; ++i) tf[i] = warp_excl_scan<false>(l < NW ? sh[i * NW + l] : 0.0, d);
#pragma unroll
        for (int i = 0; i < KR; ++i) tr[i] = warp_excl_scan<true>(l < NW ? sh[(KF + i) * NW + l] : 0.0, d);
        __syncwarp();
        if (l < NW) {
#pragma unroll
            for (int i = 0; i < KF; ++i) sh[i * NW + l] = tf[i];
#pragma unroll
            for (int i = 0; i < KR; ++i) sh[(KF + i) * NW + l] = tr[i];
        }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < KF; ++i) f[i] += sh[i * NW + w];
#pragma unroll
    for (int i = 0; i < KR; ++i) r[i] += sh[(KF + i) * NW + w];
}

#ifdef VDAMP_PHASE_TIMING
__device__ long long g_prune[4096][64][10];
#define PR_MARK(i) do { if (threadIdx.x == 0 && dbg) { long long c_ = clock64(); dbg[i] = c_ - pc0_; pc0_ = c_; } } while (0)
#define PR_NOTE(i, v) do { if (threadIdx.x == 0 && dbg) dbg[i] = (v); } while (0)
#else
#define PR_MARK(i) do { } while (0)
#define PR_NOTE(i, v) do { } while (0)
#endif

// Result of the pruned selection, consumed by select_band.
struct PrOut {
    int nbelow;        // keys below the evaluated list (0: the t = 0 candidates apply)
    double m0;         // smallest key of the list
};

__device__ __forceinline__ float pr_qminf(float c, float I, float A, float B, float tau) {
    if (c <= 0.0f) return 0.0f;
    float t = tau * I * (0.5f / c);
    t = fminf(fmaxf(t, A), B);
    return t * fmaf(c, t, -tau * I);
}
__device__ __forceinline__ float pr_lbf(float pl, float c, float A, float B, float cu, float iu, float tau) {
    return pl + c * A * A + 2.0f * tau * cu + pr_qminf(cu, iu, A, B, tau);
}
__device__ __forceinline__ float pr_ubf(float pu, float cge, float A, float il, float tau) {
    return pu + cge * A * A + 2.0f * tau * cge - tau * A * il;
}

// Lower bound of the risk + n tau over t in [A, B), from: squares below >= pl,
// c keys inside (>= A^2 each), cu keys above with sum of 1/m <= iu.
__device__ __forceinline__ double pr_lb(double pl, double c, double A, double B, double cu, double iu, double tau) {
    return pl + c * A * A + 2.0 * tau * cu + pr_qmin(cu, iu, A, B, tau);
}
// Upper bound of the risk + n tau at t = A (A > 0): squares below <= pu, cge keys
// at or above A with sum of 1/m >= il.
__device__ __forceinline__ double pr_ub(double pu, double cge, double A, double il, double tau) {
    return pu + cge * A * A + 2.0 * tau * cge - tau * A * il;
}

// One bounds level over buckets [0, K*NT) of map M (K per thread, counts in cnt, only
// buckets [flo, ftop) belong to the range): exclusive scans of the edge sums, upper
// bounds of the risk at every lower edge (t = 0 exact when flo == 0; beyond the largest
// key when `top`), U = their minimum (never above Uprev), then the buckets whose lower
// bound is <= U + margin -> [w0, w1].  pbf / iaf / cblf: squares below the range,
// inverses above it, keys below it.  Returns the margin-widened U.
template <int NT, int K, typename MapT>
__device__ __forceinline__ float pr_stage(const unsigned* cnt, const MapT& M, int flo, int ftop, bool top, float pbf,
                                          float iaf, float cblf, int n, float tauf, float ntauf, float Uprev,
                                          float* shf, int& w0, int& w1) {
    const int tid = threadIdx.x;
    const int b0 = K * tid;
    float cv[K], A[K + 1], ivs[K], ibs[K];
#pragma unroll
    for (int i = 0; i <= K; ++i) A[i] = (float)M.edge(b0 + i);
    float f[3] = {0.0f, 0.0f, 0.0f}, r[2] = {0.0f, 0.0f};
#pragma unroll
    for (int i = 0; i < K; ++i) {
        const int b = b0 + i;
        const float c = (b >= flo && b < ftop) ? (float)cnt[b] : 0.0f;
        cv[i] = c;
        f[0] = fmaf(c * A[i], A[i], f[0]);
        f[1] = fmaf(c * A[i + 1], A[i + 1], f[1]);
        ivs[i] = (b >= 1 && c > 0.0f) ? c * __frcp_ru(A[i]) : 0.0f;
        ibs[i] = (b >= 1 && c > 0.0f && A[i + 1] < INFINITY) ? c * __frcp_rd(A[i + 1]) : 0.0f;
        r[0] += ivs[i];
        r[1] += ibs[i];
        f[2] += c;
    }
    const float own_b2 = f[1];
    pr_scanf<NT, 3, 2>(f, r, shf);
    float sufa[K], sufb[K];
    {
        float s2 = iaf + r[0], s3 = iaf + r[1];
#pragma unroll
        for (int i = K - 1; i >= 0; --i) { sufa[i] = s2; s2 += ivs[i]; s3 += ibs[i]; sufb[i] = s3; }
    }
    float ub = INFINITY;
    {
        float p = pbf + f[1], cbelow = cblf + f[2];
#pragma unroll
        for (int i = 0; i < K; ++i) {
            const int b = b0 + i;
            if (b >= flo && b < ftop && b >= 1)
                ub = fminf(ub, pr_ubf(p, (float)n - cbelow, A[i], sufb[i], tauf) - ntauf);
            p = fmaf(cv[i] * A[i + 1], A[i + 1], p);
            cbelow += cv[i];
        }
    }
    if (flo == 0 && tid == 0) ub = fminf(ub, 2.0f * tauf * ((float)n - cv[0]) - ntauf);   // t = 0, exact
    float scale = 0.0f, z0 = 0.0f, z1 = 0.0f;
    if (tid == NT - 1) {
        scale = pbf + f[1] + own_b2;                   // all squares below the range top, upper edges
        if (top) ub = fminf(ub, scale - ntauf);          // t beyond the largest key
    }
    pr_reducef<NT>(scale, z0, z1, ub, shf);
    const float Ulim = fminf(Uprev, ub + 1e-5f * (fabsf(ub) + 2.0f * ntauf + scale));
    w0 = 0x7fffffff;
    w1 = -1;
    {
        float p = pbf + f[0], cbelow = cblf + f[2];
#pragma unroll
        for (int i = 0; i < K; ++i) {
            const int b = b0 + i;
            const float cu = (float)n - cbelow - cv[i];
            const float lb = pr_lbf(p, cv[i], A[i], A[i + 1], cu, sufa[i], tauf) - ntauf;
            if (b >= flo && b < ftop && lb <= Ulim) { w0 = min(w0, b); w1 = max(w1, b); }
            p = fmaf(cv[i] * A[i], A[i], p);
            cbelow += cv[i];
        }
    }
    pr_minmax<NT>(w0, w1, reinterpret_cast<int*>(shf));
    return Ulim;
}

// keys: n keys of this subband at keys[KI(tid + q * NT)], q < EF (n == EF * NT), or
// (GLOBAL) at keys[e] in L2-resident global scratch with ef = n / NT at run time.
// cnt: >= PR_NC + PR_NF + 32 words.  bid: n + n/32 shorts (coarse bucket per key), or
// null (recomputed).  list: lmax + pad keys.  sh: >= 5 * NT/32 + 8 doubles.  Runs
// scan_tile over the list (S_.run, S_.totinv).  Returns false (scratch regions
// clobbered, keys intact) when the caller must sort all keys.
//
// Bounds are evaluated in float: every term of a bound is at most the sum of
// all squares plus 2 n tau in magnitude (keys above t satisfy m > t, so
// c t^2 <= their squares and tau t sum(1/m) <= n tau), and float rounding of the
// sums and products stays far below the 1e-5 relative margin added to U.
template <typename R, int NT, int EF, typename SS, bool GLOBAL = false>
__device__ bool select_pruned(int n, double tau, const R* keys, unsigned* cnt, unsigned short* bid, R* list,
                              int lmax, double* sh, typename PrT<R>::U kmn, typename PrT<R>::U kmx, SS& S_,
                              PrOut& out, long long* dbg = nullptr) {
    // four fine buckets per thread (a 512-thread CTA uses 2,048: eight would spill)
    constexpr int NF = 4 * NT;
    static_assert(PR_NC % NT == 0 && NF <= PR_NF, "whole buckets per thread");
    constexpr int KC = PR_NC / NT, KF = NF / NT;
    const int ef = GLOBAL ? n / NT : EF;
    auto key = [&](int e) -> R { if constexpr (GLOBAL) return __ldcg(keys + e); else return keys[KI(e)]; };
    typedef typename PrT<R>::U U;
#ifdef VDAMP_PHASE_TIMING
    long long pc0_ = clock64();
    PR_NOTE(8, -1);
#endif
    const int tid = threadIdx.x;
    const double ntau = (double)n * tau;
    const float tauf = (float)tau, ntauf = (float)ntau;
    unsigned* cc = cnt;                 // coarse counts
    unsigned* cf = cnt + PR_NC;         // fine counts
    unsigned* lc = cnt + PR_NC + PR_NF; // list cursor
    float* shf = reinterpret_cast<float*>(sh);
    constexpr int NW = NT / 32;

    // ---- 1. key range, coarse map, coarse histogram (bucket ids kept) --------
    for (int o = 16; o > 0; o >>= 1) {
        const U a = __shfl_xor_sync(0xffffffffu, kmn, o), b = __shfl_xor_sync(0xffffffffu, kmx, o);
        kmn = a < kmn ? a : kmn;
        kmx = b > kmx ? b : kmx;
    }
    U* ur = reinterpret_cast<U*>(sh);
    __syncthreads();
    if ((tid & 31) == 0) { ur[tid >> 5] = kmn; ur[NW + (tid >> 5)] = kmx; }
    for (int i = tid; i < PR_NC + NF; i += NT) cnt[i] = 0u;
    if (tid == 0) *lc = 1u;                      // list slot 0: the largest key below the window
    __syncthreads();
    U mn, mx;
    {
        U a = (tid & 31) < NW ? ur[tid & 31] : ~(U)0, b = (tid & 31) < NW ? ur[NW + (tid & 31)] : 0;
        for (int o = 16; o > 0; o >>= 1) {
            const U x = __shfl_xor_sync(0xffffffffu, a, o), y = __shfl_xor_sync(0xffffffffu, b, o);
            a = x < a ? x : a;
            b = y > b ? y : b;
        }
        mn = a; mx = b;
    }
    if (mn > mx) return false;                   // all keys zero: the full path handles it
    PrMap<R> C;
    C.mn = mn;
    {
        const U span = (U)PR_OCT << PrT<R>::MB;
        C.lo = C.base = (mx - mn > span) ? mx - span : mn;
        const U d = mx - C.lo;                   // smallest ls with (d >> ls) <= PR_NC - 3
        int ls = 0;
        if (d > (U)(PR_NC - 3)) {
            ls = (int)(8 * sizeof(U)) - (sizeof(U) == 4 ? __clz((unsigned)d) : __clzll((long long)d)) - 10;
            if (ls < 0) ls = 0;
            while ((d >> ls) > (U)(PR_NC - 3)) ++ls;
        }
        C.ls = ls;
        C.top = PR_NC;
    }
#pragma unroll (GLOBAL ? 4 : (EF > 16 ? 8 : EF))
    for (int q = 0; q < ef; ++q) {
        const int e = tid + q * NT;
        const int b = C.bucket(PrT<R>::bits(key(e)));
        if (bid) bid[KI(e)] = (unsigned short)b;
        atomicAdd(&cc[b], 1u);
    }
    __syncthreads();
    PR_MARK(0);

    // ---- 2. coarse bounds -> span [g0, g1] -------------------------------------
    int g0, g1;
    const float Ulim = pr_stage<NT, KC>(cc, C, 0, PR_NC, true, 0.0f, 0.0f, 0.0f, n, tauf, ntauf, INFINITY, shf, g0, g1);
    if (g1 < 0) return false;
    PR_MARK(1);

    // ---- 3. float sums outside the span, fine histogram inside ----------------
    PrMap<R> F;
    F.mn = mn;
    F.lo = C.lo;
    F.base = C.lo + ((U)(g0 >= 2 ? g0 - 2 : 0) << C.ls);
    {
        const U fe = C.lo + ((U)(g1 >= 2 ? g1 - 1 : 0) << C.ls);   // one past the span's top bit
        int ls = 0;
        if (fe > F.base)
            while (((fe - 1 - F.base) >> ls) > (U)(NF - 3)) ++ls;
        F.ls = ls;
        F.top = fe > F.base ? 3 + (int)((fe - 1 - F.base) >> ls) : 2;
    }
    const int flo = g0 >= 2 ? 2 : g0;            // first fine bucket that belongs to the span
    float pbf = 0.0f, iaf = 0.0f, cblf = 0.0f, zz = INFINITY;
#pragma unroll (GLOBAL ? 4 : (EF > 16 ? 8 : EF))
    for (int q = 0; q < ef; ++q) {
        const int e = tid + q * NT;
        const R m = key(e);
        const int b = bid ? (int)bid[KI(e)] : C.bucket(PrT<R>::bits(m));
        const float mf = (float)m;
        pbf = b < g0 ? fmaf(mf, mf, pbf) : pbf;
        cblf += b < g0 ? 1.0f : 0.0f;
        iaf += b > g1 ? __frcp_ru(mf) : 0.0f;
        if (b >= g0 && b <= g1) atomicAdd(&cf[F.bucket(PrT<R>::bits(m))], 1u);
    }
    pr_reducef<NT>(pbf, iaf, cblf, zz, shf);
    PR_MARK(2);

    // ---- 4. fine bounds -> window [f0, f1] ---------------------------------------
    int f0, f1;
    pr_stage<NT, KF>(cf, F, flo, F.top, false, pbf, iaf, cblf, n, tauf, ntauf, Ulim, shf, f0, f1);
    if (f1 < 0) return false;
    PR_MARK(3);

    // ---- 5. exact float64 offsets (all keys), list gather, sort, scan ---------
    double pre = 0.0, suf = 0.0, nbl = 0.0, nxt = INFINITY, mprev = -INFINITY;
#pragma unroll (GLOBAL ? 4 : (EF > 16 ? 8 : EF))
    for (int q = 0; q < ef; ++q) {
        const int e = tid + q * NT;
        const R m = key(e);
        const int b = bid ? (int)bid[KI(e)] : C.bucket(PrT<R>::bits(m));
        const int fb = (b < g0) ? -1 : (b > g1) ? 0x7fffffff : F.bucket(PrT<R>::bits(m));
        const double md = (double)m;
        if (fb < f0) { pre = fma(md, md, pre); nbl += 1.0; mprev = fmax(mprev, md); }
        else if (fb > f1) { suf += PrT<R>::rcp(md); nxt = fmin(nxt, md); }
        else {
            const unsigned pos = atomicAdd(lc, 1u);
            if (pos < (unsigned)lmax) list[KI(pos)] = m;
        }
    }
    pr_reduce5<NT>(pre, suf, nbl, nxt, mprev, sh);
    const int Lw = (int)*lc - 1;                 // window keys (slots 1..Lw)
    const bool prev = nbl > 0.0;                 // the largest key below leads the list
    PR_MARK(4);
    PR_NOTE(7, Lw);
    // the padded list (a power of two >= Lw + 1) must fit the list buffer
    if (Lw + 1 > lmax || Lw + (prev ? 1 : 0) < 1) return false;
    // offsets: squares below the list (all keys below but one instance of mprev, the
    // list's first element; its ties stay below), inverses above it
    const double pre_list = prev ? pre - mprev * mprev : 0.0;
    const int nb = (int)nbl - (prev ? 1 : 0);
    const int L = Lw + 1;                        // slot 0: mprev, or +inf padding (sorted last)
    int Lp = 2;
    while (Lp < L) Lp <<= 1;
    if (tid == 0) list[KI(0)] = prev ? (R)mprev : (R)INFINITY;
    for (int i = L + tid; i < Lp; i += NT) list[KI(i)] = (R)INFINITY;
    __syncthreads();
    block_sort<R, NT>(list, Lp);
    PR_MARK(5);
    if (tid == 0) S_.run = Best{INFINITY, INFINITY, 0.0, 0.0};
    const int Lr = Lw + (prev ? 1 : 0);          // real keys
    if (Lp <= 4 * NT)
        scan_tile<R, NT, 4, false, 4, true>(list, Lr, nb, n, tau, pre_list, suf, nxt, S_.sh, S_.best, &S_.run,
                                            &S_.totinv, nullptr, nullptr);
    else
        scan_tile<R, NT, 16, false, 16, true>(list, Lr, nb, n, tau, pre_list, suf, nxt, S_.sh, S_.best, &S_.run,
                                              &S_.totinv, nullptr, nullptr);
    PR_MARK(6);
    PR_NOTE(8, 1);
    out.nbelow = nb;
    out.m0 = (double)list[KI(0)];
    return true;
}
