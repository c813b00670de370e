// Lean bound-pruned exact SURE selection for fp32 subbands of 4,096..16,384 keys
// (src/denoise.py:62-118): the bounds of vdamp_prune.cuh, restated for 512-thread CTAs
// that fit two to an SM (about 90 KB of shared memory, 64 registers, no spills), so one
// CTA's block-wide scans and barriers overlap the other's key passes.
//
//  - every block-wide reduction / scan costs one barrier: warp shuffle tree, one
//    partial per warp into a double-buffered scratch, barrier, then every warp combines
//    the 16 partials itself (same fixed tree in every warp: deterministic);
//  - bucket membership is tested on the key bits against precomputed bit thresholds
//    (the bucket maps are monotone in the bits), the key passes are branch-free apart
//    from the rare list append, and the float64 reciprocals of the exact pass run as
//    independent chains (no per-key branch);
//  - reciprocal bounds use the hardware approximation (1 ulp) widened by 3 ulp instead
//    of the directed-rounding software reciprocals.
//
// Included inside namespace vdamp by vdamp_kernels.cuh (after vdamp_prune.cuh).
#pragma once
#ifndef WN_CUT
#define WN_CUT 99
#endif

// A CTA of NT threads (NT = 128 / 256 / 512) takes a subband of EF * NT keys (4,096 /
// 8,192 / 16,384): every thread owns 32 keys, so the per-CTA block-wide work (scans over
// 2 NT coarse and 4 NT fine buckets, reductions over NT / 32 warps) shrinks with the
// subband, and 1024 / NT CTAs share an SM.
constexpr int WN_MAXT = 256;           // tau column-tile partials held
template <int NT, int EF_ = 32, bool GL = false> struct Wn {
    static constexpr int EF = EF_;             // keys per thread
    static constexpr int LE = (NT >= 512 && !GL) ? 4 : 8;   // list keys per thread of the exact scan
    static constexpr int NW = NT / 32;
    static constexpr int NC = 2 * NT;          // coarse buckets (two per thread)
    static constexpr int KF = GL ? 8 : 4;      // fine buckets per thread (large subbands: as many keys per bucket)
    static constexpr int NF = KF * NT;         // fine buckets over the coarse span
    static constexpr int LOGNF = (NT == 1024 ? 10 : NT == 512 ? 9 : NT == 256 ? 8 : 7) + (GL ? 3 : 2);
    static constexpr int LMAX = LE * NT;       // keys evaluated exactly at most (else the full sort)
    static constexpr int LIST = LMAX + LMAX / 32 + 8;                 // padded list slots (KI layout)
    static constexpr int SLOT = (EF * NT + EF * NT / 32 + 2 + 3) & ~3;       // padded key slots (KI layout)
    static constexpr int LOGNC = NT == 1024 ? 11 : NT == 512 ? 10 : NT == 256 ? 9 : 8;
};

template <int NW>
struct WnScratch {                     // per-warp partials, double-buffered
    float f[2][5 * NW];
    double d[2][2 * NW];
    unsigned u[2][2 * NW];
    int i[2][2 * NW];
    int amin[2], wlo[2], whi[2];       // block min (ordered-int floats) / window bounds by shared atomics
    float scale[2];
};

// GLOBAL: the keys stay in L2-resident global scratch (subbands beyond the shared capacity).
// CS > 1 (cluster of CS CTAs per subband, GLOBAL keys): a second counter array holds the
// histograms merged over the cluster.
template <int NT, int EF, bool GLOBAL = false, int CS = 1>
__host__ __device__ constexpr size_t wn_smem_bytes() {
    typedef Wn<NT, EF, GLOBAL> W;
    return (GLOBAL ? 0 : (size_t)W::SLOT * 4) + (size_t)(W::NC + W::NF + 32) * 4 * (CS > 1 ? 2 : 1) +
           sizeof(WnScratch<NT / 32>) + (size_t)2 * W::LIST * 4;
}

// Per-CTA partial results exchanged through distributed shared memory (cluster variant):
// every CTA publishes its own and reads all of them in rank order (fixed order: deterministic,
// and identical in every CTA of the cluster)
struct WnX {
    unsigned mn, mx;                   // key-bit range of the CTA's keys
    float pbf, iaf, cblf;              // float sums outside the coarse span
    unsigned nxb, pvb;                 // first key above / largest key below the window
    double pre, suf;                   // exact sums outside the window
    double err, ref;                   // trace error sums
};

__device__ __forceinline__ float wn_rcp(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
constexpr float WN_UP = 1.0000004f, WN_DN = 0.9999996f;   // 3 ulp around the 1-ulp approximation

// float <-> int with the same order (an involution), for shared-memory atomicMin
__device__ __forceinline__ int wn_ord(float x) { const int i = __float_as_int(x); return i ^ ((i >> 31) & 0x7fffffff); }
__device__ __forceinline__ float wn_unord(int i) { return __int_as_float(i ^ ((i >> 31) & 0x7fffffff)); }

// pr_lbf with the stationary point from the approximate reciprocal: the quadratic is
// evaluated at a t within 1e-6 of its minimiser, i.e. within 1e-12 (relative) of its minimum
__device__ __forceinline__ float wn_lbf(float pl, float c, float A, float B, float cu, float iu, float tau) {
    float q = 0.0f;
    if (cu > 0.0f) {
        float t = tau * iu * (0.5f * wn_rcp(cu));
        t = fminf(fmaxf(t, A), B);
        q = t * fmaf(cu, t, -tau * iu);
    }
    return pl + c * A * A + 2.0f * tau * cu + q;
}

// Bucket map as PrMap<float>: 0 = zeros, 1 = nonzero keys below `lo`, b >= 2 linear in
// the bits from `base` with width 2^ls.
struct WnMap {
    unsigned mn, lo, base;
    int ls, top;
    __device__ __forceinline__ int bucket(unsigned k) const {
        if (!k) return 0;
        if (k < lo) return 1;
        return 2 + (int)((k - base) >> ls);
    }
    // smallest key bits that map to bucket b (b <= one past the last bucket of the map: with the
    // largest key < 2^100, select_win's guard, the sum neither wraps nor reaches +inf)
    __device__ __forceinline__ unsigned lowbits(int b) const {
        if (b <= 0) return 0u;
        if (b == 1) return 1u;
        return base + ((unsigned)(b - 2) << ls);
    }
    // lower value edge of bucket b; edge(b + 1) is its upper edge
    __device__ __forceinline__ float edge(int b) const {
        if (b <= 0) return 0.0f;
        if (b == 1) return __uint_as_float(mn);
        return __uint_as_float(lowbits(b));
    }
};

// exclusive scans in thread order: f0..f2 forward (sum over lower threads), r0, r1
// reverse (sum over higher threads); one barrier
template <int NW>
__device__ __forceinline__ void wn_scan5(float& f0, float& f1, float& f2, float& r0, float& r1, float* sh) {
    const int l = threadIdx.x & 31, w = threadIdx.x >> 5, q = l & (NW - 1);
    float t0, t1, t2, t3, t4;
    f0 = warp_excl_scanf<false>(f0, t0);
    f1 = warp_excl_scanf<false>(f1, t1);
    f2 = warp_excl_scanf<false>(f2, t2);
    r0 = warp_excl_scanf<true>(r0, t3);
    r1 = warp_excl_scanf<true>(r1, t4);
    if (l == 0) { sh[w] = t0; sh[NW + w] = t1; sh[2 * NW + w] = t2; sh[3 * NW + w] = t3; sh[4 * NW + w] = t4; }
    __syncthreads();
    t0 = q < w ? sh[q] : 0.0f; t1 = q < w ? sh[NW + q] : 0.0f; t2 = q < w ? sh[2 * NW + q] : 0.0f;
    t3 = q > w ? sh[3 * NW + q] : 0.0f; t4 = q > w ? sh[4 * NW + q] : 0.0f;
#pragma unroll
    for (int o = NW / 2; o > 0; o >>= 1) {
        t0 += __shfl_xor_sync(0xffffffffu, t0, o);
        t1 += __shfl_xor_sync(0xffffffffu, t1, o);
        t2 += __shfl_xor_sync(0xffffffffu, t2, o);
        t3 += __shfl_xor_sync(0xffffffffu, t3, o);
        t4 += __shfl_xor_sync(0xffffffffu, t4, o);
    }
    f0 += t0; f1 += t1; f2 += t2; r0 += t3; r1 += t4;
}

// block sums of a, b, c (floats); one barrier
template <int NW>
__device__ __forceinline__ void wn_sum3(float& a, float& b, float& c, float* sh) {
    const int l = threadIdx.x & 31, w = threadIdx.x >> 5, q = l & (NW - 1);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
        c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    if (l == 0) { sh[w] = a; sh[NW + w] = b; sh[2 * NW + w] = c; }
    __syncthreads();
    a = sh[q]; b = sh[NW + q]; c = sh[2 * NW + q];
#pragma unroll
    for (int o = NW / 2; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
        c += __shfl_xor_sync(0xffffffffu, c, o);
    }
}

// One bounds level (pr_stage of vdamp_prune.cuh): K buckets per thread of map M with
// counts in cnt; only buckets [flo, ftop) belong to the range.  Upper bounds of the risk
// at every lower edge (t = 0 exact when flo == 0, beyond the largest key when `top`), U =
// their minimum (never above Uprev), then the buckets whose lower bound is <= U + margin
// -> [w0, w1].  pbf / iaf / cblf: squares below the range, inverses above it, keys below
// it (all in the scaled units: edges times ksc, tau times ksc^2).  Returns the margin-widened U.
// Three barriers; the block minimum and the window bounds go
// through shared-memory integer atomics (deterministic).
template <int NT, int K>
__device__ __forceinline__ float wn_stage(const unsigned* cnt, const WnMap& M, float ksc, int flo, int ftop, bool top, float pbf,
                                          float iaf, float cblf, int n, float tauf, float ntauf, float Uprev,
                                          WnScratch<NT / 32>& sc, int& ph, int& w0, int& w1) {
    const int tid = threadIdx.x;
    const int b0 = K * tid;
    float cv[K], A[K + 1];
#pragma unroll
    for (int i = 0; i <= K; ++i) A[i] = M.edge(b0 + i) * ksc;     // edges in units of 2^e(largest key)
    // inverse-sum terms of bucket i: c / A_i rounded up (ivs), c / A_{i+1} rounded down (ibs);
    // recomputed where needed rather than held (registers)
    auto ivs = [&](int i) { return (b0 + i >= 1 && cv[i] > 0.0f) ? cv[i] * (wn_rcp(A[i]) * WN_UP) : 0.0f; };
    auto ibs = [&](int i) { return (b0 + i >= 1 && cv[i] > 0.0f) ? cv[i] * (wn_rcp(A[i + 1]) * WN_DN) : 0.0f; };
    float f0 = 0.0f, f1 = 0.0f, f2 = 0.0f, r0 = 0.0f, r1 = 0.0f;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        const int b = b0 + i;
        const float c = (b >= flo && b < ftop) ? (float)cnt[b] : 0.0f;
        cv[i] = c;
        f0 = fmaf(c * A[i], A[i], f0);
        f1 = fmaf(c * A[i + 1], A[i + 1], f1);
        r0 += ivs(i);
        r1 += ibs(i);
        f2 += c;
    }
    const float own_b2 = f1;
    if (tid == 0) { sc.amin[ph] = 0x7fffffff; sc.wlo[ph] = 0x7fffffff; sc.whi[ph] = -1; }
    wn_scan5<NT / 32>(f0, f1, f2, r0, r1, sc.f[ph]);
    // upper bounds at the lower edges (forward), with the inverse suffixes rebuilt on the way
    float ub = INFINITY;
    {
        float s3 = iaf + r1;
#pragma unroll
        for (int i = K - 1; i >= 0; --i) s3 += ibs(i);              // inverses at or above edge b0 (lower bounds)
        float p = pbf + f1, cbelow = cblf + f2;
#pragma unroll
        for (int i = 0; i < K; ++i) {
            const int b = b0 + i;
            if (b >= flo && b < ftop && b >= 1)
                ub = fminf(ub, pr_ubf(p, (float)n - cbelow, A[i], s3, tauf) - ntauf);
            s3 -= ibs(i);
            p = fmaf(cv[i] * A[i + 1], A[i + 1], p);
            cbelow += cv[i];
        }
    }
    if (flo == 0 && tid == 0) ub = fminf(ub, 2.0f * tauf * ((float)n - cv[0]) - ntauf);   // t = 0, exact
    if (tid == NT - 1) {
        const float scale = pbf + f1 + own_b2;           // all squares below the range top, upper edges
        if (top) ub = fminf(ub, scale - ntauf);          // t beyond the largest key
        sc.scale[ph] = scale;
    }
    {
        const int um = __reduce_min_sync(0xffffffffu, wn_ord(ub));      // one REDUX per warp
        if ((tid & 31) == 0) atomicMin(&sc.amin[ph], um);
    }
    __syncthreads();
    ub = wn_unord(sc.amin[ph]);
    const float scale = sc.scale[ph];
    const float Ulim = fminf(Uprev, ub + 1e-5f * (fabsf(ub) + 2.0f * ntauf + scale));
    w0 = 0x7fffffff;
    w1 = -1;
    {
        float s2 = iaf + r0;
#pragma unroll
        for (int i = K - 1; i >= 1; --i) s2 += ivs(i);              // inverses above bucket b0 (upper bounds)
        float p = pbf + f0, cbelow = cblf + f2;
#pragma unroll
        for (int i = 0; i < K; ++i) {
            const int b = b0 + i;
            const float cu = (float)n - cbelow - cv[i];
            const float lb = wn_lbf(p, cv[i], A[i], A[i + 1], cu, s2, tauf) - ntauf;
            if (b >= flo && b < ftop && lb <= Ulim) { w0 = min(w0, b); w1 = max(w1, b); }
            if (i + 1 < K) s2 -= ivs(i + 1);
            p = fmaf(cv[i] * A[i], A[i], p);
            cbelow += cv[i];
        }
    }
    w0 = __reduce_min_sync(0xffffffffu, w0);
    w1 = __reduce_max_sync(0xffffffffu, w1);
    if ((tid & 31) == 0 && w1 >= 0) { atomicMin(&sc.wlo[ph], w0); atomicMax(&sc.whi[ph], w1); }
    __syncthreads();
    w0 = sc.wlo[ph];
    w1 = sc.whi[ph];
    ph ^= 1;
    return Ulim;
}

// Exact scan of Lr <= LE * NT sorted keys (KI layout) that follow nb smaller keys of the
// subband: LE consecutive keys per thread, scan_tile's arithmetic (squares summed upwards,
// inverses downwards: no cancellation) with one-barrier block scans; the argmin (ties ->
// smaller t) is merged into S_.run by thread 0.  pre_list: squares below the list; suf:
// inverses above it; nxt: first key above it.  Two barriers.
template <int NT, int LE, typename SS>
__device__ __forceinline__ void wn_scan_list(const float* list, int Lr, int nb, int n, double tau, double pre_list,
                                             double suf, double nxt, WnScratch<NT / 32>& sc, int& ph, SS& S_) {
    constexpr int WN_NW = NT / 32;
    const int tid = threadIdx.x, l = tid & 31, w = tid >> 5, q16 = l & (WN_NW - 1);
    const int b0 = LE * tid;
    const bool act = b0 < Lr;
    double ssq = 0.0, sinv = 0.0, sreg[LE];
    if (act) {
#pragma unroll
        for (int e = LE - 1; e >= 0; --e) {
            if (b0 + e < Lr) {
                sreg[e] = sinv;
                const double m = (double)list[KI(b0 + e)];
                ssq = fma(m, m, ssq);
                if (m > 0) sinv += rcp_posf(m);
            }
        }
    }
    const bool wact = w * 32 * LE < Lr;          // warps past the list only publish identities
    double ta = 0.0, tb = 0.0, pe = 0.0, se = 0.0;
    if (wact) {
        pe = warp_excl_scan<false>(ssq, ta);
        se = warp_excl_scan<true>(sinv, tb);
    }
    if (l == 0) { sc.d[ph][w] = ta; sc.d[ph][WN_NW + w] = tb; }
    __syncthreads();
    Best best{INFINITY, INFINITY, 0.0, 0.0};
    if (wact) {
        ta = q16 < w ? sc.d[ph][q16] : 0.0;
        tb = q16 > w ? sc.d[ph][WN_NW + q16] : 0.0;
#pragma unroll
        for (int o = WN_NW / 2; o > 0; o >>= 1) {
            ta += __shfl_xor_sync(0xffffffffu, ta, o);
            tb += __shfl_xor_sync(0xffffffffu, tb, o);
        }
        pe += ta + pre_list;
        se += tb + suf;
        if (tid == 0 && nb == 0) S_.totinv = se + sinv;       // sum of all inverses
        if (act) scan_keys<float, NT, LE, false, LE, true>(list, Lr, nb, n, tau, b0, LE, pe, se, nxt, best, sreg, nullptr, nullptr);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            Best c;
            c.risk = __shfl_xor_sync(0xffffffffu, best.risk, o);
            c.t = __shfl_xor_sync(0xffffffffu, best.t, o);
            c.cnt = __shfl_xor_sync(0xffffffffu, best.cnt, o);
            c.inv = __shfl_xor_sync(0xffffffffu, best.inv, o);
            if (better(c, best)) best = c;
        }
    }
    ph ^= 1;
    if (l == 0) S_.best[w] = best;
    __syncthreads();
    if (tid < 32) {                              // warp 0: argmin over the warp winners
        Best c = S_.best[q16];
#pragma unroll
        for (int o = WN_NW / 2; o > 0; o >>= 1) {
            Best d;
            d.risk = __shfl_xor_sync(0xffffffffu, c.risk, o);
            d.t = __shfl_xor_sync(0xffffffffu, c.t, o);
            d.cnt = __shfl_xor_sync(0xffffffffu, c.cnt, o);
            d.inv = __shfl_xor_sync(0xffffffffu, c.inv, o);
            if (better(d, c)) c = d;
        }
        if (tid == 0 && better(c, S_.run)) S_.run = c;
    }
}

// keys: n = EF * NT float keys, stored linearly; thread tid owns keys KV * (tid + q * NT) + j,
// j < KV = 4 (one 16-byte access each).  cnt: NC + NF + 32 words.
// grp, list: Wn<NT, EF, GLOBAL>::LIST keys each.  Leaves the window argmin in S_.run (and
// S_.totinv).  Returns false (scratch clobbered, keys intact) when the caller must sort
// all keys.
//
// CS > 1: the subband's n = CS * EF * NT keys are spread over a cluster of CS CTAs (keys: this
// CTA's EF * NT).  Every CTA histograms its own keys; after a cluster barrier each merges all
// CS histograms into its own copy (cnt + NC + NF + 32) and runs the same bounds on it, so all
// CTAs take the same decisions without a broadcast; per-CTA sums go through X (rank order).
// Window keys are appended to rank 0's grouped list by distributed-shared-memory atomics;
// rank 0 alone ranks and scans the list.  Returns true in every CTA; S_.run / out are rank 0's.
template <int NT, int EF, bool GLOBAL, int CS = 1, typename SS>
__device__ __forceinline__ bool select_win(int n, double tau, const float* keys, unsigned* cnt, float* grp, float* list,
                                           WnScratch<NT / 32>& sc, unsigned kmn, unsigned kmx, SS& S_, PrOut& out,
                                           long long* dbg = nullptr, WnX* X = nullptr, int ef_rt = 0) {
    typedef Wn<NT, EF, GLOBAL> W;
    const int ef = EF > 0 ? EF : ef_rt;            // keys per thread (EF == 0: a launch-time value)
    namespace cg = ::cooperative_groups;
    [[maybe_unused]] cg::cluster_group cluster = cg::this_cluster();
    [[maybe_unused]] const unsigned crank = CS > 1 ? cluster.block_rank() : 0u;
    // leave together: no CTA may exit while another still reads its shared memory
    auto fail = [&]() { if constexpr (CS > 1) cluster.sync(); return false; };
    constexpr int LE = W::LE, WN_NW = W::NW, NW = WN_NW, WN_NC = W::NC, WN_NF = W::NF, WN_LMAX = W::LMAX;
    // The thread's keys: KV consecutive keys per access (one 16-byte LDS / L2 load; 8 bytes when
    // the key count per thread is only known to be even), accesses NT * KV keys apart; keys
    // stored linearly in shared memory or in global scratch read through L2.
    constexpr int KV = EF == 0 ? 2 : 4;
    typedef typename std::conditional<KV == 4, uint4, uint2>::type KVt;
    const KVt* kb = reinterpret_cast<const KVt*>(keys);
    const int nacc = ef / KV;
    auto keyv = [&](int q, unsigned (&kk)[KV]) {
        KVt t;
        if constexpr (GLOBAL) t = __ldcg(kb + threadIdx.x + q * NT);
        else t = kb[threadIdx.x + q * NT];
        kk[0] = t.x; kk[1] = t.y;
        if constexpr (KV == 4) { kk[2] = t.z; kk[3] = t.w; }
    };
#ifdef VDAMP_PHASE_TIMING
    long long pc0_ = clock64();
    PR_NOTE(8, -1);
#endif
    const int tid = threadIdx.x, l = tid & 31, w = tid >> 5, q16 = l & (WN_NW - 1);
    unsigned* cc = cnt;                    // coarse counts (this CTA's keys)
    unsigned* cf = cnt + WN_NC;            // fine counts
    // the counts the bounds run on: merged over the cluster, or the CTA's own
    unsigned* ccm = CS > 1 ? cnt + (WN_NC + WN_NF + 32) : cc;
    unsigned* cfm = ccm + WN_NC;
    int ph = 0;
    // ccm/cfm[b] = sum over the cluster's CTAs of their cc/cf[b] (after a cluster barrier)
    auto merge_counts = [&](unsigned* dst, unsigned* src, int words) {
        if constexpr (CS > 1) {
            for (int i = tid; i < words / 4; i += NT) {
                uint4 s4 = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll 8
                for (int r = 0; r < CS; ++r) {
                    const uint4 v = reinterpret_cast<const uint4*>(cluster.map_shared_rank(src, r))[i];
                    s4.x += v.x; s4.y += v.y; s4.z += v.z; s4.w += v.w;
                }
                reinterpret_cast<uint4*>(dst)[i] = s4;
            }
            __syncthreads();
        }
    };

    // ---- 1. key range, coarse map, coarse histogram ---------------------------
    kmn = __reduce_min_sync(0xffffffffu, kmn);
    kmx = __reduce_max_sync(0xffffffffu, kmx);
    if (l == 0) { sc.u[ph][w] = kmn; sc.u[ph][WN_NW + w] = kmx; }
    {
        uint4* cz = reinterpret_cast<uint4*>(cnt);                 // cnt is 16-byte aligned
        for (int i = tid; i < (WN_NC + WN_NF) / 4; i += NT) cz[i] = make_uint4(0u, 0u, 0u, 0u);
    }
    __syncthreads();
    unsigned mn = __reduce_min_sync(0xffffffffu, sc.u[ph][q16]);
    unsigned mx = __reduce_max_sync(0xffffffffu, sc.u[ph][WN_NW + q16]);
    ph ^= 1;
    if constexpr (CS > 1) {
        if (tid == 0) { X->mn = mn; X->mx = mx; }
        cluster.sync();
#pragma unroll
        for (int r = 0; r < CS; ++r) {
            const WnX* xr = cluster.map_shared_rank(X, r);
            mn = min(mn, xr->mn);
            mx = max(mx, xr->mx);
        }
        if (crank == 0 && tid == 0) {              // trace error sums of the whole subband (rank order)
            double e2 = 0.0, r2 = 0.0;
            for (int r = 0; r < CS; ++r) { const WnX* xr = cluster.map_shared_rank(X, r); e2 += xr->err; r2 += xr->ref; }
            S_.err = e2; S_.ref = r2;
        }
    }
    if (mn > mx) return fail();                    // all keys zero: the full path handles it
    // The float bounds work on keys scaled by ksc = 2^-e (e: exponent of the largest key; exact)
    // and tau scaled by ksc^2: comparing bounds is invariant under it, and squares and
    // reciprocal sums stay well inside the float range for data of any magnitude (diverged
    // runs).  Normal keys below 2^100 (bucket edges past the largest key stay finite) spanning at
    // most 100 octaves; else the full path.
    if (mn < 0x00800000u || mx >= ((127u + 100u) << 23) || (mx >> 23) - (mn >> 23) > 100u) return fail();
    const float ksc = __uint_as_float((254u - (mx >> 23)) << 23);
    const float tauf = (float)(tau * (double)ksc * (double)ksc), ntauf = (float)((double)n * tau * (double)ksc * (double)ksc);
    WnMap C;
    C.mn = mn;
    {
        const unsigned span = (unsigned)PR_OCT << 23;
        C.lo = C.base = (mx - mn > span) ? mx - span : mn;
        const unsigned d = mx - C.lo;              // smallest ls with (d >> ls) <= WN_NC - 3
        int ls = 0;
        if (d > (unsigned)(WN_NC - 3)) {
            ls = 32 - __clz(d) - W::LOGNC;
            if (ls < 0) ls = 0;
            while ((d >> ls) > (unsigned)(WN_NC - 3)) ++ls;
        }
        C.ls = ls;
        C.top = WN_NC;
    }
#pragma unroll 2
    for (int q = 0; q < nacc; ++q) {
        unsigned kk[KV];
        keyv(q, kk);
#pragma unroll
        for (int j = 0; j < KV; ++j) atomicAdd(&cc[C.bucket(kk[j])], 1u);
    }
    if constexpr (CS > 1) cluster.sync(); else __syncthreads();
    merge_counts(ccm, cc, WN_NC);
    PR_MARK(0);
    if (WN_CUT == 0) return fail();

    // ---- 2. coarse bounds -> span [g0, g1] -------------------------------------
    int g0, g1;
    const float Ulim = wn_stage<NT, WN_NC / NT>(ccm, C, ksc, 0, WN_NC, true, 0.0f, 0.0f, 0.0f, n, tauf, ntauf, INFINITY, sc, ph, g0, g1);
    if (g1 < 0) return fail();
    PR_MARK(1);
    if (WN_CUT == 1) return fail();

    // ---- 3. float sums outside the span, fine histogram inside ----------------
    WnMap F;
    F.mn = mn;
    F.lo = C.lo;
    F.base = C.lo + ((unsigned)(g0 >= 2 ? g0 - 2 : 0) << C.ls);
    const unsigned fe = C.lo + ((unsigned)(g1 >= 2 ? g1 - 1 : 0) << C.ls);   // one past the span's top bit
    {
        int ls = 0;
        if (fe > F.base) {
            const unsigned x = fe - 1u - F.base;
            ls = x ? 32 - __clz(x) - W::LOGNF : 0;
            if (ls < 0) ls = 0;
            while ((x >> ls) > (unsigned)(WN_NF - 3)) ++ls;
        }
        F.ls = ls;
        F.top = fe > F.base ? 3 + (int)((fe - 1u - F.base) >> ls) : 2;
    }
    const int flo = g0 >= 2 ? 2 : g0;              // first fine bucket that belongs to the span
    const unsigned klo = C.lowbits(g0);            // key bits below klo: below the span
    const unsigned khi = g1 >= WN_NC - 1 ? 0xffffffffu : C.lowbits(g1 + 1);   // at or above khi: above it
    float pbf = 0.0f, iaf = 0.0f, cblf = 0.0f;
#pragma unroll 2
    for (int q = 0; q < nacc; ++q) {
        unsigned kk[KV];
        keyv(q, kk);
#pragma unroll
        for (int j = 0; j < KV; ++j) {
            const unsigned k = kk[j];
            const float mf = __uint_as_float(k) * ksc;
            const bool below = k < klo, above = k >= khi;
            pbf = fmaf(below ? mf : 0.0f, mf, pbf);
            cblf += below ? 1.0f : 0.0f;
            iaf += above ? wn_rcp(mf) * WN_UP : 0.0f;
            if (!below && !above) atomicAdd(&cf[F.bucket(k)], 1u);
        }
    }
    wn_sum3<NW>(pbf, iaf, cblf, sc.f[ph]);
    ph ^= 1;
    if constexpr (CS > 1) {
        if (tid == 0) { X->pbf = pbf; X->iaf = iaf; X->cblf = cblf; }
        cluster.sync();
        pbf = iaf = cblf = 0.0f;
#pragma unroll
        for (int r = 0; r < CS; ++r) {
            const WnX* xr = cluster.map_shared_rank(X, r);
            pbf += xr->pbf; iaf += xr->iaf; cblf += xr->cblf;
        }
        merge_counts(cfm, cf, WN_NF);
    }
    PR_MARK(2);
    if (WN_CUT == 2) return fail();

    // ---- 4. fine bounds -> window [f0, f1] ---------------------------------------
    int f0, f1;
    wn_stage<NT, WN_NF / NT>(cfm, F, ksc, flo, F.top, false, pbf, iaf, cblf, n, tauf, ntauf, Ulim, sc, ph, f0, f1);
    if (f1 < 0) return fail();
    PR_MARK(3);
    if (WN_CUT == 3) return fail();

    // ---- 5. window offsets: fine-bucket cursors (exclusive scan of the window counts) ----
    const unsigned wlo = F.lowbits(f0);
    const unsigned whi = f1 + 1 >= F.top ? khi : F.lowbits(f1 + 1);
    int Lw, nbw, base;
    {
        constexpr int KF = W::KF;
        int c[KF], own = 0, bel = 0;
#pragma unroll
        for (int i = 0; i < KF; ++i) {
            const int b = KF * tid + i;
            const int v = (b >= flo && b < F.top) ? (int)cfm[b] : 0;
            c[i] = (b >= f0 && b <= f1) ? v : 0;
            own += c[i];
            bel += b < f0 ? v : 0;
        }
        int inc = own;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) { const int u = __shfl_up_sync(0xffffffffu, inc, o); if (l >= o) inc += u; }
        bel = __reduce_add_sync(0xffffffffu, bel);
        if (l == 31) sc.i[ph][w] = inc;
        if (l == 0) sc.i[ph][WN_NW + w] = bel;
        __syncthreads();
        int tw = sc.i[ph][q16], tb = sc.i[ph][WN_NW + q16];
        ph ^= 1;
        // every lane q16 holds warp q16's totals, 32 / NW copies of each
        const int pw = __reduce_add_sync(0xffffffffu, q16 < w ? tw : 0) / (32 / WN_NW);
        tw = __reduce_add_sync(0xffffffffu, tw) / (32 / WN_NW);
        tb = __reduce_add_sync(0xffffffffu, tb) / (32 / WN_NW);
        Lw = tw;                                   // window keys
        nbw = (int)cblf + tb;                      // keys below the window
        base = nbw > 0 ? 1 : 0;                    // slot 0: the largest key below the window
        PR_NOTE(7, Lw);
        if (Lw + base > WN_LMAX || Lw + base < 1) return fail();
        int run = base + pw + (inc - own);
#pragma unroll
        for (int i = 0; i < KF; ++i) {
            const int b = KF * tid + i;
            if (b >= f0 && b <= f1) cfm[b] = (unsigned)run;
            run += c[i];
        }
    }
    if constexpr (CS > 1) cluster.sync(); else __syncthreads();      // (rank 0's cursors are the cluster's)
    unsigned* cur = CS > 1 ? cluster.map_shared_rank(cfm, 0) : cfm;
    float* grp0 = CS > 1 ? cluster.map_shared_rank(grp, 0) : grp;

    // ---- 6. exact float64 offsets (all keys), window keys grouped by fine bucket ----------
    double pre = 0.0, suf = 0.0;
    unsigned nxb = 0xffffffffu, pvb = 0u;
    // branch-free arithmetic first (independent reciprocal chains of the unrolled keys) ...
#pragma unroll 1
    for (int q = 0; q < nacc; ++q) {
        unsigned kk[KV];
        keyv(q, kk);
#pragma unroll
        for (int j = 0; j < KV; ++j) {
            const unsigned k = kk[j];
            const bool below = k < wlo, above = k >= whi;
            const double md = (double)__uint_as_float(k);
            pre = fma(below ? md : 0.0, md, pre);
            pvb = below ? max(pvb, k) : pvb;
            const double rr = rcp_posf(above ? md : 1.0);
            suf += above ? rr : 0.0;
            nxb = above ? min(nxb, k) : nxb;
        }
    }
    // ... then the (few) window keys into their fine buckets
#pragma unroll 2
    for (int q = 0; q < nacc; ++q) {
        unsigned kk[KV];
        keyv(q, kk);
#pragma unroll
        for (int j = 0; j < KV; ++j) {
            const unsigned k = kk[j];
            if (k >= wlo && k < whi) {
                const unsigned pos = atomicAdd(&cur[F.bucket(k)], 1u);
                grp0[KI(pos)] = __uint_as_float(k);
            }
        }
    }
    {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            pre += __shfl_xor_sync(0xffffffffu, pre, o);
            suf += __shfl_xor_sync(0xffffffffu, suf, o);
        }
        nxb = __reduce_min_sync(0xffffffffu, nxb);
        pvb = __reduce_max_sync(0xffffffffu, pvb);
        if (l == 0) { sc.d[ph][w] = pre; sc.d[ph][WN_NW + w] = suf; sc.u[ph][w] = nxb; sc.u[ph][WN_NW + w] = pvb; }
        __syncthreads();
        pre = sc.d[ph][q16]; suf = sc.d[ph][WN_NW + q16];
        nxb = __reduce_min_sync(0xffffffffu, sc.u[ph][q16]);
        pvb = __reduce_max_sync(0xffffffffu, sc.u[ph][WN_NW + q16]);
        ph ^= 1;
#pragma unroll
        for (int o = WN_NW / 2; o > 0; o >>= 1) {
            pre += __shfl_xor_sync(0xffffffffu, pre, o);
            suf += __shfl_xor_sync(0xffffffffu, suf, o);
        }
    }
    if constexpr (CS > 1) {
        if (tid == 0) { X->pre = pre; X->suf = suf; X->nxb = nxb; X->pvb = pvb; }
        cluster.sync();                            // partials and every CTA's window keys have landed
        if (crank == 0) {
            pre = suf = 0.0;
#pragma unroll
            for (int r = 0; r < CS; ++r) {
                const WnX* xr = cluster.map_shared_rank(X, r);
                pre += xr->pre; suf += xr->suf;
                nxb = min(nxb, xr->nxb); pvb = max(pvb, xr->pvb);
            }
        }
        cluster.sync();                            // rank 0 has read them: the other CTAs are done
        if (crank != 0) return true;
    }
    const double mprev = (double)__uint_as_float(pvb);
    const double nxt = nxb == 0xffffffffu ? (double)INFINITY : (double)__uint_as_float(nxb);
    PR_MARK(4);
    if (WN_CUT == 4) return false;
    // offsets: squares below the list (all keys below but one instance of mprev, the
    // list's first element; its ties stay below), inverses above it
    const double pre_list = base ? pre - mprev * mprev : 0.0;
    const int nb = nbw - base;
    const int Lr = Lw + base;                      // keys of the list

    // ---- 7. rank every window key inside its fine bucket -> sorted list ---------------
    // (every cursor now holds its bucket's end = the next bucket's start; ties by position)
    if (tid == 0 && base) list[KI(0)] = __uint_as_float(pvb);
    for (int p = base + tid; p < Lr; p += NT) {
        const float x = grp[KI(p)];
        const int fb = F.bucket(__float_as_uint(x));
        const int e1 = (int)cfm[fb];
        const int s0 = fb == f0 ? base : (int)cfm[fb - 1];
        int rank = 0;
        for (int q = s0; q < e1; ++q) {
            const float y = grp[KI(q)];
            rank += (y < x) || (y == x && q < p);
        }
        list[KI(s0 + rank)] = x;
    }
    __syncthreads();
    PR_MARK(5);
    if (WN_CUT == 5) return false;

    // ---- 8. exact scan of the list ------------------------------------------------------
    if (tid == 0) S_.run = Best{INFINITY, INFINITY, 0.0, 0.0};
    wn_scan_list<NT, LE>(list, Lr, nb, n, tau, pre_list, suf, nxt, sc, ph, S_);
    PR_MARK(6);
    PR_NOTE(8, 1);
    out.nbelow = nb;
    out.m0 = (double)list[KI(0)];
    return true;
}

// Shared state of sure_win32 (the fields select_win / select_finish use)
template <int NT>
struct WnShared {
    double sh[66 + NT / 32 + 2];
    double tpart[WN_MAXT];
    double tau, totinv;
    Best best[NT / 32];
    Best run;
    double err, ref;
};

// One subband of n = EF * NT keys: load, |r| keys (+ trace error sums), tau,
// select_win, outputs.  Returns false when the bounds leave too many keys.
// Shared memory: keys (KI layout) | counters | scratch | grouped list | sorted list.
template <int NT, int EF, bool GLOBAL, int CS = 1>
__device__ __forceinline__ bool win_band(const Geo& g, const SelArgs<float>& a, int j, int bi, float* keys,
                                         WnShared<NT>& S_, WnX* X = nullptr) {
    typedef float2 C;
    const int tid = threadIdx.x;
    const int n = g.len[j];                                    // == CS * ef * NT
    const int ef = EF > 0 ? EF : n / (CS * NT);                // EF == 0: any subband of a multiple of CS * NT keys
    [[maybe_unused]] const unsigned crank = CS > 1 ? ::cooperative_groups::this_cluster().block_rank() : 0u;
    const long long slice = CS > 1 ? (long long)crank * (ef * NT) : 0;     // this CTA's keys of the subband
    const long long base = (long long)bi * g.N + g.off[j] + slice;
    const long long pj = (long long)bi * g.S + j;
    if (a.tau_in) {
        if (tid == 0) S_.tau = a.tau_in[pj];
    } else {
        for (int i = tid; i < a.ntiles; i += NT) S_.tpart[i] = a.taupart[((long long)bi * a.ntiles + i) * g.S + j];
    }
    const C* rs = a.r + base;
    const C* w0 = a.w0 ? a.w0 + base : nullptr;
    double err = 0.0, ref = 0.0;
    unsigned kmn = 0xffffffffu, kmx = 0u;
    typedef Wn<NT, EF, GLOBAL> W;
    unsigned* cnt = reinterpret_cast<unsigned*>(GLOBAL ? keys : keys + W::SLOT);
    WnScratch<NT / 32>& sc = *reinterpret_cast<WnScratch<NT / 32>*>(cnt + (W::NC + W::NF + 32) * (CS > 1 ? 2 : 1));
    float* grp = reinterpret_cast<float*>(&sc + 1);          // window keys grouped by fine bucket
    float* list = grp + W::LIST;                             // ... sorted
    float* kst = GLOBAL ? a.kA + base : keys;                // where the keys go
    // KV consecutive coefficients per access (KV / 2 16-byte loads), QB accesses in flight; the
    // keys are stored as the matching vector (select_win's layout)
    constexpr int KV = EF == 0 ? 2 : 4, QB = EF >= 8 ? 2 : 1, HV = KV / 2;
    typedef typename std::conditional<KV == 4, float4, float2>::type KVf;
    const float4* rs4 = reinterpret_cast<const float4*>(rs);
    const float4* w04 = reinterpret_cast<const float4*>(w0);
    KVf* kv = reinterpret_cast<KVf*>(kst);
    auto load_keys = [&](int q0) {
        float4 v[QB][HV];
#pragma unroll
        for (int u = 0; u < QB; ++u)
#pragma unroll
            for (int h = 0; h < HV; ++h) v[u][h] = rs4[HV * (tid + (q0 + u) * NT) + h];
#pragma unroll
        for (int u = 0; u < QB; ++u) {
            float m[KV];
#pragma unroll
            for (int h = 0; h < HV; ++h) {
                m[2 * h] = cmag(make_float2(v[u][h].x, v[u][h].y));
                m[2 * h + 1] = cmag(make_float2(v[u][h].z, v[u][h].w));
            }
            KVf mv;
            mv.x = m[0]; mv.y = m[1];
            if constexpr (KV == 4) { mv.z = m[2]; mv.w = m[3]; }
            if constexpr (GLOBAL) __stcg(kv + tid + (q0 + u) * NT, mv);
            else kv[tid + (q0 + u) * NT] = mv;
#pragma unroll
            for (int j = 0; j < KV; ++j) {
                const unsigned k = __float_as_uint(m[j]);
                if (k) kmn = min(kmn, k);
                kmx = max(kmx, k);
            }
        }
        if (w0) {
#pragma unroll
            for (int u = 0; u < QB; ++u)
#pragma unroll
                for (int h = 0; h < HV; ++h) {
                    const float4 wv = w04[HV * (tid + (q0 + u) * NT) + h], rv = v[u][h];
                    const double dx = (double)rv.x - (double)wv.x, dy = (double)rv.y - (double)wv.y;
                    const double ex = (double)rv.z - (double)wv.z, ey = (double)rv.w - (double)wv.w;
                    err += dx * dx + dy * dy;
                    ref += (double)wv.x * (double)wv.x + (double)wv.y * (double)wv.y;
                    err += ex * ex + ey * ey;
                    ref += (double)wv.z * (double)wv.z + (double)wv.w * (double)wv.w;
                }
        }
    };
    if constexpr (EF == 0) {
#pragma unroll 4
        for (int q0 = 0; q0 < ef / KV; q0 += QB) load_keys(q0);
    } else {
#pragma unroll 1
        for (int q0 = 0; q0 < EF / KV; q0 += QB) load_keys(q0);
    }
    __syncthreads();
    if (!a.tau_in && tid == 0) {
        double t = 0.0;
        for (int i = 0; i < a.ntiles; ++i) t += S_.tpart[i];
        S_.tau = t;
    }
    if (w0) {
        const double e2 = block_sum<NT>(err, S_.sh), r2 = block_sum<NT>(ref, S_.sh);
        if (tid == 0) {
            if constexpr (CS > 1) { X->err = e2; X->ref = r2; }    // summed over the cluster by select_win
            else { S_.err = e2; S_.ref = r2; }
        }
    }
    __syncthreads();
    const double tau = fmax(S_.tau, TAU_FLOOR);
#ifdef VDAMP_PHASE_TIMING
    long long* pdbg = (bi < 4096 && crank == 0) ? &g_prune[bi][j][0] : nullptr;
#else
    long long* pdbg = nullptr;
#endif
    PrOut po{0, 0.0};
    if (!select_win<NT, EF, GLOBAL, CS>(n, tau, kst, cnt, grp, list, sc, kmn, kmx, S_, po, pdbg, X, ef)) return false;
    if (CS > 1 && crank != 0) return true;                     // rank 0 holds the result
    select_finish<float, NT, WnShared<NT>>(g, a, j, bi, n, tau, po.nbelow == 0 ? po.m0 : 0.0, w0 != nullptr, S_);
    return true;
}

// fp32 subbands of EF * NT keys (NT = 128 / 256 / 512: 4,096 / 8,192 / 16,384 keys), one
// per CTA, 1024 / NT CTAs per SM.  A subband the bounds cannot settle (heavy ties, diverged or
// degenerate magnitudes) is flagged in a.pflag and sorted fully by the sure_select_flagged
// launch that follows.
template <int NT, int EF, bool GLOBAL = false>
__global__ void __launch_bounds__(NT, NT >= 1024 ? 1 : 1024 / NT) sure_win32(const __grid_constant__ Geo g,
                                                            const __grid_constant__ SelArgs<float> a) {
    pdl_enter();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* keys = reinterpret_cast<float*>(smem_raw);
    __shared__ WnShared<NT> S_;
    const int bi = blockIdx.x, it = blockIdx.y;
    for (int q = a.item_start[it]; q < a.item_start[it + 1]; ++q) {
        const int j = a.item_list[q];
        const bool ok = win_band<NT, EF, GLOBAL>(g, a, j, bi, keys, S_);
        if (threadIdx.x == 0) {
            a.pflag[(long long)bi * g.S + j] = ok ? 0u : 1u;
            // captured run: the flag-scan launch is the body of a conditional node, run only if set
            if (!ok && a.cond) cudaGraphSetConditional((cudaGraphConditionalHandle)a.cond, 1u);
        }
        __syncthreads();
    }
}

// The same selection with one subband of CS * EF * NT keys spread over a thread-block cluster of
// CS CTAs (keys in L2-resident global scratch, histograms merged and partial sums exchanged
// through distributed shared memory; see select_win): for batches with so few subbands of
// >= 16,384 keys that one CTA per subband would leave most SMs idle and put the whole
// subband's latency on one SM (cfg0: 1 image x 3 subbands; cfg3: 1 x 9).  Grid: (CS * B, items),
// cluster dimension (CS, 1, 1) set at launch.  EF == 0: keys per thread = len / (CS * NT) per
// subband, so one launch takes subbands of different sizes.
template <int NT, int EF, int CS>
__global__ void __launch_bounds__(NT, 1) sure_winc(const __grid_constant__ Geo g,
                                                                             const __grid_constant__ SelArgs<float> a) {
    pdl_enter();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* keys = reinterpret_cast<float*>(smem_raw);
    __shared__ WnShared<NT> S_;
    __shared__ WnX X;
    const int bi = blockIdx.x / CS, it = blockIdx.y;
    const unsigned crank = ::cooperative_groups::this_cluster().block_rank();
    for (int q = a.item_start[it]; q < a.item_start[it + 1]; ++q) {
        const int j = a.item_list[q];
        if (q > a.item_start[it]) ::cooperative_groups::this_cluster().sync();     // X and the lists are reused
        const bool ok = win_band<NT, EF, true, CS>(g, a, j, bi, keys, S_, &X);
        if (crank == 0 && threadIdx.x == 0) {
            a.pflag[(long long)bi * g.S + j] = ok ? 0u : 1u;
            if (!ok && a.cond) cudaGraphSetConditional((cudaGraphConditionalHandle)a.cond, 1u);
        }
        __syncthreads();
    }
}

// The full sort for the (rare) subbands sure_win32 flagged in a.only (heavy ties, diverged
// or degenerate magnitudes): a few 512-thread CTAs with sure_win32's shared-memory shape
// scan the flags of all B x nitems (image, single-subband item) pairs; a flagged subband of
// n = 4,096 / 8,192 / 16,384 keys is loaded, bitonic-sorted in place and scanned exactly in
// tiles of 2,048 keys (wn_scan_list).  With nothing flagged the launch costs one pass over
// the flags.
__global__ void __launch_bounds__(512, 1) sure_win_full(const __grid_constant__ Geo g,
                                                        const __grid_constant__ SelArgs<float> a, int B, int nitems) {
    constexpr int NT = 512, LE = Wn<NT>::LE, T = LE * NT;
    typedef float2 C;
    pdl_enter();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* keys = reinterpret_cast<float*>(smem_raw);
    WnScratch<NT / 32>& sc = *reinterpret_cast<WnScratch<NT / 32>*>(keys + Wn<NT, 32>::SLOT);
    __shared__ WnShared<NT> S_;
    __shared__ unsigned wmask[NT / 32];
    const int tid = threadIdx.x;
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
                const int bi = (int)(pp % B), j = a.item_list[a.item_start[(int)(pp / B)]];
                const int n = g.len[j];
                const long long base = (long long)bi * g.N + g.off[j];
                const C* rs = a.r + base;
                const C* w0 = a.w0 ? a.w0 + base : nullptr;
                double err = 0.0, ref = 0.0;
                if (a.tau_in) {
                    if (tid == 0) S_.tau = a.tau_in[(long long)bi * g.S + j];
                } else if (tid == 0) {
                    double t = 0.0;
                    for (int i = 0; i < a.ntiles; ++i) t += a.taupart[((long long)bi * a.ntiles + i) * g.S + j];
                    S_.tau = t;
                }
                for (int e = tid; e < n; e += NT) {
                    const C v = rs[e];
                    keys[KI(e)] = cmag(v);
                    if (w0) {
                        const C wv = w0[e];
                        const double dx = (double)v.x - (double)wv.x, dy = (double)v.y - (double)wv.y;
                        err += dx * dx + dy * dy;
                        ref += (double)wv.x * (double)wv.x + (double)wv.y * (double)wv.y;
                    }
                }
                __syncthreads();
                if (w0) {
                    const double e2 = block_sum<NT>(err, S_.sh), r2 = block_sum<NT>(ref, S_.sh);
                    if (tid == 0) { S_.err = e2; S_.ref = r2; }
                }
                const double tau = fmax(S_.tau, TAU_FLOOR);
                block_sort<float, NT>(keys, n);
                const int ntl = n / T;                         // 2, 4 or 8 tiles
                double* tot = S_.sh;                           // [2][8] tile totals -> offsets
                for (int t = 0; t < ntl; ++t) {
                    double q = 0.0, v = 0.0;
#pragma unroll
                    for (int e = 0; e < LE; ++e) {
                        const double mm = (double)keys[KI(t * T + LE * tid + e)];
                        q = fma(mm, mm, q);
                        if (mm > 0) v += rcp_posf(mm);
                    }
                    q = block_sum<NT>(q, S_.sh + 16);
                    v = block_sum<NT>(v, S_.sh + 16);
                    if (tid == 0) { tot[t] = q; tot[8 + t] = v; }
                }
                if (tid == 0) {
                    double acc = 0.0;
                    for (int t = 0; t < ntl; ++t) { const double q = tot[t]; tot[t] = acc; acc += q; }
                    acc = 0.0;
                    for (int t = ntl - 1; t >= 0; --t) { const double v = tot[8 + t]; tot[8 + t] = acc; acc += v; }
                    S_.run = Best{INFINITY, INFINITY, 0.0, 0.0};
                }
                __syncthreads();
                int ph = 0;
                for (int t = 0; t < ntl; ++t) {
                    const double nf = t + 1 < ntl ? (double)keys[KI((t + 1) * T)] : (double)INFINITY;
                    wn_scan_list<NT, LE>(keys + KI(t * T), T, t * T, n, tau, tot[t], tot[8 + t], nf, sc, ph, S_);
                }
                select_finish<float, NT, WnShared<NT>>(g, a, j, bi, n, tau, (double)keys[0], w0 != nullptr, S_);
                __syncthreads();
            }
        }
        __syncthreads();
    }
}
