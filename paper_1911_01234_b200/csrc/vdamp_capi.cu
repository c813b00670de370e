// C ABI of the VDAMP hot path (include/vdamp_b200.h): plan, workspace,
// launch sequences.  Host code is plain C++ over the CUDA runtime; the
// Python package binds it with ctypes.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "vdamp_b200.h"
#include "vdamp_kernels.cuh"

using namespace vdamp;

namespace {

thread_local std::string g_err;

struct Err {
    int code;
    std::string msg;
};

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e__ = (x);                                                             \
        if (e__ != cudaSuccess)                                                            \
            throw Err{e__ == cudaErrorMemoryAllocation ? VDAMP_ERR_OOM : VDAMP_ERR_CUDA,   \
                      std::string(#x) + ": " + cudaGetErrorString(e__)};                   \
    } while (0)

struct Pass {
    int a, b, k;      // Haar levels a..b handled by one strip kernel
    int Ha, Wa;       // level a-1 image dims
    int logWa;
    int nstrips;
};

struct Plan {
    int H, W, s, B, prec, dev;
    int S;
    long long N;
    Geo geo;
    std::vector<Pass> passes;       // fine -> coarse
    std::vector<int> item_start;    // SURE work items (balanced subband groups)
    std::vector<int> item_list;
    size_t csz;                     // bytes per complex element
    int cw, logcw, ntiles, rowlog;  // column tile width, row_pass rows per CTA
    int nsm = 148;                  // SMs of the device
    // device buffers
    void* r = nullptr;
    void* T1 = nullptr;
    void* T2 = nullptr;
    void* yg = nullptr;
    void* pinv = nullptr;
    std::vector<void*> scratch;     // per pass p >= 1: level a_p - 1 approx image
    double* par = nullptr;          // [B][S][3]
    double* parf = nullptr;
    double* taupart = nullptr;      // [B][ntiles][S]
    double* prow = nullptr;         // [2s][H]
    double* pcol = nullptr;         // [2s][W]
    void* prs256 = nullptr;         // H = 256: row profiles [256][npp] in the working precision
    double* nvar = nullptr;         // [B]
    long long* offs = nullptr;      // [B+1] measurement offsets
    void* twH = nullptr;
    void* twW = nullptr;
    // fp32 subbands > SCAP: value-range split over several CTAs (big_keys / big_range)
    bool bigpath = false;
    bool t2_alias = false;          // T2 is T1 (K2 in place)
    bool cluster = false;           // few subbands of >= 16,384 keys: one thread-block cluster per subband (sure_winc)
    bool cluster16 = false;         // ... of 16 CTAs for subbands of >= 131,072 keys (non-portable size, if schedulable)
    cudaStream_t side2 = nullptr;   // second fork/join stream (cluster mode: mid-size subbands)
    cudaEvent_t ev_join2 = nullptr;
    std::vector<int> large;         // subband ids
    int big_ranges = 0, big_chunks = 0;
    unsigned* bhist = nullptr;      // [B][nlarge][BIGB]
    unsigned* btick = nullptr;      // [B][nlarge]
    double* bbest = nullptr;        // [B][nlarge][ranges][4]
    double* baux = nullptr;         // [B][nlarge][2]
    double* berrp = nullptr;        // [B][nlarge][chunks][2]
    void* kA = nullptr;             // sort scratch (large subbands only)
    void* kB = nullptr;
    void* x0 = nullptr;             // ground truth image (owned copy)
    void* w0 = nullptr;             // dwt(x0)
    void* xtmp = nullptr;           // per-iteration finalize image (NMSE, direct path)
    void* x0r = nullptr;            // raw unitary FFT2 of s_in * x0 (Parseval NMSE)
    double* nmconst = nullptr;      // [B][2]: mask error constant, |x0|^2
    double* nmpart = nullptr;       // [B][ntiles]
    bool parseval = true;           // per-iteration NMSE by Parseval (one forward FFT)
    // bound-pruned exact SURE selection (vdamp_prune.cuh), bit 0: subbands of 4,096..16,384
    // keys, bit 1: larger ones (keys in global scratch).  fp64 keys: both (2x faster than
    // their bitonic / global sorts); fp32 keys: large only (the shared-memory counting sort
    // measured faster for <= 16,384 keys: 3.46 vs 3.89 ms/step cfg1).  VDAMP_PRUNE=mask
    int prune = 0;
    void* what = nullptr;           // baselines: w_hat state [B][N]
    double* btau = nullptr;         // baselines: [B][S] oracle tau
    double* berr = nullptr;         // baselines: [B][S][2] coefficient errors
    double* trtmp = nullptr;        // [B][S][TRACE_F]
    unsigned* pflag = nullptr;      // [B][S] sure_prune32 fallback flags
    // per-iteration device times (vdamp_set_iteration_timing): events around K1..K4 of
    // every iteration on the first lane's stream; images sharing that stream
    bool iter_timing = false;
    std::vector<cudaEvent_t> itev;
    int it_images = 0, it_count = 0;
    cudaStream_t side = nullptr;    // fork/join stream for the small-subband SURE kernel
    // CUDA graph of the whole vdamp_run sequence, re-captured when its key changes
    bool graphs = true;
    bool interleave = true;          // lanes launched iteration-major (VDAMP_INTERLEAVE=0: lane-major)
    cudaGraphExec_t gexec = nullptr;
    std::vector<const void*> gkey;
    long long g_launches = 0;
    long long g_cls[VDAMP_KERNEL_CLASSES] = {0};
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> gev;   // timing events inside the graph
    // graphs of other keys seen recently (a pipelined caller alternates output buffers):
    // parked instead of destroyed, at most GRAPH_PARK of them
    struct GraphSlot {
        cudaGraphExec_t gexec;
        std::vector<const void*> gkey;
        long long g_launches;
        long long g_cls[VDAMP_KERNEL_CLASSES];
        std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> gev;
    };
    std::vector<GraphSlot> gpark;
    cudaStream_t gstream = nullptr; // capture/launch stream when the caller passes the legacy default stream
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // image lanes: vdamp_run runs the batch as `lanes` contiguous image ranges on
    // their own streams, so one lane's latency-bound SURE tail overlaps the FFT
    // kernels of the others; diagnostics ride on the lanes when interleaved
    int lanes = 1;
    int Ball = 0;                    // images of the whole plan (a lane view's B is its own range)
    struct Lane {
        cudaStream_t st = nullptr, side = nullptr, side2 = nullptr;
        cudaEvent_t fork = nullptr, join = nullptr, join2 = nullptr, done = nullptr;
        cudaEvent_t nm0 = nullptr, nmr = nullptr, nmd = nullptr;
    };
    // per-iteration NMSE beside the next iteration (Seq::nmse_iter): events "thresholds ready",
    // "r consumed", "record written"; nm_pending: an NMSE pass is in flight on the side stream
    cudaEvent_t ev_nm0 = nullptr, ev_nmr = nullptr, ev_nmd = nullptr;
    bool nm_pending = false;
    bool nm_overlap = true;          // VDAMP_NMSE_OVERLAP=0: NMSE passes in line, on the iteration's stream
    std::vector<Lane> lane;
    cudaEvent_t lane_start = nullptr;
    bool have_meas = false;
    bool have_gt = false;
    // measurement validation (scatter_measurements flags, sticky until reported):
    // device word, its pinned host copy and the event after the copy
    unsigned* d_merr = nullptr;
    unsigned* h_merr = nullptr;     // mapped pinned host word
    unsigned* h_merr_dev = nullptr; // its device alias
    cudaEvent_t ev_meas = nullptr;
    bool meas_pending = false;
    bool validate_sync = true;      // vdamp_set_validation
    // pinned staging of the per-call host arrays (noise variances, offsets), two
    // slots so a call never overwrites a slot whose copy may still be queued
    double* h_stage[2] = {nullptr, nullptr};
    cudaEvent_t ev_stage[2] = {nullptr, nullptr};
    int stage_k = 0;
    size_t bytes = 0;
    long long launches = 0;
    // timing
    bool timing = false;
    cudaError_t pend = cudaSuccess;   // first launch error, raised by dispatch()
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev;
    double ms[VDAMP_KERNEL_CLASSES] = {0};
    long long cls_launches[VDAMP_KERNEL_CLASSES] = {0};
};

void* dalloc(Plan* p, size_t n) {
    void* ptr = nullptr;
    if (n == 0) return nullptr;
    CK(cudaMalloc(&ptr, n));
    p->bytes += n;
    return ptr;
}

// padded smem element count of a row buffer of n elements (SP layout)
size_t SPN(long long n) { return (size_t)(n + (n >> 4) + 1); }

int ilog2(long long v) { int l = 0; while ((1LL << l) < v) ++l; return l; }
bool pow2(long long v) { return v > 0 && (v & (v - 1)) == 0; }

// ---------------------------------------------------------------- launch --
// event record that also works inside stream capture (a real record node)
inline cudaError_t record(cudaEvent_t e, cudaStream_t s) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cs);
    return cs == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal)
                                               : cudaEventRecord(e, s);
}

// NVTX ranges (env VDAMP_NVTX=1): one per kernel launch, named by kernel class, and
// one per vdamp_run / iteration -- host-side launch ranges for nsys/ncu timelines
static bool nvtx_enabled() {
    static const bool on = [] { const char* e = getenv("VDAMP_NVTX"); return e && atoi(e) != 0; }();
    return on;
}
static const char* const kClassNames[VDAMP_KERNEL_CLASSES] = {
    "K1 synthesis+row FFT", "K2 column FFT/residual/tau", "K3 row IFFT+analysis", "K4 SURE select",
    "finalize", "other"};
struct NvtxRange {
    bool on;
    explicit NvtxRange(const char* name) : on(nvtx_enabled()) { if (on) nvtxRangePushA(name); }
    ~NvtxRange() { if (on) nvtxRangePop(); }
};

struct Launch {
    Plan* p;
    int cls;
    cudaStream_t st;
    cudaEvent_t e0 = nullptr;
    NvtxRange nv;
    Launch(Plan* p_, int c, cudaStream_t s) : p(p_), cls(c), st(s), nv(kClassNames[c]) {
        if (p->timing) {
            cudaEvent_t e1;
            CK(cudaEventCreate(&e0));
            CK(cudaEventCreate(&e1));
            CK(record(e0, st));
            p->ev.push_back({cls, {e0, e1}});
        }
    }
    ~Launch() {
        p->launches++;
        p->cls_launches[cls]++;
        if (p->timing) record(p->ev.back().second.second, st);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess && p->pend == cudaSuccess) p->pend = e;
    }
};

// Launch with programmatic dependent launch (PDL): the kernel may start while
// the previous kernel in the stream drains; every PDL kernel executes
// griddepcontrol.wait before its first global memory access, so ordering and
// visibility are those of a plain stream launch.  Off via VDAMP_PDL=0.
static bool pdl_enabled() {
    static const bool on = [] { const char* e = getenv("VDAMP_PDL"); return !(e && atoi(e) == 0); }();
    return on;
}

// Shared-memory carve-out preference of the per-iteration kernels, in percent of the SM's
// unified L1 / shared storage (VDAMP_CARVEOUT; -1 leaves the driver's per-kernel choice).
// Kernels of different lanes and of the side streams run side by side on one SM only while
// they agree on its carve-out; a CTA that needs another split waits for the SM to drain.
// One common preference for all of them removes those drains.
int carveout_pref() {
    static const int v = [] { const char* e = getenv("VDAMP_CARVEOUT"); return e ? atoi(e) : -1; }();
    return v;
}

template <typename K>
void prefer_carveout(K kern) {
    const int v = carveout_pref();
    if (v < 0) return;
    static thread_local std::vector<const void*> done;
    const void* key = reinterpret_cast<const void*>(kern);
    for (const void* d : done) if (d == key) return;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, v > 100 ? 100 : v));
    done.push_back(key);
}

template <typename... KArgs, typename... Args>
void launch(void (*k)(KArgs...), dim3 grid, dim3 block, size_t sm, cudaStream_t st, Args... args) {
    prefer_carveout(k);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = sm;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    CK(cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...));
}

// The same with a thread-block cluster of `cs` CTAs along x (cs > 8: the kernel must have been
// opted into non-portable cluster sizes)
template <typename... KArgs, typename... Args>
void launch_cluster(void (*k)(KArgs...), int cs, dim3 grid, dim3 block, size_t sm, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = sm;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    CK(cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...));
}

// Opt every kernel into the dynamic shared memory it is launched with (static
// shared memory counts against the default 48 KB too), once per kernel/size.
// add the elapsed times of recorded event pairs to the per-class totals
void accumulate(Plan* p, std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>>& ev, bool destroy) {
    for (auto& e : ev) {
        CK(cudaEventSynchronize(e.second.second));
        float t = 0;
        CK(cudaEventElapsedTime(&t, e.second.first, e.second.second));
        p->ms[e.first] += t;
        if (destroy) { cudaEventDestroy(e.second.first); cudaEventDestroy(e.second.second); }
    }
    if (destroy) ev.clear();
}

constexpr size_t GRAPH_PARK = 3;

// destroys the current graph only
void drop_current_graph(Plan* p) {
    if (p->gexec) cudaGraphExecDestroy(p->gexec);
    p->gexec = nullptr;
    p->gkey.clear();
    for (auto& e : p->gev) { cudaEventDestroy(e.second.first); cudaEventDestroy(e.second.second); }
    p->gev.clear();
}

// destroys every graph of the plan (anything baked into them changed)
void drop_graph(Plan* p) {
    drop_current_graph(p);
    for (auto& g : p->gpark) {
        if (g.gexec) cudaGraphExecDestroy(g.gexec);
        for (auto& e : g.gev) { cudaEventDestroy(e.second.first); cudaEventDestroy(e.second.second); }
    }
    p->gpark.clear();
}

// The current graph does not match `key`: park it (oldest parked one destroyed beyond
// GRAPH_PARK) and make a parked graph of that key current if there is one.
bool switch_graph(Plan* p, const std::vector<const void*>& key) {
    if (p->gexec) {
        Plan::GraphSlot g;
        g.gexec = p->gexec;
        g.gkey = p->gkey;
        g.g_launches = p->g_launches;
        for (int c = 0; c < VDAMP_KERNEL_CLASSES; ++c) g.g_cls[c] = p->g_cls[c];
        g.gev.swap(p->gev);
        p->gexec = nullptr;
        p->gkey.clear();
        p->gpark.push_back(std::move(g));
    }
    for (size_t i = 0; i < p->gpark.size(); ++i) {
        if (p->gpark[i].gkey != key) continue;
        Plan::GraphSlot g = std::move(p->gpark[i]);
        p->gpark.erase(p->gpark.begin() + (long)i);
        p->gexec = g.gexec;
        p->gkey = g.gkey;
        p->g_launches = g.g_launches;
        for (int c = 0; c < VDAMP_KERNEL_CLASSES; ++c) p->g_cls[c] = g.g_cls[c];
        p->gev.swap(g.gev);
        return true;
    }
    while (p->gpark.size() > GRAPH_PARK) {
        Plan::GraphSlot& g = p->gpark.front();
        if (g.gexec) cudaGraphExecDestroy(g.gexec);
        for (auto& e : g.gev) { cudaEventDestroy(e.second.first); cudaEventDestroy(e.second.second); }
        p->gpark.erase(p->gpark.begin());
    }
    return false;
}

template <typename K>
void set_smem(K kern, size_t bytes) {
    static thread_local std::vector<std::pair<const void*, size_t>> done;
    const void* key = reinterpret_cast<const void*>(kern);
    for (auto& d : done)
        if (d.first == key && d.second >= bytes) return;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    for (auto& d : done)
        if (d.first == key) { d.second = bytes; return; }
    done.push_back({key, bytes});
}

// ------------------------------------------------------------ sequences --
template <typename R>
struct Seq {
    typedef typename CT<R>::T C;
    typedef R Rt;
    Plan* p;
    cudaStream_t st;
    cudaStream_t& st_ = st;
    C* r() { return (C*)p->r; }

    // 256-wide rows in 16-row strips: the register row-FFT kernels (F256)
    // (VDAMP_F256=0 falls back to the generic shared-memory FFT kernels, for A/B runs)
    static bool f256_on() {
        static const bool on = [] { const char* e = getenv("VDAMP_F256"); return !(e && atoi(e) == 0); }();
        return on;
    }
    bool f256(const Pass& ps) const { return f256_on() && p->W == 256 && ps.Wa == 256 && ps.k == 4; }
    bool c256() const { return f256_on() && p->H == 256 && p->cw == 16; }
    bool f512(const Pass& ps) const { return f256_on() && p->W == 512 && ps.Wa == 512 && ps.k == 3; }
    bool c512() const { return f256_on() && p->H == 512 && p->cw == 8; }

    // Haar synthesis of coefficients `coef` with params `par`; FFT -> T1 when
    // rowfft, else the image goes to `img`.
    // early: coef was written at least two kernels before this synthesis (not by
    // the immediately preceding kernel), so synth256 may read it before its PDL wait
    void synth(const C* coef, const double* par, bool rowfft, C* img, int cls, bool early = false, C* t1 = nullptr) {
        const int P = (int)p->passes.size();
        for (int i = P - 1; i >= 0; --i) {
            const Pass& ps = p->passes[i];
            SynArgs<R> a;
            a.coef = coef; a.par = par;
            a.asrc = (i == P - 1) ? nullptr : (const C*)p->scratch[i + 1];
            a.asrc_bs = (i == P - 1) ? 0 : (long long)(p->H >> ps.b) * (p->W >> ps.b);
            a.a = ps.a; a.b = ps.b; a.k = ps.k; a.Wa = ps.Wa; a.logWa = ps.logWa;
            a.tw = (const C*)p->twW;
            const bool last = (i == 0);
            a.dst = last ? (rowfft ? (t1 ? t1 : (C*)p->T1) : img) : (C*)p->scratch[i];
            a.dst_bs = (long long)ps.Ha * ps.Wa;
            dim3 grid(ps.nstrips, p->B);
            const size_t sm = (size_t)SPN(ps.Wa << ps.k) * sizeof(C);
            Launch L(p, cls, st);
            a.early = 0;
            if (last && rowfft && f256(ps)) {
                a.early = early ? 1 : 0;
                const size_t sme = sm;                             // coefficients land in the pixel buffer
                auto k = synth256<R>;
                set_smem(k, sme);
                launch(k, grid, PNT, sme, st, p->geo, a);
            } else if (last && rowfft && f512(ps)) {
                a.early = early ? 1 : 0;
                auto k = synth512<R>;
                set_smem(k, sm);
                launch(k, grid, PNT, sm, st, p->geo, a);
            } else if (last && rowfft) {
                auto k = synth_pass<R, SYN_ROWFFT>;
                const size_t smf = sm + (size_t)p->W * sizeof(C);
                set_smem(k, smf);
                launch(k, grid, PNT, smf, st, p->geo, a);
            } else {
                auto k = synth_pass<R, SYN_PLAIN>;
                set_smem(k, sm);
                launch(k, grid, PNT, sm, st, p->geo, a);
            }
        }
    }

    // Haar analysis; input T2 (row IFFT first) when rowifft, else image `img`.
    // vdamp: coef = Onsager(coef; par) + analysis (in place).
    void analysis(const C* img, bool rowifft, C* coef, const double* par, bool vdamp_mode, int cls) {
        const int P = (int)p->passes.size();
        for (int i = 0; i < P; ++i) {
            const Pass& ps = p->passes[i];
            AnaArgs<R> a;
            const bool first = (i == 0);
            a.src = first ? (rowifft ? (const C*)p->T2 : img) : (const C*)p->scratch[i];
            a.src_bs = (long long)ps.Ha * ps.Wa;
            a.coef = coef; a.par = par;
            a.adst = (i == P - 1) ? nullptr : (C*)p->scratch[i + 1];
            a.adst_bs = (i == P - 1) ? 0 : (long long)(p->H >> ps.b) * (p->W >> ps.b);
            a.a = ps.a; a.b = ps.b; a.k = ps.k; a.Wa = ps.Wa; a.logWa = ps.logWa;
            a.tw = (const C*)p->twW;
            dim3 grid(ps.nstrips, p->B);
            size_t sm = (size_t)SPN(ps.Wa << ps.k) * sizeof(C);
            Launch L(p, cls, st);
            if (first && rowifft && f256(ps)) {
                if (vdamp_mode) {
                    if (ANA256_TMA) sm += 4096 * sizeof(C) + 16;        // old-coefficient landing zone
                    auto k = analysis256<R, ANA_OUT_VDAMP>; set_smem(k, sm);
                    launch(k, grid, PNT, sm, st, p->geo, a);
                } else {
                    auto k = analysis256<R, ANA_OUT_COEF>; set_smem(k, sm);
                    launch(k, grid, PNT, sm, st, p->geo, a);
                }
            } else if (first && rowifft && f512(ps)) {
                if (vdamp_mode) {
                    sm += 4096 * sizeof(C) + 16;                   // old-coefficient landing zone
                    auto k = analysis512<R, ANA_OUT_VDAMP>; set_smem(k, sm);
                    launch(k, grid, PNT, sm, st, p->geo, a);
                } else {
                    auto k = analysis512<R, ANA_OUT_COEF>; set_smem(k, sm);
                    launch(k, grid, PNT, sm, st, p->geo, a);
                }
            } else if (first && rowifft) {
                sm += (size_t)p->W * sizeof(C);
                if (vdamp_mode) {
                    auto k = analysis_pass<R, ANA_IN_ROWIFFT, ANA_OUT_VDAMP>; set_smem(k, sm);
                    launch(k, grid, PNT, sm, st, p->geo, a);
                } else {
                    auto k = analysis_pass<R, ANA_IN_ROWIFFT, ANA_OUT_COEF>; set_smem(k, sm);
                    launch(k, grid, PNT, sm, st, p->geo, a);
                }
            } else {
                if (vdamp_mode) {
                    auto k = analysis_pass<R, ANA_IN_PLAIN, ANA_OUT_VDAMP>; set_smem(k, sm);
                    launch(k, grid, PNT, sm, st, p->geo, a);
                } else {
                    auto k = analysis_pass<R, ANA_IN_PLAIN, ANA_OUT_COEF>; set_smem(k, sm);
                    launch(k, grid, PNT, sm, st, p->geo, a);
                }
            }
        }
    }

    size_t col_smem() const {
        // tile buffer + twiddles; the tau partials and row profiles reuse the tile
        // buffer after the outputs are stored (the NMSE mode's block sum sits past the twiddles)
        const int np = 2 * p->s;
        const size_t E = (size_t)p->H << p->logcw;
        const size_t tau = (size_t)np * PNT * sizeof(double) + (size_t)np * p->cw * sizeof(double) +
                           (size_t)np * p->H * sizeof(R);
        return std::max(E * sizeof(C), tau) + (size_t)p->H * sizeof(C) + (PNT / 32 + 2) * sizeof(double);
    }

    void col(int mode, const C* src, C* dst, int cls) {
        ColArgs<R> a;
        a.src = src; a.dst = dst;
        a.yg = (const C*)p->yg; a.pinv = (const R*)p->pinv; a.noise_var = p->nvar;
        a.prow = p->prow; a.pcol = p->pcol; a.taupart = p->taupart;
        a.tw = (const C*)p->twH; a.cw = p->cw; a.logcw = p->logcw; a.ntiles = p->ntiles;
        a.x0r = (const C*)p->x0r; a.nmsepart = p->nmpart;
        a.prs256 = (const R*)p->prs256;
        dim3 grid(p->ntiles, p->B);
        Launch L(p, cls, st);
        if (c512() && (mode == COL_VDAMP || mode == COL_FINAL || mode == COL_NMSE)) {
            const int np = 2 * p->s, npp = (np + 3) & ~3;
            const size_t sm = (size_t)col512_region0<R>(np) + (size_t)512 * npp * sizeof(R) + (size_t)np * 8 * sizeof(double);
            switch (mode) {
                case COL_VDAMP: { auto k = col_pass512<R, COL_VDAMP>; set_smem(k, sm); launch(k, grid, PNT, sm, st, p->geo, a); break; }
                case COL_NMSE:  { auto k = col_pass512<R, COL_NMSE>;  set_smem(k, sm); launch(k, grid, PNT, sm, st, p->geo, a); break; }
                default:        { auto k = col_pass512<R, COL_FINAL>; set_smem(k, sm); launch(k, grid, PNT, sm, st, p->geo, a); break; }
            }
            return;
        }
        if (c256() && (mode == COL_VDAMP || mode == COL_FINAL || mode == COL_NMSE)) {
            const int np = 2 * p->s, npp = (np + 3) & ~3;
            // transpose tile | row profiles | column profiles | tau partials [np][PNT]
            const size_t sm = (size_t)col256_region0<R>(np) + (size_t)256 * npp * sizeof(R) +
                              (size_t)np * 16 * sizeof(double) + (size_t)np * PNT * sizeof(double);
            switch (mode) {
                case COL_VDAMP: { auto k = col_pass256<R, COL_VDAMP>; set_smem(k, sm); launch(k, grid, PNT, sm, st, p->geo, a); break; }
                case COL_NMSE:  { auto k = col_pass256<R, COL_NMSE>;  set_smem(k, sm); launch(k, grid, PNT, sm, st, p->geo, a); break; }
                default:        { auto k = col_pass256<R, COL_FINAL>; set_smem(k, sm); launch(k, grid, PNT, sm, st, p->geo, a); break; }
            }
            return;
        }
        const size_t sm = col_smem();
        switch (mode) {
            case COL_FWD:   { auto k = col_pass<R, COL_FWD>;   set_smem(k, sm); launch(k, grid, PNT, sm, st, p->geo, a); break; }
            case COL_INV:   { auto k = col_pass<R, COL_INV>;   set_smem(k, sm); launch(k, grid, PNT, sm, st, p->geo, a); break; }
            case COL_VDAMP: { auto k = col_pass<R, COL_VDAMP>; set_smem(k, sm); launch(k, grid, PNT, sm, st, p->geo, a); break; }
            case COL_RAW:   { auto k = col_pass<R, COL_RAW>;   set_smem(k, sm); launch(k, grid, PNT, sm, st, p->geo, a); break; }
            case COL_NMSE:  { auto k = col_pass<R, COL_NMSE>;  set_smem(k, sm); launch(k, grid, PNT, sm, st, p->geo, a); break; }
            default:        { auto k = col_pass<R, COL_FINAL>; set_smem(k, sm); launch(k, grid, PNT, sm, st, p->geo, a); break; }
        }
    }

    template <bool INV, bool PRE, bool POST>
    void rows(const C* src, C* dst, int cls) {
        dim3 grid(p->H >> p->rowlog, p->B);
        const size_t sm = (size_t)SPN(p->W << p->rowlog) * sizeof(C) + (size_t)p->W * sizeof(C);
        auto k = row_pass<R, INV, PRE, POST>;
        set_smem(k, sm);
        Launch L(p, cls, st);
        k<<<grid, PNT, sm, st>>>(p->geo, src, dst, (const C*)p->twW, p->rowlog);
    }

    void select(const C* rr, const double* tau_in, double* trace, bool use_w0, bool onsager_par = true) {
        SelArgs<R> a;
        a.r = rr; a.taupart = p->taupart; a.tau_in = tau_in; a.ntiles = p->ntiles;
        a.par = onsager_par ? p->par : nullptr; a.parf = p->parf; a.trace = trace;
        a.w0 = use_w0 ? (const C*)p->w0 : nullptr;
        a.kA = (R*)p->kA; a.kB = (R*)p->kB;
        a.prune = p->prune;
        a.cond = 0;
        // Captured run (CUDA graph), optional: the flag-scan launch after the sure_win32 kernels becomes
        // the body of a conditional IF node whose handle the flagging kernels set, so a run in which
        // nothing is flagged (the normal case) does not pay that launch between K4 and the next K1.
        cudaGraph_t cgraph = nullptr;
        if constexpr (std::is_same<R, float>::value) {
            // Measured on cfg1: one batch at a time 557k -> 580k img-iter/s (device-resident) and 437k ->
            // 451k (synchronous calls), but back-to-back graph launches of the streaming API 538k -> 531k
            // (graphs with conditional nodes start later behind one another), 16 / 32 images 284k ->
            // 275k / 425k -> 411k, one image 16.4k -> 15.3k.  Off unless VDAMP_CONDNODE=1.
            static const int condenv = [] { const char* e = getenv("VDAMP_CONDNODE"); return e ? atoi(e) : 0; }();
            const bool condon = condenv != 0;
            cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
            if (condon && !p->timing && cudaStreamIsCapturing(st_, &cst) == cudaSuccess && cst == cudaStreamCaptureStatusActive) {
                unsigned long long cid = 0;
                const cudaGraphNode_t* deps = nullptr;
                size_t nd = 0;
                CK(cudaStreamGetCaptureInfo(st_, &cst, &cid, &cgraph, &deps, &nd));
                cudaGraphConditionalHandle h;
                CK(cudaGraphConditionalHandleCreate(&h, cgraph, 0, cudaGraphCondAssignDefault));
                a.cond = (unsigned long long)h;
            }
        }
        // big subbands: 1024-thread CTAs with the full sort workspace; small ones:
        // 128-thread CTAs with little shared memory, many per SM
        // the small-subband kernel runs on a side stream, concurrently with the
        // big one (its CTAs fill the SMs the big kernel's tail leaves idle)
        bool forked = false, forked2 = false;
        std::vector<int> win_items, win_large;     // subbands taken by sure_win32 (fp32): shared / global keys
        if constexpr (std::is_same<R, float>::value) {
            if (p->bigpath) {
                // subbands > SCAP: keys + histogram, then value ranges over several CTAs
                BigArgs b;
                b.nlarge = (int)p->large.size(); b.ranges = p->big_ranges; b.chunks = p->big_chunks;
                for (int i = 0; i < b.nlarge; ++i) b.list[i] = p->large[i];
                b.hist = p->bhist; b.tick = p->btick; b.best = p->bbest; b.aux = p->baux; b.errp = p->berrp;
                {
                    Launch L(p, 3, st_);
                    const size_t sm = (size_t)BIGB * sizeof(unsigned);
                    set_smem(big_keys, sm);
                    launch(big_keys, dim3(b.chunks, b.nlarge, p->B), 1024, sm, st_, p->geo, a, b);
                }

                {
                    Launch L(p, 3, st_);
                    const size_t slot16 = ((size_t)SCAP + SCAP / 32 + 2 + 3) & ~(size_t)3;
                    const size_t sm = 2 * slot16 * sizeof(float) + CS_WORDS * sizeof(unsigned);
                    set_smem(big_range, sm);
                    launch(big_range, dim3(b.ranges, b.nlarge, p->B), 1024, sm, st_, p->geo, a, b);
                }
            }
        }
        // the small-subband kernel is launched first (on the side stream) so its CTAs take
        // SMs before the big kernel's 200 KB CTAs do: 411k vs 399k img-iter/s (cfg1).  With
        // per-launch timing on, both run on the caller's stream (clean per-kernel times).
        a.pflag = p->pflag;
        a.only = nullptr;
        auto set_items = [&](const std::vector<int>& li) {
            a.item_start[0] = 0;
            for (size_t i = 0; i < li.size(); ++i) { a.item_start[i + 1] = (int)i + 1; a.item_list[i] = li[i]; }
        };
        for (int big = 0; big < 2; ++big) {
            std::vector<int> li;
            for (int j = 0; j < p->S; ++j)
                if ((p->geo.len[j] > SMALL_N) == (big == 1) && !(p->bigpath && p->geo.len[j] > SCAP)) li.push_back(j);
            // longest items first (grid is image-fastest, so they are all scheduled first)
            std::stable_sort(li.begin(), li.end(), [&](int x, int y) { return p->geo.len[x] > p->geo.len[y]; });
            if (li.empty()) continue;
            cudaStream_t ls = st_;
            if (!big && p->side && !p->timing && p->B * li.size() >= 64) {
                CK(cudaEventRecord(p->ev_fork, st_));
                CK(cudaStreamWaitEvent(p->side, p->ev_fork, 0));
                ls = p->side;
                forked = true;
            }
            if (!big) {
                set_items(li);
                Launch L(p, 3, ls);
                const size_t sm = (size_t)(SMALL_N + SMALL_N / 32 + 2) * sizeof(R);
                auto k = sure_select<R, SNT_SMALL>;
                set_smem(k, sm);
                launch(k, dim3(p->B, (unsigned)li.size()), SNT_SMALL, sm, ls, p->geo, a);
                continue;
            }
            const int cap = Scap<R>::v;
            const size_t slot16 = ((size_t)cap + cap / 32 + 2 + 3) & ~(size_t)3;   // kernel's SLOT
            int pm = p->prune;
            auto launch_big = [&](const std::vector<int>& items) {
                set_items(items);
                Launch L(p, 3, ls);
                const size_t slots = (size_t)(cap + cap / 32 + 1) + 1;
                size_t sm = sizeof(R) == 4 ? 2 * slot16 * sizeof(R) + CS_WORDS * sizeof(unsigned) : slots * sizeof(R);
                // large subbands: global counting sort counters + ranking tile
                const size_t gcs = sizeof(R) == 4 ? 32768 * 4 + 16384 * sizeof(R) : 8192 * 4 + 8192 * sizeof(R);
                if (sm < gcs) sm = gcs;
                // fp64 pruned path: keys | counters | bucket ids | reduction scratch + list (vdamp_prune.cuh)
                const size_t smp = slot16 * sizeof(R) + (PR_NC + PR_NF + 32) * 4 + (size_t)PR_BIDN * 2 +
                                   (5 * 32 + 8) * 8 + ((size_t)pr_lmax<R>() + pr_lmax<R>() / 32 + 8) * sizeof(R);
                if (sizeof(R) == 8 && pm && sm < smp) sm = smp;
                constexpr int BNT = sizeof(R) == 4 ? BNT32 : BNT64;
                auto k = pm == 0 ? sure_select<R, BNT, 0>
                       : pm == 1 ? sure_select<R, BNT, 1>
                       : pm == 2 ? sure_select<R, BNT, 2> : sure_select<R, BNT, 3>;
                set_smem(k, sm);
                launch(k, dim3(p->B, (unsigned)items.size()), BNT, sm, ls, p->geo, a);
            };
            // fp32 subbands of 4,096 / 8,192 / 16,384 keys: sure_win32 (vdamp_win.cuh), one subband
            // per CTA of 32 keys per thread (16 / 8 for the CTA shapes of small batches)
            if constexpr (std::is_same<R, float>::value) {
                if ((pm & 1) && p->ntiles <= WN_MAXT) {
                    // lp: keys in shared memory; lg: 32,768 .. 131,072 keys in L2-resident global
                    // scratch (1024-thread CTAs); lr: the rest (sure_select)
                    std::vector<int> lp, lg, lr, lc;
                    for (int j : li) {
                        const int n = p->geo.len[j];
                        if (p->cluster && p->kA && n >= 16384 && n <= (1 << 20) && (n & (n - 1)) == 0) lc.push_back(j);
                        else if (n == 16384 || n == 8192 || n == 4096) lp.push_back(j);
                        else if ((pm & 2) && p->kA && (n == 32768 || n == 65536 || n == 131072)) lg.push_back(j);
                        else lr.push_back(j);
                    }
                    static const int nt4 = [] { const char* e = getenv("VDAMP_WIN4"); return e ? atoi(e) : 256; }();
                    static const int wside = [] { const char* e = getenv("VDAMP_WINSIDE"); return e ? atoi(e) : 1; }();
                    const bool can_fork = wside && p->side && !p->timing && !lp.empty();
                    auto fork = [&] {
                        if (!forked) {
                            CK(cudaEventRecord(p->ev_fork, st_));
                            CK(cudaStreamWaitEvent(p->side, p->ev_fork, 0));
                            forked = true;
                        }
                    };
                    // larger subbands first (one long-running 1024-thread CTA each): the other
                    // sure_win32 launches then run beside them on the side stream
                    const bool has_large = !lr.empty() || !lg.empty() || !lc.empty();
                    if (has_large && can_fork) fork();
                    // clusters: subbands of >= 131,072 keys on 16 CTAs each (this stream), the others
                    // on 8 CTAs each (second side stream), one launch per cluster size
                    int lcmax = 0;
                    for (int j : lc) lcmax = std::max(lcmax, p->geo.len[j]);
                    if (!lc.empty() && lcmax <= 32768) {
                        // only 16,384 / 32,768-key subbands (cfg0): 512-thread CTAs with the smaller
                        // histograms (28 vs 53 us per launch for 16,384 keys)
                        for (int n : {32768, 16384}) {
                            std::vector<int> ln;
                            for (int j : lc) if (p->geo.len[j] == n) ln.push_back(j);
                            if (ln.empty()) continue;
                            set_items(ln);
                            Launch L(p, 3, ls);
                            const dim3 grid(8u * (unsigned)p->B, (unsigned)ln.size());
                            if (n == 32768) {
                                auto k = sure_winc<512, 8, 8>;
                                set_smem(k, wn_smem_bytes<512, 8, true, 8>());
                                launch_cluster(k, 8, grid, 512, wn_smem_bytes<512, 8, true, 8>(), ls, p->geo, a);
                            } else {
                                auto k = sure_winc<512, 4, 8>;
                                set_smem(k, wn_smem_bytes<512, 4, true, 8>());
                                launch_cluster(k, 8, grid, 512, wn_smem_bytes<512, 4, true, 8>(), ls, p->geo, a);
                            }
                        }
                        for (int j : lc) (p->geo.len[j] > 16384 ? win_large : win_items).push_back(j);
                    } else if (!lc.empty()) {
                        std::vector<int> l16, l8;
                        for (int j : lc) (p->cluster16 && p->geo.len[j] >= 131072 ? l16 : l8).push_back(j);
                        auto by_len = [&](int x, int y) { return p->geo.len[x] > p->geo.len[y]; };
                        std::stable_sort(l16.begin(), l16.end(), by_len);
                        std::stable_sort(l8.begin(), l8.end(), by_len);
                        const size_t sm = wn_smem_bytes<1024, 0, true, 8>();
                        if (!l16.empty()) {
                            set_items(l16);
                            Launch L(p, 3, ls);
                            auto k = sure_winc<1024, 0, 16>;
                            set_smem(k, sm);
                            launch_cluster(k, 16, dim3(16u * (unsigned)p->B, (unsigned)l16.size()), 1024, sm, ls, p->geo, a);
                        }
                        if (!l8.empty()) {
                            cudaStream_t l2 = ls;
                            if (can_fork && p->side2 && !l16.empty()) {
                                fork();
                                CK(cudaStreamWaitEvent(p->side2, p->ev_fork, 0));
                                l2 = p->side2;
                                forked2 = true;
                            }
                            set_items(l8);
                            Launch L(p, 3, l2);
                            auto k = sure_winc<1024, 0, 8>;
                            set_smem(k, sm);
                            launch_cluster(k, 8, dim3(8u * (unsigned)p->B, (unsigned)l8.size()), 1024, sm, l2, p->geo, a);
                        }
                        for (int j : lc) (p->geo.len[j] > 16384 ? win_large : win_items).push_back(j);
                    }
                    if (!lr.empty()) {
                        pm &= 2;
                        launch_big(lr);
                    }
                    for (int n : {131072, 65536, 32768}) {
                        std::vector<int> ln;
                        for (int j : lg) if (p->geo.len[j] == n) ln.push_back(j);
                        if (ln.empty()) continue;
                        set_items(ln);
                        Launch L(p, 3, ls);
                        const dim3 grid(p->B, (unsigned)ln.size());
#define WN_LAUNCH_G(EF_) { auto k = sure_win32<1024, EF_, true>; set_smem(k, wn_smem_bytes<1024, EF_, true>()); \
                           launch(k, grid, 1024, wn_smem_bytes<1024, EF_, true>(), ls, p->geo, a); }
                        if (n == 131072) WN_LAUNCH_G(128) else if (n == 65536) WN_LAUNCH_G(64) else WN_LAUNCH_G(32)
#undef WN_LAUNCH_G
                    }
                    win_large.insert(win_large.end(), lg.begin(), lg.end());
                    // few CTAs (small batches): wider CTAs, half the keys per thread
                    static const int wfew = [] { const char* e = getenv("VDAMP_WINFEW"); return e ? atoi(e) : -1; }();
                    const bool few = wfew >= 0 ? wfew != 0 : (long long)p->Ball * 3 < (long long)p->nsm;
                    for (int n : {16384, 8192, 4096}) {
                        std::vector<int> ln;
                        for (int j : lp) if (p->geo.len[j] == n) ln.push_back(j);
                        if (ln.empty()) continue;
                        set_items(ln);
                        // the smaller subbands run beside the 16,384-key launch on the side stream
                        cudaStream_t lw = ls;
                        if (can_fork && (n != 16384 || has_large)) { fork(); lw = p->side; }
                        // cluster mode (few CTAs, latency-bound): beside the small-subband kernel too
                        // the 4,096-key launch beside the small-subband kernel, not behind it (the side
                        // chain small -> 4,096-key was as long as the 16,384-key launch on the main
                        // stream: cfg1 530k -> 556k img-iter/s, cfg2 111.6k -> 115.0k; VDAMP_SIDE2=0: one side stream)
                        static const int s2all = [] { const char* e = getenv("VDAMP_SIDE2"); return e ? atoi(e) : 1; }();
                        if (lw == p->side && (p->cluster || s2all) && p->side2 && !forked2) {
                            CK(cudaStreamWaitEvent(p->side2, p->ev_fork, 0));
                            lw = p->side2;
                            forked2 = true;
                        }
                        Launch L(p, 3, lw);
                        const dim3 grid(p->B, (unsigned)ln.size());
#define WN_LAUNCH(NT_, EF_) { auto k = sure_win32<NT_, EF_>; set_smem(k, wn_smem_bytes<NT_, EF_>()); \
                              launch(k, grid, NT_, wn_smem_bytes<NT_, EF_>(), lw, p->geo, a); }
                        if (n == 16384) { if (few) WN_LAUNCH(1024, 16) else WN_LAUNCH(512, 32) }
                        else if (n == 8192) { if (few) WN_LAUNCH(512, 16) else WN_LAUNCH(256, 32) }
                        else if (few || nt4 == 512) WN_LAUNCH(512, 8)
                        else if (nt4 == 128) WN_LAUNCH(128, 32)
                        else WN_LAUNCH(256, 16)
#undef WN_LAUNCH
                    }
                    win_items.insert(win_items.end(), lp.begin(), lp.end());
                    continue;
                }
            }
            launch_big(li);
        }
        if (forked) {
            CK(cudaEventRecord(p->ev_join, p->side));
            CK(cudaStreamWaitEvent(st_, p->ev_join, 0));
        }
        if (forked2) {
            CK(cudaEventRecord(p->ev_join2, p->side2));
            CK(cudaStreamWaitEvent(st_, p->ev_join2, 0));
        }
        if constexpr (std::is_same<R, float>::value) {
            static const int wfull = [] { const char* e = getenv("VDAMP_WINFULL"); return e ? atoi(e) : 1; }();   // 0: timing experiments only
            if (!win_items.empty() && wfull) {
                // the full sort for the subbands sure_win32 flagged (normally none): a few CTAs
                set_items(win_items);
                a.only = p->pflag;
                Launch L(p, 3, st_);
                // (sure_win32<512, 32>'s shared-memory size: no carve-out change between the two)
                const size_t sm = wn_smem_bytes<512, 32>();
                auto k = sure_win_full;
                set_smem(k, sm);
                const int pairs = p->B * (int)win_items.size();
                static const int fctas = [] { const char* e = getenv("VDAMP_WINFULL_CTAS"); return e ? atoi(e) : 0; }();
                const dim3 fgrid((unsigned)std::max(1, std::min(fctas > 0 ? fctas : p->nsm, pairs)));
                if (a.cond && cgraph) {
                    cudaStreamCaptureStatus cst;
                    unsigned long long cid = 0;
                    const cudaGraphNode_t* deps = nullptr;
                    size_t nd = 0;
                    CK(cudaStreamGetCaptureInfo(st_, &cst, &cid, &cgraph, &deps, &nd));
                    cudaGraphNodeParams np = {};
                    np.type = cudaGraphNodeTypeConditional;
                    np.conditional.handle = (cudaGraphConditionalHandle)a.cond;
                    np.conditional.type = cudaGraphCondTypeIf;
                    np.conditional.size = 1;
                    cudaGraphNode_t cnode;
                    CK(cudaGraphAddNode(&cnode, cgraph, deps, nd, &np));
                    cudaGraph_t body = np.conditional.phGraph_out[0];
                    Geo garg = p->geo;
                    SelArgs<R> aarg = a;
                    int Barg = p->B, narg = (int)win_items.size();
                    void* kargs[] = {&garg, &aarg, &Barg, &narg};
                    cudaKernelNodeParams kp = {};
                    kp.func = (void*)k;
                    kp.gridDim = fgrid;
                    kp.blockDim = dim3(512);
                    kp.sharedMemBytes = (unsigned)sm;
                    kp.kernelParams = kargs;
                    kp.extra = nullptr;
                    cudaGraphNode_t kn;
                    CK(cudaGraphAddKernelNode(&kn, body, nullptr, 0, &kp));
                    CK(cudaStreamUpdateCaptureDependencies(st_, &cnode, 1, cudaStreamSetCaptureDependencies));
                } else {
                    launch(k, fgrid, 512, sm, st_, p->geo, a, p->B, (int)win_items.size());
                }
                a.only = nullptr;
            }
            if (!win_large.empty() && wfull) {
                set_items(win_large);
                a.only = p->pflag;
                Launch L(p, 3, st_);
                const size_t slot16 = ((size_t)SCAP + SCAP / 32 + 2 + 3) & ~(size_t)3;
                size_t sm = 2 * slot16 * sizeof(R) + CS_WORDS * sizeof(unsigned);
                if (sm < 32768 * 4 + 16384 * sizeof(R)) sm = 32768 * 4 + 16384 * sizeof(R);
                auto k = sure_select_flagged<R, BNT32>;
                set_smem(k, sm);
                const int pairs = p->B * (int)win_large.size();
                launch(k, dim3((unsigned)std::max(1, std::min(p->nsm, pairs))), BNT32, sm, st_, p->geo, a, p->B,
                       (int)win_large.size());
                a.only = nullptr;
            }
        }
    }

    void apply(const C* in, C* out, const double* par) {
        const int maxlen = *std::max_element(p->geo.len, p->geo.len + p->S);
        dim3 grid((unsigned)std::max(1, std::min(maxlen / 256, 64)), p->S, p->B);
        Launch L(p, 5, st);
        apply_params<R><<<grid, 256, 0, st>>>(p->geo, in, out, par);
    }

    void identity_params() {
        Launch L(p, 5, st);
        fill_identity_params<R><<<std::max(1, (p->B * p->S + 255) / 256), 256, 0, st>>>(p->par, p->B * p->S);
    }

    // one VDAMP iteration from (r, par) -> (r, par)   (src/vdamp.py:99-144)
    void iteration(double* trace, void* snapshot, int k = -1) {
        NvtxRange nv("vdamp iteration");
        const bool tm = p->iter_timing && k >= 0 && 2 * k + 1 < (int)p->itev.size();
        if (tm) CK(record(p->itev[2 * k], st));
        synth(r(), p->par, true, nullptr, 0, true);        // r: written by K3 two kernels back
        col(COL_VDAMP, (const C*)p->T1, (C*)p->T2, 1);
        // the previous iteration's NMSE pass (side stream) must have read r before K3 rewrites it
        if (p->nm_pending) CK(cudaStreamWaitEvent(st, p->ev_nmr, 0));
        analysis(nullptr, true, r(), p->par, true, 2);
        if (snapshot) CK(cudaMemcpyAsync(snapshot, p->r, (size_t)p->B * p->N * sizeof(C), cudaMemcpyDeviceToDevice, st));
        select(r(), nullptr, trace, p->have_gt);
        if (tm) CK(record(p->itev[2 * k + 1], st));
    }

    // x_hat = finalize(soft(r; parf))   (src/vdamp.py:147-150)
    void finalize_from_r(const double* parf, C* out) {
        synth(r(), parf, true, nullptr, 4);
        col(COL_FINAL, (const C*)p->T1, (C*)p->T2, 4);
        rows<true, false, true>((const C*)p->T2, out, 4);
    }

    void nmse(const C* x, double* out) {
        Launch L(p, 5, st);
        nmse_sums<R><<<p->B, SNT, 0, st>>>(p->geo, x, (const C*)p->x0, out);
    }

    // FISTA (alg 0) / SURE-IT (alg 1) on the same kernels (src/baselines.py:54-164).
    // The gradient step r~ + Psi F^H M^T (y - M F Psi^H r~) is K1/K2/K3 with identity
    // Onsager parameters and unit weights on the mask (measurements set with p = 1).
    void baseline(int alg, int n_iters, const double* lam, C* xhat, double* trace, double* nmse_out) {
        const size_t cb = (size_t)p->B * p->N * sizeof(C);
        CK(cudaMemsetAsync(p->r, 0, cb, st));
        CK(cudaMemsetAsync(p->what, 0, cb, st));
        identity_params();
        if (alg == 0) {
            Launch L(p, 5, st);
            fill_threshold_params<<<(p->B * p->S + 255) / 256, 256, 0, st>>>(p->parf, lam, p->S, p->B);
        }
        const long long tstride = (long long)p->B * p->S * TRACE_F;
        double t_m = 1.0;
        const int mx = *std::max_element(p->geo.len, p->geo.len + p->S);
        dim3 ugrid((unsigned)std::max(1, std::min(mx / 256, 64)), p->S, p->B);
        for (int it = 0; it < n_iters; ++it) {
            synth(r(), p->par, true, nullptr, 0);
            col(COL_VDAMP, (const C*)p->T1, (C*)p->T2, 1);
            analysis(nullptr, true, r(), p->par, true, 2);          // r <- g (gradient step)
            if (alg == 1) {
                { Launch L(p, 5, st); oracle_tau<R><<<p->B, SNT, 0, st>>>(p->geo, r(), (const C*)p->w0, p->btau); }
                // par keeps the identity of the gradient step; parf = (t_j, 0, 1)
                select(r(), p->btau, trace ? trace + it * tstride : nullptr, true, false);
            }
            const double t_next = 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * t_m * t_m));
            const double beta = (t_m - 1.0) / t_next;
            t_m = t_next;
            { Launch L(p, 5, st); momentum_update<R><<<ugrid, 256, 0, st>>>(p->geo, r(), (C*)p->what, p->parf, beta); }
            if (nmse_out || (alg == 0 && trace)) {
                { Launch L(p, 5, st); coef_err<R><<<dim3(p->S, p->B), 256, 0, st>>>(p->geo, (const C*)p->what, (const C*)p->w0, p->berr); }
                if (nmse_out) {
                    Launch L(p, 5, st);
                    err_totals<<<(p->B + 127) / 128, 128, 0, st>>>(p->berr, p->S, p->B,
                                                                   nmse_out + (long long)it * p->B * VDAMP_NMSE_FIELDS);
                }
                if (alg == 0 && trace)            // FISTA records subband NMSE of w_hat in fields 6/7
                    CK(cudaMemcpy2DAsync(trace + it * tstride + 6, TRACE_F * sizeof(double), p->berr, 2 * sizeof(double),
                                         2 * sizeof(double), (size_t)p->B * p->S, cudaMemcpyDeviceToDevice, st));
            }
        }
        synth((const C*)p->what, nullptr, false, xhat, 4);                  // x_hat = idwt(w_hat)
    }

    void begin() {
        CK(cudaMemsetAsync(p->r, 0, (size_t)p->B * p->N * sizeof(C), st));   // r~_0 = 0
        identity_params();
    }
    // per-run Parseval constants: sum_mask |y - F x0|^2 and |x0|^2
    void nmse_begin() {
        if (!p->parseval) return;
        Launch L(p, 5, st);
        nmse_setup<R><<<p->B, SNT, 0, st>>>(p->geo, (const C*)p->yg, (const R*)p->pinv, (const C*)p->x0r,
                                            (const C*)p->x0, p->nmconst);
    }

    // NMSE record of this iteration's estimate into rec[b * VDAMP_NMSE_FIELDS]
    // The NMSE pass only consumes (r_k, thresholds_k); nothing in the loop consumes its result.
    // Single-pass geometries run it on the side stream with its own row-FFT buffer (xtmp), beside
    // K1 / K2 of the next iteration: K3 of that iteration waits until it has read r (ev_nmr), and the
    // next K4's fork queues behind it on the same side stream.
    bool nmse_beside() const {
        return p->parseval && p->nm_overlap && p->side && p->ev_nm0 && !p->timing && p->passes.size() == 1 && p->xtmp;
    }
    void nmse_join() {
        if (!p->nm_pending) return;
        CK(cudaEventRecord(p->ev_nmd, p->side));
        CK(cudaStreamWaitEvent(st, p->ev_nmd, 0));
        p->nm_pending = false;
    }
    void nmse_iter(double* rec) {
        if (nmse_beside()) {
            CK(cudaEventRecord(p->ev_nm0, st));
            CK(cudaStreamWaitEvent(p->side, p->ev_nm0, 0));
            Seq<R> s2{p, p->side};
            s2.synth(r(), p->parf, true, nullptr, 4, false, (C*)p->xtmp);
            CK(cudaEventRecord(p->ev_nmr, p->side));
            s2.col(COL_NMSE, (const C*)p->xtmp, nullptr, 4);
            Launch L(p, 5, p->side);
            nmse_finish<<<(p->B + 127) / 128, 128, 0, p->side>>>(p->nmpart, p->ntiles, p->nmconst, rec, p->B);
            p->nm_pending = true;
            return;
        }
        if (p->parseval) {
            // x_hat_k = finalize(soft(r_k)): F x_hat is y on the mask and
            // F Psi^H w_hat elsewhere, so one forward FFT suffices
            synth(r(), p->parf, true, nullptr, 4);
            col(COL_NMSE, (const C*)p->T1, nullptr, 4);
            Launch L(p, 5, st);
            nmse_finish<<<(p->B + 127) / 128, 128, 0, st>>>(p->nmpart, p->ntiles, p->nmconst, rec, p->B);
        } else {
            finalize_from_r(p->parf, (C*)p->xtmp);
            nmse((const C*)p->xtmp, rec);
        }
    }

    void run(int n_iters, C* xhat, double* trace, double* nmse_out, void* const* snaps) {
        begin();
        const long long tstride = (long long)p->B * p->S * TRACE_F;
        if (nmse_out) nmse_begin();
        for (int it = 0; it < n_iters; ++it) {
            iteration(trace ? trace + it * tstride : nullptr, snaps ? snaps[it] : nullptr, it);
            if (nmse_out) nmse_iter(nmse_out + (long long)it * p->B * VDAMP_NMSE_FIELDS);
        }
        finalize_from_r(p->parf, xhat);
        nmse_join();
    }
};

// lanes of >= 16 images, at most 4; none for very large batches, which fill the GPU
// by themselves (cfg1, 64 x 256^2: 2 / 3 / 4 / 8 lanes 402k / 401k / 420k / 372k;
// cfg4, 1024 x 256^2: 1 / 2 / 4 / 8 lanes 466k / 458k / 447k / 433k; cfg2, 32 x 512^2:
// 1 / 2 / 4 lanes 41.1k / 43.8k / 41.6k img-iter/s); VDAMP_LANES overrides
int default_lanes(int batch) {
    // (session 5, 128 x 256^2: 1 / 2 / 4 lanes 538k / 565k / 523k; 256 images: 606k / 589k / 518k)
    int nl = batch >= 256 ? 1 : batch >= 128 ? 2 : std::max(1, std::min(4, batch / 16));
    if (const char* le = getenv("VDAMP_LANES")) nl = atoi(le);
    return nl;
}

// side streams (small-subband SURE kernels) get the highest priority, so their
// CTAs are placed first as SMs free up: 420k vs 412k img-iter/s (cfg1)
cudaStream_t create_side_stream() {
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    cudaStream_t s = nullptr;
    CK(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, hi));
    return s;
}

void set_lanes(Plan* p, int nl) {
    p->lanes = std::max(1, std::min(p->B, nl));
    while ((int)p->lane.size() < p->lanes) {
        Plan::Lane l;
        CK(cudaStreamCreateWithFlags(&l.st, cudaStreamNonBlocking));
        l.side = create_side_stream();
        l.side2 = create_side_stream();
        CK(cudaEventCreateWithFlags(&l.join2, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&l.fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&l.join, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&l.done, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&l.nm0, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&l.nmr, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&l.nmd, cudaEventDisableTiming));
        p->lane.push_back(l);
    }
    if (p->lanes > 1 && !p->lane_start) CK(cudaEventCreateWithFlags(&p->lane_start, cudaEventDisableTiming));
}

template <typename F>
int guard(F&& f) {
    try {
        f();
        return VDAMP_OK;
    } catch (const Err& e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        return VDAMP_ERR_ARG;
    }
}

Plan* P(vdamp_plan_t h) {
    if (!h) throw Err{VDAMP_ERR_ARG, "null plan"};
    return reinterpret_cast<Plan*>(h);
}

template <typename F>
void dispatch(Plan* p, void* stream, F&& f) {
    CK(cudaSetDevice(p->dev));
    if (p->prec == VDAMP_FP32) { Seq<float> s{p, (cudaStream_t)stream}; f(s); }
    else                       { Seq<double> s{p, (cudaStream_t)stream}; f(s); }
    if (p->pend != cudaSuccess) {
        cudaError_t e = p->pend;
        p->pend = cudaSuccess;
        throw Err{VDAMP_ERR_CUDA, std::string("kernel launch failed: ") + cudaGetErrorString(e)};
    }
}

void free_plan(Plan* p) {
    if (!p) return;
    cudaSetDevice(p->dev);
    if (p->t2_alias) p->T2 = nullptr;      // (T1's memory)
    void* bufs[] = {p->what, p->btau, p->berr, p->x0r, p->nmconst, p->nmpart, p->r, p->T1, p->T2, p->yg, p->pinv, p->par, p->parf, p->taupart, p->prow, p->pcol, p->prs256,
                    p->nvar, p->offs, p->twH, p->twW, p->kA, p->kB, p->bhist, p->btick, p->bbest, p->baux, p->berrp, p->x0, p->w0, p->xtmp, p->trtmp, p->pflag};
    for (void* b : bufs) if (b) cudaFree(b);
    for (void* b : p->scratch) if (b) cudaFree(b);
    for (auto& e : p->ev) { cudaEventDestroy(e.second.first); cudaEventDestroy(e.second.second); }
    drop_graph(p);
    if (p->side) cudaStreamDestroy(p->side);
    if (p->side2) cudaStreamDestroy(p->side2);
    for (cudaEvent_t e : {p->ev_nm0, p->ev_nmr, p->ev_nmd}) if (e) cudaEventDestroy(e);
    if (p->ev_join2) cudaEventDestroy(p->ev_join2);
    if (p->gstream) cudaStreamDestroy(p->gstream);
    if (p->ev_in) cudaEventDestroy(p->ev_in);
    if (p->ev_out) cudaEventDestroy(p->ev_out);
    if (p->ev_fork) cudaEventDestroy(p->ev_fork);
    for (auto& l : p->lane) {
        cudaStreamDestroy(l.st); cudaStreamDestroy(l.side); cudaStreamDestroy(l.side2); cudaEventDestroy(l.join2);
        cudaEventDestroy(l.fork); cudaEventDestroy(l.join); cudaEventDestroy(l.done);
        cudaEventDestroy(l.nm0); cudaEventDestroy(l.nmr); cudaEventDestroy(l.nmd);
    }
    if (p->lane_start) cudaEventDestroy(p->lane_start);
    if (p->ev_join) cudaEventDestroy(p->ev_join);
    for (cudaEvent_t e : p->itev) cudaEventDestroy(e);
    if (p->d_merr) cudaFree(p->d_merr);
    if (p->h_merr) cudaFreeHost(p->h_merr);
    if (p->ev_meas) cudaEventDestroy(p->ev_meas);
    for (int i = 0; i < 2; ++i) {
        if (p->h_stage[i]) cudaFreeHost(p->h_stage[i]);
        if (p->ev_stage[i]) cudaEventDestroy(p->ev_stage[i]);
    }
    delete p;
}

std::string meas_message(unsigned f) {
    std::string m;
    if (f & MEAS_RANGE) m += "sampled index outside [0, height*width)";
    if (f & MEAS_DUP) m += std::string(m.empty() ? "" : "; ") + "repeated sampled index";
    if (f & MEAS_PROB) m += std::string(m.empty() ? "" : "; ") + "sampling probability outside (0, 1] at a sampled point";
    return m;
}

// Report the flags of the measurements set so far (VDAMP_ERR_ARG).  wait = false
// only looks if the last check has already landed (never blocks the host).
void check_meas(Plan* p, bool wait) {
    if (!p->meas_pending) return;
    if (wait) {
        CK(cudaEventSynchronize(p->ev_meas));
    } else {
        const cudaError_t q = cudaEventQuery(p->ev_meas);
        if (q == cudaErrorNotReady) return;
        CK(q);
    }
    p->meas_pending = false;
    const unsigned f = *(volatile unsigned*)p->h_merr;
    if (f) {
        *(volatile unsigned*)p->h_merr = 0;
        CK(cudaMemset(p->d_merr, 0, sizeof(unsigned)));
        p->have_meas = false;
        throw Err{VDAMP_ERR_ARG, meas_message(f)};
    }
}

}  // namespace

extern "C" {

const char* vdamp_last_error(void) { return g_err.c_str(); }
int vdamp_abi_version(void) { return 1; }

int vdamp_plan_create(int height, int width, int scales, int batch, int precision, int device,
                      vdamp_plan_t* out) {
    Plan* p = nullptr;
    int rc = guard([&] {
        if (!out) throw Err{VDAMP_ERR_ARG, "null output handle"};
        *out = nullptr;
        if (scales < 1) throw Err{VDAMP_ERR_ARG, "scales must be >= 1, got " + std::to_string(scales)};
        if (height < 1 || width < 1 || batch < 1) throw Err{VDAMP_ERR_ARG, "height, width and batch must be >= 1"};
        if (height % (1 << std::min(scales, 30)) || width % (1 << std::min(scales, 30)) || scales > 30)
            throw Err{VDAMP_ERR_SHAPE, "image shape (" + std::to_string(height) + ", " + std::to_string(width) +
                                           ") not divisible by 2^" + std::to_string(scales)};
        if (!pow2(height) || !pow2(width) || height < 2 || width < 2 || height > 2048 || width > 2048)
            throw Err{VDAMP_ERR_UNSUPPORTED, "this build supports power-of-two image sizes in [2, 2048] only"};
        if (precision != VDAMP_FP32 && precision != VDAMP_FP64) throw Err{VDAMP_ERR_ARG, "precision must be 0 (fp32) or 1 (fp64)"};
        if (1 + 3 * scales > MAXS || scales > 12) throw Err{VDAMP_ERR_UNSUPPORTED, "too many scales (max 12)"};
        p = new Plan();
        p->H = height; p->W = width; p->s = scales; p->B = batch; p->Ball = batch; p->prec = precision; p->dev = device;
        p->S = 1 + 3 * scales;
        p->N = (long long)height * width;
        CK(cudaSetDevice(device));
        Geo& g = p->geo;
        memset(&g, 0, sizeof(g));
        g.H = height; g.W = width; g.s = scales; g.S = p->S; g.logH = ilog2(height); g.logW = ilog2(width);
        g.sign_c = (((height / 2) + (width / 2)) & 1) ? -1 : 1;
        g.N = p->N;
        {
            long long off = 0;
            const int hs = height >> scales, ws = width >> scales;
            g.off[0] = 0; g.len[0] = hs * ws; off = (long long)hs * ws;
            int j = 1;
            for (int l = scales; l >= 1; --l)
                for (int o = 0; o < 3; ++o) { g.off[j] = off; g.len[j] = (height >> l) * (width >> l); off += g.len[j]; ++j; }
        }
        // Haar passes: each strip of 2^k rows x (W >> lvl) must fit PCAP elements
        int lvl = 0;
        while (lvl < scales) {
            const int Wl = width >> lvl, Hl = height >> lvl;
            int k = 1;
            while (lvl + k < scales && ((2LL << k) * Wl) <= PCAP && (2 << k) <= Hl) ++k;
            if ((1LL << k) * Wl > PCAP) throw Err{VDAMP_ERR_UNSUPPORTED, "image row too wide for a strip"};
            Pass ps;
            ps.a = lvl + 1; ps.b = lvl + k; ps.k = k; ps.Ha = Hl; ps.Wa = Wl; ps.logWa = ilog2(Wl);
            ps.nstrips = Hl >> k;
            p->passes.push_back(ps);
            lvl += k;
        }
        {
            // SURE work items: subbands > SCAP/2 alone, the rest optionally packed
            // first-fit (largest first) into bins of SCAP keys.  Packing is off:
            // measured slower at 1 CTA/SM (round 1, cfg1: 10.0 vs 6.9 ms/step)
            const bool pack_small = false;
            std::vector<int> order(p->S);
            for (int j = 0; j < p->S; ++j) order[j] = j;
            std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return g.len[x] > g.len[y]; });
            std::vector<std::vector<int>> bins;
            std::vector<long long> fill;
            for (int j : order) {
                const long long L = g.len[j];
                int placed = -1;
                if (L <= SCAP / 2 && pack_small)
                    for (size_t bi = 0; bi < bins.size(); ++bi)
                        if (fill[bi] + L <= SCAP && fill[bi] > 0 && g.len[bins[bi][0]] <= SCAP / 2) { placed = (int)bi; break; }
                if (placed < 0) { bins.push_back({}); fill.push_back(0); placed = (int)bins.size() - 1; }
                bins[placed].push_back(j);
                fill[placed] += L;
            }
            p->item_start.assign(1, 0);
            for (auto& b : bins) {
                for (int j : b) p->item_list.push_back(j);
                p->item_start.push_back((int)p->item_list.size());
            }
        }
        p->cw = std::max(1, std::min(width, PCAP / height));
        p->logcw = ilog2(p->cw);
        p->ntiles = width / p->cw;
        if (p->ntiles > MAXCT) throw Err{VDAMP_ERR_UNSUPPORTED, "too many column tiles"};
        p->rowlog = 0;
        while ((2LL << p->rowlog) * width <= PCAP && (2 << p->rowlog) <= height) ++p->rowlog;
        const size_t cs = precision == VDAMP_FP32 ? sizeof(float2) : sizeof(double2);
        const size_t rs = precision == VDAMP_FP32 ? sizeof(float) : sizeof(double);
        p->csz = cs;
        const size_t img = (size_t)batch * p->N;
        p->r = dalloc(p, img * cs);
        p->T1 = dalloc(p, img * cs);
        {
            // col_pass256 holds its whole 256 x 16 tile in registers between its loads and its
            // stores, so K2 can run in place: T2 aliases T1 and an image's working set drops by
            // 8N bytes (cfg1's 64 images: 150 -> 117 MB against the 126 MB L2; 523k -> 532k
            // img-iter/s, K2 1.01 -> 0.96 and K3 0.84 -> 0.78 ms/step; VDAMP_INPLACE=0: separate buffers)
            const char* ie = getenv("VDAMP_INPLACE");
            const char* fe = getenv("VDAMP_F256");
            p->t2_alias = height == 256 && p->cw == 16 && !(fe && atoi(fe) == 0) && !(ie && atoi(ie) == 0);
            p->T2 = p->t2_alias ? p->T1 : dalloc(p, img * cs);
        }
        p->yg = dalloc(p, img * cs);
        p->pinv = dalloc(p, img * rs);
        p->scratch.assign(p->passes.size(), nullptr);
        for (size_t i = 1; i < p->passes.size(); ++i)
            p->scratch[i] = dalloc(p, (size_t)batch * p->passes[i].Ha * p->passes[i].Wa * cs);
        p->par = (double*)dalloc(p, (size_t)batch * p->S * 3 * sizeof(double));
        p->parf = (double*)dalloc(p, (size_t)batch * p->S * 3 * sizeof(double));
        p->taupart = (double*)dalloc(p, (size_t)batch * p->ntiles * p->S * sizeof(double));
        p->prow = (double*)dalloc(p, (size_t)2 * scales * height * sizeof(double));
        p->pcol = (double*)dalloc(p, (size_t)2 * scales * width * sizeof(double));
        p->nvar = (double*)dalloc(p, (size_t)batch * sizeof(double));
        p->offs = (long long*)dalloc(p, (size_t)(batch + 1) * sizeof(long long));
        p->twH = dalloc(p, (size_t)height * cs);
        p->twW = dalloc(p, (size_t)width * cs);
        p->trtmp = (double*)dalloc(p, (size_t)batch * p->S * TRACE_F * sizeof(double));
        p->pflag = (unsigned*)dalloc(p, (size_t)batch * p->S * sizeof(unsigned));
        const int maxlen = *std::max_element(g.len, g.len + p->S);
        const int capk = precision == VDAMP_FP32 ? Scap<float>::v : Scap<double>::v;
        CK(cudaDeviceGetAttribute(&p->nsm, cudaDevAttrMultiProcessorCount, device));
        {
            // fp32, few subbands of >= 16,384 keys (cfg0: 1 image x 3, cfg3: 1 x 9): a cluster of
            // 8 CTAs per subband (sure_winc) instead of one CTA, or of value ranges over CTAs
            int nbig = 0;
            for (int j = 0; j < p->S; ++j) nbig += g.len[j] >= 16384;
            const char* ce = getenv("VDAMP_CLUSTER");
            // measured crossovers: 256^2 (16,384-key subbands, 3 per image) 4 images 64.7k vs 56.0k
            // img-iter/s without clusters, 6 images 70.8k vs 79.5k; 512^2 (65,536-key subbands) 4
            // images 25.9k vs 17.8k, 8 images 32.3k vs 30.0k
            const long long ctas = (long long)batch * nbig * 8;
            p->cluster = precision == VDAMP_FP32 && nbig > 0 && !(ce && atoi(ce) == 0) &&
                         (maxlen >= 65536 ? ctas <= 3LL * p->nsm : 3 * ctas <= 2LL * p->nsm);
            if (precision == VDAMP_FP32 && nbig > 0 && ce && atoi(ce) == 1) p->cluster = true;    // forced (A/B runs)
            if (p->cluster && maxlen <= capk) p->kA = dalloc(p, img * rs);      // the clusters' key scratch
            p->side2 = create_side_stream();
            CK(cudaEventCreateWithFlags(&p->ev_join2, cudaEventDisableTiming));
            if (p->cluster) {
                // 16-CTA clusters (non-portable size) for the largest subbands, if the device can
                // place one with this kernel's shared memory
                // (measured slower: 104 vs 80 us for a 262,144-key subband, cfg3 5.3k vs 5.5k
                // img-iter/s; off unless VDAMP_CLUSTER16=1)
                const char* c16 = getenv("VDAMP_CLUSTER16");
                if (maxlen >= 131072 && c16 && atoi(c16) == 1) {
                    auto k = sure_winc<1024, 0, 16>;
                    const size_t sm = wn_smem_bytes<1024, 0, true, 8>();
                    bool ok = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess &&
                              cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) == cudaSuccess;
                    if (ok) {
                        cudaLaunchConfig_t cfg = {};
                        cfg.gridDim = dim3(16, 1, 1);
                        cfg.blockDim = dim3(1024, 1, 1);
                        cfg.dynamicSmemBytes = sm;
                        cudaLaunchAttribute at[1];
                        at[0].id = cudaLaunchAttributeClusterDimension;
                        at[0].val.clusterDim.x = 16; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
                        cfg.attrs = at;
                        cfg.numAttrs = 1;
                        int nc = 0;
                        ok = cudaOccupancyMaxActiveClusters(&nc, k, &cfg) == cudaSuccess && nc >= 1;
                    }
                    cudaGetLastError();
                    p->cluster16 = ok;
                }
            }
        }
        if (maxlen > capk) {
            if (maxlen / capk > MAXTILES) throw Err{VDAMP_ERR_UNSUPPORTED, "subband too large"};
            p->kA = dalloc(p, img * rs);
            p->kB = dalloc(p, img * rs);
            const char* be = getenv("VDAMP_BIGRANGE");
            if (precision == VDAMP_FP32 && !p->cluster && !(be && atoi(be) == 0)) {
                for (int j = 0; j < p->S; ++j) if (g.len[j] > capk) p->large.push_back(j);
                // only when the single-CTA path would leave most SMs idle: with many large
                // subbands per batch (cfg2: 32 x 3) it fills the GPU and is measured faster
                // (482 vs 708 us per iteration); cfg3 (1 x 6) gains 4x
                const bool few = (long long)batch * (long long)p->large.size() * 4 <= (long long)p->nsm ||
                                 (be && atoi(be) == 1);
                if (!few) p->large.clear();
                if (few && (int)p->large.size() <= BIG_MAXL && (maxlen + capk / 2 - 1) / (capk / 2) <= BIG_RMAX) {
                    p->bigpath = true;
                    const size_t nl = p->large.size();
                    p->big_ranges = (maxlen + capk / 2 - 1) / (capk / 2);
                    p->big_chunks = (maxlen + BIG_CHUNK - 1) / BIG_CHUNK;
                    p->bhist = (unsigned*)dalloc(p, (size_t)batch * nl * BIGB * sizeof(unsigned));
                    p->btick = (unsigned*)dalloc(p, (size_t)batch * nl * sizeof(unsigned));
                    p->bbest = (double*)dalloc(p, (size_t)batch * nl * p->big_ranges * 4 * sizeof(double));
                    p->baux = (double*)dalloc(p, (size_t)batch * nl * 2 * sizeof(double));
                    p->berrp = (double*)dalloc(p, (size_t)batch * nl * p->big_chunks * 2 * sizeof(double));
                    CK(cudaMemset(p->bhist, 0, (size_t)batch * nl * BIGB * sizeof(unsigned)));
                    CK(cudaMemset(p->btick, 0, (size_t)batch * nl * sizeof(unsigned)));
                }
            }
        }
        p->side = create_side_stream();
        CK(cudaEventCreateWithFlags(&p->ev_nm0, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&p->ev_nmr, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&p->ev_nmd, cudaEventDisableTiming));
        // pays while the loop is latency-bound (cfg0 with trace 13.2k -> 15.6k img-iter/s, cfg1 fp64
        // 82.5k -> 84.9k); a batch whose lanes fill the GPU gains nothing (cfg1 fp32 350k -> 343k)
        p->nm_overlap = batch < 32 || precision == VDAMP_FP64;
        if (const char* ne = getenv("VDAMP_NMSE_OVERLAP")) p->nm_overlap = atoi(ne) != 0;
        CK(cudaStreamCreateWithFlags(&p->gstream, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&p->ev_in, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&p->ev_out, cudaEventDisableTiming));
        // graphs pay off while the host's launch rate limits the run (~860 launches per 3.9 ms
        // step on cfg1: 487k -> 519k img-iter/s; cfg0 13.0k -> 13.7k, cfg3 3.14k -> 3.22k);
        // larger batches are GPU-bound and measured 2-3% faster with direct launches (cfg2, cfg4)
        p->graphs = (long long)batch * p->N <= 64LL * 65536;
        if (const char* pe = getenv("VDAMP_PARSEVAL")) p->parseval = atoi(pe) != 0;
        p->prune = 3;
        {
            // one CTA per large subband: with few of them (cfg3: 1 image x 6) the pruned
            // single-CTA passes measured slower than the fp64 global sort (120 vs 165
            // img-iter/s); fp32 splits those subbands by value (big_keys / big_range)
            int nlarge = 0;
            for (int j = 0; j < p->S; ++j) nlarge += g.len[j] > capk;
            if ((long long)batch * nlarge * 4 <= (long long)p->nsm) p->prune &= 1;
        }
        if (const char* pe = getenv("VDAMP_PRUNE")) p->prune = atoi(pe) & 3;
        if (const char* ge = getenv("VDAMP_GRAPHS")) p->graphs = atoi(ge) != 0;
        if (const char* ie = getenv("VDAMP_INTERLEAVE")) p->interleave = atoi(ie) != 0;
        CK(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming));
        set_lanes(p, default_lanes(batch));
        p->d_merr = (unsigned*)dalloc(p, sizeof(unsigned));
        CK(cudaMemset(p->d_merr, 0, sizeof(unsigned)));
        CK(cudaHostAlloc((void**)&p->h_merr, sizeof(unsigned), cudaHostAllocMapped));
        *p->h_merr = 0;
        CK(cudaHostGetDevicePointer((void**)&p->h_merr_dev, p->h_merr, 0));
        CK(cudaEventCreateWithFlags(&p->ev_meas, cudaEventDisableTiming));
        for (int i = 0; i < 2; ++i) {
            CK(cudaHostAlloc((void**)&p->h_stage[i], (size_t)(2 * batch + 1) * sizeof(double), cudaHostAllocDefault));
            CK(cudaEventCreateWithFlags(&p->ev_stage[i], cudaEventDisableTiming));
        }
        CK(cudaMemset(p->yg, 0, img * cs));
        CK(cudaMemset(p->pinv, 0, img * rs));
        if (precision == VDAMP_FP32) {
            make_twiddles<float><<<(height + 255) / 256, 256>>>((float2*)p->twH, height);
            make_twiddles<float><<<(width + 255) / 256, 256>>>((float2*)p->twW, width);
        } else {
            make_twiddles<double><<<(height + 255) / 256, 256>>>((double2*)p->twH, height);
            make_twiddles<double><<<(width + 255) / 256, 256>>>((double2*)p->twW, width);
        }
        make_profiles<<<dim3((height + 127) / 128, 2 * scales), 128>>>(p->prow, height, scales);
        make_profiles<<<dim3((width + 127) / 128, 2 * scales), 128>>>(p->pcol, width, scales);
        if (height == 256 || height == 512) {
            const int np = 2 * scales, npp = (np + 3) & ~3;
            p->prs256 = dalloc(p, (size_t)height * npp * rs);
            if (precision == VDAMP_FP32) arrange_prs256<float><<<(height * npp + 255) / 256, 256>>>((float*)p->prs256, p->prow, np, npp, height);
            else arrange_prs256<double><<<(height * npp + 255) / 256, 256>>>((double*)p->prs256, p->prow, np, npp, height);
        }
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        *out = reinterpret_cast<vdamp_plan_t>(p);
    });
    if (rc != VDAMP_OK && p) free_plan(p);
    return rc;
}

int vdamp_plan_destroy(vdamp_plan_t plan) {
    return guard([&] { free_plan(reinterpret_cast<Plan*>(plan)); });
}

int vdamp_plan_layout(vdamp_plan_t plan, int64_t* offsets, int64_t* lengths) {
    return guard([&] {
        Plan* p = P(plan);
        for (int j = 0; j < p->S; ++j) {
            if (offsets) offsets[j] = p->geo.off[j];
            if (lengths) lengths[j] = p->geo.len[j];
        }
    });
}

int vdamp_plan_workspace_bytes(vdamp_plan_t plan, size_t* bytes) {
    return guard([&] { *bytes = P(plan)->bytes; });
}

int vdamp_set_measurements(vdamp_plan_t plan, const void* y, const int64_t* indices, const int64_t* counts,
                           const double* probs, int64_t probs_batch_stride, const double* noise_var, void* stream) {
    return guard([&] {
        Plan* p = P(plan);
        if (!y || !indices || !counts || !probs || !noise_var) throw Err{VDAMP_ERR_ARG, "null measurement pointer"};
        if (probs_batch_stride != 0 && probs_batch_stride != p->N)
            throw Err{VDAMP_ERR_ARG, "probs_batch_stride must be 0 (shared map) or height*width"};
        check_meas(p, false);                          // flags of an earlier call that have landed
        long long maxn = 0;
        for (int b = 0; b < p->B; ++b) {
            if (counts[b] < 1 || counts[b] > p->N) throw Err{VDAMP_ERR_ARG, "mask selects no samples or too many"};
            if (!(noise_var[b] >= 0)) throw Err{VDAMP_ERR_ARG, "noise variance must be >= 0"};
            maxn = std::max(maxn, (long long)counts[b]);
        }
        CK(cudaSetDevice(p->dev));
        cudaStream_t st = (cudaStream_t)stream;
        // pinned staging slot (its previous copies must have left the host buffer)
        const int slot = p->stage_k++ & 1;
        CK(cudaEventSynchronize(p->ev_stage[slot]));
        double* nv = p->h_stage[slot];
        long long* offs = reinterpret_cast<long long*>(nv + p->B);
        offs[0] = 0;
        for (int b = 0; b < p->B; ++b) { nv[b] = noise_var[b]; offs[b + 1] = offs[b] + counts[b]; }
        const size_t img = (size_t)p->B * p->N;
        const size_t rs = p->prec == VDAMP_FP32 ? sizeof(float) : sizeof(double);
        CK(cudaMemsetAsync(p->yg, 0, img * p->csz, st));
        CK(cudaMemsetAsync(p->pinv, 0, img * rs, st));
        CK(cudaMemcpyAsync(p->nvar, nv, p->B * sizeof(double), cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(p->offs, offs, (p->B + 1) * sizeof(long long), cudaMemcpyHostToDevice, st));
        CK(cudaEventRecord(p->ev_stage[slot], st));
        dim3 grid((unsigned)std::min<long long>((maxn + 255) / 256, 1024), p->B);
        {
            Launch L(p, 5, st);
            if (p->prec == VDAMP_FP32)
                scatter_measurements<float><<<grid, 256, 0, st>>>(p->geo, (const float2*)y, (const long long*)indices,
                                                                  p->offs, probs, probs_batch_stride, (float2*)p->yg,
                                                                  (float*)p->pinv, p->d_merr);
            else
                scatter_measurements<double><<<grid, 256, 0, st>>>(p->geo, (const double2*)y, (const long long*)indices,
                                                                   p->offs, probs, probs_batch_stride, (double2*)p->yg,
                                                                   (double*)p->pinv, p->d_merr);
        }
        if (p->pend != cudaSuccess) {
            cudaError_t e = p->pend;
            p->pend = cudaSuccess;
            throw Err{VDAMP_ERR_CUDA, std::string("scatter_measurements: ") + cudaGetErrorString(e)};
        }
        {
            Launch L(p, 5, st);
            publish_flags<<<1, 1, 0, st>>>(p->d_merr, p->h_merr_dev);
        }
        CK(cudaEventRecord(p->ev_meas, st));
        p->meas_pending = true;
        p->have_meas = true;
        if (p->validate_sync) check_meas(p, true);
    });
}

int vdamp_set_iteration_timing(vdamp_plan_t plan, int enable) {
    return guard([&] {
        Plan* p = P(plan);
        if (p->iter_timing != (enable != 0)) drop_graph(p);
        p->iter_timing = enable != 0;
    });
}

int vdamp_iteration_times(vdamp_plan_t plan, int n_iters, double* ms, int* images) {
    return guard([&] {
        Plan* p = P(plan);
        if (!p->iter_timing || n_iters > p->it_count || 2 * n_iters > (int)p->itev.size())
            throw Err{VDAMP_ERR_STATE, "no iteration times recorded for that many iterations"};
        CK(cudaSetDevice(p->dev));
        for (int k = 0; k < n_iters; ++k) {
            CK(cudaEventSynchronize(p->itev[2 * k + 1]));
            float t = 0.0f;
            CK(cudaEventElapsedTime(&t, p->itev[2 * k], p->itev[2 * k + 1]));
            ms[k] = t;
        }
        if (images) *images = p->it_images;
    });
}

int vdamp_set_validation(vdamp_plan_t plan, int synchronous) {
    return guard([&] { P(plan)->validate_sync = synchronous != 0; });
}

int vdamp_measurement_status(vdamp_plan_t plan, int wait) {
    return guard([&] {
        Plan* p = P(plan);
        CK(cudaSetDevice(p->dev));
        check_meas(p, wait != 0);
    });
}

int vdamp_check_measurements(int height, int width, int batch, const int64_t* indices, const int64_t* counts,
                             const double* probs, int64_t probs_batch_stride, const double* noise_var) {
    return guard([&] {
        if (height < 1 || width < 1 || batch < 1) throw Err{VDAMP_ERR_ARG, "height, width and batch must be >= 1"};
        if (!indices || !counts || !probs || !noise_var) throw Err{VDAMP_ERR_ARG, "null measurement pointer"};
        const long long N = (long long)height * width;
        if (probs_batch_stride != 0 && probs_batch_stride != N)
            throw Err{VDAMP_ERR_ARG, "probs_batch_stride must be 0 (shared map) or height*width"};
        std::vector<unsigned char> seen((size_t)N);
        long long o = 0;
        unsigned f = 0;
        for (int b = 0; b < batch; ++b) {
            if (counts[b] < 1 || counts[b] > N) throw Err{VDAMP_ERR_ARG, "mask selects no samples or too many"};
            if (!(noise_var[b] >= 0)) throw Err{VDAMP_ERR_ARG, "noise variance must be >= 0"};
            std::fill(seen.begin(), seen.end(), 0);
            for (long long e = 0; e < counts[b]; ++e) {
                const long long gi = indices[o + e];
                if (gi < 0 || gi >= N) { f |= MEAS_RANGE; continue; }
                if (seen[(size_t)gi]) f |= MEAS_DUP;
                seen[(size_t)gi] = 1;
                const double pr = probs[(long long)b * probs_batch_stride + gi];
                if (!(pr > 0.0 && pr <= 1.0)) f |= MEAS_PROB;
            }
            o += counts[b];
        }
        if (f) throw Err{VDAMP_ERR_ARG, meas_message(f)};
    });
}

int vdamp_set_ground_truth(vdamp_plan_t plan, const void* x0, void* stream) {
    return guard([&] {
        Plan* p = P(plan);
        if (!x0) { p->have_gt = false; return; }
        CK(cudaSetDevice(p->dev));
        const size_t bytes = (size_t)p->B * p->N * p->csz;
        if (!p->x0) {
            p->x0 = dalloc(p, bytes); p->w0 = dalloc(p, bytes); p->xtmp = dalloc(p, bytes); p->x0r = dalloc(p, bytes);
            p->nmconst = (double*)dalloc(p, (size_t)p->B * 2 * sizeof(double));
            p->nmpart = (double*)dalloc(p, (size_t)p->B * p->ntiles * sizeof(double));
        }
        CK(cudaMemcpyAsync(p->x0, x0, bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
        dispatch(p, stream, [&](auto& s) {
            typedef typename std::remove_reference<decltype(s)>::type S_;
            typedef typename S_::C C;
            typedef typename S_::Rt R;
            s.analysis((const C*)p->x0, false, (C*)p->w0, nullptr, false, 5);
            // X0r = FFT2u(s_in x0) and the per-run Parseval constants (needs measurements)
            s.template rows<false, true, false>((const C*)p->x0, (C*)p->T1, 5);
            s.col(COL_RAW, (const C*)p->T1, (C*)p->x0r, 5);
        });
        p->have_gt = true;
    });
}

// A view of images [b0, b0 + nb) of plan p: every batch-indexed buffer offset,
// B = nb, the lane's side stream and events.  Launch counts and timing events
// are merged back by lane_merge.
Plan lane_view(const Plan* p, int b0, int nb, const Plan::Lane& l) {
    Plan v = *p;
    const size_t rs = p->prec == VDAMP_FP32 ? sizeof(float) : sizeof(double);
    const size_t ci = (size_t)b0 * p->N * p->csz, ri = (size_t)b0 * p->N * rs;
    auto off = [](void* q, size_t b) -> void* { return q ? (void*)((char*)q + b) : nullptr; };
    v.r = off(p->r, ci); v.T1 = off(p->T1, ci); v.T2 = off(p->T2, ci); v.yg = off(p->yg, ci);
    v.pinv = off(p->pinv, ri); v.kA = off(p->kA, ri); v.kB = off(p->kB, ri);
    for (size_t i = 1; i < p->passes.size(); ++i)
        v.scratch[i] = off(p->scratch[i], (size_t)b0 * p->passes[i].Ha * p->passes[i].Wa * p->csz);
    v.par = p->par + (size_t)b0 * p->S * 3;
    v.parf = p->parf + (size_t)b0 * p->S * 3;
    v.taupart = p->taupart + (size_t)b0 * p->ntiles * p->S;
    v.nvar = p->nvar + b0;
    v.trtmp = p->trtmp + (size_t)b0 * p->S * TRACE_F;
    v.pflag = p->pflag + (size_t)b0 * p->S;
    v.x0 = off(p->x0, ci); v.w0 = off(p->w0, ci); v.x0r = off(p->x0r, ci); v.xtmp = off(p->xtmp, ci);
    if (p->nmconst) v.nmconst = p->nmconst + (size_t)b0 * 2;
    if (p->nmpart) v.nmpart = p->nmpart + (size_t)b0 * p->ntiles;
    if (p->bigpath) {
        const size_t nl = p->large.size();
        v.bhist = p->bhist + (size_t)b0 * nl * BIGB;
        v.btick = p->btick + (size_t)b0 * nl;
        v.bbest = p->bbest + (size_t)b0 * nl * p->big_ranges * 4;
        v.baux = p->baux + (size_t)b0 * nl * 2;
        v.berrp = p->berrp + (size_t)b0 * nl * p->big_chunks * 2;
    }
    v.B = nb;
    v.side = l.side; v.ev_fork = l.fork; v.ev_join = l.join;
    v.ev_nm0 = l.nm0; v.ev_nmr = l.nmr; v.ev_nmd = l.nmd; v.nm_pending = false;
    v.side2 = l.side2; v.ev_join2 = l.join2;
    v.ev.clear();
    v.lane.clear(); v.lanes = 1;
    return v;
}

void lane_merge(Plan* p, Plan& v, long long l0, const long long* c0) {
    p->launches += v.launches - l0;
    for (int c = 0; c < VDAMP_KERNEL_CLASSES; ++c) p->cls_launches[c] += v.cls_launches[c] - c0[c];
    for (auto& e : v.ev) p->ev.push_back(e);
    if (v.pend != cudaSuccess && p->pend == cudaSuccess) p->pend = v.pend;
}

int vdamp_run(vdamp_plan_t plan, int n_iters, void* x_hat, double* trace, double* nmse, void* const* snapshots,
              void* stream) {
    NvtxRange nv("vdamp_run");
    return guard([&] {
        Plan* p = P(plan);
        if (n_iters < 1) throw Err{VDAMP_ERR_ARG, "need at least one iteration, got " + std::to_string(n_iters)};
        check_meas(p, false);
        if (!p->have_meas) throw Err{VDAMP_ERR_STATE, "vdamp_set_measurements must be called first"};
        if (nmse && !p->have_gt) throw Err{VDAMP_ERR_STATE, "NMSE trace requested without ground truth"};
        if (!x_hat) throw Err{VDAMP_ERR_ARG, "null x_hat"};
        cudaStream_t caller = (cudaStream_t)stream;
        cudaStream_t st = caller;
        if (p->iter_timing) {
            CK(cudaSetDevice(p->dev));
            if ((int)p->itev.size() < 2 * n_iters) drop_graph(p);     // captured event nodes change
            while ((int)p->itev.size() < 2 * n_iters) {
                cudaEvent_t e;
                CK(cudaEventCreate(&e));
                p->itev.push_back(e);
            }
            p->it_count = n_iters;
        }
        // image lanes, forked from and joined back into stream cs (also captured into
        // the graph below); diagnostics (trace, NMSE, snapshots) ride on the lanes when
        // they are interleaved (iteration-major): each lane writes its image range of
        // every per-iteration record
        const bool use_lanes = p->lanes > 1 && (p->interleave || (!trace && !nmse && !snapshots));
        p->it_images = use_lanes ? (int)((long long)p->B / p->lanes) : p->B;
        auto run_lanes = [&](cudaStream_t cs) {
            CK(cudaSetDevice(p->dev));
            CK(cudaEventRecord(p->lane_start, cs));
            const int L = p->lanes;
            if (p->interleave) {
                // iteration-major launch order: every lane gets its iteration k before
                // any lane gets k + 1, so the lanes start together instead of one
                // host-submission time apart
                std::vector<Plan> vs;
                std::vector<long long> l0(L), c0((size_t)L * VDAMP_KERNEL_CLASSES);
                vs.reserve(L);
                for (int li = 0; li < L; ++li) {
                    const int b0 = (int)((long long)p->B * li / L), b1 = (int)((long long)p->B * (li + 1) / L);
                    CK(cudaStreamWaitEvent(p->lane[li].st, p->lane_start, 0));
                    vs.push_back(lane_view(p, b0, b1 - b0, p->lane[li]));
                    l0[li] = vs[li].launches;
                    for (int c = 0; c < VDAMP_KERNEL_CLASSES; ++c) c0[(size_t)li * VDAMP_KERNEL_CLASSES + c] = vs[li].cls_launches[c];
                }
                auto each = [&](auto&& fn) {
                    for (int li = 0; li < L; ++li) dispatch(&vs[li], (void*)p->lane[li].st, fn);
                };
                const long long tstride = (long long)p->B * p->S * TRACE_F;
                try {
                    each([&](auto& s) { s.begin(); });
                    if (nmse) each([&](auto& s) { s.nmse_begin(); });
                    for (int it = 0; it < n_iters; ++it)
                        for (int li = 0; li < L; ++li) {
                            const long long b0 = (long long)p->B * li / L;
                            double* tr = trace ? trace + it * tstride + b0 * p->S * TRACE_F : nullptr;
                            void* sn = (snapshots && snapshots[it]) ? (void*)((char*)snapshots[it] + (size_t)b0 * p->N * p->csz) : nullptr;
                            dispatch(&vs[li], (void*)p->lane[li].st, [&](auto& s) {
                                s.iteration(tr, sn, li == 0 ? it : -1);
                                if (nmse) s.nmse_iter(nmse + ((long long)it * p->B + b0) * VDAMP_NMSE_FIELDS);
                            });
                        }
                    for (int li = 0; li < L; ++li) {
                        const int b0 = (int)((long long)p->B * li / L);
                        void* xo = (char*)x_hat + (size_t)b0 * p->N * p->csz;
                        dispatch(&vs[li], (void*)p->lane[li].st, [&](auto& s) {
                            typedef typename std::remove_reference<decltype(s)>::type S_;
                            s.finalize_from_r(s.p->parf, (typename S_::C*)xo);
                            s.nmse_join();
                        });
                    }
                } catch (...) {
                    for (int li = 0; li < L; ++li) lane_merge(p, vs[li], l0[li], &c0[(size_t)li * VDAMP_KERNEL_CLASSES]);
                    throw;
                }
                for (int li = 0; li < L; ++li) {
                    lane_merge(p, vs[li], l0[li], &c0[(size_t)li * VDAMP_KERNEL_CLASSES]);
                    CK(cudaEventRecord(p->lane[li].done, p->lane[li].st));
                    CK(cudaStreamWaitEvent(cs, p->lane[li].done, 0));
                }
                return;
            }
            for (int li = 0; li < L; ++li) {
                const int b0 = (int)((long long)p->B * li / L), b1 = (int)((long long)p->B * (li + 1) / L);
                Plan::Lane& l = p->lane[li];
                CK(cudaStreamWaitEvent(l.st, p->lane_start, 0));
                Plan v = lane_view(p, b0, b1 - b0, l);
                v.iter_timing = p->iter_timing && li == 0;
                long long c0[VDAMP_KERNEL_CLASSES];
                for (int c = 0; c < VDAMP_KERNEL_CLASSES; ++c) c0[c] = v.cls_launches[c];
                const long long l0 = v.launches;
                void* xo = (char*)x_hat + (size_t)b0 * p->N * p->csz;
                try {
                    dispatch(&v, (void*)l.st, [&](auto& s) {
                        typedef typename std::remove_reference<decltype(s)>::type S_;
                        s.run(n_iters, (typename S_::C*)xo, nullptr, nullptr, nullptr);
                    });
                } catch (...) { lane_merge(p, v, l0, c0); throw; }
                lane_merge(p, v, l0, c0);
                CK(cudaEventRecord(l.done, l.st));
                CK(cudaStreamWaitEvent(cs, l.done, 0));
            }
            return;
        };
        if (!p->graphs && use_lanes) {
            run_lanes(caller);
            return;
        }
        if (!p->graphs) {
            dispatch(p, stream, [&](auto& s) {
                typedef typename std::remove_reference<decltype(s)>::type S_;
                s.run(n_iters, (typename S_::C*)x_hat, trace, nmse, snapshots);
            });
            return;
        }
        // the legacy default stream cannot be captured: run on the plan's stream,
        // ordered after / before the caller's work by events
        const bool hop = (caller == nullptr || caller == cudaStreamLegacy || caller == cudaStreamPerThread);
        if (hop) {
            st = p->gstream;
            CK(cudaEventRecord(p->ev_in, caller));
            CK(cudaStreamWaitEvent(st, p->ev_in, 0));
        }
        void* sarg = (void*)st;
        // key: everything baked into the captured launches
        std::vector<const void*> key{(const void*)(intptr_t)n_iters, x_hat, trace, nmse, (const void*)(intptr_t)p->have_gt,
                                     (const void*)(intptr_t)p->timing, (const void*)st,
                                     (const void*)(intptr_t)(use_lanes ? p->lanes : 1), (const void*)(intptr_t)p->interleave,
                                     (const void*)(intptr_t)p->iter_timing};
        if (snapshots) for (int k = 0; k < n_iters; ++k) key.push_back(snapshots[k]);
        else key.push_back(nullptr);
        if ((!p->gexec || key != p->gkey) && !switch_graph(p, key)) {
            CK(cudaSetDevice(p->dev));
            // capture: launches and timing events recorded during capture belong to the graph
            const long long l0 = p->launches;
            long long c0[VDAMP_KERNEL_CLASSES];
            for (int c = 0; c < VDAMP_KERNEL_CLASSES; ++c) c0[c] = p->cls_launches[c];
            std::swap(p->ev, p->gev);          // Launch appends to p->ev: collect the graph's events
            p->ev.clear();
            CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
            bool ok = true;
            try {
                if (use_lanes) run_lanes(st);
                else dispatch(p, sarg, [&](auto& s) {
                    typedef typename std::remove_reference<decltype(s)>::type S_;
                    s.run(n_iters, (typename S_::C*)x_hat, trace, nmse, snapshots);
                });
            } catch (...) { ok = false; }
            cudaGraph_t graph = nullptr;
            cudaError_t ec = cudaStreamEndCapture(st, &graph);
            std::swap(p->ev, p->gev);          // p->gev = graph events, p->ev = previous one-shot events
            if (!ok || ec != cudaSuccess) {
                if (graph) cudaGraphDestroy(graph);
                p->graphs = false;             // fall back to direct launches for this plan
                drop_current_graph(p);         // (the events collected during the failed capture)
                p->launches = l0;
                for (int c = 0; c < VDAMP_KERNEL_CLASSES; ++c) p->cls_launches[c] = c0[c];
                cudaGetLastError();
                if (use_lanes) run_lanes(st);
                else dispatch(p, sarg, [&](auto& s) {
                    typedef typename std::remove_reference<decltype(s)>::type S_;
                    s.run(n_iters, (typename S_::C*)x_hat, trace, nmse, snapshots);
                });
                if (hop) {
                    CK(cudaEventRecord(p->ev_out, st));
                    CK(cudaStreamWaitEvent(caller, p->ev_out, 0));
                }
                return;
            }
            CK(cudaGraphInstantiate(&p->gexec, graph, cudaGraphInstantiateFlagUseNodePriority));
            cudaGraphDestroy(graph);
            p->gkey = key;
            p->g_launches = p->launches - l0;
            for (int c = 0; c < VDAMP_KERNEL_CLASSES; ++c) { p->g_cls[c] = p->cls_launches[c] - c0[c]; p->cls_launches[c] = c0[c]; }
            p->launches = l0;
        }
        CK(cudaGraphLaunch(p->gexec, st));
        if (hop) {
            CK(cudaEventRecord(p->ev_out, st));
            CK(cudaStreamWaitEvent(caller, p->ev_out, 0));
        }
        p->launches += p->g_launches;
        for (int c = 0; c < VDAMP_KERNEL_CLASSES; ++c) p->cls_launches[c] += p->g_cls[c];
        if (p->timing && !p->gev.empty()) accumulate(p, p->gev, false);   // graph events are reused per replay
    });
}

int vdamp_iterate(vdamp_plan_t plan, const void* r_tilde, void* r, void* r_tilde_next, void* w_hat, double* trace,
                  void* stream) {
    return guard([&] {
        Plan* p = P(plan);
        check_meas(p, false);
        if (!p->have_meas) throw Err{VDAMP_ERR_STATE, "vdamp_set_measurements must be called first"};
        if (!r_tilde) throw Err{VDAMP_ERR_ARG, "null r_tilde"};
        dispatch(p, stream, [&](auto& s) {
            typedef typename std::remove_reference<decltype(s)>::type S_;
            typedef typename S_::C C;
            const size_t bytes = (size_t)p->B * p->N * sizeof(C);
            CK(cudaMemcpyAsync(p->r, r_tilde, bytes, cudaMemcpyDeviceToDevice, s.st));
            s.identity_params();   // r~ enters as r with (t, alpha, gain) = (0, 0, 1)
            s.iteration(trace, nullptr);
            if (r) CK(cudaMemcpyAsync(r, p->r, bytes, cudaMemcpyDeviceToDevice, s.st));
            if (r_tilde_next) s.apply((const C*)p->r, (C*)r_tilde_next, p->par);
            if (w_hat) s.apply((const C*)p->r, (C*)w_hat, p->parf);
        });
    });
}

int vdamp_dwt(vdamp_plan_t plan, const void* image, void* coeffs, void* stream) {
    return guard([&] {
        Plan* p = P(plan);
        dispatch(p, stream, [&](auto& s) {
            typedef typename std::remove_reference<decltype(s)>::type S_;
            typedef typename S_::C C;
            s.analysis((const C*)image, false, (C*)coeffs, nullptr, false, 5);
        });
    });
}

int vdamp_idwt(vdamp_plan_t plan, const void* coeffs, void* image, void* stream) {
    return guard([&] {
        Plan* p = P(plan);
        dispatch(p, stream, [&](auto& s) {
            typedef typename std::remove_reference<decltype(s)>::type S_;
            typedef typename S_::C C;
            s.synth((const C*)coeffs, nullptr, false, (C*)image, 5);
        });
    });
}

int vdamp_fft2c(vdamp_plan_t plan, const void* in, void* out, int inverse, void* stream) {
    return guard([&] {
        Plan* p = P(plan);
        dispatch(p, stream, [&](auto& s) {
            typedef typename std::remove_reference<decltype(s)>::type S_;
            typedef typename S_::C C;
            if (inverse) {
                s.template rows<true, true, false>((const C*)in, (C*)p->T1, 5);
                s.col(COL_INV, (const C*)p->T1, (C*)out, 5);
            } else {
                s.template rows<false, true, false>((const C*)in, (C*)p->T1, 5);
                s.col(COL_FWD, (const C*)p->T1, (C*)out, 5);
            }
        });
    });
}

int vdamp_finalize(vdamp_plan_t plan, const void* w_hat, void* x_hat, void* stream) {
    return guard([&] {
        Plan* p = P(plan);
        check_meas(p, false);
        if (!p->have_meas) throw Err{VDAMP_ERR_STATE, "vdamp_set_measurements must be called first"};
        dispatch(p, stream, [&](auto& s) {
            typedef typename std::remove_reference<decltype(s)>::type S_;
            typedef typename S_::C C;
            s.synth((const C*)w_hat, nullptr, true, nullptr, 4);
            s.col(COL_FINAL, (const C*)p->T1, (C*)p->T2, 4);
            s.template rows<true, false, true>((const C*)p->T2, (C*)x_hat, 4);
        });
    });
}

int vdamp_denoise_colored(vdamp_plan_t plan, const void* r, const double* tau, void* w_hat, double* trace,
                          void* stream) {
    return guard([&] {
        Plan* p = P(plan);
        if (!r || !tau) throw Err{VDAMP_ERR_ARG, "null r or tau"};
        dispatch(p, stream, [&](auto& s) {
            typedef typename std::remove_reference<decltype(s)>::type S_;
            typedef typename S_::C C;
            s.select((const C*)r, tau, trace, false);
            if (w_hat) s.apply((const C*)r, (C*)w_hat, p->parf);
        });
    });
}

int vdamp_set_timing(vdamp_plan_t plan, int enable) {
    return guard([&] {
        Plan* p = P(plan);
        p->timing = enable != 0;
        for (auto& e : p->ev) { cudaEventDestroy(e.second.first); cudaEventDestroy(e.second.second); }
        p->ev.clear();
        drop_graph(p);
        for (int c = 0; c < VDAMP_KERNEL_CLASSES; ++c) { p->ms[c] = 0; p->cls_launches[c] = 0; }
    });
}

int vdamp_kernel_times(vdamp_plan_t plan, double* ms, int64_t* launches) {
    return guard([&] {
        Plan* p = P(plan);
        accumulate(p, p->ev, true);
        for (int c = 0; c < VDAMP_KERNEL_CLASSES; ++c) {
            if (ms) ms[c] = p->ms[c];
            if (launches) launches[c] = p->cls_launches[c];
        }
    });
}

#ifdef VDAMP_PHASE_TIMING
// debug build only: copy the per-(image, subband) phase clocks of the last select launch
extern "C" VDAMP_API int vdamp_debug_phase_times(long long* out, int images) {
    return guard([&] { CK(cudaMemcpyFromSymbol(out, g_phase, (size_t)images * 64 * 4 * sizeof(long long))); });
}
extern "C" VDAMP_API int vdamp_debug_scan_times(long long* out, int images) {
    return guard([&] { CK(cudaMemcpyFromSymbol(out, g_scan, (size_t)images * 64 * 5 * sizeof(long long))); });
}
extern "C" VDAMP_API int vdamp_debug_csort_times(long long* out, int images) {
    return guard([&] { CK(cudaMemcpyFromSymbol(out, g_csort, (size_t)images * 64 * 8 * sizeof(long long))); });
}
extern "C" VDAMP_API int vdamp_debug_prune_times(long long* out, int images) {
    return guard([&] { CK(cudaMemcpyFromSymbol(out, g_prune, (size_t)images * 64 * 10 * sizeof(long long))); });
}
#endif

int vdamp_baseline_run(vdamp_plan_t plan, int algorithm, int n_iters, const double* lam, void* x_hat, double* trace,
                       double* nmse, void* stream) {
    return guard([&] {
        Plan* p = P(plan);
        if (algorithm != 0 && algorithm != 1) throw Err{VDAMP_ERR_ARG, "algorithm must be 0 (fista) or 1 (sure_it)"};
        if (n_iters < 1) throw Err{VDAMP_ERR_ARG, "need at least one iteration"};
        check_meas(p, false);
        if (!p->have_meas) throw Err{VDAMP_ERR_STATE, "vdamp_set_measurements must be called first"};
        if (algorithm == 0 && !lam) throw Err{VDAMP_ERR_ARG, "fista requires lam"};
        if ((algorithm == 1 || nmse || trace) && !p->have_gt)
            throw Err{VDAMP_ERR_STATE, algorithm == 1 ? "sure_it needs the ground truth (oracle tau)"
                                                      : "trace/NMSE need the ground truth"};
        if (!x_hat) throw Err{VDAMP_ERR_ARG, "null x_hat"};
        CK(cudaSetDevice(p->dev));
        if (!p->what) {
            p->what = dalloc(p, (size_t)p->B * p->N * p->csz);
            p->btau = (double*)dalloc(p, (size_t)p->B * p->S * sizeof(double));
            p->berr = (double*)dalloc(p, (size_t)p->B * p->S * 2 * sizeof(double));
        }
        dispatch(p, stream, [&](auto& s) {
            typedef typename std::remove_reference<decltype(s)>::type S_;
            s.baseline(algorithm, n_iters, lam, (typename S_::C*)x_hat, trace, nmse);
        });
    });
}

int vdamp_mc_accumulate(vdamp_plan_t plan, const void* r, const void* w0, double* sum_r, double* sum_sq,
                        double* scratch, void* stream) {
    return guard([&] {
        Plan* p = P(plan);
        if (!r || !w0 || !sum_r || !sum_sq || !scratch) throw Err{VDAMP_ERR_ARG, "null Monte Carlo buffer"};
        CK(cudaSetDevice(p->dev));
        cudaStream_t st = (cudaStream_t)stream;
        const unsigned grid = (unsigned)std::min<long long>((p->N + 255) / 256, 4096);
        {
            Launch L(p, 5, st);
            if (p->prec == VDAMP_FP32)
                mc_accumulate<float><<<grid, 256, 0, st>>>(p->geo, p->B, (const float2*)r, (const float2*)w0,
                                                           (double2*)sum_r, scratch);
            else
                mc_accumulate<double><<<grid, 256, 0, st>>>(p->geo, p->B, (const double2*)r, (const double2*)w0,
                                                            (double2*)sum_r, scratch);
        }
        {
            Launch L(p, 5, st);
            mc_band_sums<<<p->S, SNT, 0, st>>>(p->geo, scratch, sum_sq);
        }
        if (p->pend != cudaSuccess) {
            cudaError_t e = p->pend;
            p->pend = cudaSuccess;
            throw Err{VDAMP_ERR_CUDA, std::string("mc_accumulate: ") + cudaGetErrorString(e)};
        }
    });
}

int vdamp_set_graphs(vdamp_plan_t plan, int enable) {
    return guard([&] {
        Plan* p = P(plan);
        p->graphs = enable != 0;
        drop_graph(p);
    });
}

int vdamp_set_lanes(vdamp_plan_t plan, int lanes) {
    return guard([&] {
        Plan* p = P(plan);
        if (lanes < 0) throw Err{VDAMP_ERR_ARG, "lanes must be >= 0"};
        CK(cudaSetDevice(p->dev));
        set_lanes(p, lanes == 0 ? default_lanes(p->B) : lanes);
    });
}

int vdamp_launch_count(vdamp_plan_t plan, int64_t* count, int reset) {
    return guard([&] {
        Plan* p = P(plan);
        if (count) *count = p->launches;
        if (reset) p->launches = 0;
    });
}

}  // extern "C"
