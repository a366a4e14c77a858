// C ABI of the cvsr library (include/cvsr.h): validation, contexts, code
// layout (B1), the BP iteration scheduler (B3) and the multi-stage slice
// driver (PAPER.md:114 steps 4-6).
#include <stdarg.h>
#include <stdlib.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

using namespace cvsr;

namespace {

thread_local std::string g_err;

cvsr_status fail(cvsr_status st, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

#define CK(call)                                                                                      \
    do {                                                                                              \
        cudaError_t e_ = (call);                                                                      \
        if (e_ != cudaSuccess) return fail(CVSR_ECUDA, "%s: %s", #call, cudaGetErrorString(e_));      \
    } while (0)

struct DeviceGuard {
    int prev = -1;
    bool ok = true;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) ok = (cudaSetDevice(dev) == cudaSuccess);
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

constexpr int RING = 8;
constexpr int LOOKAHEAD = 3;

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// bump allocator over the scratch arena
struct Carve {
    char *base;
    size_t off = 0;
    template <typename P>
    P *take(size_t bytes) {
        P *p = reinterpret_cast<P *>(base + off);
        off += align_up(bytes);
        return p;
    }
};

}  // namespace

struct cvsr_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t cap_stream = nullptr;   // capture-only stream for CUDA graphs (created on first use)
    void *scratch = nullptr;
    size_t scratch_cap = 0;
    int32_t *host_counts = nullptr;      // mapped pinned: [n_act, n_ret, lanes, epoch]
    int32_t *host_counts_dev = nullptr;  // device alias of host_counts
    int32_t epoch = 0;
    cudaEvent_t ring[RING] = {};
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    unsigned long long *acc = nullptr;   // device accumulators for stats [32]
    float *llr_tab = nullptr;            // tabulated conditional LLR (grow-only)
    size_t llr_tab_cap = 0;
    uint32_t *bob_bits = nullptr;        // packed slice bits for the syndrome (grow-only)
    size_t bob_bits_cap = 0;
    int64_t launches = 0;
    // optional per-kernel-class timing (CUDA events around launches)
    bool profiling = false;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    std::vector<std::pair<int, size_t>> prof;  // (class, index of start event; stop = index + 1)
};

struct cvsr_code {
    int device = 0;
    CodeDev d{};
    void *mem = nullptr;
};

namespace {

// kernel classes for cvsr_ctx_kernel_times
enum { KC_CN = 0, KC_VN = 1, KC_INIT = 2, KC_CTRL = 3, KC_N = 4 };

void prof_begin(cvsr_ctx *ctx, int cls) {
    if (!ctx->profiling) return;
    while (ctx->ev_pool.size() < ctx->ev_used + 2) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) {
            ctx->profiling = false;
            return;
        }
        ctx->ev_pool.push_back(e);
    }
    ctx->prof.push_back({cls, ctx->ev_used});
    cudaEventRecord(ctx->ev_pool[ctx->ev_used], ctx->stream);
    ctx->ev_used += 2;
}

void prof_end(cvsr_ctx *ctx) {
    if (!ctx->profiling || ctx->prof.empty()) return;
    cudaEventRecord(ctx->ev_pool[ctx->prof.back().second + 1], ctx->stream);
}

cvsr_status check_launch(cvsr_ctx *ctx, int n_launched) {
    ctx->launches += n_launched;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(CVSR_ECUDA, "kernel launch: %s", cudaGetErrorString(e));
    return CVSR_OK;
}

cvsr_status scratch_reserve(cvsr_ctx *ctx, size_t bytes, char **out) {
    if (bytes > ctx->scratch_cap) {
        CK(cudaStreamSynchronize(ctx->stream));
        if (ctx->scratch) CK(cudaFree(ctx->scratch));
        ctx->scratch = nullptr;
        ctx->scratch_cap = 0;
        cudaError_t e = cudaMalloc(&ctx->scratch, bytes);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(CVSR_ENOMEM, "scratch arena of %zu bytes: %s", bytes, cudaGetErrorString(e));
        }
        ctx->scratch_cap = bytes;
    }
    *out = static_cast<char *>(ctx->scratch);
    return CVSR_OK;
}

// Experimental fused iteration scheduler (k_iter), opt-in with CVSR_FUSED=1.  Measured
// on B200 for C2 it is slower than the per-pass kernels (170 ms vs 105 ms per step:
// the C2V lines do not survive in L2 between a tile's CN and VN phases, DRAM traffic
// per iteration rose from 7.8 to 10 GB, and the persistent grid runs at 24 warps/SM
// with per-item barriers), so the default is the per-pass path.
bool fused_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("CVSR_FUSED");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}

// Process-default BP schedule: CVSR_SCHEDULE=layered selects the row-layered schedule (reading
// R-9), anything else the flooding schedule (reading A-8); per call, cvsr_decode_opts.flags wins.
bool layered_env() {
    static const int v = [] {
        const char *e = getenv("CVSR_SCHEDULE");
        return (e && strcmp(e, "layered") == 0) ? 1 : 0;
    }();
    return v != 0;
}

bool layered_requested(int32_t flags) {
    const int sch = flags & CVSR_SCHED_MASK;
    if (sch == CVSR_SCHED_LAYERED) return true;
    if (sch == CVSR_SCHED_FLOODING) return false;
    return layered_env();
}

// frames per lane: choose_subs(frames), narrowed in fused mode so that one tile's
// message lines (E x 128 S bytes) stay well inside L2 for the CN -> VN hand-off.
// layered: the schedule that will actually run for this code (after the fallback).
int pick_subs(int32_t frames, int64_t E, bool layered, int32_t max_dc) {
    int s = choose_subs(frames);
    static int forced = -1;
    if (forced < 0) {
        const char *e = getenv("CVSR_SUBS");  // tuning switch: force 1, 2 or 4 frames per lane
        forced = e ? atoi(e) : 0;
    }
    if (forced == 1 || forced == 2 || forced == 4) return std::min(forced, s == 4 ? 4 : std::max(s, forced));
    if (layered) s = std::min(s, layer_subs(max_dc));  // layer_kernels.cu
    static double cap = -1.0;
    if (cap < 0.0) {
        const char *e = getenv("CVSR_FUSED_MB");  // experiment switch: per-tile L2 budget (MB)
        cap = e ? atof(e) : 40.0;
    }
    if (fused_enabled())
        while (s > 1 && (double)E * LANES * s * 4 > cap * 1.0e6) s >>= 1;
    return s;
}

int tiles_for(int32_t frames, int subs) { return (frames + LANES * subs - 1) / (LANES * subs); }


// frame compaction (second arena) on/off: CVSR_COMPACT=0 disables
// CUDA-graph replay of the iteration loop for small batches (launch-bound): CVSR_GRAPH=0 disables
bool graph_enabled() {
    static const int v = [] {
        const char *e = getenv("CVSR_GRAPH");
        return (e && *e) ? atoi(e) : 1;
    }();
    return v != 0;
}
// one-CTA-per-frame shared-memory decoder for small codes: CVSR_SMEM=0 disables,
// CVSR_SMEM_KB sets the largest per-frame footprint that takes it (default 40 KB: measured
// crossover)
bool smem_enabled() {
    static const int v = [] {
        const char *e = getenv("CVSR_SMEM");
        return (e && *e) ? atoi(e) : 1;
    }();
    return v != 0;
}
size_t smem_limit() {
    static const size_t v = [] {
        const char *e = getenv("CVSR_SMEM_KB");
        return (size_t)((e && *e) ? atoi(e) : 40) * 1024;
    }();
    return v;
}
constexpr int GRAPH_ITERS = 8;      // iterations per captured graph
constexpr int GRAPH_MAX_TILES = 2;  // batches of at most this many tiles take the graph path

bool compact_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("CVSR_COMPACT");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1 && !fused_enabled();
}

// compact when the active frames fill at most this fraction of the active tiles
double compact_frac() {
    static double v = -1.0;
    if (v < 0.0) {
        const char *e = getenv("CVSR_COMPACT_FRAC");  // tuning switch
        v = e ? atof(e) : 0.65;
    }
    return v;
}

// compaction only when it frees at least this many tiles: at C4 (125 frames, 2 tiles) the 2 -> 1
// compaction moved 1.1 GB per slice to save half of a few tail iterations whose cost is mostly
// per-launch (C4 99.7 ms with, 98.6 ms without; C2's 32 tiles still gain: 41.8 vs 44.9 ms)
int compact_min_free() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("CVSR_COMPACT_MIN_FREE");  // tuning switch
        v = e ? atoi(e) : 2;
    }
    return v;
}

// second arena for frame compaction (see bp_kernels.cu "frame compaction")
struct CompactArena {
    float *msg = nullptr, *L = nullptr;
    uint4 *hb = nullptr, *st = nullptr;
    int32_t *slot_frame[2] = {nullptr, nullptr};
    int32_t *dst_src = nullptr;
};

size_t compact_bytes(int tiles, int subs, int64_t n, int64_t M, int64_t E) {
    const size_t T = (size_t)LANES * subs;
    return align_up((size_t)tiles * E * T * 4) + align_up((size_t)tiles * n * T * 4) +
           align_up((size_t)tiles * n * sizeof(uint4)) + align_up((size_t)tiles * M * sizeof(uint4)) +
           3 * align_up((size_t)tiles * T * sizeof(int32_t));
}

CompactArena carve_compact(Carve &cv, int tiles, int subs, int64_t n, int64_t M, int64_t E) {
    const size_t T = (size_t)LANES * subs;
    CompactArena c;
    c.msg = cv.take<float>((size_t)tiles * E * T * 4);
    c.L = cv.take<float>((size_t)tiles * n * T * 4);
    c.hb = cv.take<uint4>((size_t)tiles * n * sizeof(uint4));
    c.st = cv.take<uint4>((size_t)tiles * M * sizeof(uint4));
    c.slot_frame[0] = cv.take<int32_t>((size_t)tiles * T * sizeof(int32_t));
    c.slot_frame[1] = cv.take<int32_t>((size_t)tiles * T * sizeof(int32_t));
    c.dst_src = cv.take<int32_t>((size_t)tiles * T * sizeof(int32_t));
    return c;
}

size_t decstate_bytes(int tiles, int frames, int subs, int64_t n, int64_t M, int64_t E) {
    const size_t T = (size_t)LANES * subs;
    size_t b = 0;
    b += align_up((size_t)tiles * E * T * sizeof(float));
    b += align_up((size_t)tiles * n * T * sizeof(float));
    b += 2 * align_up((size_t)tiles * n * sizeof(uint4));
    b += align_up((size_t)tiles * M * sizeof(uint4));
    b += 2 * align_up((size_t)tiles * sizeof(int32_t)) + align_up(sizeof(int32_t));
    b += 5 * align_up((size_t)tiles * sizeof(uint4));
    b += align_up(16 * sizeof(int32_t));
    b += align_up((size_t)frames * sizeof(int32_t));
    b += align_up((size_t)frames);
    return b;
}

DecState carve_decstate(Carve &cv, int tiles, int frames, int subs, int64_t n, int64_t M, int64_t E, int32_t *iters_user,
                        uint8_t *conv_user) {
    DecState ds{};
    ds.tiles = tiles;
    ds.frames = frames;
    ds.subs = subs;
    ds.tile_frames = LANES * ds.subs;
    const size_t T = (size_t)ds.tile_frames;
    ds.msg = cv.take<float>((size_t)tiles * E * T * sizeof(float));
    ds.L = cv.take<float>((size_t)tiles * n * T * sizeof(float));
    ds.hb = cv.take<uint4>((size_t)tiles * n * sizeof(uint4));
    ds.hb2 = cv.take<uint4>((size_t)tiles * n * sizeof(uint4));
    ds.cn_done = cv.take<int32_t>((size_t)tiles * sizeof(int32_t));
    ds.cn_ready = cv.take<int32_t>((size_t)tiles * sizeof(int32_t));
    ds.fused_work = cv.take<int32_t>(sizeof(int32_t));
    ds.st = cv.take<uint4>((size_t)tiles * M * sizeof(uint4));
    ds.tile_active = cv.take<uint4>((size_t)tiles * sizeof(uint4));
    ds.tile_unsat = cv.take<uint4>((size_t)tiles * sizeof(uint4));
    ds.tile_newly = cv.take<uint4>((size_t)tiles * sizeof(uint4));
    ds.active_list = cv.take<int32_t>((size_t)tiles * sizeof(int32_t));
    ds.retire_list = cv.take<int32_t>((size_t)tiles * sizeof(int32_t));
    ds.counts = cv.take<int32_t>(16 * sizeof(int32_t));
    int32_t *it = cv.take<int32_t>((size_t)frames * sizeof(int32_t));
    uint8_t *cvb = cv.take<uint8_t>((size_t)frames);
    ds.iters = iters_user ? iters_user : it;
    ds.conv = conv_user ? conv_user : cvb;
    return ds;
}

// Flooding BP iterations with per-frame early termination (B3).  Expects
// ds.L, ds.st, tile state and counts initialised.  Host control: iterations
// are launched LOOKAHEAD ahead of a mapped-memory progress counter written by
// the status kernel; the counter also bounds the grid's tile dimension.
cvsr_status run_decode(cvsr_ctx *ctx, const cvsr_code *code, const DecState &ds0, int max_iter, float qmax,
                       uint32_t *bits_out, const CompactArena *ca, bool layered, bool hb_ready = false) {
    cudaStream_t s = ctx->stream;
    const CodeDev &cd = code->d;
    volatile int32_t *hc = ctx->host_counts;
    // the mapped counter is only read after an event of THIS run completed;
    // every status/list kernel of this run writes it, so stale values are impossible.
    const bool fused = fused_enabled();
    const FusedPlan plan = fused ? make_plan(cd, ds0.subs) : FusedPlan{};
    uint4 *hbuf[2] = {ds0.hb, ds0.hb2};
    DecState ds = ds0;
    ds.slot_frame = nullptr;
    // compaction arenas: index 0 = ds0's buffers, 1 = ca's; slot_frame alternates between ca's two maps
    int arena = 0, n_compact = 0;
    const int T = ds0.tile_frames;
    layered = layered && layered_supported(cd);  // otherwise flooding (cvsr_decode_opts doc)
    if (!layered && smem_enabled() && !fused && decode_smem_bytes(cd) <= smem_limit() &&
        launch_decode_smem(cd, ds0, max_iter, qmax, bits_out, s))
        return check_launch(ctx, 1);
    CK(cudaMemsetAsync(ds0.counts + 3, 0, sizeof(int32_t), s));  // device iteration counter (k_status)
    prof_begin(ctx, KC_INIT);
    int launched = 0;
    if (layered) {  // r = 0, post = L (ds.L), decision 0 = [L < 0]
        if (!layers_zero_first()) CK(cudaMemsetAsync(ds.msg, 0, (size_t)ds.tiles * cd.E * T * sizeof(float), s));
        if (!hb_ready) {  // (the reconcile LLR kernel writes the initial decisions itself)
            launch_layer_init(cd, ds, ds.tiles, s);
            launched = 1;
        }
    } else {
        launched = launch_vn(cd, ds, ds.tiles, qmax, true, nullptr, s);  // decision 0 -> hbuf[0]
    }
    prof_end(ctx);
    int bound = ds.tiles;
    // Host look-ahead check (counts of iteration k - LOOKAHEAD + 1 are upper bounds of the
    // current ones) and frame compaction.  Returns false when every frame has stopped.  In the
    // per-pass path it runs between the status/retire of iteration k and VN_k, so the hard
    // decisions need not be moved (VN_k rewrites them for every active frame).
    auto check_and_compact = [&](int k, bool move_hb) -> bool {
        if (k < LOOKAHEAD) return true;
        if (cudaEventSynchronize(ctx->ring[(k - LOOKAHEAD + 1) % RING]) != cudaSuccess) return true;
        const int32_t na = hc[0];
        const int32_t lanes = hc[2];
        if (lanes == 0) return false;
        bound = std::min(bound, std::max(na, 1));
        // compaction: the active frames fill at most compact_frac of the active tiles
        if (ca && k < max_iter && na >= 2 && (double)lanes <= compact_frac() * (double)na * T &&
            na - (lanes + T - 1) / T >= compact_min_free()) {
            DecState dst = ds;
            if (arena == 0) {
                dst.msg = ca->msg;
                dst.L = ca->L;
                dst.hb = ca->hb;
                dst.st = ca->st;
            } else {
                dst.msg = ds0.msg;
                dst.L = ds0.L;
                dst.hb = ds0.hb;
                dst.st = ds0.st;
            }
            dst.slot_frame = ca->slot_frame[n_compact & 1];
            prof_begin(ctx, KC_CTRL);
            launched += launch_compact(cd, ds, dst, ca->dst_src, std::max(1, (lanes + T - 1) / T),
                                       ctx->host_counts_dev, move_hb, s);
            prof_end(ctx);
            ds = dst;
            arena ^= 1;
            ++n_compact;
            bound = std::max(1, (lanes + T - 1) / T);
        }
        return true;
    };
    int k = 1;
    if (layered) {
        // iteration k: syndrome test of decision k-1 (k_synd_test), status/retire, then the
        // layers (reading R-9); compaction moves r (msg), post (L), hb and st of active frames
        for (; k <= max_iter + 1; ++k) {
            const int final_pass = (k == max_iter + 1);
            prof_begin(ctx, KC_CN);
            launch_synd_test(cd, ds, bound, s);
            prof_end(ctx);
            prof_begin(ctx, KC_CTRL);
            launch_status(ds, k, max_iter, final_pass, ctx->host_counts_dev, s);
            launch_retire(ds, cd.n, bound, bits_out, s);
            prof_end(ctx);
            launched += 3;
            if (final_pass) {
                CK(cudaEventRecord(ctx->ring[k % RING], s));
                break;
            }
            if (!check_and_compact(k, true)) break;
            prof_begin(ctx, KC_VN);
            launched += launch_layers(cd, ds, bound, qmax, k == 1, s);
            prof_end(ctx);
            CK(cudaEventRecord(ctx->ring[k % RING], s));
        }
        return check_launch(ctx, launched);
    }
    // Small batches are launch-bound: capture GRAPH_ITERS plain iterations (CN, status with the
    // device iteration counter, retire, VN; grids sized for all tiles, kernels exit on the
    // device counts) once and replay the graph, checking the mapped counters one graph behind.
    const bool use_graph = graph_enabled() && !fused && !ca && !ctx->profiling && ds.tiles <= GRAPH_MAX_TILES &&
                           max_iter >= 2 * GRAPH_ITERS;
    if (use_graph) {
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
        // captured on a private stream (the context stream may be the legacy default stream,
        // which cannot capture); the graph is launched on the context stream
        if (!ctx->cap_stream) CK(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
        cudaStream_t cs = ctx->cap_stream;
        CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        for (int i = 0; i < GRAPH_ITERS; ++i) {
            launch_cn(cd, ds, ds.tiles, qmax, 0, cs);
            launch_status(ds, -1, max_iter, 0, ctx->host_counts_dev, cs);
            launch_retire(ds, cd.n, ds.tiles, bits_out, cs);
            launch_vn(cd, ds, ds.tiles, qmax, false, nullptr, cs);
        }
        const cudaError_t ce = cudaStreamEndCapture(cs, &graph);
        if (ce != cudaSuccess) return fail(CVSR_ECUDA, "graph capture: %s", cudaGetErrorString(ce));
        if (cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) {
            cudaGraphDestroy(graph);
            return fail(CVSR_ECUDA, "graph instantiate: %s", cudaGetErrorString(cudaGetLastError()));
        }
        bool done = false;
        int chunk = 0;
        while (k + GRAPH_ITERS - 1 <= max_iter) {
            CK(cudaGraphLaunch(exec, s));
            CK(cudaEventRecord(ctx->ring[chunk % RING], s));
            launched += GRAPH_ITERS * (3 + cd.n_vclass);
            k += GRAPH_ITERS;
            if (++chunk >= 2) {
                CK(cudaEventSynchronize(ctx->ring[(chunk - 2) % RING]));
                if (hc[2] == 0) {
                    done = true;
                    break;
                }
            }
        }
        CK(cudaStreamSynchronize(s));  // the graph objects may be freed once the replays finished
        cudaGraphExecDestroy(exec);
        cudaGraphDestroy(graph);
        if (done || hc[2] == 0) return check_launch(ctx, launched);
    }
    for (; k <= max_iter + 1; ++k) {
        const int final_pass = (k == max_iter + 1);
        if (fused && !final_pass) {
            // CN_k (tests decision k-1 in hbuf[(k-1)&1]) + per-tile status + VN_k (writes hbuf[k&1])
            DecState dsc = ds0, dsv = ds0;
            dsc.hb = hbuf[(k - 1) & 1];
            dsv.hb = hbuf[k & 1];
            prof_begin(ctx, KC_CN);
            launch_iter(cd, dsc, dsv, plan, k, qmax, s);
            prof_end(ctx);
            prof_begin(ctx, KC_CTRL);
            launch_list(dsc, ctx->host_counts_dev, s);
            launch_retire(dsc, cd.n, bound, bits_out, s);
            prof_end(ctx);
            launched += 3;
            CK(cudaEventRecord(ctx->ring[k % RING], s));
            if (!check_and_compact(k, true)) break;
            continue;
        }
        if (fused) ds.hb = hbuf[(k - 1) & 1];  // (per-pass path: ds.hb follows compaction)
        prof_begin(ctx, KC_CN);
        launch_cn(cd, ds, bound, qmax, final_pass, s);
        prof_end(ctx);
        prof_begin(ctx, KC_CTRL);
        launch_status(ds, k, max_iter, final_pass, ctx->host_counts_dev, s);
        launch_retire(ds, cd.n, bound, bits_out, s);
        prof_end(ctx);
        launched += 3;
        if (final_pass) {
            CK(cudaEventRecord(ctx->ring[k % RING], s));
            break;
        }
        if (!check_and_compact(k, fused)) break;
        prof_begin(ctx, KC_VN);
        launched += launch_vn(cd, ds, bound, qmax, false, nullptr, s);
        prof_end(ctx);
        CK(cudaEventRecord(ctx->ring[k % RING], s));
    }
    return check_launch(ctx, launched);
}

cvsr_status check_ctx(cvsr_ctx *ctx) {
    if (!ctx) return fail(CVSR_EINVAL, "null context");
    return CVSR_OK;
}

cvsr_status check_quantiser(const cvsr_quantiser *q) {
    if (!q) return fail(CVSR_EINVAL, "null quantiser");
    if (q->m < 1 || q->m > 8) return fail(CVSR_EINVAL, "quantiser m=%d outside [1,8]", q->m);
    const int ne = (1 << q->m) - 1;
    for (int i = 0; i < ne; ++i) {
        if (!(q->edges[i] == q->edges[i]) || q->edges[i] == INFINITY || q->edges[i] == -INFINITY)
            return fail(CVSR_EINVAL, "quantiser edge %d not finite", i);
        if (i > 0 && !(q->edges[i] > q->edges[i - 1]))
            return fail(CVSR_EINVAL, "quantiser edges not strictly ascending at %d", i);
    }
    return CVSR_OK;
}

}  // namespace

// internal accessors for session.cu (not part of the ABI)
cudaStream_t cvsr_internal_ctx_stream(cvsr_ctx *ctx) { return ctx->stream; }
cvsr_status cvsr_internal_fail(cvsr_status st, const char *msg) { return fail(st, "%s", msg); }
cvsr_status cvsr_internal_launched(cvsr_ctx *ctx, int n) { return check_launch(ctx, n); }
int cvsr_internal_ctx_device(cvsr_ctx *ctx) { return ctx->device; }

// =================================================================== ABI

extern "C" {

const char *cvsr_last_error(void) { return g_err.c_str(); }

int32_t cvsr_abi_version(void) { return CVSR_ABI_VERSION; }

cvsr_status cvsr_ctx_create(int32_t device, void *cuda_stream, cvsr_ctx **out) {
    if (!out) return fail(CVSR_EINVAL, "null out");
    *out = nullptr;
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(CVSR_EINVAL, "device %d not in [0,%d)", device, ndev);
    DeviceGuard g(device);
    if (!g.ok) return fail(CVSR_ECUDA, "cudaSetDevice(%d) failed", device);
    cvsr_ctx *c = new cvsr_ctx();
    c->device = device;
    c->stream = static_cast<cudaStream_t>(cuda_stream);
    cudaError_t e = cudaHostAlloc(reinterpret_cast<void **>(&c->host_counts), 16 * sizeof(int32_t),
                                  cudaHostAllocMapped);
    if (e == cudaSuccess) e = cudaHostGetDevicePointer(reinterpret_cast<void **>(&c->host_counts_dev), c->host_counts, 0);
    for (int i = 0; i < RING && e == cudaSuccess; ++i) e = cudaEventCreateWithFlags(&c->ring[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreate(&c->t0);
    if (e == cudaSuccess) e = cudaEventCreate(&c->t1);
    if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void **>(&c->acc), 32 * sizeof(unsigned long long));
    if (e != cudaSuccess) {
        cvsr_ctx_destroy(c);
        return fail(CVSR_ECUDA, "context setup: %s", cudaGetErrorString(e));
    }
    memset(c->host_counts, 0, 16 * sizeof(int32_t));
    *out = c;
    return CVSR_OK;
}

cvsr_status cvsr_ctx_set_stream(cvsr_ctx *ctx, void *cuda_stream) {
    if (cvsr_status st = check_ctx(ctx)) return st;
    ctx->stream = static_cast<cudaStream_t>(cuda_stream);
    return CVSR_OK;
}

cvsr_status cvsr_ctx_sync(cvsr_ctx *ctx) {
    if (cvsr_status st = check_ctx(ctx)) return st;
    DeviceGuard g(ctx->device);
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaGetLastError());
    return CVSR_OK;
}

int64_t cvsr_ctx_launch_count(const cvsr_ctx *ctx) { return ctx ? ctx->launches : -1; }

cvsr_status cvsr_ctx_set_profiling(cvsr_ctx *ctx, int32_t enable) {
    if (cvsr_status st = check_ctx(ctx)) return st;
    ctx->profiling = enable != 0;
    return CVSR_OK;
}

cvsr_status cvsr_ctx_kernel_times(cvsr_ctx *ctx, double *ms_out, int64_t *launches_out) {
    if (cvsr_status st = check_ctx(ctx)) return st;
    if (!ms_out || !launches_out) return fail(CVSR_EINVAL, "null output");
    DeviceGuard g(ctx->device);
    CK(cudaStreamSynchronize(ctx->stream));
    for (int c = 0; c < KC_N; ++c) {
        ms_out[c] = 0.0;
        launches_out[c] = 0;
    }
    for (const auto &pr : ctx->prof) {
        float ms = 0.0f;
        CK(cudaEventElapsedTime(&ms, ctx->ev_pool[pr.second], ctx->ev_pool[pr.second + 1]));
        ms_out[pr.first] += ms;
        launches_out[pr.first] += 1;
    }
    ctx->prof.clear();
    ctx->ev_used = 0;
    return CVSR_OK;
}

void cvsr_ctx_destroy(cvsr_ctx *ctx) {
    if (!ctx) return;
    DeviceGuard g(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    else cudaDeviceSynchronize();
    if (ctx->scratch) cudaFree(ctx->scratch);
    if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
    if (ctx->host_counts) cudaFreeHost(ctx->host_counts);
    for (int i = 0; i < RING; ++i)
        if (ctx->ring[i]) cudaEventDestroy(ctx->ring[i]);
    if (ctx->t0) cudaEventDestroy(ctx->t0);
    if (ctx->t1) cudaEventDestroy(ctx->t1);
    if (ctx->acc) cudaFree(ctx->acc);
    for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
    if (ctx->llr_tab) cudaFree(ctx->llr_tab);
    if (ctx->bob_bits) cudaFree(ctx->bob_bits);
    delete ctx;
}

cvsr_status cvsr_code_load(cvsr_ctx *ctx, int32_t n_vars, int32_t n_checks, const int32_t *row_ptr,
                           const int32_t *col_idx, cvsr_code **out) {
    if (cvsr_status st = check_ctx(ctx)) return st;
    if (!out || !row_ptr || (!col_idx && n_checks > 0)) return fail(CVSR_EINVAL, "null argument");
    *out = nullptr;
    if (n_vars <= 0 || n_checks <= 0) return fail(CVSR_EINVAL, "n_vars=%d n_checks=%d must be > 0", n_vars, n_checks);
    if (row_ptr[0] != 0) return fail(CVSR_ECODE, "row_ptr[0] = %d != 0", row_ptr[0]);
    for (int32_t c = 0; c < n_checks; ++c)
        if (row_ptr[c + 1] < row_ptr[c]) return fail(CVSR_ECODE, "row_ptr decreasing at %d", c);
    const int64_t E = row_ptr[n_checks];
    if (E <= 0) return fail(CVSR_ECODE, "matrix has no edges");
    std::vector<int32_t> col_cnt(n_vars + 1, 0);
    std::vector<int32_t> mark(n_vars, -1);
    int32_t max_dc = 0;
    for (int32_t c = 0; c < n_checks; ++c) {
        max_dc = std::max(max_dc, row_ptr[c + 1] - row_ptr[c]);
        if (row_ptr[c + 1] - row_ptr[c] > MAX_DC)
            return fail(CVSR_ECODE, "row %d has degree %d > %d (unsupported)", c, row_ptr[c + 1] - row_ptr[c], MAX_DC);
        for (int32_t e = row_ptr[c]; e < row_ptr[c + 1]; ++e) {
            const int32_t v = col_idx[e];
            if (v < 0 || v >= n_vars) return fail(CVSR_ECODE, "col_idx[%d] = %d out of range", e, v);
            if (mark[v] == c) return fail(CVSR_ECODE, "duplicate column %d in row %d", v, c);
            mark[v] = c;
            col_cnt[v + 1]++;
        }
    }
    // CSC by variable with the CSR position of each entry (edge permutation)
    std::vector<int32_t> col_ptr(n_vars + 1, 0);
    int32_t max_dv = 0;
    for (int32_t v = 0; v < n_vars; ++v) {
        col_ptr[v + 1] = col_ptr[v] + col_cnt[v + 1];
        max_dv = std::max(max_dv, col_cnt[v + 1]);
    }
    std::vector<int32_t> fill(col_ptr.begin(), col_ptr.end() - 1);
    std::vector<int32_t> csc_slot((size_t)E);
    for (int32_t c = 0; c < n_checks; ++c)
        for (int32_t e = row_ptr[c]; e < row_ptr[c + 1]; ++e) csc_slot[fill[col_idx[e]]++] = e;

    // degree classes: distinct degrees ascending; beyond MAX_VCLASS-1 distinct
    // degrees the remaining variables form one mixed class (generic VN path)
    std::vector<int32_t> degs;
    for (int32_t v = 0; v < n_vars; ++v) degs.push_back(col_cnt[v + 1]);
    std::vector<int32_t> distinct(degs);
    std::sort(distinct.begin(), distinct.end());
    distinct.erase(std::unique(distinct.begin(), distinct.end()), distinct.end());
    const int n_exact = (int)std::min<size_t>(distinct.size(), MAX_VCLASS - 1);
    const int n_cls = (int)distinct.size() <= MAX_VCLASS - 1 ? (int)distinct.size() : MAX_VCLASS;
    auto cls_of = [&](int32_t d) {
        const int i = (int)(std::lower_bound(distinct.begin(), distinct.end(), d) - distinct.begin());
        return i < n_exact ? i : MAX_VCLASS - 1;
    };
    std::vector<int32_t> vc_vars;
    vc_vars.reserve(n_vars);
    std::vector<int32_t> vc_slots;
    vc_slots.reserve((size_t)E);
    int32_t vc_deg[MAX_VCLASS], vc_off[MAX_VCLASS], vc_cnt[MAX_VCLASS];
    int64_t vc_soff[MAX_VCLASS];
    for (int k = 0; k < n_cls; ++k) {
        const int cls = (k < n_exact) ? k : MAX_VCLASS - 1;
        vc_deg[k] = (k < n_exact) ? distinct[k] : -1;
        vc_off[k] = (int32_t)vc_vars.size();
        vc_soff[k] = (int64_t)vc_slots.size();
        for (int32_t v = 0; v < n_vars; ++v) {
            if (cls_of(degs[v]) != cls) continue;
            vc_vars.push_back(v);
            for (int32_t p = col_ptr[v]; p < col_ptr[v + 1]; ++p) vc_slots.push_back(csc_slot[p]);
        }
        vc_cnt[k] = (int32_t)vc_vars.size() - vc_off[k];
    }

    // row-layered schedule (reading R-9): greedy colouring in check order, check c takes the
    // smallest colour not taken by an earlier check sharing a variable (bitmask per variable)
    std::vector<uint64_t> taken((size_t)n_vars, 0ull);
    std::vector<int32_t> colour((size_t)n_checks);
    int32_t n_layers = 0;
    for (int32_t c = 0; c < n_checks && n_layers >= 0; ++c) {
        uint64_t m = 0ull;
        for (int32_t e = row_ptr[c]; e < row_ptr[c + 1]; ++e) m |= taken[col_idx[e]];
        const int k = __builtin_ctzll(~m);
        if (k >= MAX_LAYERS) {
            n_layers = -1;  // too many colours: flooding only
            break;
        }
        colour[c] = k;
        for (int32_t e = row_ptr[c]; e < row_ptr[c + 1]; ++e) taken[col_idx[e]] |= 1ull << k;
        n_layers = std::max(n_layers, k + 1);
    }
    if (n_layers < 0) n_layers = 0;
    std::vector<int32_t> layer_off(MAX_LAYERS + 1, 0), layer_chk;
    if (n_layers > 0) {
        for (int32_t c = 0; c < n_checks; ++c) layer_off[colour[c] + 1]++;
        for (int l = 0; l < MAX_LAYERS; ++l) layer_off[l + 1] += layer_off[l];
        layer_chk.resize((size_t)n_checks);
        std::vector<int32_t> at(layer_off.begin(), layer_off.end() - 1);
        for (int32_t c = 0; c < n_checks; ++c) layer_chk[at[colour[c]]++] = c;
        // within a layer, checks by degree (descending, then index): the checks of a layer share no
        // variable, so their order is free; grouping equal degrees keeps a warp's consecutive checks
        // on one exact-degree body of k_layer_tma
        for (int l = 0; l < n_layers; ++l)
            std::stable_sort(layer_chk.begin() + layer_off[l], layer_chk.begin() + layer_off[l + 1],
                             [&](int32_t a, int32_t b) {
                                 return row_ptr[a + 1] - row_ptr[a] > row_ptr[b + 1] - row_ptr[b];
                             });
    }

    // layer-ordered check descriptors + padded column table (layered kernels; CodeDev comment)
    const int32_t ldc = n_layers > 0 ? layer_width(max_dc) : 0;
    std::vector<int32_t> ldesc, lcol;
    if (ldc > 0) {
        ldesc.resize((size_t)n_checks * 4);
        lcol.assign((size_t)n_checks * ldc, 0);
        for (int32_t i = 0; i < n_checks; ++i) {
            const int32_t c = layer_chk[i], lo = row_ptr[c], deg = row_ptr[c + 1] - lo;
            ldesc[(size_t)i * 4 + 0] = lo;
            ldesc[(size_t)i * 4 + 1] = deg;
            ldesc[(size_t)i * 4 + 2] = c;
            ldesc[(size_t)i * 4 + 3] = 0;
            for (int32_t k = 0; k < deg; ++k) lcol[(size_t)i * ldc + k] = col_idx[lo + k];
        }
    }
    DeviceGuard g(ctx->device);
    cvsr_code *code = new cvsr_code();
    code->device = ctx->device;
    const size_t b_rp = align_up((size_t)(n_checks + 1) * 4), b_ci = align_up((size_t)E * 4);
    const size_t b_cp = align_up((size_t)(n_vars + 1) * 4), b_cs = align_up((size_t)E * 4);
    const size_t b_vv = align_up((size_t)n_vars * 4), b_vs = align_up((size_t)E * 4);
    const size_t b_lc = align_up((size_t)n_checks * 4);
    const size_t b_ld = align_up(ldesc.size() * 4), b_lcol = align_up(lcol.size() * 4);
    const size_t b_lp = ldc > 0 ? b_lc : 0;
    cudaError_t e = cudaMalloc(&code->mem, b_rp + b_ci + b_cp + b_cs + b_vv + b_vs + b_lc + b_ld + b_lcol + b_lp);
    if (e != cudaSuccess) {
        delete code;
        cudaGetLastError();
        return fail(CVSR_ENOMEM, "code arrays: %s", cudaGetErrorString(e));
    }
    char *base = static_cast<char *>(code->mem);
    int32_t *d_rp = reinterpret_cast<int32_t *>(base);
    int32_t *d_ci = reinterpret_cast<int32_t *>(base + b_rp);
    int32_t *d_cp = reinterpret_cast<int32_t *>(base + b_rp + b_ci);
    int32_t *d_cs = reinterpret_cast<int32_t *>(base + b_rp + b_ci + b_cp);
    int32_t *d_vv = reinterpret_cast<int32_t *>(base + b_rp + b_ci + b_cp + b_cs);
    int32_t *d_vs = reinterpret_cast<int32_t *>(base + b_rp + b_ci + b_cp + b_cs + b_vv);
    cudaError_t e1 = cudaMemcpy(d_rp, row_ptr, (size_t)(n_checks + 1) * 4, cudaMemcpyHostToDevice);
    cudaError_t e2 = cudaMemcpy(d_ci, col_idx, (size_t)E * 4, cudaMemcpyHostToDevice);
    cudaError_t e3 = cudaMemcpy(d_cp, col_ptr.data(), (size_t)(n_vars + 1) * 4, cudaMemcpyHostToDevice);
    cudaError_t e4 = cudaMemcpy(d_cs, csc_slot.data(), (size_t)E * 4, cudaMemcpyHostToDevice);
    cudaError_t e5 = cudaMemcpy(d_vv, vc_vars.data(), (size_t)n_vars * 4, cudaMemcpyHostToDevice);
    cudaError_t e6 = cudaMemcpy(d_vs, vc_slots.data(), (size_t)E * 4, cudaMemcpyHostToDevice);
    int32_t *d_lc = reinterpret_cast<int32_t *>(base + b_rp + b_ci + b_cp + b_cs + b_vv + b_vs);
    if (e6 == cudaSuccess && n_layers > 0)
        e6 = cudaMemcpy(d_lc, layer_chk.data(), (size_t)n_checks * 4, cudaMemcpyHostToDevice);
    int4 *d_ld = reinterpret_cast<int4 *>(base + b_rp + b_ci + b_cp + b_cs + b_vv + b_vs + b_lc);
    int32_t *d_lcol = reinterpret_cast<int32_t *>(base + b_rp + b_ci + b_cp + b_cs + b_vv + b_vs + b_lc + b_ld);
    if (e6 == cudaSuccess && ldc > 0) e6 = cudaMemcpy(d_ld, ldesc.data(), ldesc.size() * 4, cudaMemcpyHostToDevice);
    if (e6 == cudaSuccess && ldc > 0) e6 = cudaMemcpy(d_lcol, lcol.data(), lcol.size() * 4, cudaMemcpyHostToDevice);
    int32_t *d_lp = reinterpret_cast<int32_t *>(base + b_rp + b_ci + b_cp + b_cs + b_vv + b_vs + b_lc + b_ld + b_lcol);
    if (e6 == cudaSuccess && ldc > 0) {
        std::vector<int32_t> lpos((size_t)n_checks);
        for (int32_t i = 0; i < n_checks; ++i) lpos[layer_chk[i]] = i;
        e6 = cudaMemcpy(d_lp, lpos.data(), (size_t)n_checks * 4, cudaMemcpyHostToDevice);
    }
    if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess || e4 != cudaSuccess || e5 != cudaSuccess ||
        e6 != cudaSuccess) {
        cudaFree(code->mem);
        delete code;
        return fail(CVSR_ECUDA, "code upload failed");
    }
    CodeDev d{};
    d.n = n_vars;
    d.M = n_checks;
    d.E = E;
    d.row_ptr = d_rp;
    d.col_idx = d_ci;
    d.col_ptr = d_cp;
    d.csc_slot = d_cs;
    d.max_dc = max_dc;
    d.max_dv = max_dv;
    d.vc_vars = d_vv;
    d.vc_slots = d_vs;
    d.n_vclass = n_cls;
    for (int k = 0; k < MAX_VCLASS; ++k) {
        d.vc_deg[k] = k < n_cls ? vc_deg[k] : 0;
        d.vc_off[k] = k < n_cls ? vc_off[k] : 0;
        d.vc_cnt[k] = k < n_cls ? vc_cnt[k] : 0;
        d.vc_soff[k] = k < n_cls ? vc_soff[k] : 0;
    }
    d.layer_chk = d_lc;
    d.n_layers = n_layers;
    d.layer_desc = ldc > 0 ? d_ld : nullptr;
    d.layer_col = ldc > 0 ? d_lcol : nullptr;
    d.layer_pos = ldc > 0 ? d_lp : nullptr;
    d.layer_dc = ldc;
    for (int l = 0; l <= MAX_LAYERS; ++l) d.layer_off[l] = layer_off[l];
    for (int l = 0; l < MAX_LAYERS; ++l) {
        int32_t nb = 0;
        if (l < n_layers)
            for (int32_t i = layer_off[l]; i < layer_off[l + 1]; ++i)
                nb += (row_ptr[layer_chk[i] + 1] - row_ptr[layer_chk[i]]) > 2;
        d.layer_nbig[l] = nb;
    }
    code->d = d;
    *out = code;
    return CVSR_OK;
}

cvsr_status cvsr_code_info(const cvsr_code *code, int32_t *n_vars, int32_t *n_checks, int64_t *n_edges) {
    if (!code) return fail(CVSR_EINVAL, "null code");
    if (n_vars) *n_vars = code->d.n;
    if (n_checks) *n_checks = code->d.M;
    if (n_edges) *n_edges = code->d.E;
    return CVSR_OK;
}

void cvsr_code_free(cvsr_code *code) {
    if (!code) return;
    DeviceGuard g(code->device);
    cudaDeviceSynchronize();
    cudaFree(code->mem);
    delete code;
}

cvsr_status cvsr_quantise(cvsr_ctx *ctx, const cvsr_quantiser *q, const float *y, int64_t count, uint8_t *label_out) {
    if (cvsr_status st = check_ctx(ctx)) return st;
    if (cvsr_status st = check_quantiser(q)) return st;
    if (count < 0) return fail(CVSR_ESHAPE, "count < 0");
    if (count == 0) return CVSR_OK;
    if (!y || !label_out) return fail(CVSR_EINVAL, "null buffer");
    DeviceGuard g(ctx->device);
    launch_quantise(q->edges, q->m, y, count, label_out, ctx->stream);
    return check_launch(ctx, 1);
}

cvsr_status cvsr_slice_bits(cvsr_ctx *ctx, const uint8_t *label, int32_t frames, int32_t n, int32_t slice_j,
                            uint32_t *bits_out) {
    if (cvsr_status st = check_ctx(ctx)) return st;
    if (frames < 0 || n <= 0) return fail(CVSR_ESHAPE, "frames=%d n=%d", frames, n);
    if (slice_j < 0 || slice_j > 7) return fail(CVSR_EINVAL, "slice_j=%d", slice_j);
    if (frames == 0) return CVSR_OK;
    if (!label || !bits_out) return fail(CVSR_EINVAL, "null buffer");
    DeviceGuard g(ctx->device);
    launch_slice_bits(label, frames, n, slice_j, bits_out, ctx->stream);
    return check_launch(ctx, 1);
}

cvsr_status cvsr_syndrome(cvsr_ctx *ctx, const cvsr_code *code, const uint8_t *label, int32_t frames,
                          int32_t slice_j, uint32_t *synd_out) {
    if (cvsr_status st = check_ctx(ctx)) return st;
    if (!code) return fail(CVSR_EINVAL, "null code");
    if (code->device != ctx->device) return fail(CVSR_EINVAL, "code and context on different devices");
    if (frames < 0) return fail(CVSR_ESHAPE, "frames < 0");
    if (slice_j < 0 || slice_j > 7) return fail(CVSR_EINVAL, "slice_j=%d", slice_j);
    if (frames == 0) return CVSR_OK;
    if (!label || !synd_out) return fail(CVSR_EINVAL, "null buffer");
    DeviceGuard g(ctx->device);
    // pack S_j first (coalesced), then the bit-sliced transpose of the packed rows and one 16-byte
    // gather per edge for 128 frames (launch_syndrome_bits)
    const size_t bits_bytes = (((size_t)frames * words_of(code->d.n) * sizeof(uint32_t)) + 255) & ~(size_t)255;
    const size_t need = bits_bytes + (size_t)code->d.n * syndrome_sliced_groups(frames) * sizeof(uint32_t);
    if (need > ctx->bob_bits_cap) {
        CK(cudaStreamSynchronize(ctx->stream));
        if (ctx->bob_bits) CK(cudaFree(ctx->bob_bits));
        ctx->bob_bits = nullptr;
        ctx->bob_bits_cap = 0;
        cudaError_t e = cudaMalloc(reinterpret_cast<void **>(&ctx->bob_bits), need);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(CVSR_ENOMEM, "syndrome scratch: %s", cudaGetErrorString(e));
        }
        ctx->bob_bits_cap = need;
    }
    launch_slice_bits(label, frames, code->d.n, slice_j, ctx->bob_bits, ctx->stream);
    uint32_t *sliced = reinterpret_cast<uint32_t *>(reinterpret_cast<unsigned char *>(ctx->bob_bits) + bits_bytes);
    const int k = launch_syndrome_bits(code->d, ctx->bob_bits, frames, synd_out, sliced, ctx->stream);
    return check_launch(ctx, 1 + k);
}

// builds the LLR table for p on the context stream (p.table stays null when the grid
// would be too coarse for sigma_n; the kernels then evaluate exactly)
static cvsr_status prepare_llr_table(cvsr_ctx *ctx, LlrParams &p, int *launched) {
    p.table = nullptr;
    p.table4 = nullptr;
    const size_t combos = (size_t)1 << __builtin_popcount(p.known_mask);
    const size_t scalar_bytes = (combos * LLR_NTAB * sizeof(float) + 255) & ~(size_t)255;
    const size_t need = scalar_bytes + combos * LLR_NWIN * sizeof(float4);
    if (need > ctx->llr_tab_cap) {
        CK(cudaStreamSynchronize(ctx->stream));
        if (ctx->llr_tab) CK(cudaFree(ctx->llr_tab));
        ctx->llr_tab = nullptr;
        ctx->llr_tab_cap = 0;
        cudaError_t e = cudaMalloc(reinterpret_cast<void **>(&ctx->llr_tab), need);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(CVSR_ENOMEM, "LLR table: %s", cudaGetErrorString(e));
        }
        ctx->llr_tab_cap = need;
    }
    float4 *win = reinterpret_cast<float4 *>(reinterpret_cast<unsigned char *>(ctx->llr_tab) + scalar_bytes);
    if (launch_llr_table(p, ctx->llr_tab, win, ctx->stream)) {
        p.table = ctx->llr_tab;
        p.table4 = win;
        *launched += 2;
    }
    return CVSR_OK;
}

static void fill_llr_params(LlrParams &p, const cvsr_quantiser *q, int j, uint32_t mask, float sigma_n, float llr_max) {
    memset(&p, 0, sizeof(p));
    p.m = q->m;
    p.j = j;
    p.known_mask = mask;
    for (int jj = 0; jj < q->m; ++jj)
        if ((mask >> jj) & 1u) p.kj[p.nk++] = jj;
    p.sigma_n = sigma_n;
    p.inv_sigma = 1.0f / sigma_n;
    p.llr_max = llr_max;
    for (int i = 0; i < (1 << q->m) - 1; ++i) p.edges[i] = q->edges[i];
}

cvsr_status cvsr_llr_slice(cvsr_ctx *ctx, const cvsr_quantiser *q, const float *x, int32_t frames, int32_t n,
                           float sigma_n, int32_t slice_j, uint32_t known_mask, const uint8_t *known_label,
                           float llr_max, float *llr_out) {
    if (cvsr_status st = check_ctx(ctx)) return st;
    if (cvsr_status st = check_quantiser(q)) return st;
    if (frames < 0 || n <= 0) return fail(CVSR_ESHAPE, "frames=%d n=%d", frames, n);
    if (slice_j < 0 || slice_j >= q->m) return fail(CVSR_EINVAL, "slice_j=%d not in [0,m)", slice_j);
    if ((known_mask >> slice_j) & 1u) return fail(CVSR_EINVAL, "known_mask contains slice_j");
    if (known_mask >> q->m) return fail(CVSR_EINVAL, "known_mask has bits >= m");
    if (known_mask && !known_label) return fail(CVSR_EINVAL, "known_label required when known_mask != 0");
    if (!(sigma_n > 0.0f) || !(llr_max > 0.0f)) return fail(CVSR_EINVAL, "sigma_n and llr_max must be > 0");
    if (frames == 0) return CVSR_OK;
    if (!x || !llr_out) return fail(CVSR_EINVAL, "null buffer");
    DeviceGuard g(ctx->device);
    LlrParams p;
    fill_llr_params(p, q, slice_j, known_mask, sigma_n, llr_max);
    int launched = 1;
    if (cvsr_status st = prepare_llr_table(ctx, p, &launched)) return st;
    launch_llr_slice(p, x, known_label, frames, n, llr_out, ctx->stream);
    return check_launch(ctx, launched);
}

cvsr_status cvsr_llr_biawgn(cvsr_ctx *ctx, const float *y, int64_t count, float sigma2, float llr_max,
                            float *llr_out) {
    if (cvsr_status st = check_ctx(ctx)) return st;
    if (count < 0) return fail(CVSR_ESHAPE, "count < 0");
    if (!(sigma2 > 0.0f) || !(llr_max > 0.0f)) return fail(CVSR_EINVAL, "sigma2 and llr_max must be > 0");
    if (count == 0) return CVSR_OK;
    if (!y || !llr_out) return fail(CVSR_EINVAL, "null buffer");
    DeviceGuard g(ctx->device);
    launch_llr_biawgn(y, count, sigma2, llr_max, llr_out, ctx->stream);
    return check_launch(ctx, 1);
}

static cvsr_status check_opts(const cvsr_decode_opts *o) {
    if (!o) return fail(CVSR_EINVAL, "null decode opts");
    if (o->max_iter < 0 || o->max_iter > 1000000) return fail(CVSR_EINVAL, "max_iter=%d", o->max_iter);
    if (!(o->msg_clamp > 0.0f)) return fail(CVSR_EINVAL, "msg_clamp must be > 0");
    if ((o->flags & ~CVSR_SCHED_MASK) || (o->flags & CVSR_SCHED_MASK) == CVSR_SCHED_MASK)
        return fail(CVSR_EINVAL, "flags=%d: unknown bits", o->flags);
    return CVSR_OK;
}

cvsr_status cvsr_decode(cvsr_ctx *ctx, const cvsr_code *code, const float *llr, const uint32_t *synd,
                        int32_t frames, const cvsr_decode_opts *opts, uint32_t *bits_out, uint8_t *converged_out,
                        int32_t *iters_out) {
    if (cvsr_status st = check_ctx(ctx)) return st;
    if (!code) return fail(CVSR_EINVAL, "null code");
    if (code->device != ctx->device) return fail(CVSR_EINVAL, "code and context on different devices");
    if (cvsr_status st = check_opts(opts)) return st;
    if (frames < 0) return fail(CVSR_ESHAPE, "frames < 0");
    if (frames == 0) return CVSR_OK;
    if (!llr || !synd || !bits_out || !converged_out || !iters_out) return fail(CVSR_EINVAL, "null buffer");
    DeviceGuard g(ctx->device);
    const CodeDev &cd = code->d;
    const bool layered = layered_requested(opts->flags) && layered_supported(cd);
    const int subs = pick_subs(frames, cd.E, layered, cd.max_dc);
    const int tiles = tiles_for(frames, subs);
    const bool comp = compact_enabled() && tiles >= 1 + compact_min_free();
    char *base;
    if (cvsr_status st = scratch_reserve(ctx, decstate_bytes(tiles, frames, subs, cd.n, cd.M, cd.E) +
                                                  (comp ? compact_bytes(tiles, subs, cd.n, cd.M, cd.E) : 0),
                                         &base))
        return st;
    Carve cv{base};
    DecState ds = carve_decstate(cv, tiles, frames, subs, cd.n, cd.M, cd.E, iters_out, converged_out);
    CompactArena ca;
    if (comp) ca = carve_compact(cv, tiles, subs, cd.n, cd.M, cd.E);
    cudaStream_t s = ctx->stream;
    launch_to_interleaved(llr, ds.L, frames, cd.n, tiles, ds.subs, LOG2E, s);
    launch_synd_transpose(synd, frames, cd.M, ds.subs, ds.st, tiles, layered ? cd.layer_pos : nullptr, s);
    launch_init_tiles(ds, nullptr, s);
    launch_set_counts(ds, tiles, s);
    if (cvsr_status st = check_launch(ctx, 4)) return st;
    return run_decode(ctx, code, ds, opts->max_iter, opts->msg_clamp, bits_out, comp ? &ca : nullptr, layered);
}

cvsr_status cvsr_decode_trace(cvsr_ctx *ctx, const cvsr_code *code, const float *llr, const uint32_t *synd,
                              int32_t frames, int32_t k_iters, float msg_clamp, int32_t flags, float *c2v_out,
                              float *post_out) {
    if (cvsr_status st = check_ctx(ctx)) return st;
    if (!code) return fail(CVSR_EINVAL, "null code");
    if (code->device != ctx->device) return fail(CVSR_EINVAL, "code and context on different devices");
    if (k_iters < 1) return fail(CVSR_EINVAL, "k_iters must be >= 1");
    if (!(msg_clamp > 0.0f)) return fail(CVSR_EINVAL, "msg_clamp must be > 0");
    if ((flags & ~CVSR_SCHED_MASK) || (flags & CVSR_SCHED_MASK) == CVSR_SCHED_MASK)
        return fail(CVSR_EINVAL, "flags=%d: unknown bits", flags);
    const CodeDev &cd = code->d;
    const bool layered = layered_requested(flags);
    if (layered && !layered_supported(cd))
        return fail(CVSR_EINVAL, "layered trace: code needs more than %d layers or has check degree %d > 12",
                    MAX_LAYERS, cd.max_dc);
    if (frames < 0) return fail(CVSR_ESHAPE, "frames < 0");
    if (frames == 0) return CVSR_OK;
    if (!llr || !synd) return fail(CVSR_EINVAL, "null buffer");
    DeviceGuard g(ctx->device);
    const int subs = layered ? pick_subs(frames, cd.E, true, cd.max_dc) : choose_subs(frames);
    const int tiles = tiles_for(frames, subs);
    const size_t post_bytes = align_up((size_t)tiles * cd.n * LANES * subs * sizeof(float));
    char *base;
    if (cvsr_status st = scratch_reserve(ctx, decstate_bytes(tiles, frames, subs, cd.n, cd.M, cd.E) + post_bytes, &base))
        return st;
    Carve cv{base};
    DecState ds = carve_decstate(cv, tiles, frames, subs, cd.n, cd.M, cd.E, nullptr, nullptr);
    float *post_il = cv.take<float>(post_bytes);
    cudaStream_t s = ctx->stream;
    launch_to_interleaved(llr, ds.L, frames, cd.n, tiles, ds.subs, LOG2E, s);
    launch_synd_transpose(synd, frames, cd.M, ds.subs, ds.st, tiles, layered ? cd.layer_pos : nullptr, s);
    launch_init_tiles(ds, nullptr, s);
    launch_set_counts(ds, tiles, s);
    int launched = 4;
    if (layered) {
        // r = 0, post = L; k sweeps over the layers; r_e is in ds.msg (CSR slots), post_v in ds.L
        if (!layers_zero_first()) CK(cudaMemsetAsync(ds.msg, 0, (size_t)tiles * cd.E * LANES * subs * sizeof(float), s));
        launch_layer_init(cd, ds, tiles, s);
        ++launched;
        for (int k = 1; k <= k_iters; ++k) launched += launch_layers(cd, ds, tiles, msg_clamp, k == 1, s);
        if (c2v_out) {
            launch_from_interleaved(ds.msg, c2v_out, frames, cd.E, tiles, ds.subs, LN2, s);
            ++launched;
        }
        if (post_out) {
            launch_from_interleaved(ds.L, post_out, frames, cd.n, tiles, ds.subs, LN2, s);
            ++launched;
        }
        return check_launch(ctx, launched);
    }
    launched += launch_vn(cd, ds, tiles, msg_clamp, true, nullptr, s);
    for (int k = 1; k <= k_iters; ++k) {
        launch_cn(cd, ds, tiles, msg_clamp, 0, s);
        ++launched;
        if (k == k_iters && c2v_out) {
            launch_from_interleaved(ds.msg, c2v_out, frames, cd.E, tiles, ds.subs, LN2, s);
            ++launched;
        }
        launched += launch_vn(cd, ds, tiles, msg_clamp, false, (k == k_iters) ? post_il : nullptr, s);
    }
    if (post_out) {
        launch_from_interleaved(post_il, post_out, frames, cd.n, tiles, ds.subs, LN2, s);
        ++launched;
    }
    return check_launch(ctx, launched);
}

cvsr_status cvsr_reconcile(cvsr_ctx *ctx, int32_t m, const cvsr_code *const *codes, const int32_t *order,
                           const cvsr_quantiser *q, float sigma_n, const float *x, const uint32_t *const *synd,
                           int32_t frames, int32_t n, const cvsr_decode_opts *opts, uint8_t *label_out,
                           uint8_t *frame_ok, int32_t *iters, cvsr_stats *stats_out) {
    if (cvsr_status st = check_ctx(ctx)) return st;
    if (cvsr_status st = check_quantiser(q)) return st;
    if (cvsr_status st = check_opts(opts)) return st;
    if (m < 1 || m > 8 || m != q->m) return fail(CVSR_EINVAL, "m=%d must be in [1,8] and equal quantiser m", m);
    if (!codes || !order || !synd) return fail(CVSR_EINVAL, "null codes/order/synd array");
    if (frames < 0 || n <= 0) return fail(CVSR_ESHAPE, "frames=%d n=%d", frames, n);
    if (!(sigma_n > 0.0f)) return fail(CVSR_EINVAL, "sigma_n must be > 0");
    uint32_t seen = 0u;
    for (int t = 0; t < m; ++t) {
        const int j = order[t];
        if (j < 0 || j >= m || ((seen >> j) & 1u)) return fail(CVSR_EINVAL, "order is not a permutation of 0..m-1");
        seen |= 1u << j;
    }
    for (int j = 0; j < m; ++j) {
        if (codes[j]) {
            if (codes[j]->device != ctx->device) return fail(CVSR_EINVAL, "code %d on another device", j);
            if (codes[j]->d.n != n) return fail(CVSR_ESHAPE, "code %d has n=%d, expected %d", j, codes[j]->d.n, n);
        }
        if (frames > 0 && !synd[j]) return fail(CVSR_EINVAL, "synd[%d] is null", j);
    }
    if (frames == 0) {
        if (stats_out) memset(stats_out, 0, sizeof(*stats_out));
        return CVSR_OK;
    }
    if (!x || !label_out || !frame_ok || !iters) return fail(CVSR_EINVAL, "null buffer");
    DeviceGuard g(ctx->device);
    // per coded slice: the schedule that runs (layered falls back to flooding for codes it does not
    // support), frames per lane and decoder state size; the decoder state of every slice is carved
    // from the same region after the per-call buffers
    const bool want_layered = layered_requested(opts->flags);
    bool lay_j[8] = {};
    int subs_j[8] = {}, tiles_j[8] = {};
    bool comp_j[8] = {};
    size_t dec_bytes = 0;
    for (int j = 0; j < m; ++j) {
        if (!codes[j]) continue;
        const CodeDev &cd = codes[j]->d;
        lay_j[j] = want_layered && layered_supported(cd);
        subs_j[j] = pick_subs(frames, cd.E, lay_j[j], cd.max_dc);
        tiles_j[j] = tiles_for(frames, subs_j[j]);
        comp_j[j] = compact_enabled() && tiles_j[j] >= 1 + compact_min_free();
        size_t b = decstate_bytes(tiles_j[j], frames, subs_j[j], n, cd.M, cd.E);
        if (comp_j[j]) b += compact_bytes(tiles_j[j], subs_j[j], n, cd.M, cd.E);
        dec_bytes = std::max(dec_bytes, b);
    }
    const int Wn = words_of(n);
    size_t bytes = (size_t)m * align_up((size_t)frames * Wn * 4) + 3 * align_up((size_t)frames) +
                   align_up((size_t)frames * sizeof(int32_t)) + align_up((size_t)frames);
    bytes += dec_bytes;
    char *base;
    if (cvsr_status st = scratch_reserve(ctx, bytes, &base)) return st;
    Carve cv{base};
    uint32_t *bits_dec[8] = {};
    for (int j = 0; j < m; ++j) bits_dec[j] = cv.take<uint32_t>((size_t)frames * Wn * 4);
    uint8_t *alive = cv.take<uint8_t>((size_t)frames);
    uint8_t *attempt = cv.take<uint8_t>((size_t)2 * frames);
    int32_t *dec_iters = cv.take<int32_t>((size_t)frames * sizeof(int32_t));
    uint8_t *dec_conv = cv.take<uint8_t>((size_t)frames);
    char *dec_base = base + cv.off;
    DecState ds0{};  // frame count for the hand-off of disclosed slices
    ds0.frames = frames;
    ds0.iters = dec_iters;
    ds0.conv = dec_conv;
    cudaStream_t s = ctx->stream;
    CK(cudaEventRecord(ctx->t0, s));
    launch_fill_i32(iters, (int64_t)frames * m, -1, s);
    launch_fill_u8(alive, frames, 1, s);
    launch_fill_u8(attempt, 2 * (int64_t)frames, 0, s);
    int launched = 3;
    const uint32_t *known_bits[8] = {};
    uint32_t known_mask = 0u;
    for (int t = 0; t < m; ++t) {
        const int j = order[t];
        if (!codes[j]) {
            launch_slice_done(ds0, m, j, 1, alive, attempt, iters, s);
            ++launched;
            known_bits[j] = synd[j];
        } else {
            const CodeDev &cd = codes[j]->d;
            Carve cvd{dec_base};
            DecState ds = carve_decstate(cvd, tiles_j[j], frames, subs_j[j], n, cd.M, cd.E, dec_iters, dec_conv);
            CompactArena ca;
            if (comp_j[j]) ca = carve_compact(cvd, tiles_j[j], subs_j[j], n, cd.M, cd.E);
            CK(cudaMemsetAsync(bits_dec[j], 0, (size_t)frames * Wn * 4, s));
            launch_init_tiles(ds, alive, s);
            launch_set_counts(ds, tiles_j[j], s);
            launch_synd_transpose(synd[j], frames, cd.M, ds.subs, ds.st, tiles_j[j], lay_j[j] ? cd.layer_pos : nullptr,
                                  s);
            LlrParams p;
            fill_llr_params(p, q, j, known_mask, sigma_n, opts->msg_clamp);
            for (int jj = 0; jj < m; ++jj) p.known_bits[jj] = known_bits[jj];
            prof_begin(ctx, KC_INIT);
            if (cvsr_status st = prepare_llr_table(ctx, p, &launched)) return st;
            launch_llr_interleaved(p, x, frames, n, tiles_j[j], ds.subs, ds.L, lay_j[j] ? ds.hb : nullptr,
                                   ds.tile_active, s);
            prof_end(ctx);
            launched += 4;
            if (cvsr_status st = check_launch(ctx, 0)) return st;
            if (cvsr_status st = run_decode(ctx, codes[j], ds, opts->max_iter, opts->msg_clamp, bits_dec[j],
                                            comp_j[j] ? &ca : nullptr, lay_j[j], lay_j[j]))
                return st;
            launch_slice_done(ds, m, j, 0, alive, attempt, iters, s);
            ++launched;
            known_bits[j] = bits_dec[j];
        }
        known_mask |= 1u << j;
    }
    launch_assemble(known_bits, m, attempt, frames, n, label_out, s);
    CK(cudaMemcpyAsync(frame_ok, alive, (size_t)frames, cudaMemcpyDeviceToDevice, s));
    ++launched;
    CK(cudaEventRecord(ctx->t1, s));
    if (cvsr_status st = check_launch(ctx, launched)) return st;
    if (stats_out) {
        CK(cudaMemsetAsync(ctx->acc, 0, 32 * sizeof(unsigned long long), s));
        launch_frame_stats(alive, attempt, iters, frames, m, ctx->acc, s);
        if (cvsr_status st = check_launch(ctx, 1)) return st;
        unsigned long long acc[32];
        CK(cudaMemcpyAsync(acc, ctx->acc, sizeof(acc), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        memset(stats_out, 0, sizeof(*stats_out));
        stats_out->frames = frames;
        stats_out->frames_ok = (int64_t)acc[0];
        stats_out->bits_reconciled = (int64_t)acc[0] * m * (int64_t)n;
        for (int j = 0; j < m; ++j) {
            stats_out->attempted[j] = (int64_t)acc[1 + j];
            stats_out->converged[j] = (int64_t)acc[9 + j];
            stats_out->iters_sum[j] = (int64_t)acc[17 + j];
            stats_out->edge_iters[j] = codes[j] ? (int64_t)acc[17 + j] * codes[j]->d.E : 0;
            stats_out->schedule[j] = codes[j] ? (lay_j[j] ? CVSR_SCHED_LAYERED : CVSR_SCHED_FLOODING) : 0;
        }
        float ms = 0.0f;
        CK(cudaEventElapsedTime(&ms, ctx->t0, ctx->t1));
        stats_out->alice_seconds = ms * 1e-3;
    }
    return CVSR_OK;
}

cvsr_status cvsr_frame_hash(cvsr_ctx *ctx, const uint8_t *label, int32_t frames, int32_t n, uint64_t key,
                            uint64_t *hash_out) {
    if (cvsr_status st = check_ctx(ctx)) return st;
    if (frames < 0 || n <= 0) return fail(CVSR_ESHAPE, "frames=%d n=%d", frames, n);
    if (key == 0 || key >= ((1ull << 61) - 1ull)) return fail(CVSR_EINVAL, "key must be in [1, 2^61 - 2]");
    if (frames == 0) return CVSR_OK;
    if (!label || !hash_out) return fail(CVSR_EINVAL, "null buffer");
    DeviceGuard g(ctx->device);
    launch_frame_hash(label, frames, n, key, reinterpret_cast<unsigned long long *>(hash_out), ctx->stream);
    return check_launch(ctx, 1);
}

cvsr_status cvsr_verify(cvsr_ctx *ctx, const uint8_t *label_alice, const uint8_t *label_bob, const uint8_t *frame_ok,
                        int32_t frames, int32_t n, const uint64_t *keys, uint8_t *verified_out, uint64_t *hash_alice_out,
                        uint64_t *hash_bob_out) {
    if (cvsr_status st = check_ctx(ctx)) return st;
    if (frames < 0 || n <= 0) return fail(CVSR_ESHAPE, "frames=%d n=%d", frames, n);
    if (!keys) return fail(CVSR_EINVAL, "null keys");
    for (int q = 0; q < CVSR_HASH_KEYS; ++q)
        if (keys[q] == 0 || keys[q] >= ((1ull << 61) - 1ull)) return fail(CVSR_EINVAL, "key %d not in [1, 2^61 - 2]", q);
    if (frames == 0) return CVSR_OK;
    if (!label_alice || !label_bob || !frame_ok || !verified_out) return fail(CVSR_EINVAL, "null buffer");
    DeviceGuard g(ctx->device);
    unsigned long long k[CVSR_HASH_KEYS];
    for (int q = 0; q < CVSR_HASH_KEYS; ++q) k[q] = keys[q];
    launch_verify(label_alice, label_bob, frame_ok, frames, n, k, verified_out,
                  reinterpret_cast<unsigned long long *>(hash_alice_out),
                  reinterpret_cast<unsigned long long *>(hash_bob_out), ctx->stream);
    return check_launch(ctx, 1);
}

cvsr_status cvsr_count_errors(cvsr_ctx *ctx, const uint8_t *label_alice, const uint8_t *label_bob,
                              const uint8_t *frame_ok, int32_t frames, int32_t n, int64_t *counts_out) {
    if (cvsr_status st = check_ctx(ctx)) return st;
    if (!counts_out) return fail(CVSR_EINVAL, "null counts_out");
    if (frames < 0 || n <= 0) return fail(CVSR_ESHAPE, "frames=%d n=%d", frames, n);
    counts_out[0] = counts_out[1] = counts_out[2] = 0;
    if (frames == 0) return CVSR_OK;
    if (!label_alice || !label_bob || !frame_ok) return fail(CVSR_EINVAL, "null buffer");
    DeviceGuard g(ctx->device);
    cudaStream_t s = ctx->stream;
    CK(cudaMemsetAsync(ctx->acc, 0, 4 * sizeof(unsigned long long), s));
    launch_count_errors(label_alice, label_bob, frame_ok, frames, n, ctx->acc, s);
    if (cvsr_status st = check_launch(ctx, 1)) return st;
    unsigned long long acc[4];
    CK(cudaMemcpyAsync(acc, ctx->acc, sizeof(acc), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (int i = 0; i < 3; ++i) counts_out[i] = (int64_t)acc[i];
    return CVSR_OK;
}

}  // extern "C"
