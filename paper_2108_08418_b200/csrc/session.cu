// Whole-step session (include/cvsr.h "session"): device buffers for one batch
// plus Bob (quantise, syndromes / disclosed bits) and Alice (cvsr_reconcile)
// in one call, optionally from and to HOST buffers.
#include <string.h>

#include <cuda_runtime.h>

#include "common.cuh"

struct cvsr_session {
    cvsr_ctx *ctx = nullptr;
    int device = 0;
    int32_t m = 0, n = 0, frames = 0;
    const cvsr_code *codes[8] = {};
    int32_t order[8] = {};
    int32_t n_checks[8] = {};
    cvsr_quantiser q{};
    float sigma_n = 0.0f;
    cvsr_decode_opts opts{};
    bool verify = false;               // frame_ok &= hash check under verify_keys (cvsr_session_set_verify)
    uint64_t verify_keys[CVSR_HASH_KEYS] = {};
    void *mem = nullptr;
    cudaStream_t copy = nullptr;       // H2D / D2H stream of run_host
    cudaEvent_t ev_in[8] = {}, ev_out[8] = {};
    float *x = nullptr, *y = nullptr;
    uint8_t *label_bob = nullptr, *label_alice = nullptr, *frame_ok = nullptr;
    int32_t *iters = nullptr;
    uint32_t *synd[8] = {};
    // second input/output set + D2H stream of cvsr_session_run_host_stream (allocated on first use)
    void *mem2 = nullptr;
    float *x2 = nullptr, *y2 = nullptr;
    uint8_t *label_alice2 = nullptr, *frame_ok2 = nullptr;
    int32_t *iters2 = nullptr;
    cudaStream_t copy_out = nullptr;
    cudaEvent_t ev_done[2] = {}, ev_d2h[2] = {};
};

namespace {
size_t al(size_t b) { return (b + 255) & ~size_t(255); }
}  // namespace

cudaStream_t cvsr_internal_ctx_stream(cvsr_ctx *ctx);          // api.cu
cvsr_status cvsr_internal_fail(cvsr_status st, const char *msg);  // api.cu (sets cvsr_last_error)

extern "C" {

cvsr_status cvsr_session_create(cvsr_ctx *ctx, int32_t m, const cvsr_code *const *codes, const int32_t *order,
                                const cvsr_quantiser *q, float sigma_n, int32_t n, int32_t frames,
                                const cvsr_decode_opts *opts, cvsr_session **out) {
    if (!ctx || !codes || !order || !q || !opts || !out) return cvsr_internal_fail(CVSR_EINVAL, "null argument");
    *out = nullptr;
    if (m < 1 || m > 8 || q->m != m || n <= 0 || frames <= 0)
        return cvsr_internal_fail(CVSR_ESHAPE, "session: bad m / n / frames");
    cvsr_session *s = new cvsr_session();
    s->ctx = ctx;
    s->m = m;
    s->n = n;
    s->frames = frames;
    s->q = *q;
    s->sigma_n = sigma_n;
    s->opts = *opts;
    size_t bytes = 2 * al((size_t)frames * n * 4) + 2 * al((size_t)frames * n) + al(frames) + al((size_t)frames * m * 4);
    for (int j = 0; j < m; ++j) {
        s->codes[j] = codes[j];
        s->order[j] = order[j];
        int32_t nv = n, nc = 0;
        int64_t e = 0;
        if (codes[j]) {
            if (cvsr_status st = cvsr_code_info(codes[j], &nv, &nc, &e)) {
                delete s;
                return st;
            }
            if (nv != n) {
                delete s;
                return cvsr_internal_fail(CVSR_ESHAPE, "session: code length differs from n");
            }
        }
        s->n_checks[j] = nc;
        bytes += al((size_t)frames * cvsr::words_of(codes[j] ? nc : n) * 4);
    }
    int dev = 0;
    cudaGetDevice(&dev);
    s->device = dev;
    if (cudaMalloc(&s->mem, bytes) != cudaSuccess) {
        cudaGetLastError();
        delete s;
        return cvsr_internal_fail(CVSR_ENOMEM, "session buffers");
    }
    char *p = static_cast<char *>(s->mem);
    auto take = [&](size_t b) {
        char *r = p;
        p += al(b);
        return r;
    };
    s->x = reinterpret_cast<float *>(take((size_t)frames * n * 4));
    s->y = reinterpret_cast<float *>(take((size_t)frames * n * 4));
    s->label_bob = reinterpret_cast<uint8_t *>(take((size_t)frames * n));
    s->label_alice = reinterpret_cast<uint8_t *>(take((size_t)frames * n));
    s->frame_ok = reinterpret_cast<uint8_t *>(take(frames));
    s->iters = reinterpret_cast<int32_t *>(take((size_t)frames * m * 4));
    for (int j = 0; j < m; ++j)
        s->synd[j] = reinterpret_cast<uint32_t *>(take((size_t)frames * cvsr::words_of(codes[j] ? s->n_checks[j] : n) * 4));
    if (cudaStreamCreateWithFlags(&s->copy, cudaStreamNonBlocking) != cudaSuccess) {
        cudaFree(s->mem);
        delete s;
        return cvsr_internal_fail(CVSR_ECUDA, "session copy stream");
    }
    for (int i = 0; i < 8; ++i) {
        cudaEventCreateWithFlags(&s->ev_in[i], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&s->ev_out[i], cudaEventDisableTiming);
    }
    *out = s;
    return CVSR_OK;
}

// Bob + Alice for frames [f0, f0 + nf) of the session's buffers
static cvsr_status run_range(cvsr_session *s, const float *x, const float *y, int32_t f0, int32_t nf,
                             cvsr_stats *stats_out, uint8_t *label_alice = nullptr, uint8_t *frame_ok = nullptr,
                             int32_t *iters = nullptr) {
    if (!label_alice) label_alice = s->label_alice;
    if (!frame_ok) frame_ok = s->frame_ok;
    if (!iters) iters = s->iters;
    const size_t off = (size_t)f0 * s->n;
    if (cvsr_status st = cvsr_quantise(s->ctx, &s->q, y + off, (int64_t)nf * s->n, s->label_bob + off)) return st;
    const uint32_t *sy[8];
    for (int j = 0; j < s->m; ++j) {
        const int32_t W = cvsr::words_of(s->codes[j] ? s->n_checks[j] : s->n);
        uint32_t *dst = s->synd[j] + (size_t)f0 * W;
        cvsr_status st = s->codes[j] ? cvsr_syndrome(s->ctx, s->codes[j], s->label_bob + off, nf, j, dst)
                                     : cvsr_slice_bits(s->ctx, s->label_bob + off, nf, s->n, j, dst);
        if (st) return st;
        sy[j] = dst;
    }
    if (cvsr_status st = cvsr_reconcile(s->ctx, s->m, s->codes, s->order, &s->q, s->sigma_n, x + off, sy, nf, s->n,
                                        &s->opts, label_alice + off, frame_ok + f0, iters + (size_t)f0 * s->m,
                                        stats_out))
        return st;
    if (!s->verify) return CVSR_OK;
    return cvsr_verify(s->ctx, label_alice + off, s->label_bob + off, frame_ok + f0, nf, s->n, s->verify_keys,
                       frame_ok + f0, nullptr, nullptr);
}

cvsr_status cvsr_session_set_verify(cvsr_session *s, const uint64_t *keys) {
    if (!s) return cvsr_internal_fail(CVSR_EINVAL, "null session");
    if (!keys) {
        s->verify = false;
        return CVSR_OK;
    }
    for (int q = 0; q < CVSR_HASH_KEYS; ++q)
        if (keys[q] == 0 || keys[q] >= ((1ull << 61) - 1ull))
            return cvsr_internal_fail(CVSR_EINVAL, "keys must be in [1, 2^61 - 2]");
    for (int q = 0; q < CVSR_HASH_KEYS; ++q) s->verify_keys[q] = keys[q];
    s->verify = true;
    return CVSR_OK;
}

cvsr_status cvsr_session_run(cvsr_session *s, const float *x, const float *y, cvsr_stats *stats_out) {
    if (!s || !x || !y) return cvsr_internal_fail(CVSR_EINVAL, "null session or buffer");
    return run_range(s, x, y, 0, s->frames, stats_out);
}

// The batch is processed in up to 4 frame chunks: chunk c+1's inputs are copied in
// (copy stream) while chunk c is reconciled (context stream), and chunk c's results
// are copied out while chunk c+1 runs.  Per-frame results do not depend on the
// chunking.  stats_out (if requested) is accumulated over the chunks.
cvsr_status cvsr_session_run_host(cvsr_session *s, const float *x_host, const float *y_host, uint8_t *label_host,
                                  uint8_t *frame_ok_host, int32_t *iters_host, cvsr_stats *stats_out) {
    if (!s || !x_host || !y_host || !frame_ok_host) return cvsr_internal_fail(CVSR_EINVAL, "null session or buffer");
    cudaStream_t st = cvsr_internal_ctx_stream(s->ctx);
    cudaStream_t cs = s->copy;
    const int chunks = s->frames >= 4 * 128 ? 4 : 1;
    int32_t b[9];
    for (int c = 0; c <= chunks; ++c) b[c] = (int32_t)((int64_t)s->frames * c / chunks);
    if (stats_out) memset(stats_out, 0, sizeof(*stats_out));
    // inputs must not be overwritten while the previous call's work still reads them
    if (cudaStreamSynchronize(st) != cudaSuccess) return cvsr_internal_fail(CVSR_ECUDA, "session: CUDA copy or synchronisation failed");
    auto h2d = [&](int c) -> bool {
        const size_t off = (size_t)b[c] * s->n, bytes = (size_t)(b[c + 1] - b[c]) * s->n * 4;
        return cudaMemcpyAsync(s->x + off, x_host + off, bytes, cudaMemcpyHostToDevice, cs) == cudaSuccess &&
               cudaMemcpyAsync(s->y + off, y_host + off, bytes, cudaMemcpyHostToDevice, cs) == cudaSuccess &&
               cudaEventRecord(s->ev_in[c], cs) == cudaSuccess;
    };
    if (!h2d(0)) return cvsr_internal_fail(CVSR_ECUDA, "session: CUDA copy or synchronisation failed");
    for (int c = 0; c < chunks; ++c) {
        if (c + 1 < chunks && !h2d(c + 1)) return cvsr_internal_fail(CVSR_ECUDA, "session: CUDA copy or synchronisation failed");
        if (cudaStreamWaitEvent(st, s->ev_in[c], 0) != cudaSuccess) return cvsr_internal_fail(CVSR_ECUDA, "session: CUDA copy or synchronisation failed");
        cvsr_stats cst;
        if (cvsr_status r = run_range(s, s->x, s->y, b[c], b[c + 1] - b[c], stats_out ? &cst : nullptr)) return r;
        if (stats_out) {
            stats_out->frames += cst.frames;
            stats_out->frames_ok += cst.frames_ok;
            stats_out->bits_reconciled += cst.bits_reconciled;
            for (int j = 0; j < 8; ++j) {
                stats_out->attempted[j] += cst.attempted[j];
                stats_out->converged[j] += cst.converged[j];
                stats_out->iters_sum[j] += cst.iters_sum[j];
                stats_out->edge_iters[j] += cst.edge_iters[j];
                stats_out->schedule[j] = cst.schedule[j];
            }
            stats_out->alice_seconds += cst.alice_seconds;
        }
        if (cudaEventRecord(s->ev_out[c], st) != cudaSuccess || cudaStreamWaitEvent(cs, s->ev_out[c], 0) != cudaSuccess)
            return cvsr_internal_fail(CVSR_ECUDA, "session: CUDA copy or synchronisation failed");
        const int32_t f0 = b[c], nf = b[c + 1] - b[c];
        if (label_host && cudaMemcpyAsync(label_host + (size_t)f0 * s->n, s->label_alice + (size_t)f0 * s->n,
                                          (size_t)nf * s->n, cudaMemcpyDeviceToHost, cs) != cudaSuccess)
            return cvsr_internal_fail(CVSR_ECUDA, "session: CUDA copy or synchronisation failed");
        if (cudaMemcpyAsync(frame_ok_host + f0, s->frame_ok + f0, nf, cudaMemcpyDeviceToHost, cs) != cudaSuccess)
            return cvsr_internal_fail(CVSR_ECUDA, "session: CUDA copy or synchronisation failed");
        if (iters_host && cudaMemcpyAsync(iters_host + (size_t)f0 * s->m, s->iters + (size_t)f0 * s->m,
                                          (size_t)nf * s->m * 4, cudaMemcpyDeviceToHost, cs) != cudaSuccess)
            return cvsr_internal_fail(CVSR_ECUDA, "session: CUDA copy or synchronisation failed");
    }
    if (cudaStreamSynchronize(cs) != cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess) return cvsr_internal_fail(CVSR_ECUDA, "session: CUDA copy or synchronisation failed");
    return CVSR_OK;
}

// Batches back to back, double-buffered: batch b+1's inputs are copied in (copy
// stream) while batch b is reconciled (context stream), and batch b's results are
// copied out (copy_out stream) while batch b+1 runs.  Whole batches are decoded
// (no chunking), so only the first batch's input copy and the last batch's
// result copy are exposed.
cvsr_status cvsr_session_run_host_stream(cvsr_session *s, int32_t n_batches, const float *const *x_host,
                                         const float *const *y_host, uint8_t *const *label_host,
                                         uint8_t *const *frame_ok_host) {
    if (!s || n_batches < 0 || (n_batches > 0 && (!x_host || !y_host || !frame_ok_host)))
        return cvsr_internal_fail(CVSR_EINVAL, "null session or buffer list");
    for (int32_t b = 0; b < n_batches; ++b)
        if (!x_host[b] || !y_host[b] || !frame_ok_host[b]) return cvsr_internal_fail(CVSR_EINVAL, "null batch buffer");
    const size_t F = (size_t)s->frames, n = (size_t)s->n;
    if (!s->mem2) {
        const size_t bytes = 2 * al(F * n * 4) + al(F * n) + al(F) + al(F * s->m * 4);
        if (cudaMalloc(&s->mem2, bytes) != cudaSuccess) {
            cudaGetLastError();
            s->mem2 = nullptr;
            return cvsr_internal_fail(CVSR_ENOMEM, "session stream buffers");
        }
        char *p = static_cast<char *>(s->mem2);
        auto take = [&](size_t b) {
            char *r = p;
            p += al(b);
            return r;
        };
        s->x2 = reinterpret_cast<float *>(take(F * n * 4));
        s->y2 = reinterpret_cast<float *>(take(F * n * 4));
        s->label_alice2 = reinterpret_cast<uint8_t *>(take(F * n));
        s->frame_ok2 = reinterpret_cast<uint8_t *>(take(F));
        s->iters2 = reinterpret_cast<int32_t *>(take(F * s->m * 4));
        if (cudaStreamCreateWithFlags(&s->copy_out, cudaStreamNonBlocking) != cudaSuccess)
            return cvsr_internal_fail(CVSR_ECUDA, "session copy-out stream");
        for (int i = 0; i < 2; ++i) {
            cudaEventCreateWithFlags(&s->ev_done[i], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&s->ev_d2h[i], cudaEventDisableTiming);
        }
    }
    float *xs[2] = {s->x, s->x2}, *ys[2] = {s->y, s->y2};
    uint8_t *labs[2] = {s->label_alice, s->label_alice2}, *oks[2] = {s->frame_ok, s->frame_ok2};
    int32_t *its[2] = {s->iters, s->iters2};
    cudaStream_t st = cvsr_internal_ctx_stream(s->ctx), cin = s->copy, cout = s->copy_out;
    const char *emsg = "session stream: CUDA copy or synchronisation failed";
    if (cudaStreamSynchronize(st) != cudaSuccess) return cvsr_internal_fail(CVSR_ECUDA, emsg);
    auto h2d = [&](int32_t b) -> bool {
        const int k = b & 1;
        return cudaMemcpyAsync(xs[k], x_host[b], F * n * 4, cudaMemcpyHostToDevice, cin) == cudaSuccess &&
               cudaMemcpyAsync(ys[k], y_host[b], F * n * 4, cudaMemcpyHostToDevice, cin) == cudaSuccess &&
               cudaEventRecord(s->ev_in[k], cin) == cudaSuccess;
    };
    if (n_batches > 0 && !h2d(0)) return cvsr_internal_fail(CVSR_ECUDA, emsg);
    for (int32_t b = 0; b < n_batches; ++b) {
        const int k = b & 1;
        if (b + 1 < n_batches) {
            // set (b+1)&1 was last read by batch b-1's kernels
            if (b >= 1 && cudaStreamWaitEvent(cin, s->ev_done[(b + 1) & 1], 0) != cudaSuccess)
                return cvsr_internal_fail(CVSR_ECUDA, emsg);
            if (!h2d(b + 1)) return cvsr_internal_fail(CVSR_ECUDA, emsg);
        }
        if (cudaStreamWaitEvent(st, s->ev_in[k], 0) != cudaSuccess) return cvsr_internal_fail(CVSR_ECUDA, emsg);
        // set k's results of batch b-2 must have left the device
        if (b >= 2 && cudaStreamWaitEvent(st, s->ev_d2h[k], 0) != cudaSuccess)
            return cvsr_internal_fail(CVSR_ECUDA, emsg);
        if (cvsr_status r = run_range(s, xs[k], ys[k], 0, s->frames, nullptr, labs[k], oks[k], its[k])) return r;
        if (cudaEventRecord(s->ev_done[k], st) != cudaSuccess || cudaStreamWaitEvent(cout, s->ev_done[k], 0) != cudaSuccess)
            return cvsr_internal_fail(CVSR_ECUDA, emsg);
        if (label_host && label_host[b] &&
            cudaMemcpyAsync(label_host[b], labs[k], F * n, cudaMemcpyDeviceToHost, cout) != cudaSuccess)
            return cvsr_internal_fail(CVSR_ECUDA, emsg);
        if (cudaMemcpyAsync(frame_ok_host[b], oks[k], F, cudaMemcpyDeviceToHost, cout) != cudaSuccess ||
            cudaEventRecord(s->ev_d2h[k], cout) != cudaSuccess)
            return cvsr_internal_fail(CVSR_ECUDA, emsg);
    }
    if (cudaStreamSynchronize(cin) != cudaSuccess || cudaStreamSynchronize(cout) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return cvsr_internal_fail(CVSR_ECUDA, emsg);
    return CVSR_OK;
}

cvsr_status cvsr_session_buffers(const cvsr_session *s, uint8_t **label_bob, uint8_t **label_alice,
                                 uint8_t **frame_ok, int32_t **iters) {
    if (!s) return cvsr_internal_fail(CVSR_EINVAL, "null session");
    if (label_bob) *label_bob = s->label_bob;
    if (label_alice) *label_alice = s->label_alice;
    if (frame_ok) *frame_ok = s->frame_ok;
    if (iters) *iters = s->iters;
    return CVSR_OK;
}

void cvsr_session_destroy(cvsr_session *s) {
    if (!s) return;
    cvsr_ctx_sync(s->ctx);
    if (s->copy) {
        cudaStreamSynchronize(s->copy);
        cudaStreamDestroy(s->copy);
    }
    if (s->copy_out) {
        cudaStreamSynchronize(s->copy_out);
        cudaStreamDestroy(s->copy_out);
    }
    for (int i = 0; i < 8; ++i) {
        if (s->ev_in[i]) cudaEventDestroy(s->ev_in[i]);
        if (s->ev_out[i]) cudaEventDestroy(s->ev_out[i]);
    }
    for (int i = 0; i < 2; ++i) {
        if (s->ev_done[i]) cudaEventDestroy(s->ev_done[i]);
        if (s->ev_d2h[i]) cudaEventDestroy(s->ev_d2h[i]);
    }
    if (s->mem2) cudaFree(s->mem2);
    cudaFree(s->mem);
    delete s;
}

}  // extern "C"
