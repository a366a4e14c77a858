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
    void *mem = nullptr;
    float *x = nullptr, *y = nullptr;
    uint8_t *label_bob = nullptr, *label_alice = nullptr, *frame_ok = nullptr;
    int32_t *iters = nullptr;
    uint32_t *synd[8] = {};
};

namespace {
size_t al(size_t b) { return (b + 255) & ~size_t(255); }
}  // namespace

cudaStream_t cvsr_internal_ctx_stream(cvsr_ctx *ctx);  // api.cu

extern "C" {

cvsr_status cvsr_session_create(cvsr_ctx *ctx, int32_t m, const cvsr_code *const *codes, const int32_t *order,
                                const cvsr_quantiser *q, float sigma_n, int32_t n, int32_t frames,
                                const cvsr_decode_opts *opts, cvsr_session **out) {
    if (!ctx || !codes || !order || !q || !opts || !out) return CVSR_EINVAL;
    *out = nullptr;
    if (m < 1 || m > 8 || q->m != m || n <= 0 || frames <= 0) return CVSR_ESHAPE;
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
                return CVSR_ESHAPE;
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
        return CVSR_ENOMEM;
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
    *out = s;
    return CVSR_OK;
}

cvsr_status cvsr_session_run(cvsr_session *s, const float *x, const float *y, cvsr_stats *stats_out) {
    if (!s || !x || !y) return CVSR_EINVAL;
    if (cvsr_status st = cvsr_quantise(s->ctx, &s->q, y, (int64_t)s->frames * s->n, s->label_bob)) return st;
    for (int j = 0; j < s->m; ++j) {
        cvsr_status st = s->codes[j] ? cvsr_syndrome(s->ctx, s->codes[j], s->label_bob, s->frames, j, s->synd[j])
                                     : cvsr_slice_bits(s->ctx, s->label_bob, s->frames, s->n, j, s->synd[j]);
        if (st) return st;
    }
    const uint32_t *sy[8];
    for (int j = 0; j < s->m; ++j) sy[j] = s->synd[j];
    return cvsr_reconcile(s->ctx, s->m, s->codes, s->order, &s->q, s->sigma_n, x, sy, s->frames, s->n, &s->opts,
                          s->label_alice, s->frame_ok, s->iters, stats_out);
}

cvsr_status cvsr_session_run_host(cvsr_session *s, const float *x_host, const float *y_host, uint8_t *label_host,
                                  uint8_t *frame_ok_host, int32_t *iters_host, cvsr_stats *stats_out) {
    if (!s || !x_host || !y_host || !frame_ok_host) return CVSR_EINVAL;
    cudaStream_t st = cvsr_internal_ctx_stream(s->ctx);
    const size_t xb = (size_t)s->frames * s->n * 4;
    if (cudaMemcpyAsync(s->x, x_host, xb, cudaMemcpyHostToDevice, st) != cudaSuccess) return CVSR_ECUDA;
    if (cudaMemcpyAsync(s->y, y_host, xb, cudaMemcpyHostToDevice, st) != cudaSuccess) return CVSR_ECUDA;
    if (cvsr_status r = cvsr_session_run(s, s->x, s->y, stats_out)) return r;
    if (label_host &&
        cudaMemcpyAsync(label_host, s->label_alice, (size_t)s->frames * s->n, cudaMemcpyDeviceToHost, st) != cudaSuccess)
        return CVSR_ECUDA;
    if (cudaMemcpyAsync(frame_ok_host, s->frame_ok, s->frames, cudaMemcpyDeviceToHost, st) != cudaSuccess)
        return CVSR_ECUDA;
    if (iters_host && cudaMemcpyAsync(iters_host, s->iters, (size_t)s->frames * s->m * 4, cudaMemcpyDeviceToHost,
                                      st) != cudaSuccess)
        return CVSR_ECUDA;
    if (cudaStreamSynchronize(st) != cudaSuccess) return CVSR_ECUDA;
    return CVSR_OK;
}

cvsr_status cvsr_session_buffers(const cvsr_session *s, uint8_t **label_bob, uint8_t **label_alice,
                                 uint8_t **frame_ok, int32_t **iters) {
    if (!s) return CVSR_EINVAL;
    if (label_bob) *label_bob = s->label_bob;
    if (label_alice) *label_alice = s->label_alice;
    if (frame_ok) *frame_ok = s->frame_ok;
    if (iters) *iters = s->iters;
    return CVSR_OK;
}

void cvsr_session_destroy(cvsr_session *s) {
    if (!s) return;
    cvsr_ctx_sync(s->ctx);
    cudaFree(s->mem);
    delete s;
}

}  // extern "C"
