// abi.cu -- si_spmm dispatch (include/sparseinfer_b200.h).
//
// Replaces spmm_exec (spmm.py:283-333): the reference validates the plan
// against the activation and picks a task kernel by the program's output
// dtype, then fans tasks out on its thread pool; here the plan image picks
// the epilogue form and the shape picks K1 (gather, CUDA cores), K3 (2:4
// sparse tensor cores, X-stationary) or K2 (dense-expanded tensor-core
// tiles).  All launches are on the caller's stream.
#include <cuda_runtime.h>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/sparseinfer_b200.h"
#include "si_internal.h"

namespace {

const SiImage *check_image(const void *host_image)
{
    const SiImage *h = (const SiImage *)host_image;
    if (!h || h->magic != SI_IMG_MAGIC || h->version != SI_IMG_VERSION) {
        si_set_error("not a plan image (magic/version mismatch)");
        return nullptr;
    }
    return h;
}

int32_t pick_kernel(const SiImage *h, int64_t n, int32_t layout, int32_t kernel, const void *x, int64_t ldx,
                    int64_t ldo)
{
    if (kernel != SI_KERNEL_AUTO) return kernel;
    // one wave of the staged gather kernel on a very sparse weight beats the
    // tensor-core kernel's fixed cost (small N, >= 85-90% sparsity)
    if (k1s_preferred(h, n, layout, x, ldx)) return SI_KERNEL_GATHER;
    // tensor cores whenever TMA-legal, except tiny weights at small N where
    // the gather kernel's single wave is shorter (all 140 config-2 cells,
    // CUDA-graph replay: profiles/r01b_config2_*.md, DESIGN.md "Kernel
    // selection")
    if (n >= 1024 || (int64_t)h->M * h->K >= (1 << 18)) {
        if (k2_supported(h, n, layout, x, ldx, ldo)) return SI_KERNEL_TC;
    }
    return SI_KERNEL_GATHER;
}

uint64_t kernel_workspace(const SiImage *h, int64_t n, int32_t layout, int32_t k)
{
    return k == SI_KERNEL_GATHER ? k1_workspace(h, n, layout) : k == SI_KERNEL_TC ? k2_workspace(h, n, layout) : 0;
}

}  // namespace

extern "C" int32_t si_spmm_workspace_size(const void *host_image, int64_t n, int32_t x_layout, int32_t kernel,
                                          uint64_t *bytes)
{
    const SiImage *h = check_image(host_image);
    if (!h) return SI_EINVAL;
    if (!bytes) {
        si_set_error("null output pointer");
        return SI_EINVAL;
    }
    if (kernel == SI_KERNEL_AUTO) {
        // AUTO falls back to K1 for activations the tensor-core kernels cannot
        // read (unaligned base or leading dimension), which this query cannot
        // see: report what either kernel needs
        const uint64_t k1 = k1_workspace(h, n, x_layout), k2 = k2_workspace(h, n, x_layout);
        *bytes = k1 > k2 ? k1 : k2;
        return SI_OK;
    }
    *bytes = kernel_workspace(h, n, x_layout, kernel);
    return SI_OK;
}

extern "C" int32_t si_spmm_launch_count(const void *host_image, int64_t n, int32_t x_layout, int32_t kernel)
{
    const SiImage *h = check_image(host_image);
    if (!h) return -1;
    int32_t k = pick_kernel(h, n, x_layout, kernel, nullptr, x_layout == SI_ACT_KN ? n : h->K, h->M);
    return k == SI_KERNEL_GATHER ? k1_launch_count(h, x_layout) : k == SI_KERNEL_TC ? k2_launch_count(h, x_layout) : 1;
}

extern "C" int32_t si_spmm(const void *host_image, const void *dev_image, const void *x, int32_t x_layout,
                           int64_t ldx, int64_t n, const float *sides, void *out, int64_t ldo, void *workspace,
                           uint64_t workspace_bytes, int32_t kernel, void *stream)
{
    const SiImage *h = check_image(host_image);
    if (!h) return SI_EINVAL;
    if (!dev_image || !x || !out || n <= 0) {
        si_set_error("null pointer or N <= 0");
        return SI_EINVAL;
    }
    if (((uintptr_t)dev_image) % 16) {
        si_set_error("device image must be 16-byte aligned");
        return SI_EINVAL;
    }
    if (x_layout != SI_ACT_KN && x_layout != SI_ACT_NK) {
        si_set_error("bad activation layout");
        return SI_EINVAL;
    }
    if ((x_layout == SI_ACT_KN && ldx < n) || (x_layout == SI_ACT_NK && ldx < h->K) || ldo < h->M) {
        si_set_error("leading dimension smaller than the row");
        return SI_EINVAL;
    }
    if (h->n_sides > 0 && !sides) {
        si_set_error("program needs side inputs");
        return SI_EINVAL;
    }
    if (kernel < SI_KERNEL_AUTO || kernel > SI_KERNEL_WS) {
        si_set_error("unknown kernel id");
        return SI_EINVAL;
    }
    int32_t k = pick_kernel(h, n, x_layout, kernel, x, ldx, ldo);
    uint64_t need = kernel_workspace(h, n, x_layout, k);
    if (workspace_bytes < need || (need && !workspace)) {
        si_set_error("workspace too small: need " + std::to_string(need) + " bytes");
        return SI_ENOSPACE;
    }
    if (k == SI_KERNEL_TC && !k2_supported(h, n, x_layout, x, ldx, ldo)) {
        si_set_error("tensor-core kernel does not support this shape/layout");
        return SI_EUNSUPPORTED;
    }
    if (k == SI_KERNEL_SP && !k3_supported(h, n, x_layout, x, ldx)) {
        si_set_error("2:4 kernel needs token-major 16-byte-aligned activations, K <= 1024, >= 2 row tiles");
        return SI_EUNSUPPORTED;
    }
    if (k == SI_KERNEL_WS && !k4_supported(h, n, x_layout, x, ldx)) {
        si_set_error("W-stationary 2:4 kernel needs token-major 16-byte-aligned activations, K <= 1024, >= 2 row tiles");
        return SI_EUNSUPPORTED;
    }
    SpmmArgs a{h, dev_image, (const uint8_t *)x, x_layout, ldx, n, sides, out, ldo, workspace, workspace_bytes,
               stream};
    int err = k == SI_KERNEL_GATHER ? k1_launch(a)
            : k == SI_KERNEL_TC     ? k2_launch(a)
            : k == SI_KERNEL_SP     ? k3_launch(a)
            : k == SI_KERNEL_WS     ? k4_launch(a)
                                    : kref_launch(a);
    if (err != cudaSuccess) {
        si_set_error(std::string("CUDA launch failed: ") + cudaGetErrorString((cudaError_t)err));
        return SI_ECUDA;
    }
    return SI_OK;
}

// ---- host-buffer entry points ----------------------------------------------------
// The reference's spmm_exec takes host arrays; si_spmm_host is that boundary
// for callers without device buffers.  Token chunks are pipelined: while the
// kernel runs on chunk i (caller's stream), chunk i+1 is copied in on one
// internal stream and chunk i-1 copied out on another, with a 4-deep ring of
// device chunks in the caller's workspace.  si_spmm_host_batch runs several
// independent SpMMs (e.g. the Q/K/V projections, or config 5's linear set)
// as one chunk sequence, so the copy directions of consecutive jobs overlap.
namespace {

constexpr uint64_t WS_ALIGN = 256;
uint64_t align_up(uint64_t v, uint64_t a) { return (v + a - 1) / a * a; }

int out_elem_bytes(const SiImage *h) { return (h->out_dtype == 0 || h->out_dtype == 3) ? 4 : 1; }

struct HostLayout {
    int64_t chunk, ldx_dev, ldo_dev;
    uint64_t x_bytes, o_bytes, k_bytes;
};

HostLayout host_layout(const SiImage *h, int64_t chunk_n, int32_t x_layout)
{
    HostLayout L;
    L.chunk = (int64_t)align_up((uint64_t)chunk_n, 256);
    L.ldx_dev = x_layout == SI_ACT_KN ? L.chunk : (int64_t)align_up((uint64_t)h->K, 16);
    L.ldo_dev = (int64_t)align_up((uint64_t)h->M, 16);
    L.x_bytes = align_up(x_layout == SI_ACT_KN ? (uint64_t)h->K * L.chunk : (uint64_t)L.chunk * L.ldx_dev, WS_ALIGN);
    L.o_bytes = align_up((uint64_t)L.chunk * L.ldo_dev * out_elem_bytes(h), WS_ALIGN);
    // a short last chunk may select K1: reserve what either kernel needs
    const uint64_t k1 = k1_workspace(h, L.chunk, x_layout), k2 = k2_workspace(h, L.chunk, x_layout);
    L.k_bytes = align_up(k1 > k2 ? k1 : k2, WS_ALIGN);
    return L;
}

// Copy streams for the host pipeline come from a per-device pool: a call
// takes a private pair for its duration, so concurrent host-buffer calls
// (each with its own workspace) never share an in-flight copy stream.
struct CopyStreams {
    int dev = -1;
    cudaStream_t in = nullptr, out = nullptr;
};
std::mutex g_stream_mu;
std::vector<CopyStreams> g_stream_pool;

bool acquire_copy_streams(CopyStreams &cs)
{
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return false;
    {
        std::lock_guard<std::mutex> lk(g_stream_mu);
        for (size_t i = 0; i < g_stream_pool.size(); ++i)
            if (g_stream_pool[i].dev == dev) {
                cs = g_stream_pool[i];
                g_stream_pool.erase(g_stream_pool.begin() + (long)i);
                return true;
            }
    }
    cs.dev = dev;
    if (cudaStreamCreateWithFlags(&cs.in, cudaStreamNonBlocking) != cudaSuccess) return false;
    if (cudaStreamCreateWithFlags(&cs.out, cudaStreamNonBlocking) != cudaSuccess) {
        cudaStreamDestroy(cs.in);
        return false;
    }
    return true;
}

void release_copy_streams(const CopyStreams &cs)
{
    std::lock_guard<std::mutex> lk(g_stream_mu);
    g_stream_pool.push_back(cs);
}

// Token chunks of one job.  The batch's first job ramps up (chunk/8, /4, /2
// before full chunks) and its last job ramps down the same way, so the
// copy-out stream starts early and the final copy-out is short: with full
// chunks only, the first H2D and the last D2H run alone on the link.
std::vector<std::pair<int64_t, int64_t>> job_chunks(int64_t n, int64_t chunk, bool ramp_up, bool ramp_down)
{
    std::vector<int64_t> head, tail;
    for (int d = 8; d >= 2; d /= 2) {
        const int64_t c = (chunk / d) / 256 * 256;
        if (c >= 256) {
            if (ramp_up) head.push_back(c);
            if (ramp_down) tail.insert(tail.begin(), c);
        }
    }
    int64_t edges = 0;
    for (int64_t c : head) edges += c;
    for (int64_t c : tail) edges += c;
    std::vector<std::pair<int64_t, int64_t>> out;
    if (n <= edges + chunk) {   // too short to ramp: plain chunks
        for (int64_t n0 = 0; n0 < n; n0 += chunk) out.emplace_back(n0, n - n0 < chunk ? n - n0 : chunk);
        return out;
    }
    int64_t n0 = 0;
    for (int64_t c : head) { out.emplace_back(n0, c); n0 += c; }
    int64_t tail_sum = 0;
    for (int64_t c : tail) tail_sum += c;
    const int64_t body_end = n - tail_sum;   // tokens before the ramp-down
    for (; n0 < body_end; n0 += chunk) out.emplace_back(n0, body_end - n0 < chunk ? body_end - n0 : chunk);
    n0 = body_end;
    for (int64_t c : tail) { out.emplace_back(n0, c); n0 += c; }
    return out;
}

int32_t check_job(const si_host_job &j, const SiImage *&h)
{
    h = check_image(j.host_image);
    if (!h) return SI_EINVAL;
    if (!j.dev_image || !j.x_host || !j.out_host || j.n <= 0) {
        si_set_error("null pointer or N <= 0");
        return SI_EINVAL;
    }
    if (j.x_layout != SI_ACT_KN && j.x_layout != SI_ACT_NK) {
        si_set_error("bad activation layout");
        return SI_EINVAL;
    }
    if ((j.x_layout == SI_ACT_KN && j.ldx < j.n) || (j.x_layout == SI_ACT_NK && j.ldx < h->K) || j.ldo < h->M) {
        si_set_error("leading dimension smaller than the row");
        return SI_EINVAL;
    }
    if (h->n_sides > 0 && !j.sides_host) {
        si_set_error("program needs side inputs");
        return SI_EINVAL;
    }
    return SI_OK;
}

// workspace: [x 0..RING-1][out 0..RING-1][sides 0..RING-1][kernel], each the
// max over the jobs.
// A ring deeper than two lets the copy-in stream run ahead of a job whose
// copy-out is the long direction (5b writes 4x what it reads, 5c the reverse).
constexpr int RING = 4;

struct BatchLayout {
    uint64_t x_bytes = 0, o_bytes = 0, s_bytes = 0, k_bytes = 0, total = 0;
};

// per-chunk side-input buffer: f32 [n_sides][chunk][M]
uint64_t side_bytes(const SiImage *h, int64_t chunk)
{
    return align_up((uint64_t)h->n_sides * (uint64_t)chunk * (uint64_t)h->M * 4, WS_ALIGN);
}

void add_job_layout(const SiImage *h, int64_t chunk_n, int32_t x_layout, BatchLayout &B)
{
    const HostLayout L = host_layout(h, chunk_n, x_layout);
    const uint64_t sb = side_bytes(h, L.chunk);
    B.x_bytes = L.x_bytes > B.x_bytes ? L.x_bytes : B.x_bytes;
    B.o_bytes = L.o_bytes > B.o_bytes ? L.o_bytes : B.o_bytes;
    B.s_bytes = sb > B.s_bytes ? sb : B.s_bytes;
    B.k_bytes = L.k_bytes > B.k_bytes ? L.k_bytes : B.k_bytes;
    B.total = RING * (B.x_bytes + B.o_bytes + B.s_bytes) + B.k_bytes;
}

int32_t batch_layout(const si_host_job *jobs, int32_t count, int64_t chunk_n, BatchLayout &B)
{
    if (count <= 0 || !jobs || chunk_n <= 0) {
        si_set_error("empty batch or chunk <= 0");
        return SI_EINVAL;
    }
    for (int32_t i = 0; i < count; ++i) {
        const SiImage *h = nullptr;
        int32_t rc = check_job(jobs[i], h);
        if (rc != SI_OK) return rc;
        add_job_layout(h, chunk_n, jobs[i].x_layout, B);
    }
    return SI_OK;
}

}  // namespace

extern "C" int32_t si_spmm_host_batch_workspace_size(const si_host_job *jobs, int32_t count, int64_t chunk_n,
                                                     uint64_t *bytes)
{
    BatchLayout B;
    int32_t rc = batch_layout(jobs, count, chunk_n, B);
    if (rc == SI_OK) *bytes = B.total;
    return rc;
}

extern "C" int32_t si_spmm_host_batch(const si_host_job *jobs, int32_t count, void *workspace,
                                      uint64_t workspace_bytes, int64_t chunk_n, int32_t kernel, void *stream)
{
    BatchLayout B;
    int32_t rc = batch_layout(jobs, count, chunk_n, B);
    if (rc != SI_OK) return rc;
    if (workspace_bytes < B.total || !workspace) {
        si_set_error("workspace too small: need " + std::to_string(B.total) + " bytes");
        return SI_ENOSPACE;
    }
    cudaStream_t s_cmp = (cudaStream_t)stream;
    CopyStreams cs;
    if (!acquire_copy_streams(cs)) {
        si_set_error("cannot create copy streams");
        return SI_ECUDA;
    }
    cudaStream_t s_in = cs.in, s_out = cs.out;
    uint8_t *ws = (uint8_t *)workspace;
    uint8_t *xbuf[RING], *obuf[RING];
    float *sbuf[RING];
    for (int r = 0; r < RING; ++r) {
        xbuf[r] = ws + r * B.x_bytes;
        obuf[r] = ws + RING * B.x_bytes + r * B.o_bytes;
        sbuf[r] = (float *)(ws + RING * (B.x_bytes + B.o_bytes) + r * B.s_bytes);
    }
    void *kws = B.k_bytes ? ws + RING * (B.x_bytes + B.o_bytes + B.s_bytes) : nullptr;

    cudaEvent_t ev_entry, ev_in_end, ev_out_end, in_done[RING], cmp_done[RING], out_done[RING];
    cudaEventCreateWithFlags(&ev_entry, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev_in_end, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev_out_end, cudaEventDisableTiming);
    for (int r = 0; r < RING; ++r) {
        cudaEventCreateWithFlags(&in_done[r], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&cmp_done[r], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&out_done[r], cudaEventDisableTiming);
    }
    // the workspace may still be in use by work queued earlier on the caller's stream
    cudaEventRecord(ev_entry, s_cmp);
    cudaStreamWaitEvent(s_in, ev_entry, 0);
    int64_t seq = 0;   // chunk sequence number across the batch (buffer = seq % RING)
    for (int32_t jb = 0; jb < count && rc == SI_OK; ++jb) {
        const si_host_job &J = jobs[jb];
        const SiImage *h = (const SiImage *)J.host_image;
        const HostLayout L = host_layout(h, chunk_n, J.x_layout);
        const int eb = out_elem_bytes(h);
        const uint8_t *xh = (const uint8_t *)J.x_host;
        uint8_t *oh = (uint8_t *)J.out_host;
        const int ns = h->n_sides;
        const auto chunks = job_chunks(J.n, L.chunk, jb == 0, jb == count - 1);
        for (size_t ci = 0; ci < chunks.size() && rc == SI_OK; ++ci, ++seq) {
            const int b = (int)(seq % RING);
            const int64_t n0 = chunks[ci].first, nc = chunks[ci].second;
            // copy in: buffer b is free once the kernel RING chunks back finished
            if (seq >= RING) cudaStreamWaitEvent(s_in, cmp_done[b], 0);
            cudaError_t e;
            if (J.x_layout == SI_ACT_KN)
                e = cudaMemcpy2DAsync(xbuf[b], (size_t)L.ldx_dev, xh + n0, (size_t)J.ldx, (size_t)nc, (size_t)h->K,
                                      cudaMemcpyHostToDevice, s_in);
            else
                e = cudaMemcpy2DAsync(xbuf[b], (size_t)L.ldx_dev, xh + n0 * J.ldx, (size_t)J.ldx, (size_t)h->K,
                                      (size_t)nc, cudaMemcpyHostToDevice, s_in);
            // side inputs: rows n0 .. n0+nc of each [N, M] side, packed [ns][nc][M]
            for (int sd = 0; sd < ns && e == cudaSuccess; ++sd)
                e = cudaMemcpyAsync(sbuf[b] + (size_t)sd * nc * h->M,
                                    J.sides_host + ((size_t)sd * J.n + n0) * h->M, (size_t)nc * h->M * 4,
                                    cudaMemcpyHostToDevice, s_in);
            if (e != cudaSuccess) {
                rc = SI_ECUDA;
                si_set_error(std::string("H2D: ") + cudaGetErrorString(e));
                break;
            }
            cudaEventRecord(in_done[b], s_in);
            // compute: after its input arrived and the output buffer was drained
            cudaStreamWaitEvent(s_cmp, in_done[b], 0);
            if (seq >= RING) cudaStreamWaitEvent(s_cmp, out_done[b], 0);
            rc = si_spmm(J.host_image, J.dev_image, xbuf[b], J.x_layout, L.ldx_dev, nc, ns ? sbuf[b] : nullptr,
                         obuf[b], L.ldo_dev, kws, B.k_bytes, kernel, s_cmp);
            if (rc != SI_OK) break;
            cudaEventRecord(cmp_done[b], s_cmp);
            // copy out
            cudaStreamWaitEvent(s_out, cmp_done[b], 0);
            e = cudaMemcpy2DAsync(oh + n0 * J.ldo * eb, (size_t)J.ldo * eb, obuf[b], (size_t)L.ldo_dev * eb,
                                  (size_t)h->M * eb, (size_t)nc, cudaMemcpyDeviceToHost, s_out);
            if (e != cudaSuccess) {
                rc = SI_ECUDA;
                si_set_error(std::string("D2H: ") + cudaGetErrorString(e));
                break;
            }
            cudaEventRecord(out_done[b], s_out);
        }
    }
    // join both copy streams -- on the error paths too, so no copy queued by
    // this call still touches the caller's host buffers or the workspace once
    // it returns; later work on the caller's stream is ordered after them
    cudaEventRecord(ev_in_end, s_in);
    cudaEventRecord(ev_out_end, s_out);
    cudaStreamWaitEvent(s_cmp, ev_in_end, 0);
    cudaStreamWaitEvent(s_cmp, ev_out_end, 0);
    const cudaError_t e_in = cudaStreamSynchronize(s_in);
    const cudaError_t e_out = cudaStreamSynchronize(s_out);
    if (rc == SI_OK && (e_in != cudaSuccess || e_out != cudaSuccess)) {
        rc = SI_ECUDA;
        si_set_error(std::string("host pipeline: ") + cudaGetErrorString(e_in != cudaSuccess ? e_in : e_out));
    }
    release_copy_streams(cs);
    cudaEventDestroy(ev_entry);
    cudaEventDestroy(ev_in_end);
    cudaEventDestroy(ev_out_end);
    for (int r = 0; r < RING; ++r) {
        cudaEventDestroy(in_done[r]);
        cudaEventDestroy(cmp_done[r]);
        cudaEventDestroy(out_done[r]);
    }
    return rc;
}

extern "C" int32_t si_spmm_host_workspace_size(const void *host_image, int64_t chunk_n, int32_t x_layout,
                                               int32_t kernel, uint64_t *bytes)
{
    (void)kernel;
    const SiImage *h = check_image(host_image);
    if (!h) return SI_EINVAL;
    if (chunk_n <= 0 || !bytes || (x_layout != SI_ACT_KN && x_layout != SI_ACT_NK)) {
        si_set_error("bad chunk size, layout or output pointer");
        return SI_EINVAL;
    }
    // the same layout si_spmm_host_batch uses for a one-job batch
    BatchLayout B;
    add_job_layout(h, chunk_n, x_layout, B);
    *bytes = B.total;
    return SI_OK;
}

extern "C" int32_t si_spmm_host(const void *host_image, const void *dev_image, const void *x_host, int32_t x_layout,
                                int64_t ldx, int64_t n, const float *sides_host, void *out_host, int64_t ldo,
                                void *workspace, uint64_t workspace_bytes, int64_t chunk_n, int32_t kernel,
                                void *stream)
{
    const si_host_job j{host_image, dev_image, x_host, x_layout, ldx, n, out_host, ldo, sides_host};
    return si_spmm_host_batch(&j, 1, workspace, workspace_bytes, chunk_n, kernel, stream);
}
