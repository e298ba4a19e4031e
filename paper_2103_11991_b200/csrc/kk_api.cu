// kk_api.cu -- C ABI (include/kk_spgemm.h): handle, workspace, phase orchestration.
//
// Symbolic: init status -> a4 check/compress B -> a1 row flops + bins
// -> a2 scan of flops -> a3 stable binning -> host read of the symbolic bin sizes (sync 1:
// empty bins are not launched and grids are sized to their bins) -> a5 per-bin symbolic
// kernels -> a6 scan of counts into the caller's row map -> numeric bins from exact counts
// -> device->host copy of the status block + stream sync (sync 2: nnz(C) must reach the
// host before C's arrays can be allocated).
// Numeric: per-bin numeric kernels with the fused sort; asynchronous.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <array>
#include <atomic>
#include <memory>
#include <chrono>
#include <thread>
#include <cstring>
#include <string>
#include <algorithm>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/kk_spgemm.h"
#include "kk_internal.cuh"

using kk::DevStatus;
using kk::MatView;

namespace {

struct Buf {
    void* p = nullptr;
    size_t bytes = 0;
};

}  // namespace

// Per-kernel CUDA-event timing (opts.timing): events are recorded around each launch on
// its stream and resolved lazily, so the launches themselves stay asynchronous.
struct kk::KTimer {
    struct Rec {
        const char* name;
        cudaEvent_t a, b;
    };
    struct Acc {
        std::string name;
        int64_t n = 0;
        double tot = 0, mx = 0;
    };
    std::vector<Rec> pending;
    std::vector<cudaEvent_t> pool;
    std::vector<Acc> acc;
    cudaEvent_t get() {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
        cudaEvent_t e = nullptr;
        cudaEventCreate(&e);
        return e;
    }
    void resolve() {
        for (Rec& r : pending) {
            if (!r.b) continue;
            cudaEventSynchronize(r.b);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, r.a, r.b);
            Acc* a = nullptr;
            for (Acc& x : acc)
                if (x.name == r.name) a = &x;
            if (!a) {
                acc.push_back(Acc());
                a = &acc.back();
                a->name = r.name;
            }
            a->n += 1;
            a->tot += ms;
            if (ms > a->mx) a->mx = ms;
            pool.push_back(r.a);
            pool.push_back(r.b);
        }
        pending.clear();
    }
    ~KTimer() {
        resolve();
        for (cudaEvent_t e : pool) cudaEventDestroy(e);
    }
};

void kk::ktimer_begin(KTimer* t, const char* name, cudaStream_t s) {
    if (t->pending.size() > 4096) t->resolve();
    KTimer::Rec r{name, t->get(), nullptr};
    cudaEventRecord(r.a, s);
    t->pending.push_back(r);
}

void kk::ktimer_end(KTimer* t, cudaStream_t s) {
    KTimer::Rec& r = t->pending.back();
    r.b = t->get();
    cudaEventRecord(r.b, s);
}

struct kk_spgemm_handle_s {
    int device = 0;
    int num_sms = 148;
    kk_spgemm_opts_t opts;
    std::string err;
    long long launches = 0;
    // workspace
    Buf flops, fscan, binid, perm_sym, perm_num, counts, binscratch, binstart, bc_len, pairs, cursors, partial,
        status, bmeta, wlo, pat, pat_off, pat_len, diagchk, apos, bpos, spdup, spflag, status_aux, workctr, retry;
    // every workspace buffer, for destroy and stats (one list, so neither can miss one)
    Buf* all_bufs[26] = {&flops,   &fscan,   &binid,   &perm_sym, &perm_num, &counts, &binscratch, &binstart,
                         &bc_len,  &pairs,   &cursors, &partial,  &status,   &bmeta,  &wlo,        &pat,
                         &pat_off, &pat_len, &diagchk, &apos,     &bpos,     &spdup,  &spflag,     &status_aux,
                         &workctr, &retry};
    // B_C of a B prefix kept between the blocks of kk_spgemm_multiply_host (armed only there)
    struct BcCarry {
        bool armed = false, valid = false;
        const void *brm = nullptr, *bent = nullptr, *bmeta = nullptr, *bc_len = nullptr, *pairs = nullptr;
        int64_t rows = 0, k = 0;
        int comp_mode = 0, validate = 0;
        kk::StatusCarry c;
    } bcc;
    DevStatus* h_status = nullptr;  // pinned, mapped (d_status: its device address)
    DevStatus* d_status = nullptr;
    // small status reads of the other entry points (pinned, mapped; d_aux: device address)
    struct Aux {
        DevStatus st;
        int flag;
        int missing;
    };
    Aux* h_aux = nullptr;
    Aux* d_aux = nullptr;
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // record of the last symbolic (stale-handle check)
    struct Rec {
        bool valid = false;
        int64_t m = 0, n = 0, k = 0, nnzA = 0, nnzB = 0, nnzC = 0;
        const void *arm = nullptr, *aent = nullptr, *brm = nullptr, *bent = nullptr, *crm = nullptr;
        int offt = 0;
    } rec;
    // record of the last fused triple-product symbolic
    struct RapRec {
        bool valid = false;
        int64_t mc = 0, nnzR = 0, nnzA = 0, nnzP = 0, nnzC = 0;
        const void *rrm = nullptr, *arm = nullptr, *prm = nullptr, *crm = nullptr;
        int offt = 0;
    } raprec;
    // record of the last SpAdd symbolic
    struct AddRec {
        bool valid = false;
        int64_t m = 0, k = 0, nnzA = 0, nnzB = 0, nnzC = 0;
        const void *arm = nullptr, *aent = nullptr, *brm = nullptr, *bent = nullptr, *crm = nullptr;
        int offt = 0;
    } addrec;
    int host_num_bin_start[kk::NB + 1] = {0};
    kk_spgemm_stats_t stats;
    kk::KTimer* timer = nullptr;
    // kk_spgemm_multiply_host: streams, events, device staging (B; two slots of A blocks and
    // C blocks), pinned host staging (rebased row maps; C's entries and values, grow-only)
    struct HostPath {
        cudaStream_t s_in = nullptr, s_out = nullptr, s_a = nullptr;
        Buf brm, bent, bval, arm[2], aent[2], aval[2], crm[2], cent[2], cval[2];
        void* h_cent = nullptr;
        size_t h_cent_bytes = 0;
        void* h_cval = nullptr;
        size_t h_cval_bytes = 0;
    } hp;
    // texture objects over the last B of a numeric call (pointer, count, value type)
    struct TexB {
        const void *ent = nullptr, *val = nullptr;
        int64_t nnz = 0;
        int vt = -1;
        cudaTextureObject_t te = 0, tv = 0;
    } texb;
};

static void tex_release(kk_spgemm_handle_t h) {
    if (h->texb.te) cudaDestroyTextureObject(h->texb.te);
    if (h->texb.tv) cudaDestroyTextureObject(h->texb.tv);
    h->texb = kk_spgemm_handle_s::TexB();
}

// texture objects for B's entries and values (1-D linear; made once per B, kept in the handle)
static void tex_for(kk_spgemm_handle_t h, const kk_csr_t* B, unsigned long long* te, unsigned long long* tv) {
    *te = *tv = 0;
    auto& T = h->texb;
    // a texture spanning more of the same arrays serves a B that is a prefix of them (the host
    // path's row-chunked B)
    if (T.ent == B->entries && T.val == B->values && T.nnz >= B->nnz && T.vt == (int)B->value_type) {
        *te = T.te;
        *tv = T.tv;
        return;
    }
    tex_release(h);
    int maxw = 0;
    cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxTexture1DLinearWidth, h->device);
    if (B->nnz <= 0 || B->nnz > (int64_t)maxw) return;
    auto make = [&](const void* p, size_t bytes, cudaChannelFormatDesc fd) -> cudaTextureObject_t {
        cudaResourceDesc rd = {};
        rd.resType = cudaResourceTypeLinear;
        rd.res.linear.devPtr = const_cast<void*>(p);
        rd.res.linear.desc = fd;
        rd.res.linear.sizeInBytes = bytes;
        cudaTextureDesc td = {};
        td.readMode = cudaReadModeElementType;
        cudaTextureObject_t t = 0;
        if (cudaCreateTextureObject(&t, &rd, &td, nullptr) != cudaSuccess) {
            cudaGetLastError();
            t = 0;
        }
        return t;
    };
    T.ent = B->entries;
    T.val = B->values;
    T.nnz = B->nnz;
    T.vt = (int)B->value_type;
    T.te = make(B->entries, (size_t)B->nnz * 4, cudaCreateChannelDesc<int>());
    T.tv = make(B->values, (size_t)B->nnz * (B->value_type == KK_F64 ? 8 : 4),
                B->value_type == KK_F64 ? cudaCreateChannelDesc<int2>() : cudaCreateChannelDesc<float>());
    if (!T.te || !T.tv) {
        tex_release(h);
        return;
    }
    *te = T.te;
    *tv = T.tv;
}

// NVTX ranges around the entry points and the symbolic steps (visible in nsys / ncu range
// filters; header-only NVTX v3, no-ops without a tool attached)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

static kk_status_t fail(kk_spgemm_handle_t h, kk_status_t s, const char* fmt, ...) {
    if (h) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof(buf), fmt, ap);
        va_end(ap);
        h->err = buf;
    }
    return s;
}

static kk_status_t cuda_check(kk_spgemm_handle_t h, cudaError_t e, const char* what) {
    if (e == cudaSuccess) return KK_OK;
    cudaGetLastError();
    if (e == cudaErrorMemoryAllocation) return fail(h, KK_ERR_OUT_OF_MEMORY, "%s: %s", what, cudaGetErrorString(e));
    return fail(h, KK_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

static kk_status_t ensure(kk_spgemm_handle_t h, Buf& b, size_t bytes, cudaStream_t s) {
    if (bytes == 0) bytes = 16;
    if (b.bytes >= bytes) return KK_OK;
    bytes = bytes + bytes / 8 + 256;
    if (b.p) {
        if (h->opts.free)
            h->opts.free(b.p, b.bytes, s, h->opts.alloc_ctx);
        else
            cudaFreeAsync(b.p, s);
        b.p = nullptr;
        b.bytes = 0;
    }
    void* p = nullptr;
    if (h->opts.alloc) {
        p = h->opts.alloc(bytes, s, h->opts.alloc_ctx);
        if (!p) return fail(h, KK_ERR_OUT_OF_MEMORY, "workspace allocation of %zu bytes failed", bytes);
    } else {
        cudaError_t e = cudaMallocAsync(&p, bytes, s);
        if (e != cudaSuccess) return cuda_check(h, e, "cudaMallocAsync(workspace)");
    }
    b.p = p;
    b.bytes = bytes;
    return KK_OK;
}

static void release(kk_spgemm_handle_t h, Buf& b) {
    if (!b.p) return;
    if (h->opts.free)
        h->opts.free(b.p, b.bytes, nullptr, h->opts.alloc_ctx);
    else
        cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
}

static kk_status_t check_csr(kk_spgemm_handle_t h, const kk_csr_t* M, const char* name, bool need_values) {
    if (!M) return fail(h, KK_ERR_INVALID_ARG, "%s is NULL", name);
    if (M->nrows < 0 || M->ncols < 0 || M->nnz < 0)
        return fail(h, KK_ERR_INVALID_ARG, "%s has a negative size", name);
    if (M->nrows >= INT32_MAX || M->ncols >= INT32_MAX)
        return fail(h, KK_ERR_INVALID_ARG, "%s: dimensions must be < 2^31", name);
    if (M->offset_type != KK_I32 && M->offset_type != KK_I64)
        return fail(h, KK_ERR_UNSUPPORTED_TYPE, "%s: bad offset_type", name);
    if (M->value_type != KK_F32 && M->value_type != KK_F64)
        return fail(h, KK_ERR_UNSUPPORTED_TYPE, "%s: bad value_type", name);
    if (!M->row_map) return fail(h, KK_ERR_INVALID_ARG, "%s.row_map is NULL", name);
    if (M->nnz > 0 && !M->entries) return fail(h, KK_ERR_INVALID_ARG, "%s.entries is NULL", name);
    if (need_values && M->nnz > 0 && !M->values) return fail(h, KK_ERR_INVALID_ARG, "%s.values is NULL", name);
    if (M->offset_type == KK_I32 && M->nnz > INT32_MAX)
        return fail(h, KK_ERR_INDEX_OVERFLOW, "%s: nnz exceeds int32 offsets", name);
    return KK_OK;
}

static kk_status_t check_pair(kk_spgemm_handle_t h, const kk_csr_t* A, const kk_csr_t* B, bool need_values) {
    kk_status_t s;
    if ((s = check_csr(h, A, "A", need_values)) != KK_OK) return s;
    if ((s = check_csr(h, B, "B", need_values)) != KK_OK) return s;
    if (A->ncols != B->nrows)
        return fail(h, KK_ERR_DIM_MISMATCH, "A.ncols (%lld) != B.nrows (%lld)", (long long)A->ncols,
                    (long long)B->nrows);
    if (A->offset_type != B->offset_type)
        return fail(h, KK_ERR_UNSUPPORTED_TYPE, "A and B must use the same offset type");
    if (need_values && A->value_type != B->value_type)
        return fail(h, KK_ERR_UNSUPPORTED_TYPE, "A and B must use the same value type");
    return KK_OK;
}

static MatView view(const kk_csr_t* M) {
    MatView v;
    v.nrows = M->nrows;
    v.ncols = M->ncols;
    v.nnz = M->nnz;
    v.row_map = M->row_map;
    v.entries = M->entries;
    v.values = M->values;
    return v;
}

static int pick_logG(double avg) {
    // lanes per B row: smallest power of two >= 0.75 * average row length, in [4, 32]
    double want = avg * 0.75;
    int lg = 2;
    while (lg < 5 && (double)(1 << lg) < want) ++lg;
    return lg;
}

extern "C" {

void kk_spgemm_opts_default(kk_spgemm_opts_t* o) {
    if (!o) return;
    memset(o, 0, sizeof(*o));
    o->sort_rows = 1;
    o->compression = -1;
    o->validate = 0;
    o->num_streams = 2;
    o->patterns = 1;
}

const char* kk_status_string(kk_status_t s) {
    switch (s) {
        case KK_OK: return "KK_OK";
        case KK_ERR_INVALID_ARG: return "KK_ERR_INVALID_ARG";
        case KK_ERR_DIM_MISMATCH: return "KK_ERR_DIM_MISMATCH";
        case KK_ERR_UNSUPPORTED_TYPE: return "KK_ERR_UNSUPPORTED_TYPE";
        case KK_ERR_INDEX_OVERFLOW: return "KK_ERR_INDEX_OVERFLOW";
        case KK_ERR_STALE_HANDLE: return "KK_ERR_STALE_HANDLE";
        case KK_ERR_OUT_OF_MEMORY: return "KK_ERR_OUT_OF_MEMORY";
        case KK_ERR_CUDA: return "KK_ERR_CUDA";
    }
    return "KK_ERR_UNKNOWN";
}

const char* kk_last_error_detail(kk_spgemm_handle_t h) { return h ? h->err.c_str() : "null handle"; }

kk_status_t kk_spgemm_create(kk_spgemm_handle_t* out, int device, const kk_spgemm_opts_t* opts) {
    if (!out) return KK_ERR_INVALID_ARG;
    *out = nullptr;
    if (device < 0) return KK_ERR_INVALID_ARG;
    kk_spgemm_opts_t o;
    kk_spgemm_opts_default(&o);
    if (opts) o = *opts;
    if (o.compression < -1 || o.compression > 1) return KK_ERR_INVALID_ARG;
    if ((o.alloc == nullptr) != (o.free == nullptr)) return KK_ERR_INVALID_ARG;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device >= ndev) {
        cudaGetLastError();
        return KK_ERR_CUDA;
    }
    cudaSetDevice(device);
    kk_spgemm_handle_t h = new kk_spgemm_handle_s();
    h->device = device;
    h->opts = o;
    cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device);
    if (cudaHostAlloc((void**)&h->h_status, sizeof(DevStatus), cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer((void**)&h->d_status, h->h_status, 0) != cudaSuccess ||
        cudaHostAlloc((void**)&h->h_aux, sizeof(*h->h_aux), cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer((void**)&h->d_aux, h->h_aux, 0) != cudaSuccess) {
        cudaGetLastError();
        if (h->h_status) cudaFreeHost(h->h_status);
        if (h->h_aux) cudaFreeHost(h->h_aux);
        delete h;
        return KK_ERR_OUT_OF_MEMORY;
    }
    memset(h->h_status, 0, sizeof(DevStatus));
    memset(h->h_aux, 0, sizeof(*h->h_aux));
    if (o.num_streams > 1) {
        cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking);
        cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming);
    }
    memset(&h->stats, 0, sizeof(h->stats));
    if (o.timing) h->timer = new kk::KTimer();
    *out = h;
    return KK_OK;
}

kk_status_t kk_spgemm_destroy(kk_spgemm_handle_t h) {
    if (!h) return KK_ERR_INVALID_ARG;
    cudaSetDevice(h->device);
    cudaDeviceSynchronize();
    for (Buf* b : h->all_bufs) release(h, *b);
    tex_release(h);
    {
        auto& P = h->hp;
        Buf* hb[] = {&P.brm, &P.bent, &P.bval, &P.arm[0], &P.arm[1], &P.aent[0], &P.aent[1], &P.aval[0],
                     &P.aval[1], &P.crm[0], &P.crm[1], &P.cent[0], &P.cent[1], &P.cval[0], &P.cval[1]};
        for (Buf* b : hb) release(h, *b);
        if (P.h_cent) cudaFreeHost(P.h_cent);
        if (P.h_cval) cudaFreeHost(P.h_cval);
        if (P.s_in) cudaStreamDestroy(P.s_in);
        if (P.s_out) cudaStreamDestroy(P.s_out);
        if (P.s_a) cudaStreamDestroy(P.s_a);
    }
    delete h->timer;
    if (h->h_status) cudaFreeHost(h->h_status);
    if (h->h_aux) cudaFreeHost(h->h_aux);
    if (h->side) cudaStreamDestroy(h->side);
    if (h->ev_fork) cudaEventDestroy(h->ev_fork);
    if (h->ev_join) cudaEventDestroy(h->ev_join);
    cudaGetLastError();
    delete h;
    return KK_OK;
}

static kk::Launch make_launch(kk_spgemm_handle_t h, cudaStream_t s) {
    kk::Launch L;
    L.stream = s;
    L.num_sms = h->num_sms;
    L.launches = &h->launches;
    L.timer = h->timer;
    return L;
}

// the status block (and an optional flag word) to the handle's mapped host copy, then one sync
static kk_status_t read_status(kk_spgemm_handle_t h, cudaStream_t s, const DevStatus* dst, const int* dflag,
                               const char* what) {
    kk::Launch L = make_launch(h, s);
    void* d[2] = {&h->d_aux->st, &h->d_aux->flag};
    const void* src[2] = {dst, dflag};
    const size_t nb[2] = {sizeof(DevStatus), sizeof(int)};
    kk::post_words(L, dflag ? 2 : 1, d, src, nb);
    kk_status_t st;
    if ((st = cuda_check(h, cudaGetLastError(), what)) != KK_OK) return st;
    return cuda_check(h, cudaStreamSynchronize(s), what);
}

kk_status_t kk_spgemm_compress(kk_spgemm_handle_t h, const kk_csr_t* B, int32_t* len, uint64_t* pairs,
                               void* stream) {
    NvtxRange nvtx_("kk_spgemm_compress");
    if (!h) return KK_ERR_INVALID_ARG;
    kk_status_t st;
    if ((st = check_csr(h, B, "B", false)) != KK_OK) return st;
    if (B->nrows > 0 && !len) return fail(h, KK_ERR_INVALID_ARG, "len is NULL");
    if (B->nnz > 0 && !pairs) return fail(h, KK_ERR_INVALID_ARG, "pairs is NULL");
    cudaSetDevice(h->device);
    cudaStream_t s = (cudaStream_t)stream;
    // a status block of its own: the symbolic state numeric reads (B flags) stays intact
    if ((st = ensure(h, h->status_aux, sizeof(DevStatus), s)) != KK_OK) return st;
    kk::Launch L = make_launch(h, s);
    DevStatus* dst = (DevStatus*)h->status_aux.p;
    kk::init_status(L, dst);
    kk::check_compress(L, B->offset_type == KK_I64, view(B), B->ncols, true, h->opts.validate != 0, len,
                       (uint2*)pairs, nullptr, dst);
    return cuda_check(h, cudaGetLastError(), "kk_spgemm_compress launch");
}

kk_status_t kk_spgemm_row_flops(kk_spgemm_handle_t h, const kk_csr_t* A, const kk_csr_t* B, int64_t* flops,
                                int64_t* flops_scan, int64_t* total, void* stream) {
    NvtxRange nvtx_("kk_spgemm_row_flops");
    if (!h) return KK_ERR_INVALID_ARG;
    kk_status_t st;
    if ((st = check_pair(h, A, B, false)) != KK_OK) return st;
    cudaSetDevice(h->device);
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t m = A->nrows;
    const bool off64 = A->offset_type == KK_I64;
    if ((st = ensure(h, h->status_aux, sizeof(DevStatus), s)) != KK_OK) return st;
    if ((st = ensure(h, h->binid, (size_t)m, s)) != KK_OK) return st;
    if ((st = ensure(h, h->counts, (size_t)m * 4, s)) != KK_OK) return st;
    if ((st = ensure(h, h->partial, (size_t)kk::scan_partial_len(m) * 8, s)) != KK_OK) return st;
    int64_t* f = flops;
    if (!f) {
        if ((st = ensure(h, h->flops, (size_t)m * 8, s)) != KK_OK) return st;
        f = (int64_t*)h->flops.p;
    }
    kk::Launch L = make_launch(h, s);
    DevStatus* dst = (DevStatus*)h->status_aux.p;
    kk::init_status(L, dst);
    kk::row_flops_bin(L, off64, view(A), view(B), B->ncols, 0, h->opts.validate != 0, nullptr, nullptr, f,
                      (uint8_t*)h->binid.p, (int32_t*)h->counts.p, nullptr, dst);
    if (flops_scan) kk::exclusive_scan(L, true, f, true, flops_scan, m, (int64_t*)h->partial.p, nullptr, nullptr);
    if ((st = cuda_check(h, cudaGetLastError(), "kk_spgemm_row_flops launch")) != KK_OK) return st;
    if (total) {
        if ((st = read_status(h, s, dst, nullptr, "kk_spgemm_row_flops sync")) != KK_OK) return st;
        const DevStatus hs = h->h_aux->st;
        if (h->opts.validate && hs.bad_index) return fail(h, KK_ERR_INDEX_OVERFLOW, "column index of A out of range");
        *total = (int64_t)hs.total_flops;
    }
    return KK_OK;
}

kk_status_t kk_spgemm_symbolic(kk_spgemm_handle_t h, const kk_csr_t* A, const kk_csr_t* B, void* c_row_map,
                               int64_t* c_nnz, void* stream) {
    NvtxRange nvtx_("kk_spgemm_symbolic");
    if (!h) return KK_ERR_INVALID_ARG;
    h->rec.valid = false;
    kk_status_t st;
    if ((st = check_pair(h, A, B, false)) != KK_OK) return st;
    if (!c_row_map) return fail(h, KK_ERR_INVALID_ARG, "c_row_map is NULL");
    if (!c_nnz) return fail(h, KK_ERR_INVALID_ARG, "c_nnz is NULL");
    cudaSetDevice(h->device);
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t m = A->nrows, n = B->nrows, k = B->ncols;
    const bool off64 = A->offset_type == KK_I64;
    const int comp_mode = h->opts.compression;
    // workspace
    if ((st = ensure(h, h->status, sizeof(DevStatus), s)) != KK_OK) return st;
    if ((st = ensure(h, h->flops, (size_t)m * 8, s)) != KK_OK) return st;
    if ((st = ensure(h, h->fscan, (size_t)(m + 1) * 8, s)) != KK_OK) return st;
    if ((st = ensure(h, h->binid, (size_t)m, s)) != KK_OK) return st;
    if ((st = ensure(h, h->perm_sym, (size_t)m * 4, s)) != KK_OK) return st;
    if ((st = ensure(h, h->perm_num, (size_t)m * 4, s)) != KK_OK) return st;
    if ((st = ensure(h, h->counts, (size_t)m * 4, s)) != KK_OK) return st;
    if ((st = ensure(h, h->binscratch, (size_t)kk::bin_scratch_len(m) * 4, s)) != KK_OK) return st;
    if ((st = ensure(h, h->binstart, sizeof(int) * 2 * (kk::NB + 1), s)) != KK_OK) return st;
    if ((st = ensure(h, h->partial, (size_t)kk::scan_partial_len(m) * 8, s)) != KK_OK) return st;
    if ((st = ensure(h, h->cursors, (size_t)A->nnz * 4, s)) != KK_OK) return st;
    if ((st = ensure(h, h->bmeta, (size_t)n * 16, s)) != KK_OK) return st;
    if ((st = ensure(h, h->wlo, (size_t)m * 4, s)) != KK_OK) return st;
    const bool keep_pat = h->opts.patterns != 0;
    const int64_t pat_cap = keep_pat ? 48 * m : 0;
    if (keep_pat) {
        if ((st = ensure(h, h->pat, (size_t)pat_cap * 8, s)) != KK_OK) return st;
        if ((st = ensure(h, h->pat_off, (size_t)m * 8, s)) != KK_OK) return st;
        if ((st = ensure(h, h->pat_len, (size_t)m * 4, s)) != KK_OK) return st;
    }
    if (comp_mode != 0) {
        if ((st = ensure(h, h->bc_len, (size_t)n * 4, s)) != KK_OK) return st;
        if ((st = ensure(h, h->pairs, (size_t)B->nnz * 8, s)) != KK_OK) return st;
    }
    DevStatus* dst = (DevStatus*)h->status.p;
    int* sym_start = (int*)h->binstart.p;
    int* num_start = sym_start + (kk::NB + 1);
    kk::Launch L = make_launch(h, s);
    const MatView Av = view(A), Bv = view(B);

    // inside kk_spgemm_multiply_host, B is the same staging copy growing by row chunks: its rows
    // compressed by the previous block (outputs and flags) are kept
    auto& Cc = h->bcc;
    kk::StatusCarry carry;
    int64_t row0 = 0;
    if (Cc.armed && Cc.valid && Cc.brm == B->row_map && Cc.bent == B->entries && Cc.rows <= n && Cc.k == k &&
        Cc.comp_mode == comp_mode && Cc.validate == h->opts.validate && Cc.bmeta == h->bmeta.p &&
        Cc.bc_len == h->bc_len.p && Cc.pairs == h->pairs.p) {
        row0 = Cc.rows;
        carry = Cc.c;
    }
    Cc.valid = false;
    kk::init_status(L, dst, &carry);
    nvtxRangePushA("a4 compress + a1 flops + a2 scan + a3 bins");
    // a4: sortedness flags (+ B_C unless compression is off)
    kk::check_compress(L, off64, Bv, k, comp_mode != 0, h->opts.validate != 0, (int32_t*)h->bc_len.p,
                       (uint2*)h->pairs.p, (int4*)h->bmeta.p, dst, row0);
    // a1: flops per row, symbolic bins
    kk::row_flops_bin(L, off64, Av, Bv, k, comp_mode, h->opts.validate != 0, (const int32_t*)h->bc_len.p,
                      (const int4*)h->bmeta.p, (int64_t*)h->flops.p,
                      (uint8_t*)h->binid.p, (int32_t*)h->counts.p, (int32_t*)h->wlo.p, dst,
                      keep_pat ? (long long*)h->pat_off.p : nullptr);
    // a2: F = exclusive scan of flops (kept in the handle for flop-balanced partitioning)
    kk::exclusive_scan(L, true, h->flops.p, true, h->fscan.p, m, (int64_t*)h->partial.p, nullptr, nullptr);
    // a3: bin rows by symbolic work
    kk::bin_rows(L, m, (const uint8_t*)h->binid.p, (int32_t*)h->binscratch.p, (int32_t*)h->perm_sym.p, sym_start);
    // the symbolic bin sizes on the host (one sync): empty bins are not launched and grids
    // are sized to their bins
    {
        void* d = h->d_status->sym_bin_start;
        const void* src = sym_start;
        const size_t nb = sizeof(int) * (kk::NB + 1);
        kk::post_words(L, 1, &d, &src, &nb);
    }
    nvtxRangePop();
    if ((st = cuda_check(h, cudaStreamSynchronize(s), "kk_spgemm_symbolic bins")) != KK_OK) return st;
    NvtxRange nvtx_a5("a5 symbolic bins + a6 row map");
    // a5: symbolic kernels per bin (dense bin on the side stream)
    kk::SymArgs sa;
    sa.off64 = off64;
    sa.A = Av;
    sa.B = Bv;
    sa.k = k;
    sa.bc_len = (const int32_t*)h->bc_len.p;
    sa.pairs = (const uint2*)h->pairs.p;
    sa.perm = (const int32_t*)h->perm_sym.p;
    sa.bin_start = sym_start;
    sa.counts = (int32_t*)h->counts.p;
    sa.cursors = (int32_t*)h->cursors.p;
    sa.wlo = (const int32_t*)h->wlo.p;
    sa.host_bin_start = h->h_status->sym_bin_start;
    sa.pat.pat = keep_pat ? (uint2*)h->pat.p : nullptr;
    sa.pat.cap = pat_cap;
    sa.pat.off = keep_pat ? (long long*)h->pat_off.p : nullptr;
    sa.pat.len = keep_pat ? (int*)h->pat_len.p : nullptr;
    sa.st = dst;
    sa.comp_mode = comp_mode;
    if ((st = ensure(h, h->retry, (size_t)(m + 8) * 4, s)) != KK_OK) return st;
    sa.retry = (int*)h->retry.p;
    sa.logG = pick_logG(n > 0 ? (double)B->nnz / (double)n / (comp_mode != 0 ? 2.0 : 1.0) : 1.0);
    cudaStream_t side = nullptr;
    if (h->side) {
        cudaEventRecord(h->ev_fork, s);
        cudaStreamWaitEvent(h->side, h->ev_fork, 0);
        side = h->side;
    }
    kk::symbolic_bins(L, sa, side);
    if (side) {
        cudaEventRecord(h->ev_join, side);
        cudaStreamWaitEvent(s, h->ev_join, 0);
    }
    // a6: row map of C = exclusive scan of counts (overflow check for int32 offsets)
    kk::exclusive_scan(L, false, h->counts.p, off64, c_row_map, m, (int64_t*)h->partial.p, &dst->nnz_c,
                       &dst->overflow);
    // numeric bins from exact counts
    // pattern rows only where the numeric walks B rows of ~11+ entries one per warp step
    const bool use_pat = keep_pat && pick_logG(n > 0 ? (double)B->nnz / (double)n : 1.0) >= 4;
    kk::numeric_binid(L, m, (const int32_t*)h->counts.p, use_pat ? (const long long*)h->pat_off.p : nullptr,
                      (const int*)h->pat_len.p, (const uint2*)h->pat.p, (const int64_t*)h->flops.p,
                      (uint8_t*)h->binid.p, dst);
    kk::bin_rows(L, m, (const uint8_t*)h->binid.p, (int32_t*)h->binscratch.p, (int32_t*)h->perm_num.p, num_start);
    // the status words and both bins' starts to the mapped host copy (one CTA's stores), then
    // the phase's second sync
    {
        void* d[3] = {h->d_status, h->d_status->sym_bin_start, h->d_status->num_bin_start};
        const void* src[3] = {dst, sym_start, num_start};
        const size_t nb[3] = {offsetof(DevStatus, sym_bin_start), sizeof(int) * (kk::NB + 1),
                              sizeof(int) * (kk::NB + 1)};
        kk::post_words(L, 3, d, src, nb);
    }
    if ((st = cuda_check(h, cudaGetLastError(), "kk_spgemm_symbolic launch")) != KK_OK) return st;
    if ((st = cuda_check(h, cudaStreamSynchronize(s), "kk_spgemm_symbolic sync")) != KK_OK) return st;
    const DevStatus& hs = *h->h_status;
    if (h->opts.validate && hs.bad_index) return fail(h, KK_ERR_INDEX_OVERFLOW, "column index out of range");
    if (Cc.armed) {
        Cc.valid = true;
        Cc.brm = B->row_map;
        Cc.bent = B->entries;
        Cc.rows = n;
        Cc.k = k;
        Cc.comp_mode = comp_mode;
        Cc.validate = h->opts.validate;
        Cc.bmeta = h->bmeta.p;
        Cc.bc_len = h->bc_len.p;
        Cc.pairs = h->pairs.p;
        Cc.c.b_sorted = hs.b_sorted;
        Cc.c.b_strict = hs.b_strict;
        Cc.c.bad_index = hs.bad_index;
        Cc.c.total_words = hs.total_words;
    }
    if (hs.overflow)
        return fail(h, KK_ERR_INDEX_OVERFLOW, "nnz(C) = %llu exceeds int32 row offsets; use KK_I64",
                    (unsigned long long)hs.nnz_c);
    if (h->opts.deterministic && !hs.b_strict && A->nrows > 0 && B->nnz > 0)
        return fail(h, KK_ERR_UNSUPPORTED_TYPE,
                    "deterministic mode needs strictly increasing B rows (sorted, no duplicate columns)");
    *c_nnz = (int64_t)hs.nnz_c;
    // record for numeric
    h->rec.valid = true;
    h->rec.m = m;
    h->rec.n = n;
    h->rec.k = k;
    h->rec.nnzA = A->nnz;
    h->rec.nnzB = B->nnz;
    h->rec.nnzC = (int64_t)hs.nnz_c;
    h->rec.arm = A->row_map;
    h->rec.aent = A->entries;
    h->rec.brm = B->row_map;
    h->rec.bent = B->entries;
    h->rec.crm = c_row_map;
    h->rec.offt = (int)A->offset_type;
    memcpy(h->host_num_bin_start, hs.num_bin_start, sizeof(h->host_num_bin_start));
    // stats
    kk_spgemm_stats_t& S = h->stats;
    S.muladds = (int64_t)hs.total_flops;
    S.nnz_c = (int64_t)hs.nnz_c;
    S.compression_used = hs.use_comp;
    S.compressed_words = hs.use_comp ? (int64_t)hs.total_words : 0;
    S.b_sorted = hs.b_sorted;
    S.b_strict = hs.b_strict;
    S.num_symbolic_bins = kk::SYM_NBINS;
    S.num_numeric_bins = kk::NUM_NBINS;
    static_assert(kk::NB <= KK_STATS_MAX_BINS, "stats arrays must hold every bin");
    for (int b = 0; b < KK_STATS_MAX_BINS; ++b) {
        S.symbolic_bin_rows[b] = b < kk::SYM_NBINS ? hs.sym_bin_start[b + 1] - hs.sym_bin_start[b] : 0;
        S.numeric_bin_rows[b] = b < kk::NUM_NBINS ? hs.num_bin_start[b + 1] - hs.num_bin_start[b] : 0;
    }
    return KK_OK;
}

static kk_status_t numeric_impl(kk_spgemm_handle_t h, const kk_csr_t* A, const kk_csr_t* B, const void* c_row_map,
                                int32_t* c_entries, void* c_values, void* stream, const void* dinv, double omega) {
    NvtxRange nvtx_(dinv ? "kk_spgemm_jacobi_numeric" : "kk_spgemm_numeric");
    if (!h) return KK_ERR_INVALID_ARG;
    kk_status_t st;
    if ((st = check_pair(h, A, B, true)) != KK_OK) return st;
    const auto& R = h->rec;
    if (!R.valid || R.m != A->nrows || R.n != B->nrows || R.k != B->ncols || R.nnzA != A->nnz ||
        R.nnzB != B->nnz || R.arm != A->row_map || R.aent != A->entries || R.brm != B->row_map ||
        R.bent != B->entries || R.crm != c_row_map || R.offt != (int)A->offset_type)
        return fail(h, KK_ERR_STALE_HANDLE, "numeric: no matching symbolic for these matrices / row map");
    if (R.nnzC > 0 && (!c_entries || !c_values)) return fail(h, KK_ERR_INVALID_ARG, "c_entries/c_values is NULL");
    cudaSetDevice(h->device);
    cudaStream_t s = (cudaStream_t)stream;
    kk::Launch L = make_launch(h, s);
    kk::NumArgs na;
    na.off64 = A->offset_type == KK_I64;
    na.f64 = A->value_type == KK_F64;
    na.sort = h->opts.sort_rows != 0;
    na.strict = h->stats.b_strict != 0;
    na.sorted = h->stats.b_sorted != 0;
    na.det = h->opts.deterministic != 0;
    tex_for(h, B, &na.tex_ent, &na.tex_val);
    if ((st = ensure(h, h->workctr, 16, s)) != KK_OK) return st;
    na.work_ctr = (int*)h->workctr.p;
    na.wlo = (const int32_t*)h->wlo.p;
    na.pat = (const uint2*)h->pat.p;
    na.pat_off = (const long long*)h->pat_off.p;
    na.pat_len = (const int*)h->pat_len.p;
    na.A = view(A);
    na.B = view(B);
    na.k = B->ncols;
    na.c_row_map = c_row_map;
    na.c_entries = c_entries;
    na.c_values = c_values;
    na.perm = (const int32_t*)h->perm_num.p;
    na.bin_start = (const int*)h->binstart.p + (kk::NB + 1);
    na.host_bin_start = h->host_num_bin_start;
    na.cursors = (int32_t*)h->cursors.p;
    na.st = (const DevStatus*)h->status.p;
    na.logG = pick_logG(B->nrows > 0 ? (double)B->nnz / (double)B->nrows : 1.0);
    // deterministic: one B row per warp step in the warp tables (plain adds, step order)
    if (na.det) na.logG = 5;
    na.dinv = dinv;
    na.omega = omega;
    cudaStream_t side = nullptr;
    const bool dense = h->host_num_bin_start[kk::NUM_DENSE_BIN + 1] > h->host_num_bin_start[kk::NUM_DENSE_BIN];
    if (dinv) {
        if (h->opts.validate) {
            int missing = 0;
            if ((st = ensure(h, h->diagchk, sizeof(int), s)) != KK_OK) return st;
            if (!kk::check_diagonal(L, A->offset_type == KK_I64, A->nrows, A->row_map, A->entries, (int*)h->diagchk.p,
                                    &h->h_aux->missing, &h->d_aux->missing))
                return fail(h, KK_ERR_CUDA, "jacobi numeric: diagonal check failed");
            missing = h->h_aux->missing;
            if (missing)
                return fail(h, KK_ERR_INVALID_ARG, "jacobi numeric: A(i,i) is not stored in %d rows (PAPER.md:194)",
                            missing);
        }
    }
    if (h->side && dense) {
        cudaEventRecord(h->ev_fork, s);
        cudaStreamWaitEvent(h->side, h->ev_fork, 0);
        side = h->side;
    }
    kk::numeric_bins(L, na, side);
    if (side) {
        cudaEventRecord(h->ev_join, side);
        cudaStreamWaitEvent(s, h->ev_join, 0);
    }
    return cuda_check(h, cudaGetLastError(), "kk_spgemm_numeric launch");
}

kk_status_t kk_spgemm_numeric(kk_spgemm_handle_t h, const kk_csr_t* A, const kk_csr_t* B, const void* c_row_map,
                              int32_t* c_entries, void* c_values, void* stream) {
    return numeric_impl(h, A, B, c_row_map, c_entries, c_values, stream, nullptr, 0.0);
}

kk_status_t kk_spgemm_jacobi_numeric(kk_spgemm_handle_t h, double omega, const void* dinv, const kk_csr_t* A,
                                     const kk_csr_t* B, const void* c_row_map, int32_t* c_entries, void* c_values,
                                     void* stream) {
    if (!h) return KK_ERR_INVALID_ARG;
    if (!A || !B) return fail(h, KK_ERR_INVALID_ARG, "A or B is NULL");
    if (A->nrows != A->ncols || B->nrows != A->nrows)
        return fail(h, KK_ERR_DIM_MISMATCH, "jacobi numeric: A must be m x m and B m x k (A %lld x %lld, B %lld rows)",
                    (long long)A->nrows, (long long)A->ncols, (long long)B->nrows);
    if (!dinv && A->nrows > 0) return fail(h, KK_ERR_INVALID_ARG, "jacobi numeric: dinv is NULL");
    return numeric_impl(h, A, B, c_row_map, c_entries, c_values, stream, dinv ? dinv : (const void*)h, omega);
}

kk_status_t kk_spgemm_kernel_times(kk_spgemm_handle_t h, kk_kernel_time_t* out, int* count_inout) {
    if (!h || !count_inout || (*count_inout > 0 && !out)) return KK_ERR_INVALID_ARG;
    if (!h->timer) return fail(h, KK_ERR_INVALID_ARG, "timing is off (kk_spgemm_opts_t.timing = 0)");
    cudaSetDevice(h->device);
    h->timer->resolve();
    const int n = (int)h->timer->acc.size();
    const int w = *count_inout < n ? *count_inout : n;
    for (int i = 0; i < w; ++i) {
        const auto& a = h->timer->acc[i];
        memset(out[i].name, 0, sizeof(out[i].name));
        strncpy(out[i].name, a.name.c_str(), sizeof(out[i].name) - 1);
        out[i].launches = a.n;
        out[i].total_ms = a.tot;
        out[i].max_ms = a.mx;
    }
    *count_inout = n;
    return cuda_check(h, cudaGetLastError(), "kk_spgemm_kernel_times");
}

kk_status_t kk_spgemm_timing_reset(kk_spgemm_handle_t h) {
    if (!h) return KK_ERR_INVALID_ARG;
    if (!h->timer) return fail(h, KK_ERR_INVALID_ARG, "timing is off (kk_spgemm_opts_t.timing = 0)");
    cudaSetDevice(h->device);
    h->timer->resolve();
    h->timer->acc.clear();
    return cuda_check(h, cudaGetLastError(), "kk_spgemm_timing_reset");
}

kk_status_t kk_spgemm_stats(kk_spgemm_handle_t h, kk_spgemm_stats_t* out) {
    if (!h || !out) return KK_ERR_INVALID_ARG;
    *out = h->stats;
    out->kernel_launches = h->launches;
    int64_t ws = 0;
    for (const Buf* b : h->all_bufs) ws += (int64_t)b->bytes;
    {
        const auto& P = h->hp;
        const Buf* hb[] = {&P.brm, &P.bent, &P.bval, &P.arm[0], &P.arm[1], &P.aent[0], &P.aent[1], &P.aval[0],
                           &P.aval[1], &P.crm[0], &P.crm[1], &P.cent[0], &P.cent[1], &P.cval[0], &P.cval[1]};
        for (const Buf* b : hb) ws += (int64_t)b->bytes;
    }
    out->workspace_bytes = ws;
    return KK_OK;
}

// ---- C = A*B from host memory (PAPER.md:169-174 on host buffers) -------------------------
// A runs in contiguous row blocks, each an independent product (Eq. 1):
// block q's host->device copies, its symbolic + numeric phases (the caller's stream) and the
// device->host copy of its rows of C (stream s_out) overlap the neighbouring blocks' (two
// staging slots, events between the streams).  B is copied once, in row chunks (stream s_in),
// and a block waits only for the prefix of B's rows its columns reach; A's blocks go on s_a
// (or, for A == B, are taken from B's device copy).  Without a block count the first block is
// small and the rest are planned from its output size: about KK_HOST_BLOCK_BYTES (48 MB) of traffic
// per block (each block's fixed cost is ~25 launches, slow while PCIe is saturated).  The
// global row map is the blocks' row maps shifted on the device by the nnz before them; status
// reads go through mapped memory (no copy engine), so the copy-out of C runs back to back.
static kk_status_t ensure_host(kk_spgemm_handle_t h, void** p, size_t* have, size_t need, bool keep, size_t used) {
    if (*have >= need) return KK_OK;
    const size_t bytes = need + need / 4 + 256;
    void* q = nullptr;
    if (cudaHostAlloc(&q, bytes, cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        return fail(h, KK_ERR_OUT_OF_MEMORY, "pinned host allocation of %zu bytes failed", bytes);
    }
    if (keep && *p && used) memcpy(q, *p, used);
    if (*p) cudaFreeHost(*p);
    *p = q;
    *have = bytes;
    return KK_OK;
}

// grow a staging buffer outside stream order (its old contents may be in use on any of the
// host path's streams: they are drained first; a warm handle never gets here)
static kk_status_t ensure_now(kk_spgemm_handle_t h, Buf& b, size_t bytes, cudaStream_t s) {
    if (bytes == 0) bytes = 16;
    if (b.bytes >= bytes) return KK_OK;
    auto& P = h->hp;
    cudaStreamSynchronize(s);
    cudaStreamSynchronize(P.s_in);
    cudaStreamSynchronize(P.s_a);
    cudaStreamSynchronize(P.s_out);
    release(h, b);
    bytes = bytes + bytes / 8 + 256;
    void* p = nullptr;
    if (h->opts.alloc) {
        p = h->opts.alloc(bytes, s, h->opts.alloc_ctx);
        if (!p) return fail(h, KK_ERR_OUT_OF_MEMORY, "staging allocation of %zu bytes failed", bytes);
        cudaStreamSynchronize(s);
    } else {
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e != cudaSuccess) return cuda_check(h, e, "cudaMalloc(staging)");
    }
    b.p = p;
    b.bytes = bytes;
    return KK_OK;
}

extern "C" kk_status_t kk_spgemm_multiply_host(kk_spgemm_handle_t h, const kk_csr_t* A, const kk_csr_t* B,
                                              void* c_row_map, int64_t* c_nnz, int32_t** c_entries, void** c_values,
                                              int blocks, void* stream) {
    NvtxRange nvtx_("kk_spgemm_multiply_host");
    if (!h) return KK_ERR_INVALID_ARG;
    kk_status_t st;
    if ((st = check_pair(h, A, B, true)) != KK_OK) return st;
    if (!c_row_map || !c_nnz || !c_entries || !c_values) return fail(h, KK_ERR_INVALID_ARG, "NULL output pointer");
    cudaSetDevice(h->device);
    auto& P = h->hp;
    cudaStream_t s = (cudaStream_t)stream;
    if (!P.s_in) {
        cudaStreamCreateWithFlags(&P.s_in, cudaStreamNonBlocking);
        cudaStreamCreateWithFlags(&P.s_out, cudaStreamNonBlocking);
        cudaStreamCreateWithFlags(&P.s_a, cudaStreamNonBlocking);
    }
    const int64_t m = A->nrows, n = B->nrows;
    const size_t osz = A->offset_type == KK_I64 ? 8 : 4, vsz = A->value_type == KK_F64 ? 8 : 4;
    auto rmv = [&](const void* rm, int64_t i) -> int64_t {
        return osz == 8 ? ((const int64_t*)rm)[i] : (int64_t)((const int32_t*)rm)[i];
    };
    // C = A*A with one host matrix (the squaring the paper benchmarks): A's blocks are copied from
    // the device copy of B instead of crossing PCIe again
    const bool alias = A->row_map == B->row_map && A->entries == B->entries && A->values == B->values &&
                       A->offset_type == B->offset_type && A->nnz == B->nnz && A->nrows == B->nrows;
    // row cuts: fixed for a given block count (the first two a quarter and a half of the others
    // when there are 4+); planned after block 0 otherwise
    const bool adaptive = blocks <= 0 && m >= 65536;
    std::vector<int64_t> cuts{0};
    if (adaptive) {
        cuts.push_back(std::max<int64_t>(1, m / 64));
    } else {
        blocks = (int)std::max<int64_t>(1, std::min<int64_t>(blocks <= 0 ? 1 : blocks, std::max<int64_t>(m, 1)));
        std::vector<double> w(blocks, 1.0);
        if (blocks >= 4) w[0] = 0.25, w[1] = 0.5;
        double wt = 0.0, acc = 0.0;
        for (double x : w) wt += x;
        for (int q = 1; q < blocks; ++q) {
            acc += w[q - 1];
            cuts.push_back(std::max(cuts.back(), std::min<int64_t>(m, (int64_t)((double)m * acc / wt))));
        }
        cuts.push_back(m);
    }
    auto nblocks = [&]() { return (int)cuts.size() - 1; };
    // the caller's row map as device-writable mapped memory, when it is pinned
    void* rm_dev = nullptr;
    {
        cudaPointerAttributes pa;
        if (cudaPointerGetAttributes(&pa, c_row_map) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
            pa.devicePointer != nullptr)
            rm_dev = pa.devicePointer;
        cudaGetLastError();
    }
    if ((st = ensure(h, P.brm, (n + 1) * osz, s)) != KK_OK) return st;
    if ((st = ensure(h, P.bent, B->nnz * 4, s)) != KK_OK) return st;
    if ((st = ensure(h, P.bval, B->nnz * vsz, s)) != KK_OK) return st;
    // the B_C workspace sized for all of B, so the blocks' symbolic phases compress only the
    // rows their prefix adds (kk_spgemm_symbolic keeps the rest while armed)
    h->bcc = kk_spgemm_handle_s::BcCarry();
    const bool carry_ok = ensure(h, h->bmeta, (size_t)n * 16, s) == KK_OK &&
                          ensure(h, h->bc_len, (size_t)n * 4, s) == KK_OK &&
                          ensure(h, h->pairs, (size_t)B->nnz * 8, s) == KK_OK;
    cudaStreamSynchronize(s);  // the workspace may have been (re)allocated on s
    h->bcc.armed = carry_ok;
    // KK_HOST_TRACE=1: per-block copy/compute completion times on stderr (diagnostic)
    static const bool trace = getenv("KK_HOST_TRACE") && atoi(getenv("KK_HOST_TRACE")) > 0;
    const unsigned evflags = trace ? cudaEventDefault : cudaEventDisableTiming;
    const auto t_host0 = std::chrono::steady_clock::now();
    auto host_ms = [&]() {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_host0).count();
    };
    std::vector<std::array<double, 3>> hts;
    cudaEvent_t ev_t0 = nullptr;
    if (trace) {
        cudaEventCreate(&ev_t0);
        cudaEventRecord(ev_t0, P.s_in);
    }
    // B's row chunks, issued on s_in in the order the blocks need them
    const int nch = (int)std::max<int64_t>(1, std::min<int64_t>(16, n));
    std::vector<int64_t> bcut(nch + 1);
    for (int c = 0; c <= nch; ++c) bcut[c] = n * c / nch;
    std::vector<cudaEvent_t> ev_bc(nch);
    for (int c = 0; c < nch; ++c) cudaEventCreateWithFlags(&ev_bc[c], evflags);
    int b_issued = 0;
    auto issue_b = [&](int upto) {
        for (; b_issued <= upto; ++b_issued) {
            const int64_t lo = bcut[b_issued], hi = bcut[b_issued + 1];
            const int64_t e_lo = rmv(B->row_map, lo), e_hi = rmv(B->row_map, hi);
            cudaMemcpyAsync((char*)P.brm.p + lo * osz, (const char*)B->row_map + lo * osz, (hi - lo + 1) * osz,
                            cudaMemcpyHostToDevice, P.s_in);
            cudaMemcpyAsync((char*)P.bent.p + e_lo * 4, B->entries + e_lo, (e_hi - e_lo) * 4, cudaMemcpyHostToDevice,
                            P.s_in);
            cudaMemcpyAsync((char*)P.bval.p + e_lo * vsz, (const char*)B->values + e_lo * vsz, (e_hi - e_lo) * vsz,
                            cudaMemcpyHostToDevice, P.s_in);
            cudaEventRecord(ev_bc[b_issued], P.s_in);
        }
    };
    // the largest column of every group of G rows of A, from helper threads running ahead of
    // the blocks (group g on thread g % T; a group's pass stops once it reaches B's last chunk)
    constexpr int64_t G = 4096;
    const int64_t ngr = (m + G - 1) / G;
    std::vector<int32_t> gmax(std::max<int64_t>(ngr, 1), -1);
    std::unique_ptr<std::atomic<int>[]> gready(new std::atomic<int>[std::max<int64_t>(ngr, 1)]);
    for (int64_t g = 0; g < ngr; ++g) gready[g].store(0, std::memory_order_relaxed);
    std::atomic<bool> stop{false};
    const char* ts = getenv("KK_HOST_SCAN_THREADS");
    const int nthr = (int)std::max<int64_t>(
        1, std::min<int64_t>({ts && atoi(ts) > 0 ? atoi(ts) : 4, (int64_t)std::thread::hardware_concurrency() / 2,
                              (ngr + 7) / 8}));
    std::vector<std::thread> scanners;
    for (int t = 0; t < nthr; ++t)
        scanners.emplace_back([&, t]() {
            const int32_t last = (int32_t)std::min<int64_t>(bcut[nch - 1], INT32_MAX);
            const int32_t* ent = A->entries;
            for (int64_t g = t; g < ngr && !stop.load(std::memory_order_relaxed); g += nthr) {
                const int64_t e0 = rmv(A->row_map, g * G), e1 = rmv(A->row_map, std::min<int64_t>(m, (g + 1) * G));
                int32_t mx = -1;
                for (int64_t i0 = e0; i0 < e1 && mx < last; i0 += 8192) {
                    const int64_t i1 = std::min<int64_t>(e1, i0 + 8192);
                    int32_t m8 = -1;
                    for (int64_t i = i0; i < i1; ++i) m8 = ent[i] > m8 ? ent[i] : m8;
                    mx = std::max(mx, m8);
                }
                gmax[g] = mx;
                gready[g].store(1, std::memory_order_release);
            }
        });
    // the chunk holding every B row rows [r0, r1) of A read (and, for A == B, the rows themselves)
    auto need_chunk = [&](int64_t r0, int64_t r1) {
        int64_t rows = alias ? r1 : 0;
        if (r1 > r0) {
            for (int64_t g = r0 / G; g <= (r1 - 1) / G; ++g) {
                while (!gready[g].load(std::memory_order_acquire)) std::this_thread::yield();
                rows = std::max<int64_t>(rows, (int64_t)gmax[g] + 1);
            }
        }
        int c = 0;
        while (c < nch - 1 && bcut[c + 1] < rows) ++c;
        return c;
    };
    std::vector<cudaEvent_t> ev_in, ev_c, ev_out;
    std::vector<int> bneed;
    std::vector<kk_csr_t> Ab, Bq;
    auto add_events = [&]() {  // per-block records for the blocks cut so far
        while ((int)ev_in.size() < nblocks()) {
            cudaEvent_t e[3];
            for (auto& x : e) cudaEventCreateWithFlags(&x, evflags);
            ev_in.push_back(e[0]);
            ev_c.push_back(e[1]);
            ev_out.push_back(e[2]);
            bneed.push_back(nch - 1);
            Ab.emplace_back();
            Bq.emplace_back();
            if (trace) hts.push_back({0.0, 0.0, 0.0});
        }
    };
    add_events();
    // host side of block q: its B prefix, then (A != B) its rows' copies into slot q % 2
    auto load_block = [&](int q) -> kk_status_t {
        const int sl = q % 2;
        const int64_t r0 = cuts[q], r1 = cuts[q + 1];
        const int64_t e0 = rmv(A->row_map, r0), e1 = rmv(A->row_map, r1);
        kk_status_t e;
        if ((e = ensure_now(h, P.arm[sl], (r1 - r0 + 1) * osz, s)) != KK_OK) return e;
        if ((e = ensure_now(h, P.crm[sl], (r1 - r0 + 1) * osz, s)) != KK_OK) return e;
        if ((e = ensure_now(h, P.aent[sl], (e1 - e0) * 4, s)) != KK_OK) return e;
        if ((e = ensure_now(h, P.aval[sl], (e1 - e0) * vsz, s)) != KK_OK) return e;
        bneed[q] = need_chunk(r0, r1);
        issue_b(bneed[q]);
        kk_csr_t b = *B;  // the prefix of B's rows the block reads
        b.nrows = bcut[bneed[q] + 1];
        b.nnz = rmv(B->row_map, b.nrows);
        b.row_map = P.brm.p;
        b.entries = (const int32_t*)P.bent.p;
        b.values = P.bval.p;
        Bq[q] = b;
        if (!alias) {
            // the block's row map as is (rebased to 0 on the device), entries, values
            if (q >= 2) cudaStreamWaitEvent(P.s_a, ev_c[q - 2], 0);  // slot free once block q-2 is computed
            cudaMemcpyAsync(P.arm[sl].p, (const char*)A->row_map + r0 * osz, (r1 - r0 + 1) * osz,
                            cudaMemcpyHostToDevice, P.s_a);
            cudaMemcpyAsync(P.aent[sl].p, A->entries + e0, (e1 - e0) * 4, cudaMemcpyHostToDevice, P.s_a);
            cudaMemcpyAsync(P.aval[sl].p, (const char*)A->values + e0 * vsz, (e1 - e0) * vsz,
                            cudaMemcpyHostToDevice, P.s_a);
        }
        cudaEventRecord(ev_in[q], alias ? P.s_in : P.s_a);
        kk_csr_t a = *A;
        a.nrows = r1 - r0;
        a.ncols = b.nrows;
        a.nnz = e1 - e0;
        a.row_map = P.arm[sl].p;
        a.entries = (const int32_t*)P.aent[sl].p;
        a.values = P.aval[sl].p;
        Ab[q] = a;
        return KK_OK;
    };
    // the rest of the rows after block 0, from block 0's output size: blocks of about
    // KK_HOST_BLOCK_BYTES (default 48 MB) of host<->device traffic, the first half size
    auto plan = [&](int64_t nnz0) {
        const char* tb = getenv("KK_HOST_BLOCK_BYTES");
        const double target = tb && atof(tb) > 0 ? atof(tb) : 48e6;
        const int64_t r0 = cuts[1], rows0 = std::max<int64_t>(cuts[1], 1);
        if (r0 >= m) return;
        const double out = (double)nnz0 * (double)(4 + vsz) / (double)rows0 * (double)(m - r0) +
                           (double)(m - r0) * osz;
        const double ina = alias ? 0.0 : (double)(rmv(A->row_map, m) - rmv(A->row_map, r0)) * (4.0 + vsz) +
                                             (double)(m - r0) * osz;
        const double inb = (double)(B->nnz - rmv(B->row_map, bcut[bneed[0] + 1])) * (4.0 + vsz);
        const int nb = (int)std::max<double>(1.0, std::min<double>(64.0, std::ceil((out + ina + inb) / target)));
        const double wt = nb - 0.5;
        double acc = 0.0;
        for (int q = 0; q < nb - 1; ++q) {
            acc += q == 0 ? 0.5 : 1.0;
            cuts.push_back(std::max(cuts.back(), std::min<int64_t>(m, r0 + (int64_t)((double)(m - r0) * acc / wt))));
        }
        cuts.push_back(m);
        add_events();
    };
    {
        // B's texture objects sized for all of it, so the blocks' prefixes share them
        kk_csr_t bf = *B;
        bf.row_map = P.brm.p;
        bf.entries = (const int32_t*)P.bent.p;
        bf.values = P.bval.p;
        unsigned long long te, tv;
        tex_for(h, &bf, &te, &tv);
    }
    std::vector<int64_t> nnz_off{0};
    st = load_block(0);
    for (int q = 0; q < nblocks() && st == KK_OK; ++q) {
        const int sl = q % 2;
        const int64_t r0 = cuts[q], r1 = cuts[q + 1];
        cudaStreamWaitEvent(s, ev_in[q], 0);
        cudaStreamWaitEvent(s, ev_bc[bneed[q]], 0);
        if (q >= 2) cudaStreamWaitEvent(s, ev_out[q - 2], 0);  // C slot drained to the host
        {
            // the block's row map rebased to 0 on the device; for A == B (same host matrix) its rows
            // come from the device copy of B.  Slot sl is free: block q-2 was computed earlier on
            // this stream.
            kk::Launch L = make_launch(h, s);
            const int64_t e0 = rmv(A->row_map, r0), e1 = rmv(A->row_map, r1);
            if (alias) {
                kk::copy_rows(L, osz == 8, P.arm[sl].p, (const char*)P.brm.p + r0 * osz, r1 - r0 + 1, e0,
                              P.aent[sl].p, (const char*)P.bent.p + e0 * 4, (e1 - e0) * 4, P.aval[sl].p,
                              (const char*)P.bval.p + e0 * vsz, (e1 - e0) * vsz);
            } else {
                kk::rebase_row_map(L, osz == 8, P.arm[sl].p, P.arm[sl].p, r1 - r0 + 1, e0);
            }
        }
        int64_t nnz = 0;
        if (trace) hts[q][0] = host_ms();
        if ((st = kk_spgemm_symbolic(h, &Ab[q], &Bq[q], P.crm[sl].p, &nnz, s)) != KK_OK) break;
        if (trace) hts[q][1] = host_ms();
        if (q == 0) {
            if (adaptive) plan(nnz);
            // block 1 as soon as block 0's symbolic phase has run
            if (nblocks() > 1 && (st = load_block(1)) != KK_OK) break;
        }
        if ((st = ensure(h, P.cent[sl], nnz * 4, s)) != KK_OK) break;
        if ((st = ensure(h, P.cval[sl], nnz * vsz, s)) != KK_OK) break;
        if ((st = kk_spgemm_numeric(h, &Ab[q], &Bq[q], P.crm[sl].p, (int32_t*)P.cent[sl].p, P.cval[sl].p, s)) !=
            KK_OK)
            break;
        nnz_off.push_back(nnz_off[q] + nnz);
        if (osz == 4 && nnz_off[q + 1] > INT32_MAX) {
            st = fail(h, KK_ERR_INDEX_OVERFLOW, "nnz(C) exceeds int32 row offsets; use KK_I64");
            break;
        }
        {
            // the block's row map shifted to global offsets on the device (no host pass); when
            // the caller's row map is pinned (mapped) the kernel writes it there directly, one
            // copy-engine transfer less per block (each costs ~45 us of DMA restart)
            kk::Launch L = make_launch(h, s);
            kk::add_offset(L, osz == 8, (char*)P.crm[sl].p + osz, r1 - r0, nnz_off[q],
                           rm_dev ? (char*)rm_dev + (r0 + 1) * osz : nullptr);
        }
        cudaEventRecord(ev_c[q], s);
        // host output capacity (grows on a larger product: earlier blocks are kept)
        if (P.h_cent_bytes < (size_t)nnz_off[q + 1] * 4 || P.h_cval_bytes < (size_t)nnz_off[q + 1] * vsz) {
            cudaStreamSynchronize(P.s_out);
            if ((st = ensure_host(h, &P.h_cent, &P.h_cent_bytes, nnz_off[q + 1] * 4, true, nnz_off[q] * 4)) != KK_OK)
                break;
            if ((st = ensure_host(h, &P.h_cval, &P.h_cval_bytes, nnz_off[q + 1] * vsz, true, nnz_off[q] * vsz)) !=
                KK_OK)
                break;
        }
        cudaStreamWaitEvent(P.s_out, ev_c[q], 0);
        // rows r0+1..r1 of the global row map (entry r0 is the previous block's end)
        if (!rm_dev)
            cudaMemcpyAsync((char*)c_row_map + (r0 + 1) * osz, (const char*)P.crm[sl].p + osz, (r1 - r0) * osz,
                            cudaMemcpyDeviceToHost, P.s_out);
        cudaMemcpyAsync((char*)P.h_cent + nnz_off[q] * 4, P.cent[sl].p, nnz * 4, cudaMemcpyDeviceToHost, P.s_out);
        cudaMemcpyAsync((char*)P.h_cval + nnz_off[q] * vsz, P.cval[sl].p, nnz * vsz, cudaMemcpyDeviceToHost,
                        P.s_out);
        cudaEventRecord(ev_out[q], P.s_out);
        // block q+2's copies once this block's are queued (two ahead); it reuses slot q % 2, whose
        // wait is on ev_c[q], recorded above
        if (q + 2 < nblocks() && (st = load_block(q + 2)) != KK_OK) break;
        if (trace) hts[q][2] = host_ms();
    }
    stop.store(true);
    for (auto& t : scanners) t.join();
    h->bcc = kk_spgemm_handle_s::BcCarry();
    cudaStreamSynchronize(P.s_in);
    cudaStreamSynchronize(P.s_a);
    cudaStreamSynchronize(P.s_out);
    cudaStreamSynchronize(s);
    const int nbk = nblocks();
    if (trace && st == KK_OK) {
        auto at = [&](cudaEvent_t e) {
            float ms = -1.f;
            cudaEventElapsedTime(&ms, ev_t0, e);
            return ms;
        };
        fprintf(stderr, "[kk host] %d blocks%s; B in %.3f ms (%d chunks)\n", nbk, adaptive ? " (planned)" : "",
                at(ev_bc[std::min(b_issued, nch) - 1]), nch);
        for (int q = 0; q < nbk; ++q)
            fprintf(stderr,
                    "[kk host] block %d: in %.3f  computed %.3f  out %.3f ms (nnz %lld, B rows %lld)  host: "
                    "symbolic %.3f-%.3f, issued %.3f\n",
                    q, at(ev_in[q]), at(ev_c[q]), at(ev_out[q]), (long long)(nnz_off[q + 1] - nnz_off[q]),
                    (long long)Bq[q].nrows, hts[q][0], hts[q][1], hts[q][2]);
    }
    if (ev_t0) cudaEventDestroy(ev_t0);
    for (size_t q = 0; q < ev_in.size(); ++q) {
        cudaEventDestroy(ev_in[q]);
        cudaEventDestroy(ev_c[q]);
        cudaEventDestroy(ev_out[q]);
    }
    for (int c = 0; c < nch; ++c) cudaEventDestroy(ev_bc[c]);
    if (st != KK_OK) return st;
    if ((st = cuda_check(h, cudaGetLastError(), "kk_spgemm_multiply_host")) != KK_OK) return st;
    // the blocks' row maps arrived already shifted to global offsets; entry 0 is 0
    if (osz == 8)
        ((int64_t*)c_row_map)[0] = 0;
    else
        ((int32_t*)c_row_map)[0] = 0;
    *c_nnz = nnz_off[nbk];
    *c_entries = (int32_t*)P.h_cent;
    *c_values = P.h_cval;
    return KK_OK;
}

// ---- fused triple product Ac = R*A*P (NEXT-4) ----------------------
static kk_status_t check_triple(kk_spgemm_handle_t h, const kk_csr_t* R, const kk_csr_t* A, const kk_csr_t* P,
                                bool need_values) {
    kk_status_t s;
    if ((s = check_pair(h, R, A, need_values)) != KK_OK) return s;
    if ((s = check_pair(h, A, P, need_values)) != KK_OK) return s;
    return KK_OK;
}

extern "C" kk_status_t kk_spgemm_rap_symbolic(kk_spgemm_handle_t h, const kk_csr_t* R, const kk_csr_t* A,
                                             const kk_csr_t* P, void* c_row_map, int64_t* c_nnz, void* stream) {
    if (!h) return KK_ERR_INVALID_ARG;
    NvtxRange nvtx_("kk_spgemm_rap_symbolic");
    h->raprec.valid = false;
    kk_status_t st;
    if ((st = check_triple(h, R, A, P, false)) != KK_OK) return st;
    if (!c_row_map || !c_nnz) return fail(h, KK_ERR_INVALID_ARG, "c_row_map / c_nnz is NULL");
    cudaSetDevice(h->device);
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t mc = R->nrows;
    const bool off64 = R->offset_type == KK_I64;
    if ((st = ensure(h, h->status_aux, sizeof(DevStatus), s)) != KK_OK) return st;
    if ((st = ensure(h, h->counts, (size_t)mc * 4, s)) != KK_OK) return st;
    if ((st = ensure(h, h->partial, (size_t)kk::scan_partial_len(mc) * 8, s)) != KK_OK) return st;
    if ((st = ensure(h, h->spflag, sizeof(int), s)) != KK_OK) return st;
    DevStatus* dst = (DevStatus*)h->status_aux.p;
    kk::Launch L = make_launch(h, s);
    kk::init_status(L, dst);
    cudaMemsetAsync(h->spflag.p, 0, sizeof(int), s);
    kk::rap_symbolic(L, off64, view(R), view(A), view(P), (int32_t*)h->counts.p, (int*)h->spflag.p);
    kk::exclusive_scan(L, false, h->counts.p, off64, c_row_map, mc, (int64_t*)h->partial.p, &dst->nnz_c,
                       &dst->overflow);
    if ((st = read_status(h, s, dst, (const int*)h->spflag.p, "kk_spgemm_rap_symbolic sync")) != KK_OK) return st;
    const DevStatus hs = h->h_aux->st;
    const int too_many = h->h_aux->flag;
    if (too_many)
        return fail(h, KK_ERR_UNSUPPORTED_TYPE,
                    "fused R*A*P: a coarse row has more than 256 distinct columns (use two products)");
    if (hs.overflow)
        return fail(h, KK_ERR_INDEX_OVERFLOW, "nnz(Ac) = %llu exceeds int32 row offsets; use KK_I64",
                    (unsigned long long)hs.nnz_c);
    *c_nnz = (int64_t)hs.nnz_c;
    auto& Q = h->raprec;
    Q.valid = true;
    Q.mc = mc;
    Q.nnzR = R->nnz;
    Q.nnzA = A->nnz;
    Q.nnzP = P->nnz;
    Q.nnzC = (int64_t)hs.nnz_c;
    Q.rrm = R->row_map;
    Q.arm = A->row_map;
    Q.prm = P->row_map;
    Q.crm = c_row_map;
    Q.offt = (int)R->offset_type;
    return KK_OK;
}

extern "C" kk_status_t kk_spgemm_rap_numeric(kk_spgemm_handle_t h, const kk_csr_t* R, const kk_csr_t* A,
                                            const kk_csr_t* P, const void* c_row_map, int32_t* c_entries,
                                            void* c_values, void* stream) {
    if (!h) return KK_ERR_INVALID_ARG;
    NvtxRange nvtx_("kk_spgemm_rap_numeric");
    kk_status_t st;
    if ((st = check_triple(h, R, A, P, true)) != KK_OK) return st;
    const auto& Q = h->raprec;
    if (!Q.valid || Q.mc != R->nrows || Q.nnzR != R->nnz || Q.nnzA != A->nnz || Q.nnzP != P->nnz ||
        Q.rrm != R->row_map || Q.arm != A->row_map || Q.prm != P->row_map || Q.crm != c_row_map ||
        Q.offt != (int)R->offset_type)
        return fail(h, KK_ERR_STALE_HANDLE, "rap numeric: no matching rap symbolic for these matrices / row map");
    if (Q.nnzC > 0 && (!c_entries || !c_values)) return fail(h, KK_ERR_INVALID_ARG, "c_entries/c_values is NULL");
    cudaSetDevice(h->device);
    cudaStream_t s = (cudaStream_t)stream;
    kk::Launch L = make_launch(h, s);
    kk::rap_numeric(L, R->offset_type == KK_I64, R->value_type == KK_F64, view(R), view(A), view(P), c_row_map,
                    c_entries, c_values);
    return cuda_check(h, cudaGetLastError(), "kk_spgemm_rap_numeric launch");
}

// ---- SpAdd (Sec. 2.3) -------------------------------------------------
static kk_status_t check_add_pair(kk_spgemm_handle_t h, const kk_csr_t* A, const kk_csr_t* B, bool need_values) {
    kk_status_t s;
    if ((s = check_csr(h, A, "A", need_values)) != KK_OK) return s;
    if ((s = check_csr(h, B, "B", need_values)) != KK_OK) return s;
    if (A->nrows != B->nrows || A->ncols != B->ncols)
        return fail(h, KK_ERR_DIM_MISMATCH, "SpAdd: A is %lld x %lld, B is %lld x %lld", (long long)A->nrows,
                    (long long)A->ncols, (long long)B->nrows, (long long)B->ncols);
    if (A->offset_type != B->offset_type)
        return fail(h, KK_ERR_UNSUPPORTED_TYPE, "A and B must use the same offset type");
    if (need_values && A->value_type != B->value_type)
        return fail(h, KK_ERR_UNSUPPORTED_TYPE, "A and B must use the same value type");
    return KK_OK;
}

kk_status_t kk_spadd_symbolic(kk_spgemm_handle_t h, const kk_csr_t* A, const kk_csr_t* B, void* c_row_map,
                              int64_t* c_nnz, void* stream) {
    NvtxRange nvtx_("kk_spadd_symbolic");
    if (!h) return KK_ERR_INVALID_ARG;
    h->addrec.valid = false;
    kk_status_t st;
    if ((st = check_add_pair(h, A, B, false)) != KK_OK) return st;
    if (!c_row_map) return fail(h, KK_ERR_INVALID_ARG, "c_row_map is NULL");
    if (!c_nnz) return fail(h, KK_ERR_INVALID_ARG, "c_nnz is NULL");
    cudaSetDevice(h->device);
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t m = A->nrows;
    const bool off64 = A->offset_type == KK_I64;
    if ((st = ensure(h, h->status_aux, sizeof(DevStatus), s)) != KK_OK) return st;
    if ((st = ensure(h, h->counts, (size_t)m * 4, s)) != KK_OK) return st;
    if ((st = ensure(h, h->partial, (size_t)kk::scan_partial_len(m) * 8, s)) != KK_OK) return st;
    if ((st = ensure(h, h->apos, (size_t)A->nnz * 4, s)) != KK_OK) return st;
    if ((st = ensure(h, h->bpos, (size_t)B->nnz * 4, s)) != KK_OK) return st;
    if ((st = ensure(h, h->spdup, (size_t)m, s)) != KK_OK) return st;
    if ((st = ensure(h, h->spflag, sizeof(int), s)) != KK_OK) return st;
    DevStatus* dst = (DevStatus*)h->status_aux.p;
    kk::Launch L = make_launch(h, s);
    kk::init_status(L, dst);
    cudaMemsetAsync(h->spflag.p, 0, sizeof(int), s);
    kk::spadd_symbolic(L, off64, m, view(A), view(B), (int32_t*)h->counts.p, (int32_t*)h->apos.p,
                       (int32_t*)h->bpos.p, (uint8_t*)h->spdup.p, (int*)h->spflag.p);
    kk::exclusive_scan(L, false, h->counts.p, off64, c_row_map, m, (int64_t*)h->partial.p, &dst->nnz_c,
                       &dst->overflow);
    if ((st = read_status(h, s, dst, (const int*)h->spflag.p, "kk_spadd_symbolic sync")) != KK_OK) return st;
    const DevStatus hs = h->h_aux->st;
    const int too_long = h->h_aux->flag;
    if (too_long)
        return fail(h, KK_ERR_UNSUPPORTED_TYPE, "SpAdd: a row has nnz(A_i) + nnz(B_i) > 16384 (the CTA tier's shared-memory sort)");
    if (hs.overflow)
        return fail(h, KK_ERR_INDEX_OVERFLOW, "nnz(C) = %llu exceeds int32 row offsets; use KK_I64",
                    (unsigned long long)hs.nnz_c);
    *c_nnz = (int64_t)hs.nnz_c;
    auto& R = h->addrec;
    R.valid = true;
    R.nnzC = (int64_t)hs.nnz_c;
    R.m = m;
    R.k = A->ncols;
    R.nnzA = A->nnz;
    R.nnzB = B->nnz;
    R.arm = A->row_map;
    R.aent = A->entries;
    R.brm = B->row_map;
    R.bent = B->entries;
    R.crm = c_row_map;
    R.offt = (int)A->offset_type;
    return KK_OK;
}

kk_status_t kk_spadd_numeric(kk_spgemm_handle_t h, double alpha, const kk_csr_t* A, double beta, const kk_csr_t* B,
                             const void* c_row_map, int32_t* c_entries, void* c_values, void* stream) {
    NvtxRange nvtx_("kk_spadd_numeric");
    if (!h) return KK_ERR_INVALID_ARG;
    kk_status_t st;
    if ((st = check_add_pair(h, A, B, true)) != KK_OK) return st;
    const auto& R = h->addrec;
    if (!R.valid || R.m != A->nrows || R.k != A->ncols || R.nnzA != A->nnz || R.nnzB != B->nnz ||
        R.arm != A->row_map || R.aent != A->entries || R.brm != B->row_map || R.bent != B->entries ||
        R.crm != c_row_map || R.offt != (int)A->offset_type)
        return fail(h, KK_ERR_STALE_HANDLE, "spadd numeric: no matching spadd symbolic for these matrices / row map");
    if (R.nnzC > 0 && (!c_entries || !c_values)) return fail(h, KK_ERR_INVALID_ARG, "c_entries/c_values is NULL");
    cudaSetDevice(h->device);
    cudaStream_t s = (cudaStream_t)stream;
    kk::Launch L = make_launch(h, s);
    kk::spadd_numeric(L, A->offset_type == KK_I64, A->value_type == KK_F64, A->nrows, alpha, view(A), beta, view(B),
                      c_row_map, c_entries, c_values, (const int32_t*)h->apos.p, (const int32_t*)h->bpos.p,
                      (const uint8_t*)h->spdup.p);
    return cuda_check(h, cudaGetLastError(), "kk_spadd_numeric launch");
}

}  // extern "C"
