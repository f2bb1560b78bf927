// api.cu -- the C ABI of libadaptsolve.so (include/adaptsolve.h) and the
// device-resident dispatcher.
//
// Per (device, dtype, n, nrhs, lda, ldb, options) a plan owns one workspace
// and one instantiated CUDA graph that contains the whole flowchart of the
// paper:
//
//   set_args -> state_init -> detect (diag pass, tile-pair pass) -> dispatch
//   SWITCH(method) { BAND | TRI_LOWER | TRI_UPPER | CHOL(+IF fail -> LU) | LU }
//       each body = factor + rcond estimate (state machine, no host sync)
//   gate -> SWITCH(post) { nothing | primary solve (SWITCH method) |
//                          SVD fallback: QR, WHILE(Jacobi sweep), min-norm }
//   finalize -> report D2H
//
// Every branch decision is a graph conditional node whose value a kernel
// sets from device-resident flags, so a call is one graph launch and one
// stream synchronization.
#include <cuda.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <type_traits>
#include <memory>
#include <mutex>
#include <tuple>
#include <vector>

#include "factor.h"
#include "gemm.h"
#include "internal.h"
#include "rcond.h"
#include "small.h"
#include "svd.h"
#include "trsm.h"

namespace as {

struct RepOut {
    as_report rep;
    int32_t ret;
    int32_t kernel_nodes_hint;
};

// ------------------------------------------------------------------ small kernels
__global__ void set_args_kernel2(DevArgs a, DevArgs* dst) {
    *dst = a;
    // the tensor map in the argument block is consumed through the tensormap proxy (detect.cu)
    asm volatile("fence.proxy.tensormap::generic.release.gpu;" ::: "memory");
}

// 2-D tensor map of A for the detection tile pipeline (TMA 2-D tiles): dims
// (rows, columns) = (n, n), row stride lda, box 64 x 64, no swizzle, out-of-range elements read as 0.
typedef CUresult (*TmapEncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                              const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static TmapEncFn tmap_encoder() {
    static TmapEncFn enc = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess) { cudaGetLastError(); f = nullptr; }
        return (TmapEncFn)f;
    }();
    return enc;
}
// A plan takes the TMA pair pass when the shape qualifies (detect_tma_plan), A is 16-byte aligned (part of
// the plan key: the choice between the two pair kernels is made on the host) and the driver can encode maps.
static bool plan_uses_tma(int dt, int64_t n, int64_t lda, bool a16) {
    return a16 && detect_tma_plan(dt, n, lda) && tmap_encoder() != nullptr;
}
static int fill_tmap(DevArgs& a, int dt, const void* A, int64_t lda, int64_t n) {
    a.tma_ok = 0;
    const size_t es = dt == AS_F64 ? 8 : 4;
    static_assert(sizeof(CUtensorMap) == sizeof(a.tmapA), "CUtensorMap is 128 bytes");
    const cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)n}, strides[1] = {(cuuint64_t)(lda * es)};
    const cuuint32_t box[2] = {kTile, kTile}, estr[2] = {1, 1};
    CUtensorMap tm;
    const CUresult r = tmap_encoder()(&tm, dt == AS_F64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                                      const_cast<void*>(A), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        fprintf(stderr, "[adaptsolve] cuTensorMapEncodeTiled failed (%d)\n", (int)r);
        return AS_ERR_CUDA_BASE + (int)cudaErrorInvalidValue;
    }
    memcpy(a.tmapA, &tm, sizeof(tm));
    a.tma_ok = 1;
    return 0;
}
__global__ void set_cond_kernel(cudaGraphConditionalHandle h, unsigned v) {
    if (threadIdx.x == 0) cudaGraphSetConditional(h, v);
}

// triangular path prep: first exact-zero diagonal (singular), triangle 1-norm.  One CTA per column pair
// (u, n-1-u): n + 1 elements together whatever u, every load of a column in flight at once (a warp per
// column left the longest column, n / 32 dependent rounds on one warp, as the kernel's critical path);
// the eight warp sums of a column are added in a fixed order (no floating-point atomics: Z25).
template <typename T>
__global__ void __launch_bounds__(256) tri_prep_kernel(const DevArgs* args, int64_t lda, int64_t n, DevState* st, int upper) {
    const T* A = (const T*)args->A;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ T wsum[2][8];
    double best = 0.0;
    unsigned long long info = ~0ull;
    for (int64_t u = blockIdx.x; u < (n + 1) / 2; u += gridDim.x) {
        T s[2] = {T(0), T(0)};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t j = h ? n - 1 - u : u;
            if (h && j == u) break;
            const int64_t i0 = upper ? 0 : j, i1 = upper ? j : n - 1;
            const T* col = A + j * lda;
            T a0 = T(0), a1 = T(0), a2 = T(0), a3 = T(0);
            for (int64_t i = i0 + threadIdx.x; i <= i1; i += 4 * 256) {
                const T v0 = col[i];
                const T v1 = i + 256 <= i1 ? col[i + 256] : T(0);
                const T v2 = i + 512 <= i1 ? col[i + 512] : T(0);
                const T v3 = i + 768 <= i1 ? col[i + 768] : T(0);
                a0 += v0 < T(0) ? -v0 : v0; a1 += v1 < T(0) ? -v1 : v1;
                a2 += v2 < T(0) ? -v2 : v2; a3 += v3 < T(0) ? -v3 : v3;
            }
            s[h] = warp_sum((a0 + a1) + (a2 + a3));
        }
        __syncthreads();                 // the previous pair's sums have been read
        if (lane == 0) { wsum[0][warp] = s[0]; wsum[1][warp] = s[1]; }
        __syncthreads();
        if (threadIdx.x == 0) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t j = h ? n - 1 - u : u;
                if (h && j == u) break;
                T t = T(0);
#pragma unroll
                for (int w = 0; w < 8; ++w) t += wsum[h][w];
                if ((double)t > best || t != t) best = (double)t;
                if (A[j + j * lda] == T(0) && (unsigned long long)(j + 1) < info) info = (unsigned long long)(j + 1);
            }
        }
    }
    if (threadIdx.x == 0) {
        if (best > 0.0) atomicMax(&st->anorm_bits, dbits(best));
        if (info != ~0ull) atomicMin(&st->info, info);
    }
}

__global__ void gate_kernel(DevState* st, cudaGraphConditionalHandle h_post) {
    if (threadIdx.x != 0) return;
    if (st->flags & AS_FLAG_NONFINITE) {   // AS_OPT_CHECK_FINITE rejected the input (Z28): nothing runs
        st->post = 0;
        if (h_post) cudaGraphSetConditional(h_post, 0u);
        return;
    }
    const bool singular = st->info != ~0ull;
    if (singular) { st->flags |= AS_FLAG_SINGULAR; st->rcond = 0.0; }
    const double r = st->rcond;
    const bool gate = singular || !(r >= st->thr);   // Z11: NaN -> gate
    unsigned post = 1;
    if (gate) {
        st->flags |= AS_FLAG_RCOND_LOW;
        if (st->opts & AS_OPT_NO_FALLBACK) {
            if (singular) { st->ret = AS_ERR_SINGULAR_NO_FALLBACK; post = 0; }
            else { st->flags |= AS_FLAG_POORLY_COND; post = 1; }
        } else {
            post = 2;
        }
    }
    st->gate = gate ? 1 : 0;
    st->post = (int)post;
    if (h_post) cudaGraphSetConditional(h_post, post);
}

__global__ void solve_dispatch_kernel(DevState* st, cudaGraphConditionalHandle h) {
    if (threadIdx.x == 0) cudaGraphSetConditional(h, (unsigned)st->method);
}

__global__ void finalize_kernel(const DevState* st, RepOut* out, const DevArgs* args) {
    if (threadIdx.x != 0) return;
    RepOut o;
    memset(&o, 0, sizeof(o));
    const bool fullscan = (st->opts & (AS_OPT_FULLSCAN | AS_OPT_FORCE_METHOD)) != 0;
    o.rep.flags = st->det_flags | ((unsigned)st->method << AS_FLAG_METHOD_SHIFT) | st->flags;
    o.rep.method = st->method;
    o.rep.primary_method = st->primary;
    o.rep.sweeps = st->sweeps;
    const bool banded = (st->det_flags & AS_FLAG_BANDED) || st->primary == AS_METHOD_BAND;
    o.rep.kl = (banded || fullscan) ? st->kl : -1;
    o.rep.ku = (banded || fullscan) ? st->ku : -1;
    o.rep.rcond = st->info != ~0ull ? 0.0 : st->rcond;
    o.rep.anorm = dfrom(st->anorm_bits);
    o.rep.rank = (st->flags & AS_FLAG_FALLBACK) ? st->rank : -1;
    o.rep.info = st->info == ~0ull ? 0 : (int64_t)st->info;
    o.rep.chol_fail_col = st->chol_failed ? st->chol_fail_col : 0;
    o.ret = st->ret;
    *out = o;
    if (args->rep_dev) *args->rep_dev = o.rep;
    if (args->ret_dev) *args->ret_dev = o.ret;
}

// ------------------------------------------------------------------ capture helpers
static int check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        fprintf(stderr, "[adaptsolve] %s: %s\n", what, cudaGetErrorString(e));
        return AS_ERR_CUDA_BASE + (int)e;
    }
    return 0;
}

static int64_t count_kernels(cudaGraph_t g);

static cudaGraphConditionalHandle make_handle(cudaStream_t s, unsigned defval) {
    cudaStreamCaptureStatus stt;
    cudaGraph_t g;
    const cudaGraphNode_t* deps;
    size_t nd;
    cudaStreamGetCaptureInfo(s, &stt, nullptr, &g, &deps, &nd);
    cudaGraphConditionalHandle h = 0;
    cudaGraphConditionalHandleCreate(&h, g, defval, cudaGraphCondAssignDefault);
    return h;
}

// adds a conditional node after the current capture frontier of s; returns its body graphs
static cudaGraph_t* add_cond(cudaStream_t s, cudaGraphConditionalHandle h, cudaGraphConditionalNodeType type,
                             unsigned size) {
    cudaStreamCaptureStatus stt;
    cudaGraph_t g;
    const cudaGraphNode_t* deps;
    size_t nd;
    cudaStreamGetCaptureInfo(s, &stt, nullptr, &g, &deps, &nd);
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = type;
    p.conditional.size = size;
    cudaGraphNode_t node;
    std::vector<cudaGraphNode_t> dv(deps, deps + nd);
    check(cudaGraphAddNode(&node, g, dv.data(), dv.size(), &p), "cudaGraphAddNode(conditional)");
    cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies);
    return p.conditional.phGraph_out;
}

struct Builder {
    Work w;
    SyncAlloc sa;
    std::vector<cudaStream_t> streams;   // capture stream per nesting depth
    int depth = 0;
    int err = 0;
    cudaStream_t cur() { return streams[depth]; }
    template <typename F>
    void body(cudaGraph_t g, F&& fn) {
        ++depth;
        cudaStream_t s = streams[depth];
        err = err ? err : check(cudaStreamBeginCaptureToGraph(s, g, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed),
                                "BeginCaptureToGraph");
        fn(s);
        cudaGraph_t out;
        err = err ? err : check(cudaStreamEndCapture(s, &out), "EndCapture(body)");
        --depth;
    }
};

// The 1-norm / zero-diagonal pass streams the whole triangle while the diagonal-block inverses touch only
// n / 64 blocks: the two run side by side (a second captured stream).  The inverses' "skip if singular"
// test may then miss a zero diagonal found concurrently; their output is unused in that case (every
// solve checks the flag itself).
struct TriStreams {
    cudaStream_t aux = nullptr;
    cudaEvent_t ev[2];
};
static TriStreams& tri_streams() {
    static thread_local TriStreams S;
    if (!S.aux) {
        cudaStreamCreateWithFlags(&S.aux, cudaStreamNonBlocking);
        for (auto& e : S.ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    }
    return S;
}
static void tri_prep(const Work& w, bool upper, cudaStream_t s) {
    TriStreams& TS = tri_streams();
    cudaEventRecord(TS.ev[0], s);
    cudaStreamWaitEvent(TS.aux, TS.ev[0], 0);
    launch_trtri_blocks(w.dtype, nullptr, w.lda, w.n, w.Dinv0, upper, false, w.st, true, w.args, TS.aux);
    cudaEventRecord(TS.ev[1], TS.aux);
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((w.n + 1) / 2, (int64_t)w.num_sms * 16));
    if (w.dtype == AS_F64) tri_prep_kernel<double><<<blocks, 256, 0, s>>>(w.args, w.lda, w.n, w.st, upper);
    else tri_prep_kernel<float><<<blocks, 256, 0, s>>>(w.args, w.lda, w.n, w.st, upper);
    cudaStreamWaitEvent(s, TS.ev[1], 0);
}

// Z = [B | e/n | alt] (ld n): the triangular path solves the primary system together with the two
// estimator applications that do not depend on its iteration (the start vector and the closing
// alternating-sign probe of xLACN2, Z13b/Z24) -- one sweep instead of three.
template <typename T>
__global__ void tri_rhs_kernel(const DevArgs* args, int64_t n, int64_t ldb, int64_t nrhs, T* Z, const int64_t* perm) {
    const T* B = (const T*)args->B;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * (nrhs + 2); e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e % n, c = e / n;
        T v;
        if (c < nrhs) v = B[(perm ? perm[i] : i) + c * ldb];      // LU: the rows of P B
        else if (c == nrhs) v = T(1) / (T)n;
        else v = ((i & 1) ? T(-1) : T(1)) * (T(1) + (T)i / (T)(n > 1 ? n - 1 : 1));
        Z[e] = v;
    }
}
// xe = M (e/n) from Z (the estimator's first result), or X = M B (the primary solution, after the gate)
template <typename T>
__global__ void tri_take_kernel(const DevArgs* args, int64_t n, int64_t ldb, int64_t nrhs, const T* Z, T* xe, int which) {
    T* X = (T*)args->X;
    const int64_t tot = which == 0 ? n : n * nrhs;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
        if (which == 0) xe[e] = Z[e + nrhs * n];
        else { const int64_t i = e % n, c = e / n; X[i + c * ldb] = Z[e]; }
    }
}
// kind KIND_TRI (the caller's triangle), KIND_CHOL (L then L^T), KIND_LU (P B; unit L then U; the
// estimator's columns without interchanges, as xGECON applies inv(U) inv(L), Z13b)
static void fused_solve(const Work& w, int kind, bool upper, SyncAlloc& sa, cudaStream_t s) {
    const int blocks = w.num_sms * 4;
    const int nz = (int)w.nrhs + 2;
    auto go = [&](auto* Z) {
        using T = std::remove_pointer_t<decltype(Z)>;
        tri_rhs_kernel<T><<<blocks, 256, 0, s>>>(w.args, w.n, w.ldb, w.nrhs, Z, kind == KIND_LU ? w.perm : nullptr);
        if (kind == KIND_TRI) {
            launch_trsm(w.dtype, nullptr, w.lda, w.Dinv0, upper, false, Z, w.n, w.n, nz, sa, -1, true, w.args, w.st, s);
        } else if (kind == KIND_CHOL) {
            launch_trsm(w.dtype, w.W, w.ldw, w.Dinv0, false, false, Z, w.n, w.n, nz, sa, -1, true, w.args, w.st, s);
            launch_trsm(w.dtype, w.W, w.ldw, w.Dinv0, false, true, Z, w.n, w.n, nz, sa, -1, true, w.args, w.st, s);
        } else {
            launch_trsm(w.dtype, w.W, w.ldw, w.Dinv0, false, false, Z, w.n, w.n, nz, sa, -1, true, w.args, w.st, s);
            launch_trsm(w.dtype, w.W, w.ldw, w.Dinv1, true, false, Z, w.n, w.n, nz, sa, -1, true, w.args, w.st, s);
        }
        tri_take_kernel<T><<<blocks, 256, 0, s>>>(w.args, w.n, w.ldb, w.nrhs, Z, (T*)w.xe, 0);
        launch_estimator(w, kind, upper, sa, s, Z + (w.nrhs + 1) * w.n);
    };
    if (w.dtype == AS_F64) go((double*)w.zx);
    else go((float*)w.zx);
}
static void tri_take_x(const Work& w, cudaStream_t s) {
    if (w.dtype == AS_F64) tri_take_kernel<double><<<w.num_sms * 4, 256, 0, s>>>(w.args, w.n, w.ldb, w.nrhs, (const double*)w.zx, nullptr, 1);
    else tri_take_kernel<float><<<w.num_sms * 4, 256, 0, s>>>(w.args, w.n, w.ldb, w.nrhs, (const float*)w.zx, nullptr, 1);
}

// ------------------------------------------------------------------ branch bodies (shared by graph and eager modes)
constexpr int kCholOk = 100;
constexpr int kBandSpike = 101;

static void body_factor(const Work& w, int m, SyncAlloc& sa, cudaStream_t s) {
    switch (m) {
    case AS_METHOD_BAND: launch_band_factor(w, s); launch_estimator(w, KIND_BAND, false, sa, s); break;  // sequential
    case kBandSpike + 0: case kBandSpike + 1: case kBandSpike + 2: case kBandSpike + 3:
        launch_band_spike(w, m - kBandSpike, s);
        break;
    // the primary solve runs with the estimator's first application (the gate may still send the
    // call to the fallback, which then overwrites X; X itself is written only after the gate)
    case AS_METHOD_TRI_LOWER: tri_prep(w, false, s); fused_solve(w, KIND_TRI, false, sa, s); break;
    case AS_METHOD_TRI_UPPER: tri_prep(w, true, s); fused_solve(w, KIND_TRI, true, sa, s); break;
    case AS_METHOD_LU: launch_lu_factor(w, s); fused_solve(w, KIND_LU, false, sa, s); break;
    case kCholOk: launch_chol_tri_prep(w, s); fused_solve(w, KIND_CHOL, false, sa, s); break;
    default: break;
    }
}

static void body_solve(const Work& w, int m, SyncAlloc& sa, cudaStream_t s) {
    switch (m) {
    case AS_METHOD_BAND: launch_band_solve(w, s); break;
    case AS_METHOD_TRI_LOWER:
    case AS_METHOD_TRI_UPPER:
        tri_take_x(w, s);          // solved with the estimator's first application (fused_solve)
        break;
    case AS_METHOD_CHOL:
    case AS_METHOD_LU: tri_take_x(w, s); break;   // solved in fused_solve
    default: break;
    }
}

// ------------------------------------------------------------------ plans
struct PlanKey {
    uintptr_t stream;    // plans (and their workspaces) are per stream: concurrent streams never share one
    int dev, dtype;
    int64_t n, nrhs, lda, ldb;
    uint32_t opts;
    int force;
    double thr, cut;
    int sweeps;
    int instrumented;
    int eager;
    int a16;             // A is 16-byte aligned (the detection pair pass is then the TMA pipeline)
    bool operator<(const PlanKey& o) const {
        return std::tie(stream, dev, dtype, n, nrhs, lda, ldb, opts, force, thr, cut, sweeps, instrumented, eager, a16) <
               std::tie(o.stream, o.dev, o.dtype, o.n, o.nrhs, o.lda, o.ldb, o.opts, o.force, o.thr, o.cut, o.sweeps,
                        o.instrumented, o.eager, o.a16);
    }
};
static int g_instrument = 0;
static int g_eager = 0;

struct Plan {
    PlanKey key{};
    Work w{};
    void* ws = nullptr;
    size_t ws_bytes = 0;
    RepOut* rep_ws = nullptr;
    RepOut* rep_pinned = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaGraphNode_t args_node = nullptr;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    // kernel-node counts per branch (for the launch count a call executes)
    int64_t nodes_top = 0, nodes_method[8] = {}, nodes_chol_lu = 0, nodes_chol_ok = 0;
    int64_t nodes_solve_hdr = 0, nodes_solve[8] = {}, nodes_fallback = 0, nodes_sweep = 0;
    std::mutex mu;
    ~Plan() {
        for (auto e : ev) if (e) cudaEventDestroy(e);
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
        if (ws) cudaFree(ws);
        if (rep_pinned) cudaFreeHost(rep_pinned);
    }
};

static std::mutex g_mu;
static std::map<PlanKey, std::unique_ptr<Plan>> g_plans;

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

static size_t layout(Work& w, uint32_t opts, char* base) {
    const size_t es = w.dtype == AS_F64 ? 8 : 4;
    const int64_t n = w.n, nr = std::max<int64_t>(w.nrhs, 1);
    const int64_t nblk = (n + kNB - 1) / kNB;
    const int64_t band_rows = (opts & AS_OPT_FORCE_METHOD) ? 3 * n : n;
    size_t off = 0;
    auto take = [&](size_t bytes) { char* p = base ? base + off : nullptr; off = align256(off + bytes); return p; };
    w.ldw = (n + 3) / 4 * 4;
    w.st = (DevState*)take(sizeof(DevState));
    w.args = (DevArgs*)take(sizeof(DevArgs));
    take(sizeof(RepOut));  // report slot follows args (see rep_ws)
    const size_t w_elems = std::max<size_t>((size_t)w.ldw * (size_t)std::max<int64_t>(band_rows, 1),
                                            (size_t)spike_scratch_elems(n, w.num_sms > 0 ? w.num_sms : 148));
    w.W = take(es * w_elems);
    w.diag = take(es * (n + kTile));   // + one tile: the TMA detection pass copies whole 64-element slices
    w.xe = take(es * n);
    w.Dinv0 = take(es * nblk * kNB * kNB);
    w.Dinv1 = take(es * nblk * kNB * kNB);
    w.vec = take(es * n * std::max<int64_t>(nr, 2));
    w.yv = take(es * n * nr);
    w.zx = take(es * n * (nr + 2));
    w.ipiv = (int64_t*)take(8 * n);
    w.perm = (int64_t*)take(8 * n);
    w.flags_ts_len = 160 * trsm_sync_words(n, (int)nr);
    w.flags_ts = (unsigned*)take(4 * w.flags_ts_len);
    w.ll_len = 100 * trsm_ll_words(n, 1) + 10 * trsm_ll_words(n, (int)nr + 2);   // + the fused solves' 2 columns
    w.ll = (unsigned long long*)take(8 * w.ll_len);
    w.bars_len = 8 + nblk + 8;
    w.bars = (unsigned*)take(4 * w.bars_len);
    w.cand = take(lu_cand_bytes());      // LU panel exchange words (headers, candidate rows, diagonal row)
    w.lfbuf = take(lu_lfbuf_bytes(n, w.dtype));
    w.linv = take(es * (size_t)((n + 127) / 128) * 128 * 128);
    w.swplan = take(lu_swplan_bytes(n));
    return off;
}

static int build_graph(Plan& P) {
    Work& w = P.w;
    Builder B;
    B.w = w;
    B.sa.base = w.flags_ts;
    B.sa.cap = w.flags_ts_len;
    B.sa.llbase = w.ll;
    B.sa.llcap = w.ll_len;
    for (int i = 0; i < 6; ++i) {
        cudaStream_t s;
        cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
        B.streams.push_back(s);
    }
    const PlanKey& k = P.key;
    cudaStream_t s0 = B.streams[0];
    cudaGraph_t g_cb0 = nullptr, g_cb1 = nullptr, g_wb = nullptr, g_sb[6] = {};
    cudaGraph_t* mb = nullptr;
    cudaGraph_t* pb = nullptr;
    int err = check(cudaStreamBeginCapture(s0, cudaStreamCaptureModeRelaxed), "BeginCapture");
    if (!err) {
        DevArgs a0{};
        set_args_kernel2<<<1, 1, 0, s0>>>(a0, w.args);
        {
            cudaStreamCaptureStatus stt;
            const cudaGraphNode_t* deps;
            size_t nd;
            cudaStreamGetCaptureInfo(s0, &stt, nullptr, nullptr, &deps, &nd);
            P.args_node = nd ? deps[0] : nullptr;
        }
        launch_state_init(w, s0, k.opts, k.force, k.thr, k.cut, k.sweeps);
        cudaMemsetAsync(w.flags_ts, 0, 4 * w.flags_ts_len, s0);
        if (k.instrumented) cudaEventRecordWithFlags(P.ev[0], s0, cudaEventRecordExternal);
        if (!(k.opts & AS_OPT_SKIP_DETECT)) launch_detect(w, s0, (k.opts & (AS_OPT_FULLSCAN | AS_OPT_FORCE_METHOD)) != 0,
                                                          (k.opts & AS_OPT_CHECK_FINITE) != 0);
        cudaGraphConditionalHandle h_method = make_handle(s0, 0);
        launch_dispatch(w, s0, h_method);
        if (k.instrumented) cudaEventRecordWithFlags(P.ev[1], s0, cudaEventRecordExternal);
        mb = add_cond(s0, h_method, cudaGraphCondTypeSwitch, 6);
        // ---- factor + estimate bodies
        for (int m : {AS_METHOD_TRI_LOWER, AS_METHOD_TRI_UPPER, AS_METHOD_LU})
            B.body(mb[m], [&](cudaStream_t s) { body_factor(w, m, B.sa, s); });
        B.body(mb[AS_METHOD_BAND], [&](cudaStream_t s) {
            launch_band_norm(w, s);
            cudaGraphConditionalHandle h_bm = make_handle(s, 0);
            launch_band_dominance(w, h_bm, s);
            // SWITCH: 0 sequential GBTRF path, 1 + c partitioned path with K class 2^c, 5 the
            // register chain for kl, ku <= 3
            cudaGraph_t* bb = add_cond(s, h_bm, cudaGraphCondTypeSwitch, 6);
            B.body(bb[0], [&](cudaStream_t s2) { body_factor(w, AS_METHOD_BAND, B.sa, s2); });
            for (int c = 0; c < 4; ++c)
                B.body(bb[1 + c], [&](cudaStream_t s2) { body_factor(w, kBandSpike + c, B.sa, s2); });
            B.body(bb[5], [&](cudaStream_t s2) { launch_band_chain(w, s2); });
        });
        B.body(mb[AS_METHOD_CHOL], [&](cudaStream_t s) {
            launch_chol_factor(w, s);
            cudaGraphConditionalHandle h_cf = make_handle(s, 0);
            launch_chol_check(w, h_cf, s);
            cudaGraph_t* cb = add_cond(s, h_cf, cudaGraphCondTypeIf, 2);
            g_cb0 = cb[0]; g_cb1 = cb[1];
            // failed: general LU on the original A
            B.body(cb[0], [&](cudaStream_t s2) { body_factor(w, AS_METHOD_LU, B.sa, s2); });
            B.body(cb[1], [&](cudaStream_t s2) { body_factor(w, kCholOk, B.sa, s2); });
        });
        // ---- gate + post
        if (k.instrumented) cudaEventRecordWithFlags(P.ev[2], s0, cudaEventRecordExternal);
        cudaGraphConditionalHandle h_post = make_handle(s0, 0);
        gate_kernel<<<1, 32, 0, s0>>>(w.st, h_post);
        pb = add_cond(s0, h_post, cudaGraphCondTypeSwitch, 3);
        B.body(pb[1], [&](cudaStream_t s) {
            cudaGraphConditionalHandle h_solve = make_handle(s, 0);
            solve_dispatch_kernel<<<1, 32, 0, s>>>(w.st, h_solve);
            cudaGraph_t* sb = add_cond(s, h_solve, cudaGraphCondTypeSwitch, 6);
            for (int m = 0; m < 6; ++m) g_sb[m] = sb[m];
            for (int m = AS_METHOD_BAND; m <= AS_METHOD_LU; ++m)
                B.body(sb[m], [&](cudaStream_t s2) { body_solve(w, m, B.sa, s2); });
        });
        B.body(pb[2], [&](cudaStream_t s) {
            launch_svd_pre(w, s);
            cudaGraphConditionalHandle h_while = make_handle(s, 1);
            set_cond_kernel<<<1, 32, 0, s>>>(h_while, 1u);
            cudaGraph_t* wb = add_cond(s, h_while, cudaGraphCondTypeWhile, 1);
            g_wb = wb[0];
            B.body(wb[0], [&](cudaStream_t s2) { launch_svd_sweep(w, h_while, s2); });
            launch_svd_post(w, s);
        });
        if (k.instrumented) cudaEventRecordWithFlags(P.ev[3], s0, cudaEventRecordExternal);
        finalize_kernel<<<1, 32, 0, s0>>>(w.st, P.rep_ws, w.args);
        cudaMemcpyAsync(P.rep_pinned, P.rep_ws, sizeof(RepOut), cudaMemcpyDeviceToHost, s0);
        err = check(cudaStreamEndCapture(s0, &P.graph), "EndCapture");
        if (!err) {
            P.nodes_top = count_kernels(P.graph);
            for (int m = 1; m < 6; ++m) P.nodes_method[m] = count_kernels(mb[m]);
            P.nodes_chol_lu = g_cb0 ? count_kernels(g_cb0) : 0;
            P.nodes_chol_ok = g_cb1 ? count_kernels(g_cb1) : 0;
            P.nodes_solve_hdr = count_kernels(pb[1]);
            for (int m = 1; m < 6; ++m) P.nodes_solve[m] = g_sb[m] ? count_kernels(g_sb[m]) : 0;
            P.nodes_fallback = count_kernels(pb[2]);
            P.nodes_sweep = g_wb ? count_kernels(g_wb) : 0;
        }
    }
    err = err ? err : B.err;
    if (!err && (B.sa.used > B.sa.cap || B.sa.llpeak > B.sa.llcap)) err = AS_ERR_CUDA_BASE + 999;
    if (!err) err = check(cudaGraphInstantiate(&P.exec, P.graph, 0), "GraphInstantiate");
    for (auto s : B.streams) cudaStreamDestroy(s);
    cudaGetLastError();
    return err;
}

static int get_plan(const PlanKey& key, Plan** out) {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_plans.find(key);
    if (it != g_plans.end()) { *out = it->second.get(); return 0; }
    auto P = std::make_unique<Plan>();
    P->key = key;
    Work& w = P->w;
    w.dtype = key.dtype; w.n = key.n; w.nrhs = key.nrhs; w.lda = key.lda; w.ldb = key.ldb;
    cudaDeviceGetAttribute(&w.num_sms, cudaDevAttrMultiProcessorCount, key.dev);
    w.det_tma = plan_uses_tma(key.dtype, key.n, key.lda, key.a16 != 0);
    const size_t bytes = layout(w, key.opts, nullptr);
    int err = check(cudaMalloc(&P->ws, bytes), "cudaMalloc(workspace)");
    if (err) return err;
    P->ws_bytes = bytes;
    layout(w, key.opts, (char*)P->ws);
    err = check(cudaMemset(P->ws, 0, bytes), "cudaMemset(workspace)");   // epoch 0, exchange words untagged
    if (err) return err;
    P->rep_ws = (RepOut*)((char*)w.args + align256(sizeof(DevArgs)));
    err = check(cudaMallocHost(&P->rep_pinned, sizeof(RepOut)), "cudaMallocHost");
    if (err) return err;
    if (key.instrumented)
        for (auto& e : P->ev) cudaEventCreate(&e);
    err = key.eager ? 0 : build_graph(*P);
    if (err) return err;
    *out = P.get();
    g_plans[key] = std::move(P);
    return 0;
}

// Eager mode (profiling / debugging): the same kernels launched directly on the
// stream with the branch decisions read back by the host.  Graph kernel nodes
// under conditional nodes cannot be profiled kernel-by-kernel by ncu; this mode
// gives the per-kernel launch list of the identical kernels.
static int run_eager(Plan& P, const DevArgs& a, cudaStream_t s) {
    Work& w = P.w;
    const PlanKey& k = P.key;
    SyncAlloc sa;
    sa.base = w.flags_ts;
    sa.cap = w.flags_ts_len;
    sa.llbase = w.ll;
    sa.llcap = w.ll_len;
    DevState h;
    auto rd = [&]() {
        cudaMemcpyAsync(&h, w.st, sizeof(DevState), cudaMemcpyDeviceToHost, s);
        return check(cudaStreamSynchronize(s), "eager sync");
    };
    set_args_kernel2<<<1, 1, 0, s>>>(a, w.args);
    launch_state_init(w, s, k.opts, k.force, k.thr, k.cut, k.sweeps);
    cudaMemsetAsync(w.flags_ts, 0, 4 * w.flags_ts_len, s);
    if (k.instrumented) cudaEventRecord(P.ev[0], s);
    if (!(k.opts & AS_OPT_SKIP_DETECT)) launch_detect(w, s, (k.opts & (AS_OPT_FULLSCAN | AS_OPT_FORCE_METHOD)) != 0,
                                                      (k.opts & AS_OPT_CHECK_FINITE) != 0);
    launch_dispatch(w, s, 0);
    if (k.instrumented) cudaEventRecord(P.ev[1], s);
    int err = rd();
    if (err) return err;
    if (h.method == AS_METHOD_CHOL) {
        launch_chol_factor(w, s);
        launch_chol_check(w, 0, s);
        if ((err = rd())) return err;
        body_factor(w, h.chol_failed ? AS_METHOD_LU : kCholOk, sa, s);
    } else if (h.method == AS_METHOD_BAND) {
        launch_band_norm(w, s);
        launch_band_dominance(w, 0, s);
        if ((err = rd())) return err;
        if (h.band_chain) launch_band_chain(w, s);
        else body_factor(w, h.band_use_spike ? kBandSpike + h.band_use_spike - 1 : AS_METHOD_BAND, sa, s);
    } else {
        body_factor(w, h.method, sa, s);
    }
    if (k.instrumented) cudaEventRecord(P.ev[2], s);
    gate_kernel<<<1, 32, 0, s>>>(w.st, 0);
    if ((err = rd())) return err;
    if (h.post == 1) {
        body_solve(w, h.method, sa, s);
    } else if (h.post == 2) {
        launch_svd_pre(w, s);
        for (;;) {
            launch_svd_sweep(w, 0, s);
            if ((err = rd())) return err;
            if (h.svd_conv || h.sweeps >= h.max_sweeps) break;
        }
        launch_svd_post(w, s);
    }
    if (k.instrumented) cudaEventRecord(P.ev[3], s);
    finalize_kernel<<<1, 32, 0, s>>>(w.st, P.rep_ws, w.args);
    cudaMemcpyAsync(P.rep_pinned, P.rep_ws, sizeof(RepOut), cudaMemcpyDeviceToHost, s);
    return check(cudaGetLastError(), "eager launch");
}

static bool is_device_ptr(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

static thread_local int64_t t_last_nodes = 0;

// The symmetric-indefinite specialisation (Z30) lives in the one-block solver (small.cu): a single
// system with AS_OPT_SYM_INDEF and n <= kSmallN runs there as a batch of one.
struct SmallOut { as_report rep; int32_t ret; int32_t pad; };
static std::mutex g_small_mu;
static std::map<std::pair<int, uintptr_t>, std::pair<SmallOut*, SmallOut*>> g_small_out;   // (device, stream) -> (dev, pinned)

static int solve_small_single(as_dtype dt, const void* A, int64_t lda, int64_t n, const void* B, int64_t ldb,
                              int64_t nrhs, void* X, const PlanKey& key, as_report* rep_host, as_report* rep_dev,
                              void* sigma, cudaStream_t stream, bool sync, int32_t* ret_dev) {
    SmallOut *d = nullptr, *h = nullptr;
    {
        std::lock_guard<std::mutex> lk(g_small_mu);
        auto& slot = g_small_out[{key.dev, (uintptr_t)stream}];
        if (!slot.first) {
            if (cudaMalloc(&slot.first, sizeof(SmallOut)) != cudaSuccess ||
                cudaMallocHost(&slot.second, sizeof(SmallOut)) != cudaSuccess) {
                cudaGetLastError();
                return AS_ERR_CUDA_BASE + (int)cudaErrorMemoryAllocation;
            }
        }
        d = slot.first;
        h = slot.second;
    }
    SmallArgs a{};
    a.A = A; a.lda = lda; a.sA = lda * n;
    a.B = B; a.ldb = ldb; a.sB = ldb * nrhs;
    a.X = X; a.ldx = ldb; a.sX = ldb * nrhs;
    a.n = (int)n; a.nrhs = (int)nrhs; a.batch = 1;
    a.opts = key.opts; a.force = key.force;
    a.thr = key.thr; a.cut = key.cut; a.max_sweeps = key.sweeps;
    a.rep = rep_dev ? rep_dev : &d->rep;
    a.ret = ret_dev ? ret_dev : &d->ret;
    a.sigma = sigma; a.sS = n;
    int err = launch_small_batched(dt, a, stream);
    if (err || !sync) return err;
    if (rep_dev) cudaMemcpyAsync(&d->rep, rep_dev, sizeof(as_report), cudaMemcpyDeviceToDevice, stream);
    if (ret_dev) cudaMemcpyAsync(&d->ret, ret_dev, sizeof(int32_t), cudaMemcpyDeviceToDevice, stream);
    cudaMemcpyAsync(h, d, sizeof(SmallOut), cudaMemcpyDeviceToHost, stream);
    err = check(cudaStreamSynchronize(stream), "cudaStreamSynchronize");
    if (err) return err;
    if (rep_host) *rep_host = h->rep;
    t_last_nodes = 1;
    return h->ret;
}
static thread_local Plan* t_last_plan = nullptr;

// kernel nodes of a graph; recursing into conditional bodies per `pick`
static int64_t count_kernels(cudaGraph_t g) {
    size_t nn = 0;
    cudaGraphGetNodes(g, nullptr, &nn);
    std::vector<cudaGraphNode_t> nodes(nn);
    cudaGraphGetNodes(g, nodes.data(), &nn);
    int64_t c = 0;
    for (auto nd : nodes) {
        cudaGraphNodeType t;
        cudaGraphNodeGetType(nd, &t);
        if (t == cudaGraphNodeTypeKernel) ++c;
    }
    return c;
}

static int solve_impl(as_dtype dt, const void* A, int64_t lda, int64_t n, const void* B, int64_t ldb, int64_t nrhs,
                      void* X, const as_options* opt, as_report* rep_host, as_report* rep_dev, void* sigma,
                      cudaStream_t stream, bool sync, int32_t* ret_dev = nullptr) {
    if (dt != AS_F64 && dt != AS_F32) return -1;
    if (n < 0) return -4;
    if (nrhs < 0) return -7;
    if (lda < std::max<int64_t>(1, n)) return -3;
    if (ldb < std::max<int64_t>(1, n)) return -6;
    if (n == 0 || nrhs == 0) {
        if (rep_host) { memset(rep_host, 0, sizeof(*rep_host)); rep_host->rcond = 1.0; rep_host->kl = rep_host->ku = -1; rep_host->rank = -1; }
        return 0;
    }
    if (!A) return -2;
    if (!B) return -5;
    if (!X) return -8;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return AS_ERR_NO_DEVICE; }
    if (!is_device_ptr(A)) return -2;
    if (!is_device_ptr(B)) return -5;
    if (!is_device_ptr(X)) return -8;
    PlanKey key{};
    key.stream = (uintptr_t)stream;
    key.dev = dev; key.dtype = dt; key.n = n; key.nrhs = nrhs; key.lda = lda; key.ldb = ldb;
    const double eps = dt == AS_F64 ? 2.220446049250313080847e-16 : 1.1920928955078125e-07;
    key.opts = opt ? opt->flags : 0u;
    key.force = (opt && (opt->flags & AS_OPT_FORCE_METHOD)) ? opt->force_method : 0;
    if (key.opts & AS_OPT_FORCE_METHOD) {
        if (key.force < AS_METHOD_BAND || (key.force > AS_METHOD_LU && key.force != AS_METHOD_LDLT)) return -9;
        if (key.force == AS_METHOD_LDLT && !((key.opts & AS_OPT_SYM_INDEF) && n <= kSmallN && nrhs <= kSmallRhs)) return -9;
    }
    if ((key.opts & AS_OPT_SKIP_DETECT) && (!(key.opts & AS_OPT_FORCE_METHOD) || key.force == AS_METHOD_BAND)) return -9;
    // the finite check rides on the detection pass, which SKIP_DETECT removes
    if ((key.opts & AS_OPT_SKIP_DETECT) && (key.opts & AS_OPT_CHECK_FINITE)) return -9;
    key.thr = (opt && opt->rcond_threshold >= 0) ? opt->rcond_threshold : 0.5 * eps;
    if (dt == AS_F32) key.thr = (double)(float)key.thr;
    key.cut = (opt && opt->lsq_cutoff >= 0) ? opt->lsq_cutoff : (double)n * eps;
    key.sweeps = (opt && opt->max_sweeps > 0) ? opt->max_sweeps : 30;
    key.instrumented = g_instrument;
    key.eager = g_eager;
    key.a16 = ((uintptr_t)A & 15) == 0;
    if ((key.opts & AS_OPT_SYM_INDEF) && n <= kSmallN && nrhs <= kSmallRhs && !(key.opts & AS_OPT_SKIP_DETECT))
        return solve_small_single(dt, A, lda, n, B, ldb, nrhs, X, key, rep_host, rep_dev, sigma, stream, sync, ret_dev);
    Plan* P = nullptr;
    int err = get_plan(key, &P);
    if (err) return err;
    std::lock_guard<std::mutex> lk(P->mu);
    DevArgs a{};
    a.A = A; a.B = B; a.X = X; a.sigma = sigma; a.rep_dev = rep_dev; a.rep_host = nullptr; a.ret_dev = ret_dev;
    if (P->w.det_tma && (err = fill_tmap(a, dt, A, lda, n)) != 0) return err;
    cudaKernelNodeParams kp = {};
    if (key.eager) {
        err = run_eager(*P, a, stream);
        if (err) return err;
        t_last_plan = P;
        if (!sync) return 0;
        if ((err = check(cudaStreamSynchronize(stream), "cudaStreamSynchronize"))) return err;
        if (rep_host) *rep_host = P->rep_pinned->rep;
        return P->rep_pinned->ret;
    }
    DevArgs* dst = P->w.args;
    void* params[2] = {&a, &dst};
    kp.func = (void*)set_args_kernel2;
    kp.gridDim = dim3(1);
    kp.blockDim = dim3(1);
    kp.kernelParams = params;
    err = check(cudaGraphExecKernelNodeSetParams(P->exec, P->args_node, &kp), "ExecKernelNodeSetParams");
    if (err) return err;
    err = check(cudaGraphLaunch(P->exec, stream), "cudaGraphLaunch");
    if (err) return err;
    t_last_plan = P;
    if (!sync) return 0;
    err = check(cudaStreamSynchronize(stream), "cudaStreamSynchronize");
    if (err) return err;
    if (rep_host) *rep_host = P->rep_pinned->rep;
    {
        const as_report& r = P->rep_pinned->rep;
        // a Cholesky failure runs the LU body inside the CHOL body's IF branch (primary_method is then LU)
        int64_t c = P->nodes_top;
        if (r.flags & AS_FLAG_CHOL_FAILED) c += P->nodes_method[AS_METHOD_CHOL] + P->nodes_chol_lu;
        else if (r.primary_method == AS_METHOD_CHOL) c += P->nodes_method[AS_METHOD_CHOL] + P->nodes_chol_ok;
        else c += P->nodes_method[r.primary_method & 7];
        if (r.flags & AS_FLAG_FALLBACK) c += P->nodes_fallback + (int64_t)r.sweeps * P->nodes_sweep;
        else if (!(P->rep_pinned->ret)) c += P->nodes_solve_hdr + P->nodes_solve[r.primary_method & 7];
        t_last_nodes = c;
    }
    return P->rep_pinned->ret;
}

// ------------------------------------------------------------------ detection-only path
struct DetPlan {
    Work w{};
    void* ws = nullptr;
    ~DetPlan() { if (ws) cudaFree(ws); }
};
static std::map<std::tuple<int, int, int64_t, int64_t, int>, std::unique_ptr<DetPlan>> g_det;

__global__ void det_out_kernel(const DevState* st, as_structure* out, int fullscan) {
    if (threadIdx.x != 0) return;
    as_structure o;
    o.flags = st->alive & ~st->pair_kill;
    // BANDED alive at the end means every tile was read: kl/ku are final, re-check the 25% rule on the pair
    if ((o.flags & AS_FLAG_BANDED) && !band_density_ok(st->n, st->kl, st->ku)) o.flags &= ~AS_FLAG_BANDED;
    o.nonfinite_seen = (st->flags & AS_FLAG_NONFINITE) ? 1 : 0;
    o.reserved = 0;
    int m;
    if (o.flags & AS_FLAG_BANDED) m = AS_METHOD_BAND;
    else if (o.flags & AS_FLAG_LOWER) m = AS_METHOD_TRI_LOWER;
    else if (o.flags & AS_FLAG_UPPER) m = AS_METHOD_TRI_UPPER;
    else if (o.flags & AS_FLAG_SPD_CANDIDATE) m = AS_METHOD_CHOL;
    else m = AS_METHOD_LU;
    o.method = m;
    const bool exact = fullscan || (o.flags & AS_FLAG_BANDED);
    o.kl = exact ? st->kl : -1;
    o.ku = exact ? st->ku : -1;
    o.max_diag = dfrom(st->max_diag);
    *out = o;
}

// device staging for as_solve_host's A, B and X (X separate from B: an in-place solve would
// exclude the speculative partitioned band path); freed by as_release_all
static std::mutex g_host_mu;
static std::map<std::tuple<int, int, int64_t, int64_t>, std::tuple<void*, void*, void*>> g_host_staging;

}  // namespace as

using namespace as;

extern "C" {

int as_solve_ex(as_dtype dt, const void* A, int64_t lda, int64_t n, const void* B, int64_t ldb, int64_t nrhs, void* X,
                const as_options* opt, as_report* rep, void* sigma_out, void* stream) {
    return solve_impl(dt, A, lda, n, B, ldb, nrhs, X, opt, rep, nullptr, sigma_out, (cudaStream_t)stream, true);
}

int as_solve(as_dtype dt, const void* A, int64_t lda, int64_t n, const void* B, int64_t ldb, int64_t nrhs, void* X,
             uint32_t* info_flags, double* rcond, void* stream) {
    as_report r;
    int ret = solve_impl(dt, A, lda, n, B, ldb, nrhs, X, nullptr, &r, nullptr, nullptr, (cudaStream_t)stream, true);
    if (ret >= 0) {
        if (info_flags) *info_flags = r.flags;
        if (rcond) *rcond = r.rcond;
    }
    return ret;
}

int as_solve_f64(const double* A, int64_t lda, int64_t n, const double* B, int64_t ldb, int64_t nrhs, double* X,
                 uint32_t* info_flags, double* rcond, void* stream) {
    return as_solve(AS_F64, A, lda, n, B, ldb, nrhs, X, info_flags, rcond, stream);
}

int as_solve_f32(const float* A, int64_t lda, int64_t n, const float* B, int64_t ldb, int64_t nrhs, float* X,
                 uint32_t* info_flags, double* rcond, void* stream) {
    return as_solve(AS_F32, A, lda, n, B, ldb, nrhs, X, info_flags, rcond, stream);
}

int as_solve_async(as_dtype dt, const void* A, int64_t lda, int64_t n, const void* B, int64_t ldb, int64_t nrhs,
                   void* X, const as_options* opt, as_report* rep_dev, void* sigma_out, void* stream) {
    return solve_impl(dt, A, lda, n, B, ldb, nrhs, X, opt, nullptr, rep_dev, sigma_out, (cudaStream_t)stream, false);
}

int as_solve_batched(as_dtype dt, int64_t n, int64_t nrhs, int64_t batch, const void* A, int64_t lda, int64_t strideA,
                     const void* B, int64_t ldb, int64_t strideB, void* X, int64_t ldx, int64_t strideX,
                     const as_options* opt, as_report* rep, int32_t* ret, void* sigma_out, void* stream) {
    if (dt != AS_F64 && dt != AS_F32) return -1;
    if (n < 0) return -2;
    if (nrhs < 0) return -3;
    if (batch < 0) return -4;
    if (lda < std::max<int64_t>(1, n)) return -6;
    if (strideA < lda * n) return -7;
    if (ldb < std::max<int64_t>(1, n)) return -9;
    if (strideB < ldb * nrhs) return -10;
    if (ldx < std::max<int64_t>(1, n)) return -12;
    if (strideX < ldx * nrhs) return -13;
    if (n == 0 || nrhs == 0 || batch == 0) return 0;
    if (!A || !is_device_ptr(A)) return -5;
    if (!B || !is_device_ptr(B)) return -8;
    if (!X || !is_device_ptr(X)) return -11;
    if (rep && !is_device_ptr(rep)) return -15;
    if (ret && !is_device_ptr(ret)) return -16;
    if (sigma_out && !is_device_ptr(sigma_out)) return -17;
    const double eps = dt == AS_F64 ? 2.220446049250313080847e-16 : 1.1920928955078125e-07;
    const uint32_t opts = opt ? opt->flags : 0u;
    const int force = (opts & AS_OPT_FORCE_METHOD) ? opt->force_method : 0;
    if ((opts & AS_OPT_FORCE_METHOD) && (force < AS_METHOD_BAND || (force > AS_METHOD_LU && force != AS_METHOD_LDLT))) return -14;
    if ((opts & AS_OPT_FORCE_METHOD) && force == AS_METHOD_LDLT && !((opts & AS_OPT_SYM_INDEF) && n <= kSmallN && nrhs <= kSmallRhs))
        return -14;
    if (opts & AS_OPT_SKIP_DETECT) return -14;   // the one-block solver always detects (it reads A once anyway)
    cudaStream_t s = (cudaStream_t)stream;
    const size_t es = dt == AS_F64 ? 8 : 4;
    if (n <= kSmallN && nrhs <= kSmallRhs) {
        SmallArgs a{};
        a.A = A; a.lda = lda; a.sA = strideA;
        a.B = B; a.ldb = ldb; a.sB = strideB;
        a.X = X; a.ldx = ldx; a.sX = strideX;
        a.n = (int)n; a.nrhs = (int)nrhs; a.batch = batch;
        a.opts = opts; a.force = force;
        a.thr = (opt && opt->rcond_threshold >= 0) ? opt->rcond_threshold : 0.5 * eps;
        if (dt == AS_F32) a.thr = (double)(float)a.thr;
        a.cut = (opt && opt->lsq_cutoff >= 0) ? opt->lsq_cutoff : (double)n * eps;
        a.max_sweeps = (opt && opt->max_sweeps > 0) ? opt->max_sweeps : 30;
        a.rep = rep; a.ret = ret;
        a.sigma = sigma_out; a.sS = n;
        return launch_small_batched(dt, a, s);
    }
    // larger systems: one graph launch of the single-system solver per system, on the stream
    if (ldx != ldb) return -12;   // the single-system path writes X with ldb
    for (int64_t b = 0; b < batch; ++b) {
        const int r = solve_impl(dt, (const char*)A + es * b * strideA, lda, n, (const char*)B + es * b * strideB, ldb,
                                 nrhs, (char*)X + es * b * strideX, opt, nullptr, rep ? rep + b : nullptr,
                                 sigma_out ? (char*)sigma_out + es * b * n : nullptr, s, false, ret ? ret + b : nullptr);
        if (r != 0) return r;
    }
    return 0;
}

int as_solve_host(as_dtype dt, const void* A, int64_t lda, int64_t n, const void* B, int64_t ldb, int64_t nrhs,
                  void* X, const as_options* opt, as_report* rep, void* stream) {
    if (dt != AS_F64 && dt != AS_F32) return -1;
    if (n < 0) return -4;
    if (nrhs < 0) return -7;
    if (lda < std::max<int64_t>(1, n)) return -3;
    if (ldb < std::max<int64_t>(1, n)) return -6;
    if (n == 0 || nrhs == 0) return as_solve_ex(dt, A, lda, n, B, ldb, nrhs, X, opt, rep, nullptr, stream);
    if (!A) return -2;
    if (!B) return -5;
    if (!X) return -8;
    const size_t es = dt == AS_F64 ? 8 : 4;
    cudaStream_t s = (cudaStream_t)stream;
    auto& bufs = g_host_staging;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_host_mu);
    auto key = std::make_tuple(dev, (int)dt, n, nrhs);
    auto it = bufs.find(key);
    if (it == bufs.end()) {
        void *dA = nullptr, *dB = nullptr, *dX = nullptr;
        if (cudaMalloc(&dA, es * n * n) != cudaSuccess || cudaMalloc(&dB, es * n * nrhs) != cudaSuccess ||
            cudaMalloc(&dX, es * n * nrhs) != cudaSuccess) {
            cudaGetLastError();
            if (dA) cudaFree(dA);
            if (dB) cudaFree(dB);
            return AS_ERR_CUDA_BASE + (int)cudaErrorMemoryAllocation;
        }
        it = bufs.emplace(key, std::make_tuple(dA, dB, dX)).first;
    }
    void* dA = std::get<0>(it->second);
    void* dB = std::get<1>(it->second);
    void* dX = std::get<2>(it->second);
    int err = check(cudaMemcpy2DAsync(dA, es * n, A, es * lda, es * n, n, cudaMemcpyHostToDevice, s), "H2D A");
    if (!err) err = check(cudaMemcpy2DAsync(dB, es * n, B, es * ldb, es * n, nrhs, cudaMemcpyHostToDevice, s), "H2D B");
    if (err) return err;
    int ret = solve_impl(dt, dA, n, n, dB, n, nrhs, dX, opt, rep, nullptr, nullptr, s, true);
    if (ret < 0) return ret;
    err = check(cudaMemcpy2DAsync(X, es * ldb, dX, es * n, es * n, nrhs, cudaMemcpyDeviceToHost, s), "D2H X");
    if (!err) err = check(cudaStreamSynchronize(s), "sync");
    return err ? err : ret;
}

int as_detect(as_dtype dt, const void* A, int64_t lda, int64_t n, uint32_t detect_flags, as_structure* out,
              void* stream) {
    if (dt != AS_F64 && dt != AS_F32) return -1;
    if (n < 0) return -4;
    if (lda < std::max<int64_t>(1, n)) return -3;
    if (!out) return -6;
    if (n == 0) { memset(out, 0, sizeof(*out)); out->kl = out->ku = -1; return 0; }
    if (!A || !is_device_ptr(A)) return -2;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaStream_t s = (cudaStream_t)stream;
    std::lock_guard<std::mutex> lk(g_mu);
    const int a16 = ((uintptr_t)A & 15) == 0;
    auto key = std::make_tuple(dev, (int)dt, n, lda, a16);
    auto it = g_det.find(key);
    if (it == g_det.end()) {
        auto D = std::make_unique<DetPlan>();
        Work& w = D->w;
        w.dtype = dt; w.n = n; w.lda = lda; w.nrhs = 1; w.ldb = n;
        cudaDeviceGetAttribute(&w.num_sms, cudaDevAttrMultiProcessorCount, dev);
        w.det_tma = plan_uses_tma(dt, n, lda, a16 != 0);
        const size_t es = dt == AS_F64 ? 8 : 4;
        size_t bytes = align256(sizeof(DevState)) + align256(sizeof(DevArgs)) + align256(sizeof(as_structure)) +
                       align256(es * (n + kTile)) + align256(64 * 4);
        int err = check(cudaMalloc(&D->ws, bytes), "cudaMalloc(detect)");
        if (err) return err;
        char* p = (char*)D->ws;
        w.st = (DevState*)p; p += align256(sizeof(DevState));
        w.args = (DevArgs*)p; p += align256(sizeof(DevArgs));
        w.cand = p; p += align256(sizeof(as_structure));
        w.diag = p; p += align256(es * (n + kTile));
        w.bars = (unsigned*)p; w.bars_len = 64;
        it = g_det.emplace(key, std::move(D)).first;
    }
    Work& w = it->second->w;
    DevArgs a{};
    a.A = A;
    if (w.det_tma) { const int e = fill_tmap(a, dt, A, lda, n); if (e) return e; }
    set_args_kernel2<<<1, 1, 0, s>>>(a, w.args);
    launch_state_init(w, s, detect_flags, 0, 0.0, 0.0, 30);
    const bool check_finite = (detect_flags & AS_OPT_CHECK_FINITE) != 0;
    const bool fullscan = (detect_flags & AS_OPT_FULLSCAN) != 0 || check_finite;
    launch_detect(w, s, fullscan, check_finite);
    det_out_kernel<<<1, 32, 0, s>>>(w.st, (as_structure*)w.cand, fullscan);
    as_structure h;
    int err = check(cudaMemcpyAsync(&h, w.cand, sizeof(h), cudaMemcpyDeviceToHost, s), "D2H structure");
    if (!err) err = check(cudaStreamSynchronize(s), "sync");
    if (err) return err;
    *out = h;
    return 0;
}

#ifdef AS_DEBUG
// Test-only: the primary factorization alone (the same launchers the solve uses), eagerly on a
// private workspace, factors copied out for the PA = LU / L L^T = A reconstruction tests.
int64_t as_debug_factor(as_dtype dt, int32_t method, const void* A, int64_t lda, int64_t n, int64_t kl, int64_t ku,
                        void* W, int64_t* ipiv, void* stream) {
    (void)kl; (void)ku;
    if (dt != AS_F64 && dt != AS_F32) return -1;
    if (method != AS_METHOD_LU && method != AS_METHOD_CHOL) return -(int64_t)AS_ERR_NOT_IMPLEMENTED;
    if (n <= 0) return -5;
    if (lda < n) return -4;
    if (!A || !is_device_ptr(A)) return -3;
    if (!W || !is_device_ptr(W)) return -8;
    if (method == AS_METHOD_LU && (!ipiv || !is_device_ptr(ipiv))) return -9;
    cudaStream_t s = (cudaStream_t)stream;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return AS_ERR_NO_DEVICE; }
    Work w{};
    w.dtype = dt; w.n = n; w.nrhs = 1; w.lda = lda; w.ldb = n;
    cudaDeviceGetAttribute(&w.num_sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t bytes = layout(w, 0, nullptr);
    void* ws = nullptr;
    int err = check(cudaMalloc(&ws, bytes), "cudaMalloc(debug workspace)");
    if (err) return err;
    layout(w, 0, (char*)ws);
    cudaMemsetAsync(ws, 0, bytes, s);
    DevArgs a{};
    a.A = A;
    set_args_kernel2<<<1, 1, 0, s>>>(a, w.args);
    launch_state_init(w, s, 0u, 0, 0.0, 0.0, 30);
    if (method == AS_METHOD_LU) launch_lu_factor(w, s);
    else launch_chol_factor(w, s);
    const size_t es = dt == AS_F64 ? 8 : 4;
    cudaMemcpy2DAsync(W, es * n, w.W, es * w.ldw, es * n, n, cudaMemcpyDeviceToDevice, s);
    if (method == AS_METHOD_LU) cudaMemcpyAsync(ipiv, w.ipiv, 8 * n, cudaMemcpyDeviceToDevice, s);
    DevState h;
    cudaMemcpyAsync(&h, w.st, sizeof(DevState), cudaMemcpyDeviceToHost, s);
    err = check(cudaStreamSynchronize(s), "debug factor");
    cudaFree(ws);
    if (err) return err;
    if (method == AS_METHOD_LU) return h.info == ~0ull ? 0 : (int64_t)h.info;
    return h.chol_failed ? h.chol_fail_col + 1 : 0;
}

#endif  // AS_DEBUG

int64_t as_workspace_bytes(as_dtype dt, int64_t n, int64_t nrhs, uint32_t opts) {
    if ((dt != AS_F64 && dt != AS_F32) || n < 0 || nrhs < 0) return -1;
    Work w{};
    w.dtype = dt; w.n = n; w.nrhs = nrhs;
    int dev = 0;
    w.num_sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&w.num_sms, cudaDevAttrMultiProcessorCount, dev);
    else cudaGetLastError();
    return (int64_t)layout(w, opts, nullptr);
}

int64_t as_last_kernel_nodes(void) { return t_last_nodes; }

void as_set_instrumentation(int enable) { g_instrument = enable ? 1 : 0; }

void as_set_exec_mode(int eager) { g_eager = eager ? 1 : 0; }

double as_bench_gemm(int dtype, int64_t M, int64_t N, int64_t K, int trans_b, int iters) {
    const size_t es = dtype == AS_F64 ? 8 : 4;
    const int64_t ld = (std::max(M, std::max(N, K)) + 3) / 4 * 4;
    void *A = nullptr, *B = nullptr, *Cm = nullptr;
    if (cudaMalloc(&A, es * ld * K) || cudaMalloc(&B, es * ld * std::max(N, K)) || cudaMalloc(&Cm, es * ld * N)) {
        cudaGetLastError();
        return -1.0;
    }
    cudaMemset(A, 0, es * ld * K);
    cudaMemset(B, 0, es * ld * std::max(N, K));
    cudaMemset(Cm, 0, es * ld * N);
    GemmArgs g{};
    g.M = M; g.N = N; g.K = K;
    g.A = A; g.lda = ld; g.TA = false;
    g.B = B; g.ldb = ld; g.TB = trans_b != 0;
    g.C = Cm; g.ldc = ld;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch_gemm_minus(dtype, g, 0);
    cudaEventRecord(e0, 0);
    for (int i = 0; i < iters; ++i) launch_gemm_minus(dtype, g, 0);
    cudaEventRecord(e1, 0);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(A); cudaFree(B); cudaFree(Cm);
    return 2.0 * (double)M * N * K * iters / (ms * 1e-3) / 1e12;
}

#ifdef AS_DEBUG
double as_debug_panel_time(int dtype, int kind, void* W, int64_t ldw, int64_t n, int64_t k0, int nbp, const void* Wsrc,
                           int iters, int dbg) {
    if (!W || !Wsrc || n <= 0 || k0 < 0 || k0 >= n || nbp <= 0 || ldw < n || iters <= 0) return -1.0;
    if (kind <= 1) return as::lu_debug_panel_time(dtype, kind, W, ldw, n, k0, nbp, Wsrc, iters, dbg);
    return as::chol_debug_panel_time(dtype, kind - 2, W, ldw, n, k0, nbp, Wsrc, iters, dbg);
}

int as_debug_lu_trace(unsigned long long* tmin, unsigned long long* tmax, int cap) {
    if (!tmin || !tmax || cap <= 0) return -1;
    return as::lu_trace_copy(tmin, tmax, cap);
}

int as_debug_timestamps(unsigned long long* out16) {
    Plan* P = t_last_plan;
    if (!P || !out16) return -1;
    DevState h;
    if (cudaMemcpy(&h, P->w.st, sizeof(DevState), cudaMemcpyDeviceToHost) != cudaSuccess) {
        cudaGetLastError();
        return -2;
    }
    memcpy(out16, h.dbg_t, sizeof(h.dbg_t));
    return 0;
}

#endif  // AS_DEBUG

double as_measure_fp64_peak(int iters, void* stream) {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1.0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return measure_fp64_peak(sms, iters, (cudaStream_t)stream);
}

int as_last_stage_ms(double* out4) {
    Plan* P = t_last_plan;
    if (!P || !P->key.instrumented || !out4) return -1;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, P->ev[0], P->ev[1]); out4[0] = ms;
    cudaEventElapsedTime(&ms, P->ev[1], P->ev[2]); out4[1] = ms;
    cudaEventElapsedTime(&ms, P->ev[2], P->ev[3]); out4[2] = ms;
    cudaEventElapsedTime(&ms, P->ev[0], P->ev[3]); out4[3] = ms;
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

void as_release_all(void) {
    {
        std::lock_guard<std::mutex> lk(g_mu);
        g_plans.clear();
        g_det.clear();
    }
    std::lock_guard<std::mutex> lk(g_host_mu);
    for (auto& kv : g_host_staging) {
        cudaFree(std::get<0>(kv.second));
        cudaFree(std::get<1>(kv.second));
        cudaFree(std::get<2>(kv.second));
    }
    g_host_staging.clear();
}

const char* as_strerror(int code) {
    if (code == 0) return "success";
    if (code < 0) return "illegal argument";
    switch (code) {
    case AS_ERR_SINGULAR_NO_FALLBACK: return "matrix is exactly singular and the SVD fallback is disabled";
    case AS_ERR_SVD_NOT_CONVERGED: return "one-sided Jacobi SVD did not converge within max_sweeps";
    case AS_ERR_NONFINITE: return "non-finite (NaN or Inf) input";
    case AS_ERR_NOT_IMPLEMENTED: return "not implemented";
    case AS_ERR_NO_DEVICE: return "no CUDA device";
    default: break;
    }
    if (code >= AS_ERR_CUDA_BASE) return cudaGetErrorString((cudaError_t)(code - AS_ERR_CUDA_BASE));
    return "unknown error";
}

int as_version(void) { return 1; }

}  // extern "C"
