// api.cu — host orchestration of the B200 JABBA path and its C ABI
// (include/jabba_b200.h). Mirrors jabba_fit (jabba.hpp:30-36) =
// partitional_compress (compression.hpp:167-193) + digitize
// (digitization.hpp:207-293), and reconstruct (inverse.hpp:127-132).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/jabba_b200.h"
#include "jb_device.hpp"

using namespace jb;

namespace jb_api {
struct MaxOp2 {};  // (placeholder to keep the named namespace non-empty)
struct MaxOp {
    __device__ int64_t operator()(int64_t a, int64_t b) const { return a > b ? a : b; }
};
}  // namespace jb_api
using jb_api::MaxOp;

// ---------------------------------------------------------------------------
// kernel-level event profiler (jb_device.hpp: prof_begin / prof_end)

#include <exception>
#include <map>
#include <mutex>
#include <thread>

namespace jb {
namespace prof_detail {
// Events come from a pool created when profiling is enabled, so a profiled
// launch costs two cudaEventRecord calls and nothing else.
struct ProfRec {
    const char* name;
    int a, b;  // pool slots
};
bool g_prof_on = false;
std::mutex g_prof_mu;
std::vector<cudaEvent_t> g_pool;
size_t g_pool_next = 0;
std::vector<ProfRec> g_prof_pending;
std::map<std::string, std::pair<double, int64_t>> g_prof_totals;
thread_local std::vector<std::pair<const char*, int>> g_prof_stack;

int take_event() {
    if (g_pool_next >= g_pool.size()) return -1;
    return (int)g_pool_next++;
}
}  // namespace prof_detail
using namespace prof_detail;

void prof_begin(const char* name, cudaStream_t st) {
    if (!g_prof_on) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    const int a = take_event();
    if (a >= 0) cudaEventRecord(g_pool[a], st);
    g_prof_stack.emplace_back(name, a);
}

void prof_end(cudaStream_t st) {
    if (!g_prof_on || g_prof_stack.empty()) return;
    auto top = g_prof_stack.back();
    g_prof_stack.pop_back();
    std::lock_guard<std::mutex> lk(g_prof_mu);
    if (top.second < 0) return;
    const int b = take_event();
    if (b < 0) return;
    cudaEventRecord(g_pool[b], st);
    g_prof_pending.push_back(ProfRec{top.first, top.second, b});
}
}  // namespace jb

using namespace jb::prof_detail;

namespace jb {
namespace cache_detail {
std::mutex g_mu;
std::map<std::pair<cudaStream_t, size_t>, std::vector<void*>> g_free;

size_t bucket(size_t bytes) {
    if (bytes <= 256) return 256;
    if (bytes < (1u << 20)) {
        size_t b = 256;
        while (b < bytes) b <<= 1;
        return b;
    }
    return (bytes + (1u << 20) - 1) & ~(size_t)((1u << 20) - 1);
}
}  // namespace cache_detail

void* dev_alloc(size_t bytes, cudaStream_t st) {
    using namespace cache_detail;
    const size_t b = bucket(bytes);
    {
        std::lock_guard<std::mutex> lk(g_mu);
        auto it = g_free.find({st, b});
        if (it != g_free.end() && !it->second.empty()) {
            void* p = it->second.back();
            it->second.pop_back();
            return p;
        }
    }
    void* p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, b, st);
    if (e == cudaErrorMemoryAllocation) {  // trim this stream's cache and retry once
        cudaGetLastError();
        dev_cache_drop(st);
        e = cudaMallocAsync(&p, b, st);
    }
    if (e != cudaSuccess)
        throw Error(CUDA_ERROR, std::string("device allocation of ") + std::to_string(b) +
                                    " bytes: " + cudaGetErrorString(e));
    return p;
}

void dev_free(void* p, size_t bytes, cudaStream_t st) {
    using namespace cache_detail;
    std::lock_guard<std::mutex> lk(g_mu);
    g_free[{st, bucket(bytes)}].push_back(p);
}

void dev_cache_drop(cudaStream_t st) {
    using namespace cache_detail;
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto it = g_free.begin(); it != g_free.end();) {
        if (it->first.first == st) {
            for (void* p : it->second) cudaFreeAsync(p, st);
            it = g_free.erase(it);
        } else {
            ++it;
        }
    }
}

void trace_mark(const char* what, cudaStream_t st) {
    static const bool on = [] {
        const char* e = getenv("JB_TRACE");
        return e && *e == '1';
    }();
    if (!on) return;
    static thread_local std::chrono::steady_clock::time_point last =
        std::chrono::steady_clock::now();
    cudaStreamSynchronize(st);
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[jb] %-28s %9.3f ms\n", what,
            std::chrono::duration<double, std::milli>(now - last).count());
    last = now;
}
}  // namespace jb

namespace {

void prof_collect() {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (auto& r : g_prof_pending) {
        cudaEventSynchronize(g_pool[r.b]);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, g_pool[r.a], g_pool[r.b]);
        auto& t = g_prof_totals[r.name];
        t.first += ms;
        t.second += 1;
    }
    g_prof_pending.clear();
    g_pool_next = 0;
}

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return JB_OK;
    } catch (const jb::Error& e) {
        return fail(e.code, e.what());
    } catch (const std::bad_alloc&) {
        return fail(JB_INTERNAL, "host allocation failed");
    } catch (const std::exception& e) {
        return fail(JB_INTERNAL, e.what());
    }
}

using Clock = std::chrono::steady_clock;
double ms_since(Clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

}  // namespace

struct jb_context {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;  // svq sampling, concurrent with scale_pieces
    cudaEvent_t side_done = nullptr;
    cudaStream_t aux = nullptr;  // scale_pieces: the increments' sums beside the lengths' sequential sum
};

struct jb_fit {
    int32_t layout = JB_LAYOUT_COLLECTION;
    bool drop_local_last = false;  // distributed univariate-partitioned: not the last rank
    int64_t piece_base = 0;        // global index of this rank's first piece
    SegTable seg;
    Pieces pieces;
    DArr<double> anchors;  // per segment (device)
    std::vector<double> h_anchors;
    DArr<uint32_t> labels;  // ranked (device)
    uint64_t k = 0;
    std::vector<double> centers, mean_lengths;  // ranked codebook (host)
    DArr<double> d_centers, d_mean_lengths;
    double scaling[3] = {1.0, 1.0, 1.0};
    // diagnostics
    uint64_t iterations = 0, sample_size = 0, draws = 0, work_tiles = 0, changed_labels = 0;
    uint64_t d2_tiles = 0;
    int32_t fix_rounds = 0, ga_rounds = 0;
    double phase_ms[5] = {0, 0, 0, 0, 0};
};

namespace {

__global__ void k_gather_anchors(const double* __restrict__ v, const int64_t* __restrict__ first,
                                 int64_t n_seg, double* __restrict__ out) {
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s < n_seg) out[s] = v[first[s]];
}

// distributed svq: sample entries whose piece this rank owns
__global__ void k_own_flags(const uint64_t* __restrict__ idx, uint64_t S, uint64_t base,
                            uint64_t n_local, uint8_t* __restrict__ flags) {
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < S;
         s += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t g = idx[s];
        flags[s] = (g >= base && g < base + n_local) ? 1 : 0;
    }
}

__global__ void k_local_idx(const uint64_t* __restrict__ idx, const uint32_t* __restrict__ gpos,
                            int64_t n, uint64_t base, uint64_t* __restrict__ lidx) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        lidx[i] = idx[gpos[i]] - base;
}

__global__ void k_iota_pos(uint32_t* __restrict__ gpos, uint64_t* __restrict__ lidx, int64_t n,
                           uint64_t base) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        gpos[i] = (uint32_t)(base + i);
        lidx[i] = (uint64_t)i;
    }
}

__global__ void k_embed_axis(const double2* __restrict__ pts, int64_t n, int axis,
                             double2* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double2 p = pts[i];
        out[i] = make_double2(axis == 0 ? p.x : p.y, 0.0);
    }
}

__global__ void k_pair_keys(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b,
                            int64_t n, unsigned long long* __restrict__ key,
                            uint32_t* __restrict__ idx) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        key[i] = ((unsigned long long)a[i] << 32) | b[i];
        idx[i] = (uint32_t)i;
    }
}

// run heads of the sorted pair keys: first appearance (stable sort keeps the
// smallest original index first in each run)
__global__ void k_pair_heads(const unsigned long long* __restrict__ skey,
                             const uint32_t* __restrict__ sidx, int64_t n,
                             int64_t* __restrict__ headpos, int64_t* __restrict__ first_flag) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
        const bool head = r == 0 || skey[r] != skey[r - 1];
        headpos[r] = head ? r : 0;
        if (head) first_flag[sidx[r]] = 1;
    }
}

__global__ void k_pair_labels(const uint32_t* __restrict__ sidx,
                              const int64_t* __restrict__ headpos_scan,
                              const int64_t* __restrict__ id_of, int64_t n,
                              uint32_t* __restrict__ labels) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t first = sidx[headpos_scan[r]];
        labels[sidx[r]] = (uint32_t)id_of[first];
    }
}


int gsz(int64_t n) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 8));
}

// ga-hier (digitization.hpp:168-195): two 1-D aggregations, pieces labeled by
// the observed (len-group, inc-group) pair in order of first appearance.
uint64_t ga_hier_device(const double* d_pts, int64_t n, const jb_config& c, const BBox& bb,
                        DArr<uint32_t>& labels, int& rounds, cudaStream_t st) {
    const double a_len = c.has_alpha_len ? c.alpha_len : c.alpha;
    const double a_inc = c.has_alpha_inc ? c.alpha_inc : c.alpha;
    DArr<double2> e(n, st);
    GAOut gl, gi;
    for (int axis = 0; axis < 2; ++axis) {
        k_embed_axis<<<gsz(n), 256, 0, st>>>(reinterpret_cast<const double2*>(d_pts), n, axis,
                                             e.p);
        JB_LAUNCH_CHECK();
        BBox eb = axis == 0 ? BBox{bb.xmin, bb.xmax, 0.0, 0.0} : BBox{bb.ymin, bb.ymax, 0.0, 0.0};
        greedy_aggregate_device(reinterpret_cast<const double*>(e.p), n,
                                axis == 0 ? a_len : a_inc, c.sort_key, c.early_stop != 0, eb,
                                axis == 0 ? gl : gi, st);
    }
    rounds = gl.rounds + gi.rounds;
    DArr<unsigned long long> key(n, st), skey(n, st);
    DArr<uint32_t> idx(n, st), sidx(n, st);
    k_pair_keys<<<gsz(n), 256, 0, st>>>(gl.labels.p, gi.labels.p, n, key.p, idx.p);
    JB_LAUNCH_CHECK();
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, key.p, skey.p, idx.p, sidx.p, n, 0, 64, st);
    DArr<uint8_t> tmp(tb, st);
    cub::DeviceRadixSort::SortPairs(tmp.p, tb, key.p, skey.p, idx.p, sidx.p, n, 0, 64, st);
    JB_LAUNCH_CHECK();
    DArr<int64_t> headpos(n, st), hscan(n, st), first_flag(n + 1, st), id_of(n + 1, st);
    first_flag.zero();
    k_pair_heads<<<gsz(n), 256, 0, st>>>(skey.p, sidx.p, n, headpos.p, first_flag.p);
    JB_LAUNCH_CHECK();
    size_t t1 = 0, t2 = 0;
    cub::DeviceScan::InclusiveScan(nullptr, t1, headpos.p, hscan.p, MaxOp(), n, st);
    cub::DeviceScan::ExclusiveSum(nullptr, t2, first_flag.p, id_of.p, n + 1, st);
    DArr<uint8_t> tmp2(std::max(t1, t2), st);
    cub::DeviceScan::InclusiveScan(tmp2.p, t1, headpos.p, hscan.p, MaxOp(), n, st);
    cub::DeviceScan::ExclusiveSum(tmp2.p, t2, first_flag.p, id_of.p, n + 1, st);
    JB_LAUNCH_CHECK();
    labels.alloc(n, st);
    k_pair_labels<<<gsz(n), 256, 0, st>>>(sidx.p, hscan.p, id_of.p, n, labels.p);
    JB_LAUNCH_CHECK();
    int64_t k = 0;
    JB_CUDA(cudaMemcpyAsync(&k, id_of.p + n, 8, cudaMemcpyDeviceToHost, st));
    JB_CUDA(cudaStreamSynchronize(st));
    return (uint64_t)k;
}

void validate_vq(const jb_config& c, double r) {
    if (c.k < 1) throw Error(INVALID_INPUT, "VQConfig: k must be >= 1");
    if (!(r > 0.0 && r <= 1.0)) throw Error(INVALID_INPUT, "VQConfig: r must be in (0,1]");
    if (c.max_iters < 1) throw Error(INVALID_INPUT, "VQConfig: max_iters must be >= 1");
    if (c.n_init < 1) throw Error(INVALID_INPUT, "VQConfig: n_init must be >= 1");
}

void validate_ga(const jb_config& c, double alpha) {
    if (!(alpha > 0.0)) throw Error(INVALID_INPUT, "GAConfig: alpha must be > 0");
    if (c.has_alpha_len && !(c.alpha_len > 0.0))
        throw Error(INVALID_INPUT, "GAConfig: alpha_len must be > 0");
    if (c.has_alpha_inc && !(c.alpha_inc > 0.0))
        throw Error(INVALID_INPUT, "GAConfig: alpha_inc must be > 0");
}

// auto_alpha (digitization.hpp:66-75), host libm exactly as the reference
double auto_alpha_host(int64_t n, int64_t N, double tol, double eta) {
    if (N < 1 || n <= N) throw Error(INVALID_INPUT, "auto_alpha: requires n > N >= 1");
    if (!(tol > 0.0)) throw Error(INVALID_INPUT, "auto_alpha: tol must be > 0");
    if (!(eta > 0.0)) throw Error(INVALID_INPUT, "auto_alpha: eta must be > 0");
    const double dn = (double)n, dN = (double)N;
    const double poly = 3.0 * dn * dn * dn * dn + 2.0 - 5.0 * dn * dn;
    const double num = 60.0 * dn * (dn - dN) * tol * tol;
    return std::pow(num / (dN * eta * eta * poly), 0.25);
}

void run_fit(jb_context* ctx, const double* values, int64_t n_values, bool on_device,
             const int64_t* seg_first, const int64_t* seg_steps, int64_t n_seg, int32_t layout,
             const jb_config& c, jb_fit* fit, const Comm& cm, int64_t n_seg_global) {
    cudaStream_t st = ctx->stream;
    JB_CUDA(cudaSetDevice(ctx->device));
    const auto t_start = Clock::now();
    // CompressionConfig::validate (compression.hpp:22-25), partitional_compress (:169)
    if (!(c.tol > 0.0)) throw Error(INVALID_INPUT, "compression tol must be > 0");
    if (c.max_piece_len < 0) throw Error(INVALID_INPUT, "max_piece_len must be >= 0");
    if (n_seg <= 0) throw Error(INVALID_INPUT, "empty dataset");
    if (layout < 0 || layout > 2) throw Error(LAYOUT_ERROR, "unknown layout");
    fit->layout = layout;
    fit->drop_local_last = layout == 0 && cm.rank + 1 < cm.world;
    SegTable& seg = fit->seg;
    seg.n_seg = n_seg;
    seg.h_first.assign(seg_first, seg_first + n_seg);
    seg.h_steps.assign(seg_steps, seg_steps + n_seg);
    int64_t max_last = 0;
    seg.total_steps = 0;
    for (int64_t s = 0; s < n_seg; ++s) {
        if (seg_steps[s] < 1)
            throw Error(INVALID_INPUT, "compression needs at least 2 samples (segment " +
                                           std::to_string(s) + ")");
        if (seg_first[s] < 0) throw Error(INVALID_INPUT, "negative segment offset");
        // piece lengths are 32-bit on the device: a segment longer than that
        // needs max_piece_len to bound them (the reference's are 64-bit)
        if (seg_steps[s] > INT32_MAX && !(c.max_piece_len > 0 && c.max_piece_len <= INT32_MAX))
            throw Error(INVALID_INPUT, "segment " + std::to_string(s) + " has more than 2^31-1 "
                                       "steps: set max_piece_len <= 2^31-1");
        max_last = std::max(max_last, seg_first[s] + seg_steps[s]);
        seg.total_steps += seg_steps[s];
    }
    if (max_last >= n_values) throw Error(INVALID_INPUT, "segment table exceeds the value buffer");
    (void)n_seg_global;
    seg.first.alloc(n_seg, st);
    seg.steps.alloc(n_seg, st);
    seg.first.upload(seg_first, n_seg);
    seg.steps.upload(seg_steps, n_seg);
    JB_TRACE("fit: start", st);
    DArr<double> dvals;
    const double* d_values = values;
    if (!on_device) {
        dvals.alloc(max_last + 1, st);
        dvals.upload(values, max_last + 1);
        d_values = dvals.p;
    }

    // svq on one GPU: the engine draws and the sample (sampling_kmeans
    // clustering.hpp:251-262) depend only on N and the seed, so they run on
    // a side stream: the draws from the start of the fit (a bound on their
    // count, S <= r * steps, is known before compression: the stream is the
    // same prefix for any count), the sample from a helper thread while
    // scale_pieces runs here; the backend joins them (and rethrows their
    // error after scale's own).
    struct SvqPre {
        DArr<uint64_t> raw, sample;
        SampleOrder jorder;
        uint64_t S = 0, raw_count = 0, cursor = 0;
        std::exception_ptr err;
        std::thread th;
        bool inline_done = false;  // JB_SERIAL_SIDE: ran on the calling thread (profilers)
        ~SvqPre() {
            if (th.joinable()) th.join();
        }
    } pre;
    const bool svq_side = c.backend == JB_BACKEND_SVQ && !cm.dist();
    if (svq_side) {
        if (!ctx->side) {
            JB_CUDA(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
            JB_CUDA(cudaEventCreateWithFlags(&ctx->side_done, cudaEventDisableTiming));
        }
        if (c.r > 0.0 && c.r <= 1.0 && c.k >= 1 && c.n_init >= 1 && c.n_init < 1000000 &&
            c.k < (1ULL << 40)) {  // the helper validates again and reports errors in order
            pre.raw_count = (uint64_t)std::llround(c.r * (double)seg.total_steps) +
                            (c.k + 1) * c.n_init + 4096;
            mt19937_64_generate(c.seed, pre.raw_count, pre.raw, ctx->side);
        }
    }

    // ---- compression (local segments) ----
    JB_TRACE("fit: values on device", st);
    compress_segments(d_values, seg, c.tol, c.max_piece_len, fit->pieces, st, &fit->fix_rounds);
    JB_TRACE("fit: compressed", st);
    fit->anchors.alloc(n_seg, st);
    k_gather_anchors<<<(int)((n_seg + 255) / 256), 256, 0, st>>>(d_values, seg.first.p, n_seg,
                                                                 fit->anchors.p);
    JB_LAUNCH_CHECK();
    fit->h_anchors = fit->anchors.to_host(n_seg);
    dvals.release();
    fit->phase_ms[0] = ms_since(t_start);

    // global piece layout: this rank's pieces are [base, base + N) of N_glob
    const int64_t N = fit->pieces.N;
    int64_t base = 0, N_glob = N, steps_glob = seg.total_steps;
    std::vector<int64_t> N_all(1, N);
    if (cm.dist()) {
        const int64_t mine[2] = {N, seg.total_steps};
        std::vector<int64_t> all(2 * cm.world);
        cm.allgather(mine, sizeof mine, all.data());
        N_all.assign(cm.world, 0);
        N_glob = steps_glob = 0;
        for (int r = 0; r < cm.world; ++r) {
            N_all[r] = all[2 * r];
            if (r < cm.rank) base += all[2 * r];
            N_glob += all[2 * r];
            steps_glob += all[2 * r + 1];
        }
    }
    fit->piece_base = base;

    if (svq_side) {
        const int dev = ctx->device;
        cudaStream_t s2 = ctx->side;
        cudaEvent_t ev = ctx->side_done;
        const int64_t Ng = N_glob;
        auto side_work = [&pre, &c, dev, s2, ev, Ng] {
            try {
                JB_CUDA(cudaSetDevice(dev));
                validate_vq(c, c.r);
                pre.S = (uint64_t)std::llround(c.r * (double)Ng);
                if (pre.S < c.k)
                    throw Error(INVALID_INPUT, "sampling_kmeans: sample of " + std::to_string(pre.S) +
                                                   " points is smaller than k=" +
                                                   std::to_string(c.k) + " (increase r)");
                const uint64_t need = pre.S + (c.k + 1) * c.n_init + 4096;
                if (pre.raw.p == nullptr || pre.raw_count < need) {  // no early draws
                    pre.raw_count = need;
                    mt19937_64_generate(c.seed, pre.raw_count, pre.raw, s2);
                }
                pre.cursor = sample_indices_device((uint64_t)Ng, pre.S, pre.raw.p, pre.raw_count,
                                                   pre.sample, s2, &pre.jorder);
                JB_CUDA(cudaEventRecord(ev, s2));
            } catch (...) {
                pre.err = std::current_exception();
            }
        };
        // JB_SERIAL_SIDE=1: no helper thread (ncu cannot replay a kernel while
        // another host thread launches); same work, same streams
        static const bool serial = getenv("JB_SERIAL_SIDE") != nullptr;
        if (serial) {
            side_work();
            pre.inline_done = true;
        } else {
            pre.th = std::thread(side_work);
        }
    }

    // ---- digitize: scale_pieces ----
    auto t1 = Clock::now();
    Scaled sc;
    if (!ctx->aux) JB_CUDA(cudaStreamCreateWithFlags(&ctx->aux, cudaStreamNonBlocking));
    scale_pieces(fit->pieces, steps_glob, c.scl, sc, st, &cm, ctx->aux);
    JB_TRACE("fit: scaled", st);
    fit->scaling[0] = sc.scl;
    fit->scaling[1] = sc.sigma_len;
    fit->scaling[2] = sc.sigma_inc;
    const BBox bb{sc.xmin, sc.xmax, sc.ymin, sc.ymax};
    PtsView pv = points_view(fit->pieces, sc);
    PieceRows rows;  // x = scl * len / sigma_len: exact row grids in k-means
    rows.len = fit->pieces.len.p;
    rows.scl = sc.scl;
    rows.sl = sc.sigma_len;
    rows.max_len = sc.max_len_global;
    fit->phase_ms[1] = ms_since(t1);

    // ---- run_backend (digitization.hpp:131-198) ----
    auto t2 = Clock::now();
    uint64_t k = 0;
    std::vector<double> backend_centers;
    DArr<uint32_t> labels;
    DArr<uint64_t> sample;         // piece index (this rank's numbering) per sample entry
    KMeansOut svq_km;              // svq: the sample's k-means (labels on demand)
    int64_t n_sample_local = 0;
    bool assign_needed = false;
    switch (c.backend) {
        case JB_BACKEND_VQ: {
            validate_vq(c, 1.0);
            if ((int64_t)c.k > N_glob) throw Error(INVALID_INPUT, "kmeans: k exceeds points");
            DArr<uint64_t> raw;
            const uint64_t raw_count = (c.k + 1) * c.n_init + 4096;
            mt19937_64_generate(c.seed, raw_count, raw, st);
            uint64_t cursor = 0;
            KMeansOut km;
            if (cm.dist()) {
                DArr<uint32_t> gpos(std::max<int64_t>(N, 1), st);
                DArr<uint64_t> lidx(std::max<int64_t>(N, 1), st);
                k_iota_pos<<<gsz(N), 256, 0, st>>>(gpos.p, lidx.p, N, (uint64_t)base);
                JB_LAUNCH_CHECK();
                lloyd_best_dist(cm, pv, lidx.p, gpos.p, N, (uint64_t)N_glob, c.k, c.max_iters,
                                c.n_init, raw.p, raw_count, &cursor, bb, km, st, rows);
            } else {
                lloyd_best_device(pv, nullptr, N, c.k, c.max_iters, c.n_init, raw.p,
                                  raw_count, &cursor, bb, km, st, rows);
            }
            k = c.k;
            backend_centers = km.centers;
            kmeans_labels(km, N, st);
            labels = std::move(km.labels);
            fit->iterations = km.iterations;
            fit->draws = cursor;
            break;
        }
        case JB_BACKEND_SVQ: {
            DArr<uint64_t> raw;
            SampleOrder jorder;  // single GPU: gather-friendly spatial pass
            uint64_t S = 0, raw_count = 0, cursor = 0;
            if (pre.th.joinable() || pre.inline_done) {  // sampled on the side stream (above)
                if (pre.th.joinable()) pre.th.join();
                if (pre.err) std::rethrow_exception(pre.err);
                JB_CUDA(cudaStreamWaitEvent(st, ctx->side_done, 0));
                S = pre.S;
                raw_count = pre.raw_count;
                cursor = pre.cursor;
                raw = std::move(pre.raw);
                sample = std::move(pre.sample);
                jorder = std::move(pre.jorder);
            } else {
                validate_vq(c, c.r);
                S = (uint64_t)std::llround(c.r * (double)N_glob);
                if (S < c.k)
                    throw Error(INVALID_INPUT, "sampling_kmeans: sample of " + std::to_string(S) +
                                                   " points is smaller than k=" +
                                                   std::to_string(c.k) + " (increase r)");
                raw_count = S + (c.k + 1) * c.n_init + 4096;
                mt19937_64_generate(c.seed, raw_count, raw, st);
                JB_TRACE("svq: engine draws", st);
                cursor = sample_indices_device((uint64_t)N_glob, S, raw.p, raw_count, sample, st,
                                               cm.dist() ? nullptr : &jorder);
            }
            JB_TRACE("svq: sample indices", st);
            KMeansOut km;
            if (cm.dist()) {  // the entries this rank owns, in sample order
                DArr<uint8_t> flags(S, st);
                k_own_flags<<<gsz((int64_t)S), 256, 0, st>>>(sample.p, S, (uint64_t)base,
                                                             (uint64_t)N, flags.p);
                JB_LAUNCH_CHECK();
                DArr<uint32_t> gpos(S, st);
                DArr<int64_t> nsel(1, st);
                size_t tb = 0;
                thrust::counting_iterator<uint32_t> it0(0);
                cub::DeviceSelect::Flagged(nullptr, tb, it0, flags.p, gpos.p, nsel.p, (int64_t)S, st);
                DArr<uint8_t> tmp(tb, st);
                cub::DeviceSelect::Flagged(tmp.p, tb, it0, flags.p, gpos.p, nsel.p, (int64_t)S, st);
                JB_LAUNCH_CHECK();
                nsel.download(&n_sample_local, 1);
                JB_CUDA(cudaStreamSynchronize(st));
                DArr<uint64_t> lidx(std::max<int64_t>(n_sample_local, 1), st);
                k_local_idx<<<gsz(n_sample_local), 256, 0, st>>>(sample.p, gpos.p, n_sample_local,
                                                                 (uint64_t)base, lidx.p);
                JB_LAUNCH_CHECK();
                lloyd_best_dist(cm, pv, lidx.p, gpos.p, n_sample_local, S, c.k, c.max_iters,
                                c.n_init, raw.p, raw_count, &cursor, bb, km, st, rows);
                sample = std::move(lidx);
            } else {
                lloyd_best_device(pv, sample.p, (int64_t)S, c.k, c.max_iters, c.n_init,
                                  raw.p, raw_count, &cursor, bb, km, st, rows, &jorder);
                n_sample_local = (int64_t)S;
            }
            k = c.k;
            backend_centers = km.centers;
            fit->work_tiles = km.work_tiles;
            fit->changed_labels = km.changed_labels;
            fit->d2_tiles = km.d2_tiles;
            fit->iterations = km.iterations;
            svq_km = std::move(km);  // sample labels: unsorted only if needed below
            labels.alloc(std::max<int64_t>(N, 1), st);
            assign_needed = true;
            fit->sample_size = S;
            fit->draws = cursor;
            break;
        }
        case JB_BACKEND_GA:
        case JB_BACKEND_GA_AUTO:
        case JB_BACKEND_GA_HIER: {
            double alpha = c.alpha;
            if (c.backend == JB_BACKEND_GA_AUTO) {
                if (!(c.eta > 0.0)) throw Error(INVALID_INPUT, "AutoDigitizeConfig: eta must be > 0");
                alpha = auto_alpha_host(steps_glob, N_glob, c.tol, c.eta);
            }
            validate_ga(c, alpha);
            // GA is one sequential sweep over all points in key order (SURVEY
            // §8e): every rank runs it on the gathered points (replicated)
            DArr<double> all_pts;
            materialize_points(fit->pieces, sc, st);  // GA sorts and sweeps the points
            pv = points_view(fit->pieces, sc);
            const double* gpts = sc.pts.p;
            if (cm.dist()) {
                int64_t mx = 0;
                for (auto v : N_all) mx = std::max(mx, v);
                std::vector<double> mine(2 * mx, 0.0), all(2 * mx * cm.world);
                if (N) {
                    JB_CUDA(cudaMemcpyAsync(mine.data(), sc.pts.p, 16 * N, cudaMemcpyDeviceToHost, st));
                    JB_CUDA(cudaStreamSynchronize(st));
                }
                cm.allgather(mine.data(), 16 * mx, all.data());
                std::vector<double> cat;
                cat.reserve(2 * N_glob);
                for (int r = 0; r < cm.world; ++r)
                    cat.insert(cat.end(), all.begin() + 2 * mx * r,
                               all.begin() + 2 * mx * r + 2 * N_all[r]);
                all_pts.alloc(2 * N_glob, st);
                all_pts.upload(cat.data(), 2 * N_glob);
                gpts = all_pts.p;
            }
            DArr<uint32_t> glabels;
            if (c.backend == JB_BACKEND_GA_HIER) {
                int rounds = 0;
                k = ga_hier_device(gpts, N_glob, c, bb, glabels, rounds, st);
                fit->ga_rounds = rounds;
            } else {
                GAOut ga;
                greedy_aggregate_device(gpts, N_glob, alpha, c.sort_key, c.early_stop != 0, bb, ga,
                                        st);
                k = ga.groups;
                glabels = std::move(ga.labels);
                fit->ga_rounds = ga.rounds;
            }
            if (cm.dist()) {
                labels.alloc(std::max<int64_t>(N, 1), st);
                if (N)
                    JB_CUDA(cudaMemcpyAsync(labels.p, glabels.p + base, 4 * N,
                                            cudaMemcpyDeviceToDevice, st));
            } else {
                labels = std::move(glabels);
            }
            break;
        }
        default:
            throw Error(INVALID_INPUT, "unknown backend");
    }
    JB_TRACE("fit: backend", st);
    fit->phase_ms[2] = ms_since(t2);

    // ---- group statistics, ranking, codebook (digitization.hpp:217-291) ----
    auto t3 = Clock::now();
    GroupStats gs;
    RangeHist xh;  // per-range (length, group) counts: the exact x sums below
    assign_and_stats(pv, fit->pieces.len.p, N, backend_centers, k, bb, assign_needed,
                     labels.p, gs, st, sc.max_len_global, sc.scl, sc.sigma_len, &cm, base,
                     k <= 2048 ? &xh : nullptr);
    // ranking (digitization.hpp:257-262) needs only the counts and first
    // indices: the labels are rewritten in rank order on the aux stream, out of
    // place, while the sequential x sums below read the backend's labels
    std::vector<uint64_t> order(k);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](uint64_t a, uint64_t b) {
        if (gs.counts[a] != gs.counts[b]) return gs.counts[a] > gs.counts[b];
        return gs.first_seen[a] < gs.first_seen[b];
    });
    std::vector<uint32_t> rank_of(k);
    for (uint64_t r = 0; r < k; ++r) rank_of[order[r]] = (uint32_t)r;
    DArr<uint32_t> ranked;
    cudaEvent_t ev_ranked = nullptr;
    if (k > 0 && N > 0) {
        ranked.alloc(N, st);
        cudaEvent_t ev;
        JB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        JB_CUDA(cudaEventRecord(ev, st));
        JB_CUDA(cudaStreamWaitEvent(ctx->aux, ev, 0));
        JB_CUDA(cudaEventDestroy(ev));
        relabel(labels.p, N, rank_of, ctx->aux, ranked.p, false);
        JB_CUDA(cudaEventCreateWithFlags(&ev_ranked, cudaEventDisableTiming));
        JB_CUDA(cudaEventRecord(ev_ranked, ctx->aux));
    }
    struct EvGuard {  // the join also runs when the sums below throw
        cudaEvent_t& e;
        cudaStream_t st;
        void join() {
            if (e) {
                cudaStreamWaitEvent(st, e, 0);
                cudaEventDestroy(e);
                e = nullptr;
            }
        }
        ~EvGuard() {
            if (e) {
                cudaEventSynchronize(e);
                cudaEventDestroy(e);
            }
        }
    } ranked_guard{ev_ranked, st};
    // the x sums bit-exact as the reference accumulates them: then the
    // codebook's x and every reconstructed length match (inverse.hpp:46,63-74)
    if (k > 0) {
        std::vector<double> sx;
        if (k <= 2048) {
            SeqTerms xt;
            xt.len = fit->pieces.len.p;
            xt.kind = SeqTerms::X;
            xt.a = sc.scl;
            xt.b = sc.sigma_len;
            sx = range_seq_sums(xh, xt, labels.p, st, &cm);
        } else {  // large alphabets (GA): sort the lengths by group, then sum
            sx = exact_group_sum_x(fit->pieces.len.p, labels.p, N, k, sc.scl, sc.sigma_len, st, &cm);
        }
        for (uint64_t g = 0; g < k; ++g) gs.sum_x[g] = sx[g];
    }
    std::vector<double> centers(2 * k), mean_lengths(k);
    bool need_sample_stats = false;
    for (uint64_t g = 0; g < k; ++g) need_sample_stats |= gs.counts[g] == 0;
    std::vector<uint64_t> sls(k, 0), slc(k, 0);
    if (need_sample_stats && c.backend == JB_BACKEND_SVQ) {
        if (n_sample_local > 0) {
            kmeans_labels(svq_km, n_sample_local, st);
            sample_len_stats(sample.p, svq_km.labels.p, n_sample_local, fit->pieces.len.p, k, sls,
                             slc, st);
        }
        if (cm.dist()) {
            auto a = cm.gather(sls), b = cm.gather(slc);
            std::fill(sls.begin(), sls.end(), 0);
            std::fill(slc.begin(), slc.end(), 0);
            for (int r = 0; r < cm.world; ++r)
                for (uint64_t g = 0; g < k; ++g) {
                    sls[g] += a[(size_t)r * k + g];
                    slc[g] += b[(size_t)r * k + g];
                }
        }
    }
    for (uint64_t g = 0; g < k; ++g) {
        if (gs.counts[g] > 0) {
            centers[2 * g] = gs.sum_x[g] / (double)gs.counts[g];
            centers[2 * g + 1] = gs.sum_y[g] / (double)gs.counts[g];
            mean_lengths[g] = (double)gs.len_sums[g] / (double)gs.counts[g];
        } else {
            centers[2 * g] = backend_centers.at(2 * g);
            centers[2 * g + 1] = backend_centers.at(2 * g + 1);
            const uint64_t lc = slc[g];
            mean_lengths[g] = lc > 0 ? (double)sls[g] / (double)lc : 1.0;
        }
    }
    fit->k = k;
    fit->centers.resize(2 * k);
    fit->mean_lengths.resize(k);
    for (uint64_t r = 0; r < k; ++r) {
        fit->centers[2 * r] = centers[2 * order[r]];
        fit->centers[2 * r + 1] = centers[2 * order[r] + 1];
        fit->mean_lengths[r] = mean_lengths[order[r]];
        if (!std::isfinite(fit->centers[2 * r]) || !std::isfinite(fit->centers[2 * r + 1]))
            throw Error(INVALID_INPUT, "codebook: non-finite center");  // core.hpp:173-175
    }
    ranked_guard.join();  // st waits for the ranked labels
    if (k > 0 && N > 0) labels = std::move(ranked);  // the old array returns to st's cache
    fit->labels = std::move(labels);
    fit->d_centers.alloc(std::max<uint64_t>(2 * k, 1), st);
    fit->d_mean_lengths.alloc(std::max<uint64_t>(k, 1), st);
    fit->d_centers.upload(fit->centers.data(), 2 * k);
    fit->d_mean_lengths.upload(fit->mean_lengths.data(), k);
    JB_CUDA(cudaStreamSynchronize(st));
    JB_TRACE("fit: stats+codebook", st);
    fit->phase_ms[3] = ms_since(t3);
    fit->phase_ms[4] = ms_since(t_start);
}

std::vector<int64_t> out_offsets_for(const std::vector<int64_t>& steps, int32_t layout,
                                     int64_t* total, bool drop_local_last = false) {
    std::vector<int64_t> off(steps.size());
    int64_t pos = 0;
    for (size_t s = 0; s < steps.size(); ++s) {
        off[s] = pos;
        const bool drop = layout == 0 && (s + 1 < steps.size() || drop_local_last);
        pos += drop ? steps[s] : steps[s] + 1;
    }
    *total = pos;
    return off;
}

}  // namespace

extern "C" {

int jb_abi_version(void) { return JB_ABI_VERSION; }
const char* jb_last_error(void) { return g_last_error.c_str(); }

void jb_config_default(jb_config* c) {
    std::memset(c, 0, sizeof *c);
    c->tol = 0.1;
    c->max_piece_len = 0;
    c->backend = JB_BACKEND_GA;
    c->scl = 1.0;
    c->k = 8;
    c->r = 1.0;
    c->max_iters = 300;
    c->n_init = 1;
    c->seed = 0;
    c->alpha = 0.5;
    c->sort_key = JB_SORT_FIRST_PRINCIPAL_COMPONENT;
    c->early_stop = 1;
    c->eta = 1.0;
    c->threads = 1;
}

jb_status jb_context_create(int device, jb_context** out) {
    return (jb_status)guarded([&] {
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
            throw Error(NO_DEVICE, "no CUDA device visible");
        if (device < 0 || device >= n) throw Error(NO_DEVICE, "device index out of range");
        JB_CUDA(cudaSetDevice(device));
        cudaMemPool_t pool;
        JB_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t thr = UINT64_MAX;
        JB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
        auto* c = new jb_context;
        c->device = device;
        JB_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        *out = c;
    });
}

void jb_context_destroy(jb_context* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    jb::dev_cache_drop(ctx->stream);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->side) {
        cudaStreamSynchronize(ctx->side);
        jb::dev_cache_drop(ctx->side);
        cudaStreamSynchronize(ctx->side);
        cudaEventDestroy(ctx->side_done);
    }
    if (ctx->aux) {
        cudaStreamSynchronize(ctx->aux);
        jb::dev_cache_drop(ctx->aux);
        cudaStreamSynchronize(ctx->aux);
        cudaStreamDestroy(ctx->aux);
    }
    // buffers of fits that outlive the context stay valid (the stream handle
    // is not destroyed: a jb_fit still references it)
    delete ctx;
}

jb_status jb_plan_segments(const int64_t* series_lengths, int64_t n_series, int32_t layout,
                           int64_t parts, int64_t* seg_first, int64_t* seg_steps,
                           int64_t* n_seg_out) {
    return (jb_status)guarded([&] {
        if (n_series <= 0) throw Error(INVALID_INPUT, "empty dataset");
        if (layout == JB_LAYOUT_UNIVARIATE_PARTITIONED && n_series != 1)
            throw Error(LAYOUT_ERROR, "univariate-partitioned dataset must hold exactly one series");
        if (layout == JB_LAYOUT_MULTIVARIATE)
            for (int64_t s = 1; s < n_series; ++s)
                if (series_lengths[s] != series_lengths[0])
                    throw Error(LAYOUT_ERROR, "multivariate dataset has ragged dimensions");
        int64_t nseg = 0, first = 0;
        for (int64_t s = 0; s < n_series; ++s) {
            const int64_t len = series_lengths[s];
            const int64_t steps = len == 0 ? 0 : len - 1;
            if (parts == 1 && layout != JB_LAYOUT_UNIVARIATE_PARTITIONED) {
                seg_first[nseg] = first;
                seg_steps[nseg] = steps;
                ++nseg;
            } else {
                if (parts <= 0) throw Error(INVALID_PARTITION, "partition count must be >= 1");
                if (parts > steps)
                    throw Error(INVALID_PARTITION, "cannot split " + std::to_string(steps) +
                                                       " steps into " + std::to_string(parts) +
                                                       " segments");
                const int64_t base = steps / parts, extra = steps % parts;
                int64_t begin = first;
                for (int64_t p = 0; p < parts; ++p) {
                    const int64_t st = base + (p < extra ? 1 : 0);
                    seg_first[nseg] = begin;
                    seg_steps[nseg] = st;
                    ++nseg;
                    begin += st;
                }
            }
            first += len;
        }
        *n_seg_out = nseg;
    });
}

jb_status jb_fit_transform(jb_context* ctx, const double* values, int64_t n_values,
                           int32_t values_on_device, const int64_t* seg_first,
                           const int64_t* seg_steps, int64_t n_seg, int32_t layout,
                           const jb_config* cfg, jb_fit** out) {
    *out = nullptr;
    jb_fit* fit = new jb_fit;
    const int rc = guarded([&] {
        run_fit(ctx, values, n_values, values_on_device != 0, seg_first, seg_steps, n_seg, layout,
                *cfg, fit, Comm{}, n_seg);
    });
    if (rc != JB_OK) {
        delete fit;
        cudaGetLastError();
        return (jb_status)rc;
    }
    *out = fit;
    return JB_OK;
}

jb_status jb_fit_transform_dist(jb_context* ctx, const jb_comm* comm, const double* values,
                                int64_t n_values, int32_t values_on_device,
                                const int64_t* seg_first, const int64_t* seg_steps,
                                int64_t n_seg_local, int64_t n_seg_global, int32_t layout,
                                const jb_config* cfg, jb_fit** out) {
    *out = nullptr;
    jb_fit* fit = new jb_fit;
    const int rc = guarded([&] {
        if (!comm || comm->world < 1 || comm->rank < 0 || comm->rank >= comm->world ||
            (comm->world > 1 && !comm->allgather))
            throw Error(INVALID_INPUT, "invalid communicator");
        Comm cm;
        cm.c = comm;
        cm.rank = comm->rank;
        cm.world = comm->world;
        run_fit(ctx, values, n_values, values_on_device != 0, seg_first, seg_steps, n_seg_local,
                layout, *cfg, fit, cm, n_seg_global);
    });
    if (rc != JB_OK) {
        delete fit;
        cudaGetLastError();
        return (jb_status)rc;
    }
    *out = fit;
    return JB_OK;
}

void jb_fit_free(jb_fit* fit) { delete fit; }

int64_t jb_fit_n_segments(const jb_fit* f) { return f->seg.n_seg; }
int64_t jb_fit_n_pieces(const jb_fit* f) { return f->pieces.N; }
uint64_t jb_fit_k(const jb_fit* f) { return f->k; }
int32_t jb_fit_layout(const jb_fit* f) { return f->layout; }

int64_t jb_fit_reconstruct_size(const jb_fit* f) {
    int64_t total = 0;
    out_offsets_for(f->seg.h_steps, f->layout, &total, f->drop_local_last);
    return total;
}

jb_status jb_fit_copy_pieces(const jb_fit* f, int64_t* piece_offsets, int64_t* len, double* inc) {
    return (jb_status)guarded([&] {
        cudaStream_t st = f->pieces.len.s;
        if (piece_offsets) f->pieces.seg_offsets.download(piece_offsets, f->seg.n_seg + 1);
        if (inc) f->pieces.inc.download(inc, f->pieces.N);
        std::vector<int32_t> l;
        if (len) l = f->pieces.len.to_host(f->pieces.N);
        JB_CUDA(cudaStreamSynchronize(st));
        if (len)
            for (int64_t i = 0; i < f->pieces.N; ++i) len[i] = l[i];
    });
}

jb_status jb_fit_copy_symbolic(const jb_fit* f, uint32_t* labels, double* centers,
                               double* mean_lengths, double* scaling, double* anchors,
                               int64_t* source_lengths) {
    return (jb_status)guarded([&] {
        if (labels) {
            f->labels.download(labels, f->pieces.N);
            JB_CUDA(cudaStreamSynchronize(f->labels.s));
        }
        if (centers) std::copy(f->centers.begin(), f->centers.end(), centers);
        if (mean_lengths) std::copy(f->mean_lengths.begin(), f->mean_lengths.end(), mean_lengths);
        if (scaling) std::copy(f->scaling, f->scaling + 3, scaling);
        if (anchors) std::copy(f->h_anchors.begin(), f->h_anchors.end(), anchors);
        if (source_lengths)
            std::copy(f->seg.h_steps.begin(), f->seg.h_steps.end(), source_lengths);
    });
}

jb_status jb_fit_stats(const jb_fit* f, uint64_t* iterations, uint64_t* sample_size,
                       uint64_t* draws, int32_t* fix_rounds, int32_t* ga_rounds,
                       double* phase_ms) {
    if (iterations) *iterations = f->iterations;
    if (sample_size) *sample_size = f->sample_size;
    if (draws) *draws = f->draws;
    if (fix_rounds) *fix_rounds = f->fix_rounds;
    if (ga_rounds) *ga_rounds = f->ga_rounds;
    if (phase_ms) std::copy(f->phase_ms, f->phase_ms + 5, phase_ms);
    if (phase_ms) {  // extended diagnostics after the 5 phase timings
        phase_ms[5] = (double)f->work_tiles;
        phase_ms[6] = (double)f->changed_labels;
        phase_ms[7] = (double)f->d2_tiles;
    }
    return JB_OK;
}

jb_status jb_fit_inverse_transform(jb_context* ctx, const jb_fit* f, double* out_values,
                                   int32_t out_on_device, int64_t* out_offsets) {
    return (jb_status)guarded([&] {
        cudaStream_t st = ctx->stream;
        JB_CUDA(cudaSetDevice(ctx->device));
        int64_t total = 0;
        const auto off = out_offsets_for(f->seg.h_steps, f->layout, &total, f->drop_local_last);
        DArr<int64_t> d_off(f->seg.n_seg, st);
        d_off.upload(off.data(), f->seg.n_seg);
        DArr<double> d_out;
        double* dst = out_values;
        if (!out_on_device) {
            d_out.alloc(total, st);
            dst = d_out.p;
        }
        // the fit's arrays were produced on the fit's stream: order after it
        JB_CUDA(cudaStreamSynchronize(f->labels.s ? f->labels.s : st));
        InverseIn in{f->labels.p,
                     f->pieces.seg_offsets.p,
                     f->anchors.p,
                     f->seg.steps.p,
                     d_off.p,
                     f->seg.n_seg,
                     f->pieces.N,
                     f->layout,
                     f->k,
                     f->d_centers.p,
                     f->d_mean_lengths.p,
                     f->scaling[0],
                     f->scaling[1],
                     f->scaling[2],
                     f->drop_local_last};
        inverse_transform_device(in, dst, st);
        if (!out_on_device) d_out.download(out_values, total);
        JB_CUDA(cudaStreamSynchronize(st));
        if (out_offsets) {
            if (f->layout == 0) {
                out_offsets[0] = 0;
                out_offsets[1] = total;
            } else {
                for (int64_t s = 0; s < f->seg.n_seg; ++s) out_offsets[s] = off[s];
                out_offsets[f->seg.n_seg] = total;
            }
        }
    });
}

int64_t jb_reconstruct_size(const int64_t* source_lengths, int64_t n_seg, int32_t layout) {
    int64_t total = 0;
    out_offsets_for(std::vector<int64_t>(source_lengths, source_lengths + n_seg), layout, &total);
    return total;
}

jb_status jb_inverse_transform(jb_context* ctx, const double* centers, const double* mean_lengths,
                               uint64_t k, const double* scaling, const uint32_t* labels,
                               const int64_t* piece_offsets, const double* anchors,
                               const int64_t* source_lengths, int64_t n_seg, int32_t layout,
                               double* out_values) {
    return (jb_status)guarded([&] {
        cudaStream_t st = ctx->stream;
        JB_CUDA(cudaSetDevice(ctx->device));
        if (layout == 0 && n_seg <= 0) throw Error(INVALID_INPUT, "stitch_partitions: no segments");
        if (n_seg < 0) throw Error(INVALID_INPUT, "negative segment count");
        if (n_seg == 0) return;
        if (piece_offsets[0] != 0) throw Error(INVALID_INPUT, "piece offsets must start at 0");
        for (int64_t s = 0; s < n_seg; ++s)
            if (piece_offsets[s + 1] < piece_offsets[s])
                throw Error(INVALID_INPUT, "piece offsets must be non-decreasing");
        const int64_t N = piece_offsets[n_seg];
        std::vector<int64_t> steps(source_lengths, source_lengths + n_seg);
        int64_t total = 0;
        const auto off = out_offsets_for(steps, layout, &total);
        DArr<uint32_t> d_lab(std::max<int64_t>(N, 1), st);
        DArr<int64_t> d_po(n_seg + 1, st), d_sl(n_seg, st), d_off(n_seg, st);
        DArr<double> d_anc(n_seg, st), d_c(std::max<uint64_t>(2 * k, 1), st),
            d_ml(std::max<uint64_t>(k, 1), st), d_out(std::max<int64_t>(total, 1), st);
        d_lab.upload(labels, N);
        d_po.upload(piece_offsets, n_seg + 1);
        d_sl.upload(source_lengths, n_seg);
        d_off.upload(off.data(), n_seg);
        d_anc.upload(anchors, n_seg);
        d_c.upload(centers, 2 * k);
        d_ml.upload(mean_lengths, k);
        InverseIn in{d_lab.p, d_po.p, d_anc.p, d_sl.p, d_off.p, n_seg, N, layout, k, d_c.p,
                     d_ml.p, scaling[0], scaling[1], scaling[2], false};
        inverse_transform_device(in, d_out.p, st);
        d_out.download(out_values, total);
        JB_CUDA(cudaStreamSynchronize(st));
    });
}

namespace jb_api {
__global__ void k_len_to_i32(const int64_t* __restrict__ in, int64_t n, int32_t* __restrict__ out,
                             int* __restrict__ bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = in[i];
        if (v < INT32_MIN || v > INT32_MAX) *bad = 1;
        out[i] = (int32_t)v;
    }
}
}  // namespace jb_api

jb_status jb_symbolize_with(jb_context* ctx, const double* centers, uint64_t k,
                            const double* scaling, const int64_t* len, const double* inc,
                            int64_t n, int32_t pieces_on_device, uint32_t* labels) {
    return (jb_status)guarded([&] {
        cudaStream_t st = ctx->stream;
        JB_CUDA(cudaSetDevice(ctx->device));
        if (k == 0) throw Error(INVALID_INPUT, "symbolize_with: empty codebook");
        if (n < 0) throw Error(INVALID_INPUT, "negative piece count");
        if (n == 0) return;
        const std::vector<double> c(centers, centers + 2 * k);
        DArr<int32_t> d_len(n, st);
        DArr<int64_t> h2d_len;
        DArr<double> d_inc;
        DArr<uint32_t> d_lab;
        DArr<int> bad(1, st);
        bad.zero();
        const int64_t* src_len = len;
        if (!pieces_on_device) {
            h2d_len.alloc(n, st);
            h2d_len.upload(len, n);
            src_len = h2d_len.p;
            d_inc.alloc(n, st);
            d_inc.upload(inc, n);
            d_lab.alloc(n, st);
        }
        jb_api::k_len_to_i32<<<gsz(n), 256, 0, st>>>(src_len, n, d_len.p, bad.p);
        JB_LAUNCH_CHECK();
        int hb = 0;
        bad.download(&hb, 1);
        JB_CUDA(cudaStreamSynchronize(st));
        if (hb) throw Error(INVALID_INPUT, "symbolize_with: piece length beyond 32 bits");
        symbolize_pieces(d_len.p, pieces_on_device ? inc : d_inc.p, n, c, k, scaling,
                         pieces_on_device ? labels : d_lab.p, st);
        if (!pieces_on_device) d_lab.download(labels, n);
        JB_CUDA(cudaStreamSynchronize(st));
    });
}

void jb_profile_enable(int32_t on) {
    prof_collect();
    if (on && g_pool.empty()) {
        g_pool.resize(1 << 15);
        for (auto& e : g_pool) cudaEventCreate(&e);
    }
    g_prof_on = on != 0;
}

void jb_profile_reset(void) {
    prof_collect();
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof_totals.clear();
}

int32_t jb_profile_read(char* names, double* total_ms, int64_t* launches, int32_t cap) {
    prof_collect();
    std::lock_guard<std::mutex> lk(g_prof_mu);
    int32_t i = 0;
    for (const auto& kv : g_prof_totals) {
        if (i >= cap) break;
        std::strncpy(names + 64 * i, kv.first.c_str(), 63);
        names[64 * i + 63] = 0;
        total_ms[i] = kv.second.first;
        launches[i] = kv.second.second;
        ++i;
    }
    return (int32_t)g_prof_totals.size();
}

jb_status jb_mt19937_64_stream(jb_context* ctx, uint64_t seed, uint64_t count, uint64_t* out) {
    return (jb_status)guarded([&] {
        JB_CUDA(cudaSetDevice(ctx->device));
        DArr<uint64_t> raw;
        mt19937_64_generate(seed, count, raw, ctx->stream);
        raw.download(out, count);
        JB_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

jb_status jb_sample_indices(jb_context* ctx, uint64_t n, uint64_t sample_size, uint64_t seed,
                            uint64_t* out) {
    return (jb_status)guarded([&] {
        JB_CUDA(cudaSetDevice(ctx->device));
        if (sample_size > n) throw Error(INVALID_INPUT, "sample larger than population");
        DArr<uint64_t> raw, idx;
        const uint64_t raw_count = sample_size + 4096;
        mt19937_64_generate(seed, raw_count, raw, ctx->stream);
        sample_indices_device(n, sample_size, raw.p, raw_count, idx, ctx->stream);
        idx.download(out, sample_size);
        JB_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

jb_status jb_kmeans(jb_context* ctx, const double* points, int64_t n, uint64_t k,
                    uint64_t max_iters, uint64_t n_init, uint64_t seed, uint32_t* labels,
                    double* centers, uint64_t* iterations) {
    return (jb_status)guarded([&] {
        JB_CUDA(cudaSetDevice(ctx->device));
        cudaStream_t st = ctx->stream;
        // VQConfig::validate (clustering.hpp:26-31) through the fit's checks
        jb_config c;
        jb_config_default(&c);
        c.k = k;
        c.max_iters = max_iters;
        c.n_init = n_init;
        validate_vq(c, 1.0);
        if (n <= 0) throw Error(INVALID_INPUT, "kmeans: no points");
        if ((int64_t)k > n) throw Error(INVALID_INPUT, "kmeans: k exceeds points");
        BBox bb{points[0], points[0], points[1], points[1]};
        for (int64_t i = 0; i < n; ++i) {
            const double x = points[2 * i], y = points[2 * i + 1];
            if (!std::isfinite(x) || !std::isfinite(y))
                throw Error(INVALID_INPUT, "kmeans: non-finite point");
            bb.xmin = std::min(bb.xmin, x);
            bb.xmax = std::max(bb.xmax, x);
            bb.ymin = std::min(bb.ymin, y);
            bb.ymax = std::max(bb.ymax, y);
        }
        DArr<double> dp(2 * n, st);
        dp.upload(points, 2 * n);
        PtsView pv;
        pv.pts = reinterpret_cast<const double2*>(dp.p);
        DArr<uint64_t> raw;
        const uint64_t raw_count = (k + 1) * n_init + 4096;
        mt19937_64_generate(seed, raw_count, raw, st);
        uint64_t cursor = 0;
        KMeansOut km;
        lloyd_best_device(pv, nullptr, n, k, max_iters, n_init, raw.p, raw_count, &cursor, bb, km,
                          st);
        kmeans_labels(km, n, st);
        km.labels.download(labels, n);
        JB_CUDA(cudaStreamSynchronize(st));
        std::copy(km.centers.begin(), km.centers.begin() + 2 * k, centers);
        *iterations = km.iterations;
    });
}

jb_status jb_mse(jb_context* ctx, const double* a, const double* b, int64_t n, int32_t on_device,
                 double* out) {
    return (jb_status)guarded([&] {
        JB_CUDA(cudaSetDevice(ctx->device));
        if (n <= 0) throw Error(INVALID_INPUT, "mse: empty series");
        DArr<double> da, db;
        const double* pa = a;
        const double* pb = b;
        if (!on_device) {
            da.alloc(n, ctx->stream);
            db.alloc(n, ctx->stream);
            da.upload(a, n);
            db.upload(b, n);
            pa = da.p;
            pb = db.p;
        }
        SeqTerms t;
        t.kind = SeqTerms::SQDIFF;
        t.w = pa;
        t.w2 = pb;
        *out = seq_sum_nonneg(t, {0, n}, ctx->stream)[0] / (double)n;
    });
}

jb_status jb_seq_sum_nonneg(jb_context* ctx, const double* terms, const int64_t* seg_off,
                            int64_t n_seg, double* out) {
    return (jb_status)guarded([&] {
        JB_CUDA(cudaSetDevice(ctx->device));
        if (n_seg < 0) throw Error(INVALID_INPUT, "negative segment count");
        std::vector<int64_t> off(seg_off, seg_off + n_seg + 1);
        for (int64_t g = 0; g < n_seg; ++g)
            if (off[g + 1] < off[g] || off[0] < 0)
                throw Error(INVALID_INPUT, "segment offsets must be non-decreasing");
        const int64_t n = n_seg > 0 ? off[n_seg] : 0;
        DArr<double> w(std::max<int64_t>(n, 1), ctx->stream);
        w.upload(terms, n);
        SeqTerms t;
        t.kind = SeqTerms::DIRECT;
        t.w = w.p;
        const std::vector<double> r = seq_sum_nonneg(t, off, ctx->stream);
        std::copy(r.begin(), r.end(), out);
    });
}

int32_t jb_symbol_token(uint64_t rank, uint64_t alphabet_size, char* buf) {
    // symbol_token (core.hpp:186-193)
    if (alphabet_size <= 94) {
        const int code = rank < 62 ? 65 + (int)rank : 33 + (int)rank - 62;
        buf[0] = (char)code;
        buf[1] = 0;
        return 1;
    }
    const std::string s = "#" + std::to_string(rank);
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return (int32_t)s.size();
}

}  // extern "C"
