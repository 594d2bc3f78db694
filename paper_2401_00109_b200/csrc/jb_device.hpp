// jb_device.hpp — stream-ordered device arrays and the kernel entry points
// shared between the translation units of libjabba_b200.so.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <utility>
#include <vector>

#include "../../include/jabba_b200.h"
#include "jb_common.cuh"

namespace jb {

// JB_DEBUG=1: host-side diagnostics on stderr (collective sequence, k-means
// seeds and per-iteration label changes) for comparing ranks / paths.
inline bool dbg_on() {
    static const bool on = getenv("JB_DEBUG") != nullptr;
    return on;
}
inline uint64_t dbg_hash(const void* p, size_t bytes) {  // FNV-1a
    uint64_t h = 1469598103934665603ULL;
    for (size_t i = 0; i < bytes; ++i) h = (h ^ static_cast<const unsigned char*>(p)[i]) * 1099511628211ULL;
    return h;
}

// Host side of the distributed fit's collectives: an exact allgather of host
// bytes (rank order). world == 1 means single-GPU.
struct Comm {
    const jb_comm* c = nullptr;
    int rank = 0, world = 1;
    bool dist() const { return world > 1; }
    void allgather(const void* send, size_t bytes, void* recv) const {
        if (!dist()) {
            memcpy(recv, send, bytes);
            return;
        }
        if (dbg_on()) {
            static int seq = 0;
            fprintf(stderr, "[jb r%d] allgather #%d: %zu bytes\n", rank, seq++, bytes);
        }
        if (c->allgather(c->user, send, bytes, recv) != 0)
            throw Error(NCCL_ERROR, "allgather callback failed");
    }
    template <class T>
    std::vector<T> gather(const std::vector<T>& v) const {
        std::vector<T> out(v.size() * world);
        allgather(v.data(), sizeof(T) * v.size(), out.data());
        return out;
    }
    // exact element-wise sum of int128 vectors held as (lo, hi) u64 pairs
    std::vector<unsigned long long> sum_i128(const std::vector<unsigned long long>& v) const {
        if (!dist()) return v;
        auto all = gather(v);
        std::vector<unsigned long long> out(v.size(), 0);
        for (int r = 0; r < world; ++r)
            for (size_t i = 0; i + 1 < v.size(); i += 2) {
                const u128 a = ((u128)out[i + 1] << 64) | out[i];
                const u128 b = ((u128)all[r * v.size() + i + 1] << 64) | all[r * v.size() + i];
                const u128 c2 = a + b;
                out[i] = (unsigned long long)c2;
                out[i + 1] = (unsigned long long)(c2 >> 64);
            }
        return out;
    }
};

// Per-stream, size-bucketed cache of device buffers (api.cu). Buffers freed
// on a stream are reused only by later work on the same stream, so reuse is
// stream-ordered and needs no sync; repeated fits of the same shape never
// touch the allocator (a cudaMallocAsync pool growth of 14 GB costs ~1 s).
void* dev_alloc(size_t bytes, cudaStream_t st);
void dev_free(void* p, size_t bytes, cudaStream_t st);
void dev_cache_drop(cudaStream_t st);  // release everything cached for st

// Move-only device array over dev_alloc/dev_free.
template <class T>
struct DArr {
    T* p = nullptr;
    size_t n = 0;
    cudaStream_t s = 0;
    DArr() = default;
    DArr(size_t count, cudaStream_t st) { alloc(count, st); }
    DArr(const DArr&) = delete;
    DArr& operator=(const DArr&) = delete;
    DArr(DArr&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
    DArr& operator=(DArr&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p;
            n = o.n;
            s = o.s;
            o.p = nullptr;
            o.n = 0;
        }
        return *this;
    }
    ~DArr() { release(); }
    void alloc(size_t count, cudaStream_t st) {
        release();
        s = st;
        n = count;
        if (count) p = static_cast<T*>(dev_alloc(sizeof(T) * count, st));
    }
    void release() {
        if (p) dev_free(p, sizeof(T) * n, s);
        p = nullptr;
        n = 0;
    }
    void zero() {
        if (n) JB_CUDA(cudaMemsetAsync(p, 0, sizeof(T) * n, s));
    }
    void upload(const T* h, size_t count) {
        if (count) JB_CUDA(cudaMemcpyAsync(p, h, sizeof(T) * count, cudaMemcpyHostToDevice, s));
    }
    void download(T* h, size_t count) const {
        if (count) JB_CUDA(cudaMemcpyAsync(h, p, sizeof(T) * count, cudaMemcpyDeviceToHost, s));
    }
    std::vector<T> to_host(size_t count) const {
        std::vector<T> h(count);
        download(h.data(), count);
        JB_CUDA(cudaStreamSynchronize(s));
        return h;
    }
};

// ---------------------------------------------------------------------------
// Kernel-level CUDA-event profiler (api.cu). When enabled, every instrumented
// launch site records an event pair on the launching stream; totals are
// collected per kernel name by jb_profile_read().

void prof_begin(const char* name, cudaStream_t st);
void prof_end(cudaStream_t st);

struct ProfScope {
    cudaStream_t st;
    ProfScope(const char* name, cudaStream_t s) : st(s) { prof_begin(name, s); }
    ~ProfScope() { prof_end(st); }
};
// host-side phase trace (env JB_TRACE=1): prints ms since the previous mark
void trace_mark(const char* what, cudaStream_t st);
#define JB_TRACE(what, st) ::jb::trace_mark(what, st)

#define JB_CAT2(a, b) a##b
#define JB_CAT(a, b) JB_CAT2(a, b)
#define JB_PROF(name, st) ::jb::ProfScope JB_CAT(jb_prof_scope_, __LINE__)(name, st)

// ---------------------------------------------------------------------------
// Compression (compress.cu)

struct SegTable {
    int64_t n_seg = 0;
    DArr<int64_t> first, steps;  // per segment: first sample index, steps
    std::vector<int64_t> h_first, h_steps;
    int64_t total_steps = 0;
};

struct Pieces {
    int64_t N = 0;
    DArr<int32_t> len;
    DArr<double> inc;
    DArr<int64_t> seg_offsets;  // n_seg + 1
    double max_abs_inc = 0.0;
    int32_t max_len = 0, min_len = 0;
};

// Compresses every segment (compression.hpp:31-83, 167-193) with the
// speculative-chunk scheme; validates finiteness. Throws jb::Error.
void compress_segments(const double* d_values, const SegTable& seg, double tol,
                       int64_t max_piece_len, Pieces& out, cudaStream_t st,
                       int* n_fix_iters = nullptr);

// ---------------------------------------------------------------------------
// Scaling (digitize.cu): scale_pieces digitization.hpp:25-59

// The scaled points (x, y) = (scl * len / sigma_len, inc / sigma_inc)
// (ScalingParams::apply core.hpp:130-132, k_scale's exact expressions),
// either materialised or computed where they are read.
struct PtsView {
    const double2* pts = nullptr;  // materialised, or null: from len / inc
    const int32_t* len = nullptr;
    const double* inc = nullptr;
    double scl = 1.0, sl = 1.0, si = 1.0;
    double rsi = 0.0;  // div_by_recip(si): y = inc / si by div_by on device
    __host__ __device__ __forceinline__ double2 at(uint64_t i) const {
        if (pts) return pts[i];
#ifdef __CUDA_ARCH__
        return make_double2(scl * (double)len[i] / sl, div_by(inc[i], si, rsi));
#else
        return make_double2(scl * (double)len[i] / sl, inc[i] / si);
#endif
    }
};

struct Scaled {
    DArr<double> pts;  // 2N interleaved (x, y): only when a backend needs them (GA)
    double scl = 1.0, sigma_len = 1.0, sigma_inc = 1.0;
    double xmin = 0, xmax = 0, ymin = 0, ymax = 0;  // bounding box of ALL points
    int64_t N_global = 0;
    int32_t max_len_global = 0;
};

// total_steps: of ALL ranks' segments; cm: null or world == 1 for one GPU.
// Computes sigma and the bounding box; the points stay virtual. aux: an
// optional second stream for the increments' sums, which then overlap the
// lengths' sequential sum on st (both joined before the call returns).
void scale_pieces(const Pieces& pc, int64_t total_steps, double scl, Scaled& out,
                  cudaStream_t st, const Comm* cm = nullptr, cudaStream_t aux = nullptr);
PtsView points_view(const Pieces& pc, const Scaled& sc);
// materialises sc.pts (GA backends sort and sweep the points many times)
void materialize_points(const Pieces& pc, Scaled& sc, cudaStream_t st);

struct BBox {
    double xmin, xmax, ymin, ymax;
};

// ---------------------------------------------------------------------------
// Exact emulation of the reference's sequential fp64 sums of non-negative
// terms (seqsum.cu): var_len (digitization.hpp:39-45) and the per-group sum
// of x (digitization.hpp:224-231).

struct SeqTerms {
    enum Kind : int { VAR_LEN = 0, X = 1, DIRECT = 2, SQDIFF = 3 };
    const int32_t* len = nullptr;  // term i from len[i]
    const double* w = nullptr;     // DIRECT: the terms themselves; SQDIFF: (w[i] - w2[i])^2
    const double* w2 = nullptr;
    int kind = VAR_LEN;
    double a = 0.0, b = 1.0;       // VAR_LEN: (len - a)^2;  X: a * len / b
};

// Segment g is the terms [seg_off[g], seg_off[g+1]); each is summed
// s = s_in[g]; s = fl(s + term) in index order, bit-exactly.
struct SeqSum {
    SeqTerms terms;
    cudaStream_t stream = 0;
    int64_t n_seg = 0, nblk = 0, n2 = 0, n3 = 0;
    std::vector<int64_t> h_off, h_blk;
    std::vector<double> local_total;  // approximate per-segment sums (prediction)
    DArr<int64_t> d_blk, d_off;
    DArr<double> bsum, gpre;
    DArr<int> bseg, be, e2, s2, e3, s3;
    DArr<unsigned long long> pe, po, pe2, po2, pe3, po3;
    void setup(const SeqTerms& t, const std::vector<int64_t>& seg_off, cudaStream_t st);
    // s_in_approx: approximate start values; terms_before: terms of the
    // sequence preceding this part (other ranks), for the error bound
    void predict(const std::vector<double>& s_in_approx, const std::vector<int64_t>& terms_before);
    std::vector<double> resolve(const std::vector<double>& s_in);
};

// Range-histogram input of an exact sum whose terms are a function of the
// piece length (seqsum.cu): for every range r of R consecutive pieces, the
// pieces of group g with length l in 1..RH are counted in
// hist[(r * RH + l - 1) * k + g]; longer pieces are listed (long_idx, any
// order); approx[r * k + g] is an approximate sum of the record's terms (a
// binade prediction only: any rounding is fine). k == 1:
// every piece is in the one group. Written by the producer kernels
// (k_var_blocks, k_assign_stats), consumed by range_seq_sums.
struct RangeHist {
    int64_t n = 0, R = 0, nr = 0;
    int k = 1, RH = 0;
    DArr<uint16_t> hist;
    DArr<double> approx;
    DArr<uint32_t> long_idx;
    DArr<unsigned long long> long_n;
    void alloc(int64_t n_, int64_t R_, int k_, int RH_, bool longs, cudaStream_t st) {
        n = n_;
        R = R_;
        k = k_;
        RH = RH_;
        nr = (n + R - 1) / R;
        hist.alloc(std::max<int64_t>(nr * RH * k, 1), st);
        approx.alloc(std::max<int64_t>(nr * k, 1), st);
        approx.zero();
        long_n.alloc(1, st);
        long_n.zero();
        if (longs) long_idx.alloc(std::max<int64_t>(n, 1), st);
        else long_idx.release();
    }
};

// Exact sequential sums of the terms of every group's pieces in index order
// (d_labels: group of each piece, null when k == 1); multi-GPU as below.
std::vector<double> range_seq_sums(const RangeHist& h, const SeqTerms& t,
                                   const uint32_t* d_labels, cudaStream_t st,
                                   const Comm* cm = nullptr);

// One call for all ranks (cm null or world 1: single GPU); rank r's terms of
// segment g follow ranks 0..r-1's. Returns the exact sums from s = 0.
std::vector<double> seq_sum_nonneg(const SeqTerms& t, const std::vector<int64_t>& seg_off,
                                   cudaStream_t st, const Comm* cm = nullptr);

// ---------------------------------------------------------------------------
// k-means family (kmeans.cu)

struct KMeansOut {
    uint64_t k = 0;
    std::vector<double> centers;  // 2k, backend cluster order
    DArr<uint32_t> labels;        // per input point, once kmeans_labels() ran
    DArr<uint32_t> slabs, sorig;  // labels in the internal (Morton) order + its
                                  // map to the input order: unsorted on demand
    uint64_t iterations = 0;
    double sse = 0.0;
    uint64_t work_tiles = 0, changed_labels = 0;  // Lloyd diagnostics (all iterations)
    uint64_t d2_tiles = 0;                        // D^2 rounds: tiles updated (persistent path)
};

// Materialises out.labels (input order) from the internal order.
void kmeans_labels(KMeansOut& out, int64_t n, cudaStream_t st);

// sample_indices (clustering.hpp:74-85) on device; idx is S entries.
// Returns the number of engine draws consumed (>= S).
// jorder (optional): the swap targets j_i sorted (stable) and the swap
// indices i in that order -- the sample in ascending piece order except the
// ~S^2/2n entries of repeated targets -- for the gather-friendly Morton pass.
struct SampleOrder {
    DArr<uint32_t> j, i;
};
uint64_t sample_indices_device(uint64_t n, uint64_t S, const uint64_t* d_raw, uint64_t raw_count,
                               DArr<uint64_t>& idx, cudaStream_t st,
                               SampleOrder* jorder = nullptr);

// Raw std::mt19937_64 stream on device.
void mt19937_64_generate(uint64_t seed, uint64_t count, DArr<uint64_t>& out, cudaStream_t st);

// Integer piece lengths behind the scaled points (x = scl * len / sl): lets
// the k-means kernels use the exact row grid (jb_rowgrid.cuh). len == null:
// 2-D grid only.
struct PieceRows {
    const int32_t* len = nullptr;  // per piece, indexed like d_pts
    double scl = 1.0, sl = 1.0;
    int32_t max_len = 0;           // global maximum piece length
};

// Best-of-n_init lloyd_once (clustering.hpp:200-236) on the points
// d_pts[d_idx[i]] (or d_pts[i] when d_idx is null), i < n; 2-interleaved
// device doubles. Draws are consumed from d_raw starting at *cursor (updated).
// out.labels are in the original point order.
void lloyd_best_device(const PtsView& pv, const uint64_t* d_idx, int64_t n, uint64_t k,
                       uint64_t max_iters, uint64_t n_init, const uint64_t* d_raw,
                       uint64_t raw_count, uint64_t* cursor, const BBox& bb, KMeansOut& out,
                       cudaStream_t st, const PieceRows& rows = PieceRows{},
                       const SampleOrder* jorder = nullptr);

// Distributed variant: this rank holds the sample entries it owns -- local
// piece index d_lidx[i] and global sample position d_gpos[i] (ascending), n
// entries -- of a global sample of S points. Same results on every rank,
// equal to lloyd_best_device on the whole sample.
void lloyd_best_dist(const Comm& cm, const PtsView& pv, const uint64_t* d_lidx,
                     const uint32_t* d_gpos, int64_t n, uint64_t S, uint64_t k, uint64_t max_iters,
                     uint64_t n_init, const uint64_t* d_raw, uint64_t raw_count, uint64_t* cursor,
                     const BBox& bb, KMeansOut& out, cudaStream_t st,
                     const PieceRows& rows = PieceRows{});

// Per-point nearest center (clustering.hpp:146-163) with exact tie rule, plus
// group statistics for digitize (digitization.hpp:217-231).
struct GroupStats {
    std::vector<uint64_t> counts, first_seen, len_sums;
    std::vector<double> sum_x, sum_y;  // rounded exact sums
};
void assign_and_stats(const PtsView& pv, const int32_t* d_len, int64_t n,
                      const std::vector<double>& centers, uint64_t k, const BBox& bb,
                      bool do_assign, uint32_t* d_labels, GroupStats& gs, cudaStream_t st,
                      int32_t max_len, double scl, double sigma_len, const Comm* cm = nullptr,
                      int64_t first_base = 0, RangeHist* rh = nullptr);

// symbolize_with (digitization.hpp:297-307) on device: labels of held-out
// pieces (len, inc) against a codebook (centers 2k, scaling scl/sl/si).
void symbolize_pieces(const int32_t* d_len, const double* d_inc, int64_t n,
                      const std::vector<double>& centers, uint64_t k, const double scaling[3],
                      uint32_t* d_labels, cudaStream_t st);

// d_out: null for in place, else a second array; sync = false leaves the
// kernel in flight on st (the caller joins the stream)
void relabel(uint32_t* d_labels, int64_t n, const std::vector<uint32_t>& rank_of,
             cudaStream_t st, uint32_t* d_out = nullptr, bool sync = true);

// The reference's sequential per-group sums of x = scl*len/sigma_len over the
// pieces in index order (digitization.hpp:224-231), bit-exact: labels are the
// backend's cluster ids (< k) of this rank's pieces.
std::vector<double> exact_group_sum_x(const int32_t* d_len, const uint32_t* d_labels, int64_t n,
                                      uint64_t k, double scl, double sigma_len, cudaStream_t st,
                                      const Comm* cm = nullptr);

// Sum of len and count over sample labels (svq empty-cluster fallback,
// digitization.hpp:240-252).
void sample_len_stats(const uint64_t* d_sample, const uint32_t* d_sample_labels, int64_t S,
                      const int32_t* d_len, uint64_t k, std::vector<uint64_t>& len_sum,
                      std::vector<uint64_t>& count, cudaStream_t st);

void gather_points(const double* d_pts, const uint64_t* d_idx, int64_t S, double* d_out,
                   cudaStream_t st);

// ---------------------------------------------------------------------------
// Greedy aggregation (ga.cu): greedy_aggregate clustering.hpp:328-375

struct GAOut {
    uint64_t groups = 0;
    DArr<uint32_t> labels;
    int rounds = 0;  // decision rounds of the parallel sweep
};
void greedy_aggregate_device(const double* d_pts, int64_t n, double alpha, int sort_key,
                             bool early_stop, const BBox& bb, GAOut& out, cudaStream_t st);

// ---------------------------------------------------------------------------
// Inverse (inverse.cu): inverse.hpp:32-132

struct InverseIn {
    const uint32_t* labels;       // N ranked labels (device)
    const int64_t* seg_offsets;   // n_seg+1 (device)
    const double* anchors;        // n_seg (device)
    const int64_t* source_lengths;// n_seg (device)
    const int64_t* out_offsets;   // n_seg (device): first output index of each segment
    int64_t n_seg, N;
    int32_t layout;
    uint64_t k;
    const double* centers;        // 2k (device)
    const double* mean_lengths;   // k (device)
    double scl, sigma_len, sigma_inc;
    bool drop_local_last;         // distributed stitched fit: this rank is not the last
};
// Writes reconstructed samples into d_out. Throws on unknown_symbol /
// invalid_piece exactly where the reference throws.
void inverse_transform_device(const InverseIn& in, double* d_out, cudaStream_t st);

}  // namespace jb
