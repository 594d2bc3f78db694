/*
 * jabba_b200.h — C ABI of the B200-native JABBA fit_transform / inverse_transform
 * path (libjabba_b200.so). Plain pointers and sizes only; no CUDA or torch
 * types cross this boundary.
 *
 * Reference interfaces replaced (paths relative to
 * /root/reference/proj/include/jabba/):
 *   jb_fit_transform      <- jabba::jabba_fit(const Dataset&, JabbaConfig)   jabba.hpp:30-36
 *                            (= partitional_compress compression.hpp:167-193
 *                               + digitize digitization.hpp:207-293)
 *   jb_inverse_transform  <- jabba::reconstruct(const SymbolicResult&)        inverse.hpp:127-132
 *   jb_fit_inverse_transform  same, on a device-resident fit (no host copy)
 *   jb_symbolize_with     <- jabba::symbolize_with(const Codebook&, const PieceSequence&)
 *                                                                             digitization.hpp:297-307
 *   jb_plan_segments      <- Dataset::partitioned/multivariate/collection     core.hpp:73-98
 *                            + detail::split_series                           compression.hpp:140-160
 *   jb_config             <- JabbaConfig jabba.hpp:17-21, CompressionConfig compression.hpp:18-26,
 *                            DigitizeConfig digitization.hpp:110-117, VQConfig clustering.hpp:19-32,
 *                            GAConfig clustering.hpp:36-48, AutoDigitizeConfig digitization.hpp:77-83
 *   jb_status             <- jabba::error hierarchy                           core.hpp:20-30
 *
 * Threading: every call is reentrant per context; a context owns one CUDA
 * stream and must not be used from two threads at once without external
 * locking. Different contexts may run concurrently.
 */
#ifndef JABBA_B200_H
#define JABBA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define JB_ABI_VERSION 1

typedef enum {
    JB_OK = 0,
    JB_INVALID_INPUT = 1,     /* jabba::invalid_input */
    JB_INVALID_PIECE = 2,     /* jabba::invalid_piece */
    JB_INVALID_PARTITION = 3, /* jabba::invalid_partition */
    JB_UNKNOWN_SYMBOL = 4,    /* jabba::unknown_symbol */
    JB_PARSE_ERROR = 5,       /* jabba::parse_error (reserved: no parsing on this path) */
    JB_LAYOUT_ERROR = 6,      /* jabba::layout_error */
    JB_VERSION_ERROR = 7,     /* jabba::version_error (reserved) */
    JB_CUDA_ERROR = 100,
    JB_NCCL_ERROR = 101,
    JB_NO_DEVICE = 102,
    JB_INTERNAL = 103
} jb_status;

typedef enum { /* core.hpp:55 */
    JB_LAYOUT_UNIVARIATE_PARTITIONED = 0,
    JB_LAYOUT_MULTIVARIATE = 1,
    JB_LAYOUT_COLLECTION = 2
} jb_layout;

typedef enum { /* digitization.hpp:88 */
    JB_BACKEND_VQ = 0,
    JB_BACKEND_SVQ = 1,
    JB_BACKEND_GA = 2,
    JB_BACKEND_GA_AUTO = 3,
    JB_BACKEND_GA_HIER = 4
} jb_backend;

typedef enum { /* clustering.hpp:34 */
    JB_SORT_FIRST_PRINCIPAL_COMPONENT = 0,
    JB_SORT_TWO_NORM = 1
} jb_sort_key;

typedef struct {
    double tol;            /* CompressionConfig::tol (> 0) */
    int64_t max_piece_len; /* CompressionConfig::max_piece_len (0 = unbounded) */
    int32_t backend;       /* jb_backend */
    double scl;            /* DigitizeConfig::scl (>= 0) */
    uint64_t k;            /* VQConfig::k */
    double r;              /* VQConfig::r, sampling ratio in (0,1] */
    uint64_t max_iters;    /* VQConfig::max_iters */
    uint64_t n_init;       /* VQConfig::n_init */
    uint64_t seed;         /* VQConfig::seed (std::mt19937_64 stream) */
    double alpha;          /* GAConfig::alpha */
    int32_t sort_key;      /* jb_sort_key */
    int32_t early_stop;    /* GAConfig::early_stop */
    int32_t has_alpha_len; /* GAConfig::alpha_len present */
    double alpha_len;
    int32_t has_alpha_inc; /* GAConfig::alpha_inc present */
    double alpha_inc;
    double eta;            /* AutoDigitizeConfig::eta */
    uint32_t threads;      /* JabbaConfig::threads (accepted; the GPU path ignores it) */
} jb_config;

/* The reference's defaults (compression.hpp:19-20, digitization.hpp:111-112,
 * clustering.hpp:20-24,37-39, digitization.hpp:78, jabba.hpp:20). */
void jb_config_default(jb_config* cfg);

typedef struct jb_context jb_context;
typedef struct jb_fit jb_fit;

int jb_abi_version(void);
/* thread-local message of the last failing call */
const char* jb_last_error(void);

/* Create a context on CUDA device `device` (owns a stream). */
jb_status jb_context_create(int device, jb_context** out);
void jb_context_destroy(jb_context* ctx);

/* Segment table for a dataset of n_series concatenated series with the given
 * lengths (samples). layout semantics as Dataset (core.hpp:73-98); `parts`
 * splits every series with split_series semantics (compression.hpp:140-160):
 * univariate-partitioned needs exactly one series; collection/multivariate
 * with parts == 1 use one segment per series (the reference's own layouts),
 * parts > 1 is the multi-series x partitions extension (configs 2 and 5).
 * seg_first/seg_steps need room for n_series * max(parts,1) entries. */
jb_status jb_plan_segments(const int64_t* series_lengths, int64_t n_series, int32_t layout,
                           int64_t parts, int64_t* seg_first, int64_t* seg_steps,
                           int64_t* n_seg_out);

/* fit_transform == jabba_fit. `values` holds every sample of every series;
 * segment s covers values[seg_first[s] .. seg_first[s] + seg_steps[s]]
 * (inclusive; split segments share their boundary sample).
 * values_on_device != 0: `values` is a device pointer on the context's GPU
 * (no H2D copy); otherwise a host pointer (copied, pinned if registered). */
jb_status jb_fit_transform(jb_context* ctx, const double* values, int64_t n_values,
                           int32_t values_on_device, const int64_t* seg_first,
                           const int64_t* seg_steps, int64_t n_seg, int32_t layout,
                           const jb_config* cfg, jb_fit** out);
void jb_fit_free(jb_fit* fit);

/* sizes */
int64_t jb_fit_n_segments(const jb_fit* fit);
int64_t jb_fit_n_pieces(const jb_fit* fit);
uint64_t jb_fit_k(const jb_fit* fit);
int32_t jb_fit_layout(const jb_fit* fit);
/* number of samples jb_fit_inverse_transform / jb_inverse_transform write */
int64_t jb_fit_reconstruct_size(const jb_fit* fit);

/* copy-outs (host buffers). CompressedBatch: per-segment piece offsets
 * (n_seg+1), lens, incs. SymbolicResult: ranked labels per piece, codebook
 * centers (2k, scaled space, ranked order), mean_lengths (k), scaling
 * {scl, sigma_len, sigma_inc}, per-segment anchors and source lengths.
 * Any pointer may be NULL to skip that array. */
jb_status jb_fit_copy_pieces(const jb_fit* fit, int64_t* piece_offsets, int64_t* len,
                             double* inc);
jb_status jb_fit_copy_symbolic(const jb_fit* fit, uint32_t* labels, double* centers,
                               double* mean_lengths, double* scaling, double* anchors,
                               int64_t* source_lengths);
/* diagnostics: Lloyd iterations, sample size, engine draws consumed,
 * compression fix-up rounds, GA decision rounds, per-phase milliseconds
 * (compress, scale, backend, stats, total) */
jb_status jb_fit_stats(const jb_fit* fit, uint64_t* iterations, uint64_t* sample_size,
                       uint64_t* draws, int32_t* fix_rounds, int32_t* ga_rounds,
                       double* phase_ms /* 8: 5 phases, Lloyd tiles processed, labels changed,
                                          D^2 tiles updated */);

/* inverse_transform on the device-resident fit. out_values: host
 * (out_on_device == 0) or device pointer with jb_fit_reconstruct_size()
 * entries; per-output-series offsets in out_offsets (n_out+1; n_out = 1 for
 * univariate-partitioned, n_seg otherwise), may be NULL. */
jb_status jb_fit_inverse_transform(jb_context* ctx, const jb_fit* fit, double* out_values,
                                   int32_t out_on_device, int64_t* out_offsets);

/* inverse_transform == reconstruct on a host SymbolicResult. */
int64_t jb_reconstruct_size(const int64_t* source_lengths, int64_t n_seg, int32_t layout);
jb_status jb_inverse_transform(jb_context* ctx, const double* centers,
                               const double* mean_lengths, uint64_t k, const double* scaling,
                               const uint32_t* labels, const int64_t* piece_offsets,
                               const double* anchors, const int64_t* source_lengths,
                               int64_t n_seg, int32_t layout, double* out_values);

/* symbolize_with: labels of n held-out pieces (len, inc) against a codebook
 * (centers 2k interleaved, scaling {scl, sigma_len, sigma_inc}):
 * Codebook::nearest(ScalingParams::apply(piece)), lowest index on ties
 * (core.hpp:130-132, 147-160). pieces_on_device != 0: len/inc/labels are
 * device pointers on the context's GPU; else host pointers. k == 0 ->
 * JB_INVALID_INPUT ("symbolize_with: empty codebook"). */
jb_status jb_symbolize_with(jb_context* ctx, const double* centers, uint64_t k,
                            const double* scaling, const int64_t* len, const double* inc,
                            int64_t n, int32_t pieces_on_device, uint32_t* labels);

/* ---- Joint fit sharded over ranks (one process per GPU) -----------------
 * Every rank passes ITS contiguous range of the global segment table (and a
 * values buffer covering it). Compression, scaling, the final assignment and
 * the inverse are local; the exchanges are tiny and exact (piece counts,
 * 128-bit fixed-point partial sums, D^2 partial sums / picks, Lloyd cluster
 * deltas, group statistics), so every rank ends with the same codebook and
 * labels bit-identical to the single-GPU fit. The only collective needed is
 * an allgather of host bytes, supplied by the caller (NCCL or gloo through
 * torch.distributed in the Python mirror). Returns a fit holding this rank's
 * segments; jb_fit_inverse_transform reconstructs them (a univariate-
 * partitioned fit drops the last sample of every rank but the last). */
typedef struct {
    void* user;
    int32_t rank, world;
    /* gather `bytes` from every rank into recv (world * bytes, rank order);
       return 0 on success */
    int32_t (*allgather)(void* user, const void* send, uint64_t bytes, void* recv);
} jb_comm;

jb_status jb_fit_transform_dist(jb_context* ctx, const jb_comm* comm, const double* values,
                                int64_t n_values, int32_t values_on_device,
                                const int64_t* seg_first, const int64_t* seg_steps,
                                int64_t n_seg_local, int64_t n_seg_global, int32_t layout,
                                const jb_config* cfg, jb_fit** out);

/* Kernel-level CUDA-event profiler: when enabled, every launch of the hot
 * kernels is bracketed by events on its stream. jb_profile_read fills up to
 * `cap` records (names: 64 bytes each) and returns the number of kernels. */
void jb_profile_enable(int32_t on);
void jb_profile_reset(void);
int32_t jb_profile_read(char* names, double* total_ms, int64_t* launches, int32_t cap);

/* Measured fp64 DFMA throughput of `device` in TFLOP/s (2 flops per DFMA):
 * the roofline denominator for fp64-bound kernels. */
jb_status jb_probe_fp64_tflops(int device, double* tflops);

/* Building blocks, exposed for parity tests against the reference's RNG use:
 * the first `count` draws of std::mt19937_64(seed) generated on the device
 * (multi-CTA jump-ahead), and detail::sample_indices (clustering.hpp:74-85)
 * resolved on the device. Host output buffers. */
jb_status jb_mt19937_64_stream(jb_context* ctx, uint64_t seed, uint64_t count, uint64_t* out);
jb_status jb_sample_indices(jb_context* ctx, uint64_t n, uint64_t sample_size, uint64_t seed,
                            uint64_t* out);

/* jabba::kmeans (clustering.hpp:224-236) on 2-D points (host, interleaved
 * x,y): D^2 seeding, Lloyd iterations and restarts on the device with the
 * reference's RNG stream; labels (n), centers (2k), iterations of the best run. */
jb_status jb_kmeans(jb_context* ctx, const double* points, int64_t n, uint64_t k,
                    uint64_t max_iters, uint64_t n_init, uint64_t seed, uint32_t* labels,
                    double* centers, uint64_t* iterations);

/* The reference's left-to-right fp64 accumulation `s += w` from s = 0 of
 * non-negative terms (scale_pieces var_len digitization.hpp:39-45, group sums
 * :224-231), reproduced bit-exactly by the parallel emulation the fit uses
 * (seqsum.cu): out[g] = sequential sum of terms[seg_off[g] .. seg_off[g+1]).
 * Terms must be >= 0 (the result is exact for any finite non-negative input). */
jb_status jb_seq_sum_nonneg(jb_context* ctx, const double* terms, const int64_t* seg_off,
                            int64_t n_seg, double* out);

/* jabba::mse (metrics.hpp:18-29) on the GPU, bit-exact: the reference's
 * left-to-right sum of (a_i - b_i)^2 (the same emulation as
 * jb_seq_sum_nonneg) divided by n. on_device != 0: a and b are device
 * pointers on the context's GPU; else host pointers. n == 0 ->
 * JB_INVALID_INPUT. */
jb_status jb_mse(jb_context* ctx, const double* a, const double* b, int64_t n, int32_t on_device,
                 double* out);

/* symbol token of cluster rank r in an alphabet of size k (core.hpp:186-193);
 * writes a NUL-terminated string into buf (>= 24 bytes); returns its length */
int32_t jb_symbol_token(uint64_t rank, uint64_t alphabet_size, char* buf);

#ifdef __cplusplus
}
#endif
#endif /* JABBA_B200_H */
