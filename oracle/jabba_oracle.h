/*
 * jabba_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference JABBA fit + inverse path
 * (/root/reference/proj/include/jabba/*.hpp), used exclusively as the
 * parity checker by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs. Nothing in the product library
 * (paper_2401_00109_b200/) links, calls or loads this code.
 *
 * Parity pinning: validated against (1) the reference's own known-answer
 * tests (tests/golden/*.json, see tests/test_oracle_golden.py) and (2) the
 * real reference headers compiled into oracle/_ref/libjabba_ref.so by
 * oracle/Makefile (tests/test_oracle_vs_ref.py).
 *
 * The flat argument conventions are identical to include/jabba_b200.h so the
 * same test vectors drive the oracle, the compiled reference and the GPU path.
 */
#ifndef JABBA_ORACLE_H
#define JABBA_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes: same numbering as jb_status in include/jabba_b200.h */
enum {
    JO_OK = 0,
    JO_INVALID_INPUT = 1,
    JO_INVALID_PIECE = 2,
    JO_INVALID_PARTITION = 3,
    JO_UNKNOWN_SYMBOL = 4,
    JO_LAYOUT_ERROR = 6,
    JO_INTERNAL = 103
};

/* mirrors jb_config (include/jabba_b200.h) field for field */
typedef struct {
    double tol;
    int64_t max_piece_len;
    int32_t backend; /* 0 vq, 1 svq, 2 ga, 3 ga-auto, 4 ga-hier */
    double scl;
    uint64_t k;
    double r;
    uint64_t max_iters;
    uint64_t n_init;
    uint64_t seed;
    double alpha;
    int32_t sort_key; /* 0 first principal component, 1 two-norm */
    int32_t early_stop;
    int32_t has_alpha_len;
    double alpha_len;
    int32_t has_alpha_inc;
    double alpha_inc;
    double eta;
    uint32_t threads;
} jo_config;

typedef struct {
    int64_t n_seg;
    int64_t n_pieces;
    int64_t* piece_offsets; /* n_seg + 1 */
    int64_t* piece_len;     /* n_pieces */
    double* piece_inc;      /* n_pieces */
    double* anchors;        /* n_seg */
    int64_t* source_lengths;/* n_seg */
    uint64_t k;
    double* centers;        /* 2k, ranked order */
    double* mean_lengths;   /* k */
    double scaling[3];      /* scl, sigma_len, sigma_inc */
    uint32_t* labels;       /* n_pieces, ranked ids */
    /* diagnostics */
    uint64_t iterations;    /* Lloyd iterations of the selected run (vq/svq) */
    uint64_t sample_size;
} jo_fit_result;

const char* jo_last_error(void);

/* segment planning: split_series / partitional_compress validation
 * (compression.hpp:140-193). layout: 0 univariate-partitioned, 1 multivariate,
 * 2 collection. parts: partitions per series. */
int jo_plan_segments(const int64_t* series_lengths, int64_t n_series, int32_t layout,
                     int64_t parts, int64_t* seg_first, int64_t* seg_steps,
                     int64_t* n_seg_out);

/* jabba_fit (jabba.hpp:30-36): compress every segment, digitize jointly */
int jo_fit(const double* values, const int64_t* seg_first, const int64_t* seg_steps,
           int64_t n_seg, const jo_config* cfg, jo_fit_result* out);
void jo_fit_free(jo_fit_result* r);

/* compression only (compression.hpp:70-83 per segment) */
int jo_compress(const double* values, const int64_t* seg_first, const int64_t* seg_steps,
                int64_t n_seg, double tol, int64_t max_piece_len, int64_t* piece_offsets,
                int64_t** piece_len, double** piece_inc);

/* reconstruct (inverse.hpp:127-132). Output: univariate-partitioned ->
 * stitched single series of sum(steps)+1 values; else per-segment
 * (steps+1) values concatenated. out_values must hold jo_reconstruct_size(). */
/* symbolize_with (digitization.hpp:297-307) of n pieces against a codebook */
int jo_symbolize_with(const double* centers, uint64_t k, const double* scaling,
                      const int64_t* len, const double* inc, int64_t n, uint32_t* labels);
int64_t jo_reconstruct_size(const int64_t* source_lengths, int64_t n_seg, int32_t layout);
int jo_reconstruct(const double* centers, const double* mean_lengths, uint64_t k,
                   const double* scaling, const uint32_t* labels, const int64_t* piece_offsets,
                   const double* anchors, const int64_t* source_lengths, int64_t n_seg,
                   int32_t layout, double* out_values);

/* building blocks exposed for known-answer tests */
void jo_quantize_lengths(const double* real_lens, int64_t n, int64_t* out);
int jo_match_total_length(int64_t* lens, int64_t n, int64_t target);
double jo_auto_alpha(int64_t n, int64_t N, double tol, double eta, int* status);
int jo_inverse_compress(const int64_t* len, const double* inc, int64_t n, double anchor,
                        double* out);
int jo_greedy_aggregate(const double* pts, int64_t n, double alpha, int32_t sort_key,
                        int32_t early_stop, uint32_t* labels, int64_t* n_groups,
                        int64_t* starting_points);
int jo_kmeans(const double* pts, int64_t n, uint64_t k, uint64_t max_iters, uint64_t n_init,
              uint64_t seed, uint32_t* labels, double* centers, uint64_t* iterations);
int jo_sample_indices(uint64_t n, uint64_t sample_size, uint64_t seed, uint64_t* out);

/* libstdc++ RNG restatement (exposed so tests can pin it against std::) */
void jo_mt_stream(uint64_t seed, uint64_t count, uint64_t* out);
uint64_t jo_uniform_int_stream(uint64_t seed, uint64_t lo, uint64_t hi, uint64_t count,
                               uint64_t* out);
void jo_uniform_real_stream(uint64_t seed, double lo, double hi, uint64_t count, double* out);

#ifdef __cplusplus
}
#endif
#endif
