// jb_rowgrid.cuh — exact nearest-center lookup for JABBA's scaled pieces.
//
// A piece's x coordinate is scl * len / sigma_len with an INTEGER len
// (digitization.hpp:97-106), so the points lie on vertical lines x_l, one per
// piece length; at config 4 ~99% of the pieces have len <= 2. The row grid
// keeps, for every length l <= R and every y cell of a fine 1-D grid, the
// candidate centers of the degenerate box {x_l} x [cell y range] under the
// same min-max pruning as jb_grid.cuh (proof there). x_l is computed by the
// very expression k_scale uses, so a point of length l lies on x_l exactly.
// A cell packs up to 4 candidate indices (ascending) in one 64-bit word; a
// cell with ONE candidate decides the label without any arithmetic. Longer
// pieces, overflowing cells (low half-word 0xFFFE) and cells not built (all
// ones: a built cell always holds >= 1 candidate) fall back to the 2-D grid.
#pragma once

#include "jb_grid.cuh"

namespace jb {

constexpr uint64_t kRowSpill = 0xFFFDull;     // low half-word of a spilled cell (5..kSpill)
constexpr uint64_t kRowOverflow = 0xFFFEull;  // low half-word of an overflowing cell
constexpr uint64_t kRowEmpty = 0xFFFFull;     // unused candidate slot
// A cell with 5..kSpill candidates keeps them in spill[cell * kSpill ..] and
// its word holds (kRowSpill | count << 16 | cell << 32): dense clusters of
// centers (config 5, k = 500 around the short rows) would otherwise send
// whole cells to the all-centers fallback.
constexpr int kSpill = 16;

struct RowGrid {
    double y0, h, invh, mh;  // y cells (same inflation rule as CandGrid)
    double scl, sl;          // x_l = scl * (double)l / sl  (k_scale's expression)
    int R, Gy;               // lengths 1..R, Gy cells per length
    uint64_t* cell;          // R * Gy packed candidate words
    uint16_t* spill;         // R * Gy * kSpill, or null (no spilling: overflow)
    double slack;            // build slack (jb_grid.cuh keep_threshold): valid while
                             // every center stays within slack / 2 of its build position
};

__host__ inline RowGrid make_row_grid_desc(double ymin, double ymax, double scl, double sl,
                                           int32_t max_len, int64_t cell_budget,
                                           int32_t max_rows = 256) {
    RowGrid g{};
    g.R = (int)std::max<int64_t>(1, std::min<int64_t>(max_len, max_rows));
    int64_t gy = 256;
    while (gy < 16384 && gy * 2 * g.R <= cell_budget) gy *= 2;
    g.Gy = (int)gy;
    const double wy = ymax - ymin;
    g.y0 = ymin;
    g.h = wy > 0 ? wy / g.Gy : 1.0;
    g.invh = 1.0 / g.h;
    g.mh = g.h * 1e-9 + 1e-15 * (std::fabs(ymin) + std::fabs(ymax));
    g.scl = scl;
    g.sl = sl;
    g.cell = nullptr;
    g.spill = nullptr;
    g.slack = 0.0;
    return g;
}

__device__ __forceinline__ double row_x(const RowGrid& g, int l) {
    return __ddiv_rn(__dmul_rn(g.scl, (double)l), g.sl);  // == k_scale: scl * (double)L / sl
}

constexpr int kRowSeg = kBuildTB;  // y cells per CTA block, one thread per cell

// one CTA per (length, kRowSeg y cells) segment; blocks: the segments to
// build (null: all of them)
__device__ __forceinline__ void row_grid_build_body(RowGrid g,
                                                                    const double* centers,
                                                                    int k, const int* __restrict__ blocks,
                                                                    int nblocks) {
    __shared__ BlockCands s;
    extern __shared__ double s_centers[];  // 2k: every cell test reads them
    for (int q = threadIdx.x; q < 2 * k; q += blockDim.x) s_centers[q] = centers[q];
    __syncthreads();
    centers = s_centers;
    const int nseg = (g.Gy + kRowSeg - 1) / kRowSeg;
    for (int bi = blockIdx.x; bi < nblocks; bi += gridDim.x) {
        const int blk = blocks ? blocks[bi] : bi;
        const int row = blk / nseg, iy0 = (blk % nseg) * kRowSeg;
        const int iy1 = min(iy0 + kRowSeg, g.Gy) - 1;
        const double x = row_x(g, row + 1);
        block_candidates(s, centers, k, x, x, g.y0 + iy0 * g.h - g.mh, g.y0 + (iy1 + 1) * g.h + g.mh,
                         g.slack);
        const int iy = iy0 + (int)threadIdx.x;
        if (iy <= iy1) {
            uint16_t tmp[kSpill];
            const int nc = thread_cell_candidates(centers, k, s, x, x, g.y0 + iy * g.h - g.mh,
                                                  g.y0 + (iy + 1) * g.h + g.mh, tmp, kSpill,
                                                  g.slack);
            const size_t cidx = (size_t)row * g.Gy + iy;
            uint64_t word;
            if (nc > 4 && nc <= kSpill && g.spill) {
                for (int j = 0; j < nc; ++j) g.spill[cidx * kSpill + j] = tmp[j];
                word = kRowSpill | ((uint64_t)nc << 16) | ((uint64_t)cidx << 32);
            } else if (nc > 4) {
                word = (~0ull << 16) | kRowOverflow;
            } else {
                word = ~0ull;
                for (int j = 0; j < nc; ++j) {
                    word &= ~(0xFFFFull << (16 * j));
                    word |= (uint64_t)tmp[j] << (16 * j);
                }
            }
            g.cell[cidx] = word;
        }
        __syncthreads();
    }
}

static __global__ void __launch_bounds__(kBuildTB) k_row_grid_build(RowGrid g,
                                                                    const double* centers,
                                                                    int k, const int* __restrict__ blocks,
                                                                    int nblocks) {
    row_grid_build_body(g, centers, k, blocks, nblocks);
}

inline int row_grid_segments(const RowGrid& g) { return g.R * ((g.Gy + kRowSeg - 1) / kRowSeg); }

inline void launch_row_grid_build(const RowGrid& g, const double* centers, int k, cudaStream_t st,
                                  const int* blocks = nullptr, int nblocks = -1) {
    if (nblocks < 0) nblocks = row_grid_segments(g);
    if (nblocks > 0)
        k_row_grid_build<<<nblocks, kBuildTB, sizeof(double) * 2 * k, st>>>(g, centers, k, blocks,
                                                                          nblocks);
}

// segments holding at least one point (length l <= R, y) -> flags[segment] = 1
static __global__ void k_row_occupancy(RowGrid g, const double2* __restrict__ pts,
                                       const int32_t* __restrict__ len, int64_t n,
                                       int* __restrict__ flags) {
    const int nseg = (g.Gy + kRowSeg - 1) / kRowSeg;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int l = len[i];
        if (l < 1 || l > g.R) continue;
        int iy = (int)((pts[i].y - g.y0) * g.invh);
        iy = min(max(iy, 0), g.Gy - 1);
        const int f = (l - 1) * nseg + iy / kRowSeg;
        if (!flags[f]) flags[f] = 1;
    }
}

// nearest center from an already loaded row-cell word (~0: no row cell)
__device__ __forceinline__ uint32_t row_nearest_w(const CandGrid& g, const uint16_t* spill,
                                                  uint64_t w, double px, double py,
                                                  const double* cx, const double* cy, int k);

__device__ __forceinline__ uint32_t row_pick(uint64_t w, const CandGrid& g, const uint16_t* spill,
                                             double px, double py, const double* cx,
                                             const double* cy, int k) {
    const uint32_t c0 = (uint32_t)(w & 0xFFFF);
    if (c0 == kRowSpill) return row_nearest_w(g, spill, w, px, py, cx, cy, k);
    if (c0 < kRowSpill) {
        uint32_t best = c0;
        const uint32_t c1 = (uint32_t)((w >> 16) & 0xFFFF);
        if (c1 == kRowEmpty) return best;  // the only possible argmin
        double bd = dist2(px, py, cx[c0], cy[c0]);
#pragma unroll
        for (int j = 1; j < 4; ++j) {
            const uint32_t c = (uint32_t)((w >> (16 * j)) & 0xFFFF);
            if (c == kRowEmpty) break;
            const double d = dist2(px, py, cx[c], cy[c]);
            if (d < bd) {
                bd = d;
                best = c;
            }
        }
        return best;
    }
    return grid_nearest(g, px, py, cx, cy, k);
}

// candidates of a built cell word: 1..4 inline, 5..kSpill spilled, 0 otherwise
__device__ __forceinline__ int row_word_count(uint64_t w) {
    const uint64_t c0 = w & 0xFFFF;
    if (c0 == kRowSpill) return (int)((w >> 16) & 0xFFFF);
    if (c0 >= kRowOverflow) return 0;
    int n = 1;
    while (n < 4 && ((w >> (16 * n)) & 0xFFFF) != kRowEmpty) ++n;
    return n;
}
__device__ __forceinline__ uint32_t row_word_cand(const uint16_t* spill, uint64_t w, int j) {
    if ((w & 0xFFFF) == kRowSpill) return __ldcg(spill + (size_t)(w >> 32) * kSpill + j);
    return (uint32_t)((w >> (16 * j)) & 0xFFFF);
}

// the row-cell word of a piece of length len at y = py (~0: no row cell,
// which row_nearest_w sends to the 2-D grid fallback). RO: the grid is
// read-only for the whole kernel, so the word may come through L1 (the final
// assignment); otherwise (grids rebuilt inside a persistent kernel) L2 only.
template <bool RO = false>
__device__ __forceinline__ uint64_t row_cell_word(const RowGrid& rg, int32_t len, double py) {
    if (len < 1 || len > rg.R) return ~0ull;
    int iy = (int)((py - rg.y0) * rg.invh);
    iy = min(max(iy, 0), rg.Gy - 1);
    const unsigned long long* w =
        reinterpret_cast<const unsigned long long*>(rg.cell) + (size_t)(len - 1) * rg.Gy + iy;
    return RO ? __ldg(w) : __ldcg(w);
}

// nearest_center (clustering.hpp:146-157) of a piece at (px, py) whose row
// cell word w was loaded ahead (row_cell_word)
__device__ __forceinline__ uint32_t row_nearest_w(const CandGrid& g, const uint16_t* spill,
                                                  uint64_t w, double px, double py,
                                                  const double* cx, const double* cy, int k) {
    const uint32_t c0 = (uint32_t)(w & 0xFFFF);
    if (c0 == kRowSpill) {
        const uint16_t* sl = spill + (size_t)(w >> 32) * kSpill;
        const int nc = (int)((w >> 16) & 0xFFFF);
        uint32_t best = __ldcg(sl);
        double bd = dist2(px, py, cx[best], cy[best]);
        for (int j = 1; j < nc; ++j) {
            const uint32_t c = __ldcg(sl + j);
            const double d = dist2(px, py, cx[c], cy[c]);
            if (d < bd) {
                bd = d;
                best = c;
            }
        }
        return best;
    }
    if (c0 < kRowSpill) {
        uint32_t best = c0;
        const uint32_t c1 = (uint32_t)((w >> 16) & 0xFFFF);
        if (c1 == kRowEmpty) return best;  // the only possible argmin
        double bd = dist2(px, py, cx[c0], cy[c0]);
#pragma unroll
        for (int j = 1; j < 4; ++j) {
            const uint32_t c = (uint32_t)((w >> (16 * j)) & 0xFFFF);
            if (c == kRowEmpty) break;
            const double d = dist2(px, py, cx[c], cy[c]);
            if (d < bd) {
                bd = d;
                best = c;
            }
        }
        return best;
    }
    return grid_nearest(g, px, py, cx, cy, k);
}

// nearest_center (clustering.hpp:146-157) of a piece of length len at (px, py)
__device__ __forceinline__ uint32_t row_nearest(const RowGrid& rg, const CandGrid& g, int32_t len,
                                                double px, double py, const double* cx,
                                                const double* cy, int k) {
    return row_nearest_w(g, rg.spill, row_cell_word(rg, len, py), px, py, cx, cy, k);
}

}  // namespace jb
