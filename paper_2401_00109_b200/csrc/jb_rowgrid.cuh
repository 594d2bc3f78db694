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
// pieces and overflowing cells fall back to the 2-D grid.
#pragma once

#include "jb_grid.cuh"

namespace jb {

constexpr uint64_t kRowOverflow = 0xFFFEull;  // low half-word of an overflowing cell
constexpr uint64_t kRowEmpty = 0xFFFFull;     // unused candidate slot

struct RowGrid {
    double y0, h, invh, mh;  // y cells (same inflation rule as CandGrid)
    double scl, sl;          // x_l = scl * (double)l / sl  (k_scale's expression)
    int R, Gy;               // lengths 1..R, Gy cells per length
    uint64_t* cell;          // R * Gy packed candidate words
};

__host__ inline RowGrid make_row_grid_desc(double ymin, double ymax, double scl, double sl,
                                           int32_t max_len, int64_t cell_budget) {
    RowGrid g{};
    g.R = (int)std::max<int64_t>(1, std::min<int64_t>(max_len, 256));
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
    return g;
}

__device__ __forceinline__ double row_x(const RowGrid& g, int l) {
    return __ddiv_rn(__dmul_rn(g.scl, (double)l), g.sl);  // == k_scale: scl * (double)L / sl
}

// one warp per cell
static __global__ void k_row_grid_build(RowGrid g, const double* __restrict__ centers, int k) {
    const int lane = threadIdx.x & 31;
    const int64_t ncell = (int64_t)g.R * g.Gy;
    for (int64_t cell = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; cell < ncell;
         cell += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int row = (int)(cell / g.Gy), iy = (int)(cell % g.Gy);
        const double x = row_x(g, row + 1);
        const double by0 = g.y0 + iy * g.h - g.mh, by1 = g.y0 + (iy + 1) * g.h + g.mh;
        double M = INFINITY;
        for (int c = lane; c < k; c += 32) {
            double dmn, dmx;
            grid_box_d2(centers[2 * c], centers[2 * c + 1], x, x, by0, by1, dmn, dmx);
            M = fmin(M, dmx);
        }
        for (int o = 16; o > 0; o >>= 1) M = fmin(M, __shfl_xor_sync(0xffffffffu, M, o));
        const double thr = M * (1.0 + 1e-12) + 1e-300;
        int nc = 0;
        uint64_t word = ~0ull;  // all slots empty
        for (int c0 = 0; c0 < k && nc <= 4; c0 += 32) {
            const int c = c0 + lane;
            bool keep = false;
            if (c < k) {
                double dmn, dmx;
                grid_box_d2(centers[2 * c], centers[2 * c + 1], x, x, by0, by1, dmn, dmx);
                keep = dmn <= thr;
            }
            unsigned m = __ballot_sync(0xffffffffu, keep);
            while (m && nc < 5) {
                const int l = __ffs(m) - 1;
                m &= m - 1;
                if (nc < 4) {
                    word &= ~(0xFFFFull << (16 * nc));
                    word |= (uint64_t)(c0 + l) << (16 * nc);
                }
                ++nc;
            }
        }
        if (nc > 4) word = (~0ull << 16) | kRowOverflow;
        if (lane == 0) g.cell[cell] = word;
    }
}

// nearest_center (clustering.hpp:146-157) of a piece of length len at (px, py)
__device__ __forceinline__ uint32_t row_nearest(const RowGrid& rg, const CandGrid& g, int32_t len,
                                                double px, double py, const double* cx,
                                                const double* cy, int k) {
    if (len >= 1 && len <= rg.R) {
        int iy = (int)((py - rg.y0) * rg.invh);
        iy = min(max(iy, 0), rg.Gy - 1);
        const uint64_t w = __ldg(reinterpret_cast<const unsigned long long*>(rg.cell) +
                                 (size_t)(len - 1) * rg.Gy + iy);
        const uint32_t c0 = (uint32_t)(w & 0xFFFF);
        if (c0 != kRowOverflow) {
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
    }
    return grid_nearest(g, px, py, cx, cy, k);
}

}  // namespace jb
