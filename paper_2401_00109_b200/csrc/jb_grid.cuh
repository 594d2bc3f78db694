// jb_grid.cuh — exact candidate grid for nearest-center queries.
//
// A uniform G x G grid over the points' bounding box. Every cell stores, in
// index order, the centers that can be the reference's nearest center
// (clustering.hpp:146-157: rounded dx*dx+dy*dy, strict <, lowest index) for
// SOME point of the cell's slightly inflated box. A center c is dropped only if
//     dmin2(c, box) > M * (1 + 1e-12),   M = min over centers of dmax2(., box);
// then for every point p of the box, with D the exact squared distance,
//     D(p,c) >= dmin2/(1+4u) > M(1+1e-12)/(1+4u) >= D(p,c*)(1+1e-12)/(1+4u)^2
// and the rounded distances (relative error <= 4u, u = 2^-53) satisfy
// d(p,c) > d(p,c*): c is neither the argmin nor a lower-index tie. Looping
// over the candidates in index order with strict < is therefore exactly the
// reference's loop over all centers. Cells with more than `cap` candidates
// fall back to all centers.
#pragma once

#include <cmath>

#include "jb_common.cuh"

namespace jb {

struct CandGrid {
    double x0, y0, w, h, invw, invh, mw, mh;
    int G, cap;
    uint16_t* cnt;   // G*G; 0xFFFF = use all centers
    uint16_t* cand;  // G*G*cap
};

__host__ inline CandGrid make_grid_desc(double xmin, double xmax, double ymin, double ymax,
                                        int G, int cap) {
    CandGrid g{};
    g.G = G;
    g.cap = cap;
    const double wx = xmax - xmin, wy = ymax - ymin;
    g.x0 = xmin;
    g.y0 = ymin;
    g.w = wx > 0 ? wx / G : 1.0;
    g.h = wy > 0 ? wy / G : 1.0;
    g.invw = 1.0 / g.w;
    g.invh = 1.0 / g.h;
    // inflation covers the rounding of the cell index and of the box corners
    g.mw = g.w * 1e-9 + 1e-15 * (std::fabs(xmin) + std::fabs(xmax));
    g.mh = g.h * 1e-9 + 1e-15 * (std::fabs(ymin) + std::fabs(ymax));
    return g;
}

__device__ __forceinline__ void grid_box_d2(double cx, double cy, double bx0, double bx1,
                                            double by0, double by1, double& dmin2,
                                            double& dmax2) {
    const double ex = fmax(fmax(bx0 - cx, cx - bx1), 0.0);
    const double ey = fmax(fmax(by0 - cy, cy - by1), 0.0);
    dmin2 = ex * ex + ey * ey;
    const double fx = fmax(fabs(bx0 - cx), fabs(bx1 - cx));
    const double fy = fmax(fabs(by0 - cy), fabs(by1 - cy));
    dmax2 = fx * fx + fy * fy;
}

// Candidate lists of a block of cells (one CTA): the centers kept for the
// block's bounding box, then every cell filtered against that short list.
// Exactly the flat per-cell result: for a cell box b inside the block box B
// (B's edges are the SAME rounded expressions as the edge cells' edges, and
// rounding is monotone), dmin2(c,b) >= dmin2(c,B) and M_b <= M_B, so a center
// dropped for B is dropped for b; and the argmin of dmax2(., b) is never
// dropped for B (dmax2(c*,b) = M_b <= M_B < dmin2(c*,B) <= dmax2(c*,b) would
// follow), so M over the short list is M_b.
constexpr int kBuildTB = 256;
constexpr int kBuildList = 512;  // block candidates kept in smem (else: all centers)

struct BlockCands {
    uint16_t list[kBuildList];
    int n;
    int wc[kBuildTB / 32];
    double wmin[kBuildTB / 32];
};

// Keep threshold on dmin2. slack > 0 keeps, in addition, every center that
// could become a candidate after the centers move by up to slack / 2 each:
// c is dropped only if dmin(c) > sqrt(M) + slack, so after moves of at most
// D = slack / 2, dmin'(c) >= dmin(c) - D > sqrt(M) + D >= sqrt(M') and c is
// still not a candidate (M' <= (sqrt(M) + D)^2). The (1 + 1e-12) factors
// cover the rounding of sqrt, the sum and the square. slack = 0: the exact
// rule of the header comment.
__device__ __forceinline__ double keep_threshold(double M, double slack) {
    if (slack <= 0.0) return M * (1.0 + 1e-12) + 1e-300;
    const double r = sqrt(M) * (1.0 + 1e-12) + slack;
    return r * r * (1.0 + 1e-12) + 1e-300;
}

// block-wide: s.list/s.n := centers kept for box (bx0,bx1,by0,by1), index order
__device__ inline void block_candidates(BlockCands& s, const double* centers, int k,
                                        double bx0, double bx1, double by0, double by1,
                                        double slack = 0.0) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double M = INFINITY;
    for (int c = threadIdx.x; c < k; c += kBuildTB) {
        double dmn, dmx;
        grid_box_d2(centers[2 * c], centers[2 * c + 1], bx0, bx1, by0, by1, dmn, dmx);
        M = fmin(M, dmx);
    }
    for (int o = 16; o > 0; o >>= 1) M = fmin(M, __shfl_xor_sync(0xffffffffu, M, o));
    if (lane == 0) s.wmin[warp] = M;
    if (threadIdx.x == 0) s.n = 0;
    __syncthreads();
    M = s.wmin[0];
    for (int w = 1; w < kBuildTB / 32; ++w) M = fmin(M, s.wmin[w]);
    const double thr = keep_threshold(M, slack);
    for (int c0 = 0; c0 < k; c0 += kBuildTB) {
        const int c = c0 + threadIdx.x;
        bool keep = false;
        if (c < k) {
            double dmn, dmx;
            grid_box_d2(centers[2 * c], centers[2 * c + 1], bx0, bx1, by0, by1, dmn, dmx);
            keep = dmn <= thr;
        }
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) s.wc[warp] = __popc(m);
        __syncthreads();
        int off = s.n;
        for (int w = 0; w < warp; ++w) off += s.wc[w];
        off += __popc(m & ((1u << lane) - 1u));
        if (keep && off < kBuildList) s.list[off] = (uint16_t)c;
        __syncthreads();
        if (threadIdx.x == 0)
            for (int w = 0; w < kBuildTB / 32; ++w) s.n += s.wc[w];
        __syncthreads();
    }
}

constexpr int kGridBlock = 16;  // cells per block side: one thread per cell

// thread-wide candidate filter of one cell box over the block list (or all k
// centers); writes up to cap indices in index order, returns the full count
__device__ __forceinline__ int thread_cell_candidates(const double* centers, int k,
                                                      const BlockCands& s, double bx0, double bx1,
                                                      double by0, double by1, uint16_t* out,
                                                      int cap, double slack = 0.0) {
    const bool all = s.n > kBuildList;
    const int m = all ? k : s.n;
    double M = INFINITY;
    for (int j = 0; j < m; ++j) {
        const int c = all ? j : s.list[j];
        double dmn, dmx;
        grid_box_d2(centers[2 * c], centers[2 * c + 1], bx0, bx1, by0, by1, dmn, dmx);
        M = fmin(M, dmx);
    }
    const double thr = keep_threshold(M, slack);
    int nc = 0;
    for (int j = 0; j < m; ++j) {
        const int c = all ? j : s.list[j];
        double dmn, dmx;
        grid_box_d2(centers[2 * c], centers[2 * c + 1], bx0, bx1, by0, by1, dmn, dmx);
        if (dmn <= thr) {
            if (nc < cap) out[nc] = (uint16_t)c;
            ++nc;
        }
    }
    return nc;
}

// one CTA per kGridBlock x kGridBlock block of cells, one thread per cell
static __global__ void __launch_bounds__(kBuildTB) k_grid_build(CandGrid g,
                                                                const double* centers,
                                                                int k) {
    __shared__ BlockCands s;
    extern __shared__ double s_centers[];  // 2k: every cell test reads them
    for (int q = threadIdx.x; q < 2 * k; q += blockDim.x) s_centers[q] = centers[q];
    __syncthreads();
    centers = s_centers;
    const int Gb = (g.G + kGridBlock - 1) / kGridBlock;
    for (int blk = blockIdx.x; blk < Gb * Gb; blk += gridDim.x) {
        const int ix0 = (blk % Gb) * kGridBlock, iy0 = (blk / Gb) * kGridBlock;
        const int ix1 = min(ix0 + kGridBlock, g.G) - 1, iy1 = min(iy0 + kGridBlock, g.G) - 1;
        block_candidates(s, centers, k, g.x0 + ix0 * g.w - g.mw, g.x0 + (ix1 + 1) * g.w + g.mw,
                         g.y0 + iy0 * g.h - g.mh, g.y0 + (iy1 + 1) * g.h + g.mh);
        const int ix = ix0 + (int)threadIdx.x % kGridBlock, iy = iy0 + (int)threadIdx.x / kGridBlock;
        if (ix <= ix1 && iy <= iy1) {
            const int cell = iy * g.G + ix;
            const int nc = thread_cell_candidates(
                centers, k, s, g.x0 + ix * g.w - g.mw, g.x0 + (ix + 1) * g.w + g.mw,
                g.y0 + iy * g.h - g.mh, g.y0 + (iy + 1) * g.h + g.mh,
                g.cand + (size_t)cell * g.cap, g.cap);
            g.cnt[cell] = nc <= g.cap ? (uint16_t)nc : (uint16_t)0xFFFF;
        }
        __syncthreads();
    }
}

inline void launch_grid_build(const CandGrid& g, const double* centers, int k, cudaStream_t st) {
    const int Gb = (g.G + kGridBlock - 1) / kGridBlock;
    k_grid_build<<<Gb * Gb, kBuildTB, sizeof(double) * 2 * k, st>>>(g, centers, k);
}

// nearest_center (clustering.hpp:146-157) through the grid; cx/cy in smem
__device__ __forceinline__ uint32_t grid_nearest(const CandGrid& g, double px, double py,
                                                 const double* cx, const double* cy, int k) {
    int n = 0xFFFF, cell = 0;  // G == 0: no grid, every center
    if (g.G > 0) {
        int ix = (int)((px - g.x0) * g.invw);
        int iy = (int)((py - g.y0) * g.invh);
        ix = min(max(ix, 0), g.G - 1);
        iy = min(max(iy, 0), g.G - 1);
        cell = iy * g.G + ix;
        n = __ldg(g.cnt + cell);
    }
    uint32_t best = 0;
    double bd = __longlong_as_double(0x7FF0000000000000LL);  // +inf
    if (n == 0xFFFF) {
        for (int c = 0; c < k; ++c) {
            const double d = dist2(px, py, cx[c], cy[c]);
            if (d < bd) {
                bd = d;
                best = (uint32_t)c;
            }
        }
        return best;
    }
    const uint16_t* cl = g.cand + (size_t)cell * g.cap;
    for (int j = 0; j < n; ++j) {
        const uint32_t c = __ldg(cl + j);
        const double d = dist2(px, py, cx[c], cy[c]);
        if (d < bd) {
            bd = d;
            best = c;
        }
    }
    return best;
}

inline int grid_side_for(uint64_t k) {
    int G = 64;
    while (G < 256 && (double)G * G < 256.0 * (double)k) G <<= 1;
    return G;
}

}  // namespace jb
