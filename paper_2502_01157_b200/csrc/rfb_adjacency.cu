// rfb_adjacency.cu -- Delaunay adjacency (the CSR the walk consumes) on the
// GPU, by per-site Voronoi cell clipping.
//
// Replaces geometry/delaunay.py:445-520 `build` (incremental Bowyer-Watson,
// exact predicates) + geometry/adjacency.py:46-64 `from_triangulation`
// (symmetrised, ascending CSR, hull flags).  Two sites are Delaunay
// neighbours iff their Voronoi cells share a face, so each site's neighbour
// list is read off its own Voronoi cell:
//
//  * one warp per site; the cell is a convex polytope kept in shared memory
//    in dual form -- a list of triangles (a, b, c) of plane indices, one per
//    polytope vertex, each with its fp64 coordinates relative to the site
//    (Ray, Sokolov, Lefebvre, Levy 2018, "Meshless Voronoi on the GPU");
//  * it starts as a box of half-width B = 1e6 x (bbox diagonal) and is
//    clipped by the bisector plane  n.x <= |n|^2/2,  n = x_j - x_i, of every
//    candidate site j: vertices beyond the plane are removed, the boundary
//    edges (u->v) of the removed triangles (edges whose reverse is not also
//    removed) each become a new triangle (u, v, P);
//  * candidates come from a uniform grid in increasing-distance order (a
//    precomputed table of cell offsets sorted by their minimum distance, then
//    Chebyshev rings to the grid's edge); a site x_j can only cut the cell
//    if |x_j - x_i| < 2 R, R = the farthest vertex, so the search stops at
//    the first batch whose lower bound reaches 2 R (security radius);
//  * neighbours = sites whose planes carry at least one final vertex, sorted
//    ascending; hull sites (unbounded cells) are those whose final cell
//    still touches the box.
// The union of the per-site lists is taken (a missing reverse edge is
// added), offsets are an exclusive scan of the degrees.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <vector>

#include "../../include/rfb.h"

namespace rfb_adj {

constexpr unsigned kFull = 0xffffffffu;
#ifndef RFB_ADJ_WARPS
#define RFB_ADJ_WARPS 2
#endif
#ifndef RFB_ADJ_MAX_PLANES
#define RFB_ADJ_MAX_PLANES 80
#endif
constexpr int kWarps = RFB_ADJ_WARPS;            // sites (warps) per block
constexpr int kMaxPlanes = RFB_ADJ_MAX_PLANES;   // pass-1 planes per cell, box included
#ifndef RFB_ADJ_MAX_VERTS
#define RFB_ADJ_MAX_VERTS 128
#endif
constexpr int kMaxVerts = RFB_ADJ_MAX_VERTS;  // polytope vertices (dual triangles)
#ifndef RFB_ADJ_CELL_SITES
#define RFB_ADJ_CELL_SITES 2.0  // mean sites per grid cell over the bounding box
#endif
#ifndef RFB_ADJ_SPIRAL_G
#define RFB_ADJ_SPIRAL_G 5
#endif
constexpr int kSpiralG = RFB_ADJ_SPIRAL_G;  // spiral table covers offsets |d|_inf <= G
constexpr int kSpiralN = (2 * kSpiralG + 1) * (2 * kSpiralG + 1) * (2 * kSpiralG + 1);

enum : int { kErrNone = 0, kErrOverflow = 1, kErrDuplicate = 2, kErrDegenerate = 4 };

// One cell under construction (shared memory).  Pass 1 uses the small
// buffer; cells that outgrow it (transiently long cells at the boundary of a
// dense region) restart in pass 2 with the large one.
template <int MP, int MV>
struct CellBuf {
    static constexpr int kPlanes = MP, kVerts = MV;
    double nx[MP], ny[MP], nz[MP], no[MP];
    double vx[MV], vy[MV], vz[MV];
    int32_t pid[MP];       // site id, or -1 for the box planes
    uint32_t tri[MV];      // a | b << 8 | c << 16
    uint16_t edge[3 * MV];
    uint32_t rmask[MV / 32];
    uint8_t used[MP];
    uint8_t pmap[MP];
};
using WarpCell = CellBuf<kMaxPlanes, kMaxVerts>;
using BigCell = CellBuf<255, 1024>;

struct Grid {
    double lo[3];
    double h;       // cubic cell edge
    int dim[3];
};

struct Args {
    const double4 *pos;      // [n] grid-sorted {x, y, z, 0}
    const int32_t *ids;      // [n] original id of sorted site k
    const int32_t *cstart;   // [ncell + 1] first sorted index of each cell
    const int4 *spiral;      // [kSpiralN] {dx, dy, dz, lb^2 in units of h^2 (as int)}
    int64_t n;
    Grid g;
    double box;              // box half-width B
    double dup2;             // duplicate tolerance squared
    int32_t cap;             // per-site row capacity
    int32_t *rows;           // [n][cap] by original id
    int32_t *deg;            // [n]
    uint8_t *hull;           // [n]
    int32_t *tail;           // [n] sorted indices of sites queued for pass 2
    float *tail_key;         // [n] their cell extent after the spiral (schedule key)
    int32_t *tail_next;      // pass-2 work counter
    int32_t *flags;          // [0]: OR of errors, [1]: sites queued for pass 2,
                             // [2]: max vertices, [3]: max planes used
};

// Warp-uniform summary of the current cell (local coordinates).
struct CellState {
    int nv, np, err;
    double R2;               // max |v|^2
    double lo[3], hi[3];     // vertex bounding box
};

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ int cell_index(const Grid &g, int ix, int iy, int iz) {
    return (iz * g.dim[1] + iy) * g.dim[0] + ix;
}

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// vertex = intersection of planes a, b, c (local coordinates)
template <class Cell>
__device__ __forceinline__ bool vertex_of(const Cell &C, int a, int b, int c, double pnx,
                                          double pny, double pnz, double po, double &x, double &y,
                                          double &z) {
    // c may be the plane being added (passed in registers, c < 0)
    const double ax = C.nx[a], ay = C.ny[a], az = C.nz[a], ao = C.no[a];
    const double bx = C.nx[b], by = C.ny[b], bz = C.nz[b], bo = C.no[b];
    double cx, cy, cz, co;
    if (c < 0) {
        cx = pnx; cy = pny; cz = pnz; co = po;
    } else {
        cx = C.nx[c]; cy = C.ny[c]; cz = C.nz[c]; co = C.no[c];
    }
    const double bcx = by * cz - bz * cy, bcy = bz * cx - bx * cz, bcz = bx * cy - by * cx;
    const double cax = cy * az - cz * ay, cay = cz * ax - cx * az, caz = cx * ay - cy * ax;
    const double abx = ay * bz - az * by, aby = az * bx - ax * bz, abz = ax * by - ay * bx;
    const double det = ax * bcx + ay * bcy + az * bcz;
    if (det == 0.0) return false;
    x = (ao * bcx + bo * cax + co * abx) / det;
    y = (ao * bcy + bo * cay + co * aby) / det;
    z = (ao * bcz + bo * caz + co * abz) / det;
    return true;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = fmax(v, __shfl_xor_sync(kFull, v, off));
    return v;
}

// Drop planes no triangle references (full-scan cells clip many transient planes).
template <class Cell>
__device__ void compact_planes(Cell &C, int lane, int nv, int &np) {
    for (int p = lane; p < np; p += 32) C.used[p] = 0;
    __syncwarp();
    for (int v = lane; v < nv; v += 32) {
        const uint32_t t = C.tri[v];
        C.used[t & 255] = 1;
        C.used[(t >> 8) & 255] = 1;
        C.used[(t >> 16) & 255] = 1;
    }
    __syncwarp();
    int kept = 0;
    for (int base = 0; base < np; base += 32) {
        const int p = base + lane;
        const bool keep = p < np && C.used[p];
        const unsigned kb = __ballot_sync(kFull, keep);
        double a = 0, b = 0, c = 0, d = 0;
        int32_t id = 0;
        if (keep) {
            a = C.nx[p]; b = C.ny[p]; c = C.nz[p]; d = C.no[p]; id = C.pid[p];
        }
        __syncwarp();
        if (keep) {
            const int dst = kept + __popc(kb & lanemask_lt());
            C.nx[dst] = a; C.ny[dst] = b; C.nz[dst] = c; C.no[dst] = d; C.pid[dst] = id;
            C.pmap[p] = (uint8_t)dst;
        }
        kept += __popc(kb);
        __syncwarp();
    }
    for (int v = lane; v < nv; v += 32) {
        const uint32_t t = C.tri[v];
        C.tri[v] = (uint32_t)C.pmap[t & 255] | ((uint32_t)C.pmap[(t >> 8) & 255] << 8) |
                   ((uint32_t)C.pmap[(t >> 16) & 255] << 16);
    }
    np = kept;
    __syncwarp();
}

// Clip the cell by n.x <= o (plane of site j).  Returns false on overflow /
// degeneracy (err set).
template <class Cell>
__device__ bool clip(Cell &C, int lane, double pnx, double pny, double pnz, double po,
                     int32_t j, CellState &S) {
    int &nv = S.nv, &np = S.np, &err = S.err;
    int nrem = 0;
    bool on = false;
    for (int base = 0; base < nv; base += 32) {
        const int v = base + lane;
        bool rem = false;
        if (v < nv) {
            const double d = pnx * C.vx[v] + pny * C.vy[v] + pnz * C.vz[v];
            rem = d > po;
            on |= d == po;
        }
        const unsigned b = __ballot_sync(kFull, rem);
        if (lane == 0) C.rmask[base >> 5] = b;
        nrem += __popc(b);
    }
    // a vertex exactly on the new plane: five or more cospherical sites (e.g. a lattice),
    // which the reference resolves by symbolic perturbation -- outside this builder's scope
    if (__any_sync(kFull, on)) {
        err |= kErrDegenerate;
        return false;
    }
    if (nrem == 0) return true;
    __syncwarp();
    if (np == Cell::kPlanes) compact_planes(C, lane, nv, np);
    if (np == Cell::kPlanes) {
        err |= kErrOverflow;
        return false;
    }
    const int P = np++;
    if (lane == 0) {
        C.nx[P] = pnx; C.ny[P] = pny; C.nz[P] = pnz; C.no[P] = po; C.pid[P] = j;
    }
    // removed triangles -> their directed edges
    int r0 = 0;
    for (int base = 0; base < nv; base += 32) {
        const unsigned b = C.rmask[base >> 5];
        const int v = base + lane;
        if ((b >> lane) & 1u) {
            const int r = r0 + __popc(b & lanemask_lt());
            const uint32_t t = C.tri[v];
            const uint32_t a = t & 255, bb = (t >> 8) & 255, c = (t >> 16) & 255;
            C.edge[3 * r] = (uint16_t)(a | (bb << 8));
            C.edge[3 * r + 1] = (uint16_t)(bb | (c << 8));
            C.edge[3 * r + 2] = (uint16_t)(c | (a << 8));
        }
        r0 += __popc(b);
    }
    __syncwarp();
    // compact the kept triangles in place
    int kept = 0;
    for (int base = 0; base < nv; base += 32) {
        const int v = base + lane;
        const bool keep = v < nv && !((C.rmask[base >> 5] >> lane) & 1u);
        const unsigned kb = __ballot_sync(kFull, keep);
        uint32_t t = 0;
        double x = 0, y = 0, z = 0;
        if (keep) {
            t = C.tri[v]; x = C.vx[v]; y = C.vy[v]; z = C.vz[v];
        }
        __syncwarp();
        if (keep) {
            const int d = kept + __popc(kb & lanemask_lt());
            C.tri[d] = t; C.vx[d] = x; C.vy[d] = y; C.vz[d] = z;
        }
        kept += __popc(kb);
        __syncwarp();
    }
    // boundary edges (reverse not removed) -> new triangles (u, v, P)
    const int ne = 3 * nrem;
    int nvn = kept;
    bool bad = false;
    for (int e0 = 0; e0 < ne; e0 += 32) {
        const int e = e0 + lane;
        bool bnd = false;
        uint32_t ed = 0;
        if (e < ne) {
            ed = C.edge[e];
            const uint16_t rev = (uint16_t)((ed >> 8) | ((ed & 255) << 8));
            bnd = true;
            for (int k = 0; k < ne; ++k)
                if (C.edge[k] == rev) {
                    bnd = false;
                    break;
                }
        }
        const unsigned bm = __ballot_sync(kFull, bnd);
        if (bnd) {
            const int d = nvn + __popc(bm & lanemask_lt());
            if (d < Cell::kVerts) {
                const int u = ed & 255, w = ed >> 8;
                double x, y, z;
                if (!vertex_of(C, u, w, -1, pnx, pny, pnz, po, x, y, z)) bad = true;
                C.tri[d] = (uint32_t)u | ((uint32_t)w << 8) | ((uint32_t)P << 16);
                C.vx[d] = x; C.vy[d] = y; C.vz[d] = z;
            }
        }
        nvn += __popc(bm);
    }
    if (__any_sync(kFull, bad)) err |= kErrDegenerate;
    if (nvn > Cell::kVerts) {
        err |= kErrOverflow;
        return false;
    }
    nv = nvn;
    __syncwarp();
    double m = 0.0, l0 = INFINITY, l1 = INFINITY, l2 = INFINITY, h0 = -INFINITY, h1 = -INFINITY,
           h2 = -INFINITY;
    for (int v = lane; v < nv; v += 32) {
        const double x = C.vx[v], y = C.vy[v], z = C.vz[v];
        m = fmax(m, x * x + y * y + z * z);
        l0 = fmin(l0, x); l1 = fmin(l1, y); l2 = fmin(l2, z);
        h0 = fmax(h0, x); h1 = fmax(h1, y); h2 = fmax(h2, z);
    }
    S.R2 = warp_max(m);
    S.lo[0] = -warp_max(-l0); S.lo[1] = -warp_max(-l1); S.lo[2] = -warp_max(-l2);
    S.hi[0] = warp_max(h0); S.hi[1] = warp_max(h1); S.hi[2] = warp_max(h2);
    return true;
}

// Offer the points of `cell` (lane-private, may be -1) to the clipper.
#ifndef RFB_ADJ_FLAT
#define RFB_ADJ_FLAT 1  // sparse spiral batches scanned as one flat candidate list (1M: 71 -> 66 ms)
#endif
#ifndef RFB_ADJ_FLAT_MAX
#define RFB_ADJ_FLAT_MAX 128  // candidates per batch up to which the flat order is used
#endif
constexpr int kFlatMax = RFB_ADJ_FLAT_MAX;
#ifndef RFB_ADJ_SORTED
#define RFB_ADJ_SORTED 1  // pass 1: offer a batch's candidates nearest first
#endif
#ifndef RFB_ADJ_PROFILE
#define RFB_ADJ_PROFILE 0  // count candidate clip tests per phase into stats[5..6]
#endif
// Necessary condition for site p (local coordinates) to cut the cell: some
// vertex v has p.v > |p|^2/2; bounded by the vertex box's support function
// (with a relative slack far above fp64 rounding, so the filter never
// rejects a candidate the exact clip test would act on).
__device__ __forceinline__ bool may_cut(const CellState &S, double dx, double dy, double dz,
                                        double d2) {
    if (!(d2 < 4.0 * S.R2 * (1.0 + 1e-12))) return false;
    const double sup = (dx > 0.0 ? dx * S.hi[0] : dx * S.lo[0]) +
                       (dy > 0.0 ? dy * S.hi[1] : dy * S.lo[1]) +
                       (dz > 0.0 ? dz * S.hi[2] : dz * S.lo[2]);
    return sup * (1.0 + 1e-12) > 0.5 * d2;
}

template <class Cell>
__device__ __forceinline__ void offer_cells(const Args &A, Cell &C, int lane, int cell,
                                            double sx, double sy, double sz, int32_t self,
                                            CellState &S, int phase) {
    int c0 = 0, c1 = 0;
    if (cell >= 0) {
        c0 = __ldg(A.cstart + cell);
        c1 = __ldg(A.cstart + cell + 1);
    }
    int cnt = c1 - c0;
    // Sparse batches (uniform scenes: ~2 sites per grid cell) are scanned as one flat list,
    // 32 candidates per round (inclusive warp scan of the counts; each lane finds the cell
    // owning its flat index by binary search over the prefix sums), instead of max-per-cell
    // rounds with most lanes idle.  Dense batches (the 3M surface shell: ~60 per cell) keep
    // the round-robin order -- one site of every cell per round, a spatially spread sample
    // that shrinks the cell fastest (flat order there is 2.3x slower).
    int incl = cnt, maxcnt = cnt;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int o = __shfl_up_sync(kFull, incl, off);
        if (lane >= off) incl += o;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) maxcnt = max(maxcnt, __shfl_xor_sync(kFull, maxcnt, off));
    const int total = __shfl_sync(kFull, incl, 31);
    const int excl = incl - cnt;
    const bool flat = RFB_ADJ_FLAT && total <= kFlatMax;
    const int rounds = flat ? (total + 31) / 32 : maxcnt;
    for (int q = 0; q < rounds; ++q) {
        bool has;
        int idx;
        if (flat) {
            const int t = q * 32 + lane;
            int lo = 0;  // owner = first lane whose inclusive prefix exceeds t
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const int probe = __shfl_sync(kFull, incl, lo + step - 1);
                if (probe <= t) lo += step;
            }
            const int oc0 = __shfl_sync(kFull, c0, lo & 31), oex = __shfl_sync(kFull, excl, lo & 31);
            has = t < total;
            idx = oc0 + (t - oex);
        } else {
            has = q < cnt;
            idx = c0 + q;
        }
        double dx = 0, dy = 0, dz = 0, d2 = 0;
        int32_t jid = -1;
        if (has) {
            const double4 p = A.pos[idx];
            jid = __ldg(A.ids + idx);
            dx = p.x - sx; dy = p.y - sy; dz = p.z - sz;
            d2 = dx * dx + dy * dy + dz * dz;
            has = jid != self && (d2 <= A.dup2 || may_cut(S, dx, dy, dz, d2));
        }
#if RFB_ADJ_SORTED
        // nearest candidate first: the cell shrinks fastest, so fewer later candidates
        // survive may_cut / cut anything
        bool pend = has;
        while (__any_sync(kFull, pend)) {
            double key = pend ? d2 : INFINITY;
            int L = lane;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const double ok = __shfl_xor_sync(kFull, key, off);
                const int oL = __shfl_xor_sync(kFull, L, off);
                if (ok < key || (ok == key && oL < L)) {
                    key = ok;
                    L = oL;
                }
            }
            if (lane == L) pend = false;
#else
        unsigned m = __ballot_sync(kFull, has);
        while (m) {
            const int L = __ffs(m) - 1;
            m &= m - 1;
#endif
            const double bx = __shfl_sync(kFull, dx, L), by = __shfl_sync(kFull, dy, L),
                         bz = __shfl_sync(kFull, dz, L), b2 = __shfl_sync(kFull, d2, L);
            const int32_t bj = __shfl_sync(kFull, jid, L);
            if (b2 <= A.dup2) {
                S.err |= kErrDuplicate;
                continue;
            }
            if (S.err == 0 && may_cut(S, bx, by, bz, b2)) {
#if RFB_ADJ_PROFILE
                if (lane == 0) atomicAdd(reinterpret_cast<unsigned long long *>(A.flags + 8) + phase, 1ull);
#endif
                clip(C, lane, bx, by, bz, 0.5 * b2, bj, S);
            }
        }
    }
}

template <class Cell>
__device__ void init_cell(Cell &C, int lane, double B, CellState &S) {
    // box: planes 0..5 = +x, -x, +y, -y, +z, -z at distance B
    if (lane < 6) {
        const double sgn = (lane & 1) ? -1.0 : 1.0;
        C.nx[lane] = lane / 2 == 0 ? 2.0 * B * sgn : 0.0;
        C.ny[lane] = lane / 2 == 1 ? 2.0 * B * sgn : 0.0;
        C.nz[lane] = lane / 2 == 2 ? 2.0 * B * sgn : 0.0;
        C.no[lane] = 2.0 * B * B;
        C.pid[lane] = -1;
    }
    if (lane < 8) {  // corner (sx, sy, sz): planes X, Y, Z oriented with det > 0
        const int bx = lane & 1, by = (lane >> 1) & 1, bz = (lane >> 2) & 1;
        const uint32_t px = bx, py = 2 + by, pz = 4 + bz;
        const bool neg = (bx + by + bz) & 1;  // det(sx ex, sy ey, sz ez) = sx sy sz
        C.tri[lane] = neg ? (py | (px << 8) | (pz << 16)) : (px | (py << 8) | (pz << 16));
        C.vx[lane] = bx ? -B : B;
        C.vy[lane] = by ? -B : B;
        C.vz[lane] = bz ? -B : B;
    }
    __syncwarp();
    S.nv = 8; S.np = 6; S.err = 0;
    S.R2 = 3.0 * B * B;
    for (int q = 0; q < 3; ++q) {
        S.lo[q] = -B;
        S.hi[q] = B;
    }
}

// Clip by the sites of the spiral table's cells, nearest first, until the
// security radius is reached.  Returns true when the cell is final.
// Does the box [l, h] (site-relative) meet a vertex ball B(v, |v|) of the cell?
// min over the box of |x - v|^2 - |v|^2 = sum_a (x_a^2 - 2 x_a v_a) at x_a = clamp(v_a);
// near-zero counts as meeting (conservative).
template <class Cell>
__device__ __forceinline__ bool box_meets_balls(const Cell &C, int nv, const double *l,
                                                const double *h) {
    for (int v = 0; v < nv; ++v) {
        const double w[3] = {C.vx[v], C.vy[v], C.vz[v]};
        double sum = 0.0, mag = 0.0;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const double xa = fmin(fmax(w[a], l[a]), h[a]);
            const double term = xa * xa - 2.0 * xa * w[a];
            sum += term;
            mag += fabs(term);
        }
        if (sum < 1e-12 * mag) return true;
    }
    return false;
}

template <class Cell>
__device__ bool spiral_phase(const Args &A, Cell &C, int lane, const double4 &s, int32_t self,
                             int ix, int iy, int iz, CellState &S) {
    const Grid &g = A.g;
    const double h2 = g.h * g.h;
    for (int s0 = 0; s0 < kSpiralN && S.err == 0; s0 += 32) {
        if ((double)__ldg(&A.spiral[s0].w) * h2 >= 4.0 * S.R2) return true;
        int cell = -1;
        if (s0 + lane < kSpiralN) {
            const int4 o = __ldg(A.spiral + s0 + lane);
            const int cx = ix + o.x, cy = iy + o.y, cz = iz + o.z;
            if (cx >= 0 && cy >= 0 && cz >= 0 && cx < g.dim[0] && cy < g.dim[1] && cz < g.dim[2])
                cell = cell_index(g, cx, cy, cz);
        }
        offer_cells(A, C, lane, cell, s.x, s.y, s.z, self, S, 0);
    }
    return false;
}

// neighbours: planes with at least one final vertex, ascending site id
template <class Cell>
__device__ void emit_site(const Args &A, Cell &C, int lane, int32_t self, const CellState &S) {
    const int nv = S.nv, np = S.np;
    int err = S.err;
    for (int p = lane; p < np; p += 32) C.used[p] = 0;
    __syncwarp();
    for (int v = lane; v < nv; v += 32) {
        const uint32_t t = C.tri[v];
        C.used[t & 255] = 1;
        C.used[(t >> 8) & 255] = 1;
        C.used[(t >> 16) & 255] = 1;
    }
    __syncwarp();
    int cnt = 0;
    bool on_hull = false;
    for (int base = 0; base < np; base += 32) {
        const int p = base + lane;
        const bool u = p < np && C.used[p];
        const bool site = u && C.pid[p] >= 0;
        cnt += __popc(__ballot_sync(kFull, site));
        on_hull |= __any_sync(kFull, u && C.pid[p] < 0);
    }
    if (cnt > A.cap) err |= kErrOverflow;
    int32_t *row = A.rows + (int64_t)self * A.cap;
    if (err == 0) {
        for (int p = lane; p < np; p += 32) {
            if (!C.used[p] || C.pid[p] < 0) continue;
            const int32_t id = C.pid[p];
            int rank = 0;
            for (int q = 0; q < np; ++q) rank += (C.used[q] && C.pid[q] >= 0 && C.pid[q] < id);
            row[rank] = id;
        }
    }
    if (lane == 0) {
        A.deg[self] = err == 0 ? cnt : 0;
        A.hull[self] = on_hull ? 1 : 0;
        if (err) atomicOr(A.flags, err);
        atomicMax(A.flags + 2, nv);
        atomicMax(A.flags + 3, np);
    }
    __syncwarp();
}

__device__ __forceinline__ void site_cell(const Grid &g, const double4 &s, int &ix, int &iy, int &iz) {
    ix = clampi((int)floor((s.x - g.lo[0]) / g.h), 0, g.dim[0] - 1);
    iy = clampi((int)floor((s.y - g.lo[1]) / g.h), 0, g.dim[1] - 1);
    iz = clampi((int)floor((s.z - g.lo[2]) / g.h), 0, g.dim[2] - 1);
}

// Pass 1: one warp per site, spiral only.  Cells not final after the
// spiral (near the hull: long or unbounded cells) are queued for pass 2.
#ifndef RFB_ADJ_MINB
#define RFB_ADJ_MINB 10  // 96 registers, 10 blocks (20 warps) per SM with the 128/80 buffers
#endif
__global__ void __launch_bounds__(32 * kWarps, RFB_ADJ_MINB) k_voronoi(Args A) {
    __shared__ WarpCell cells[kWarps];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WarpCell &C = cells[w];
    for (int64_t k = (int64_t)blockIdx.x * kWarps + w; k < A.n; k += (int64_t)gridDim.x * kWarps) {
        const double4 s = A.pos[k];
        const int32_t self = A.ids[k];
        CellState S;
        init_cell(C, lane, A.box, S);
        int ix, iy, iz;
        site_cell(A.g, s, ix, iy, iz);
        const bool done = spiral_phase(A, C, lane, s, self, ix, iy, iz, S);
        if ((done && S.err == 0) || (S.err & ~kErrOverflow)) {
            emit_site(A, C, lane, self, S);
        } else if (lane == 0) {  // not final after the spiral, or outgrew the buffer
            const int q = atomicAdd(A.flags + 1, 1);
            A.tail[q] = (int32_t)k;
            A.tail_key[q] = (float)S.R2;
        }
        __syncwarp();
    }
}

// Unbounded cells (their vertices on the box are "far") are what makes pass 2
// expensive: the far vertices' balls B(v, |v|) cover half-spaces, so the ball
// box spans the grid.  The few far vertices are kept apart; a site x (local
// coordinates) can cut the cell only if |x| < 2 Rn (Rn = farthest non-box
// vertex) or |x|^2 - 2 x.v < 0 for a far vertex v.
constexpr int kMaxFar = 32;
struct FarSet {
    double x[kMaxFar], y[kMaxFar], z[kMaxFar];
    double Rn2;  // max |v|^2 over vertices not on the box
    int n;       // far vertices, or -1 when there are too many (no pruning)
};

template <class Cell>
__device__ void far_refresh(const Cell &C, int lane, const CellState &S, FarSet &F,
                            int32_t *prof = nullptr) {
    double m = 0.0;
    int cnt = 0;
    for (int base = 0; base < S.nv; base += 32) {
        const int v = base + lane;
        bool far = false;
        double r2 = 0.0;
        if (v < S.nv) {
            const uint32_t t = C.tri[v];
            far = C.pid[t & 255] < 0 || C.pid[(t >> 8) & 255] < 0 || C.pid[(t >> 16) & 255] < 0;
            r2 = C.vx[v] * C.vx[v] + C.vy[v] * C.vy[v] + C.vz[v] * C.vz[v];
            if (!far) m = fmax(m, r2);
        }
        const unsigned fm = __ballot_sync(kFull, far);
        if (far) {
            const int slot = cnt + __popc(fm & lanemask_lt());
            if (slot < kMaxFar) {
                F.x[slot] = C.vx[v];
                F.y[slot] = C.vy[v];
                F.z[slot] = C.vz[v];
            }
        }
        cnt += __popc(fm);
    }
    m = warp_max(m);
    if (lane == 0) {
        F.Rn2 = m;
        F.n = cnt <= kMaxFar ? cnt : -1;
#if RFB_ADJ_PROFILE
        if (prof) atomicMax(prof, cnt);  // largest far-vertex count seen
#endif
    }
}

// Can any point of the local box [l, h] lie in some far ball?  (|x|^2 - 2 x.v
// minimised per axis at the box point nearest v; no |v|^2 is formed, so the
// huge radii cost no precision; the slack is relative.)
__device__ __forceinline__ bool box_meets_far(const FarSet &F, const double *l, const double *h) {
    for (int k = 0; k < F.n; ++k) {
        const double v[3] = {F.x[k], F.y[k], F.z[k]};
        double sum = 0.0, mag = 0.0;
        for (int a = 0; a < 3; ++a) {
            const double xa = fmin(fmax(v[a], l[a]), h[a]);
            const double term = xa * xa - 2.0 * xa * v[a];
            sum += term;
            mag += fabs(term);
        }
        if (sum < 1e-12 * mag) return true;
    }
    return false;
}

// Grid-cell bounds of the union of the vertex balls B(v, |v|) (warp 0).
template <class Cell>
__device__ void ball_box(const Cell &C, int lane, const CellState &S, const double4 &s,
                         const Grid &g, int *box) {
    double bl[3] = {INFINITY, INFINITY, INFINITY}, bh[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int v = lane; v < S.nv; v += 32) {
        const double x = C.vx[v], y = C.vy[v], z = C.vz[v];
        const double r = sqrt(x * x + y * y + z * z) * (1.0 + 1e-12);
        bl[0] = fmin(bl[0], x - r); bh[0] = fmax(bh[0], x + r);
        bl[1] = fmin(bl[1], y - r); bh[1] = fmax(bh[1], y + r);
        bl[2] = fmin(bl[2], z - r); bh[2] = fmax(bh[2], z + r);
    }
    const double sc[3] = {s.x, s.y, s.z};
    for (int q = 0; q < 3; ++q) {
        const double lo = -warp_max(-bl[q]) + sc[q], hi = warp_max(bh[q]) + sc[q];
        const double f0 = floor((lo - g.lo[q]) / g.h), f1 = floor((hi - g.lo[q]) / g.h);
        if (lane == 0) {
            box[q] = f0 < 0.0 ? 0 : (f0 > g.dim[q] - 1 ? g.dim[q] - 1 : (int)f0);
            box[3 + q] = f1 < 0.0 ? 0 : (f1 > g.dim[q] - 1 ? g.dim[q] - 1 : (int)f1);
        }
    }
}

// The part of Chebyshev ring r around (ix, iy, iz) inside the inclusive
// cell box `box` (lo xyz, hi xyz), as up to six face rectangles.
struct RingBox {
    int start[7];
    int fix[6];      // coordinate on the face's fixed axis
    int lo1[6], n1[6], lo2[6];
    __device__ int total() const { return start[6]; }
    __device__ void cell(int t, int &cx, int &cy, int &cz) const {
        int f = 0;
        while (t >= start[f + 1]) ++f;
        const int u = t - start[f], a = lo1[f] + u % n1[f], b = lo2[f] + u / n1[f];
        if (f < 2) { cx = fix[f]; cy = a; cz = b; }
        else if (f < 4) { cx = a; cy = fix[f]; cz = b; }
        else { cx = a; cy = b; cz = fix[f]; }
    }
};

__device__ __forceinline__ RingBox ring_box(int r, int ix, int iy, int iz, const int *box) {
    RingBox R;
    const int c[3] = {ix, iy, iz};
    int n = 0;
    for (int f = 0; f < 6; ++f) {
        const int ax = f >> 1, sgn = (f & 1) ? -1 : 1;
        const int fixv = c[ax] + sgn * r;
        // the two free axes; faces of lower axes own the shared edges
        const int a1 = ax == 0 ? 1 : 0, a2 = ax == 2 ? 1 : 2;
        const int s1 = a1 < ax ? r - 1 : r, s2 = a2 < ax ? r - 1 : r;
        const int l1 = max(c[a1] - s1, box[a1]), h1 = min(c[a1] + s1, box[3 + a1]);
        const int l2 = max(c[a2] - s2, box[a2]), h2 = min(c[a2] + s2, box[3 + a2]);
        const bool ok = fixv >= box[ax] && fixv <= box[3 + ax] && h1 >= l1 && h2 >= l2;
        R.start[f] = n;
        R.fix[f] = fixv;
        R.lo1[f] = l1;
        R.lo2[f] = l2;
        R.n1[f] = ok ? h1 - l1 + 1 : 1;
        n += ok ? (h1 - l1 + 1) * (h2 - l2 + 1) : 0;
    }
    R.start[6] = n;
    return R;
}

// Pass 2: one block per queued site.  Warp 0 rebuilds the cell (spiral)
// in the large buffer; if it is not final the whole block scans Chebyshev
// rings of grid cells outward, restricted to the grid-cell box of the
// vertex balls B(v, |v|) (every site that can still cut the cell lies in
// one of them).  Each thread tests its candidates exactly against the
// current vertices (p.v > |p|^2/2, the clip test); survivors are queued in
// shared memory and warp 0 clips by them.  After every ring the box and the
// security radius are refreshed, so a long cell that gets capped stops
// scanning early; unbounded (hull) cells scan to the grid's edge.
#ifndef RFB_ADJ_TAIL_THREADS
#define RFB_ADJ_TAIL_THREADS 128
#endif
constexpr int kTailThreads = RFB_ADJ_TAIL_THREADS;
constexpr int kTailQueue = 512;
#ifndef RFB_ADJ_COARSE
#define RFB_ADJ_COARSE 1  // pass 2 scans rings of CB^3-cell blocks pruned by the vertex balls
#endif
#ifndef RFB_ADJ_CB
#define RFB_ADJ_CB 4
#endif
constexpr int kCB = RFB_ADJ_CB;


#if RFB_ADJ_PROFILE
#define RFB_PC(i, v) do { if (A.hull[self]) atomicAdd(reinterpret_cast<unsigned long long *>(A.flags + 18 + 2 * (i)), (unsigned long long)(v)); } while (0)
#else
#define RFB_PC(i, v) ((void)0)
#endif
__global__ void __launch_bounds__(kTailThreads) k_voronoi_tail(Args A, int32_t count) {
    __shared__ BigCell C;
    __shared__ CellState SS;
    __shared__ bool fin;
    __shared__ int32_t queue[kTailQueue];
    __shared__ int qn, box[6];
    __shared__ FarSet far;
#if RFB_ADJ_COARSE
    __shared__ int live[kTailThreads], nlive;
#endif
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const Grid &g = A.g;
    const int rmax = max(max(g.dim[0], g.dim[1]), g.dim[2]);
    __shared__ int32_t s_item;
    for (;;) {
        // dynamic schedule over the queue, sorted by decreasing cell extent
        // (longest-processing-time first: the unbounded cells start first)
        if (tid == 0) s_item = atomicAdd(A.tail_next, 1);
        __syncthreads();
        const int32_t item = s_item;
        if (item >= count) break;
#if RFB_ADJ_PROFILE
        const long long clk0 = clock64();
#endif
        const int64_t k = A.tail[item];
        const double4 s = A.pos[k];
        const int32_t self = A.ids[k];
        int ix, iy, iz;
        site_cell(g, s, ix, iy, iz);
        if (warp == 0) {
            CellState S;
            init_cell(C, lane, A.box, S);
            const bool done = spiral_phase(A, C, lane, s, self, ix, iy, iz, S);
            ball_box(C, lane, S, s, g, box);
            far_refresh(C, lane, S, far, A.flags + 7);
            if (lane == 0) {
                fin = done || S.err != 0;
                SS = S;
                qn = 0;
            }
        }
        __syncthreads();
        // one grid cell's sites against the current cell (the exact clip test, or the far
        // vertices only beyond 2 Rn); survivors go to the shared queue
        auto scan_cell = [&](int cx, int cy, int cz, bool use_far) {
            const int cell = cell_index(g, cx, cy, cz);
            const int c0 = __ldg(A.cstart + cell), c1 = __ldg(A.cstart + cell + 1);
            RFB_PC(2, 1);
            RFB_PC(3, c1 - c0);
            for (int q = c0; q < c1; ++q) {
                const double4 p = A.pos[q];
                const double dx = p.x - s.x, dy = p.y - s.y, dz = p.z - s.z;
                const double d2 = dx * dx + dy * dy + dz * dz;
                if (d2 <= A.dup2) {
                    atomicOr(A.flags, kErrDuplicate);
                    continue;
                }
                if (!may_cut(SS, dx, dy, dz, d2)) continue;
                RFB_PC(4, 1);
                const double o = 0.5 * d2;
                bool cut = false;
                if (use_far && d2 >= 4.0 * far.Rn2 * (1.0 + 1e-9)) {
                    // beyond 2 Rn only the far vertices can be cut (conservative
                    // test; clip() decides exactly)
                    for (int k = 0; k < far.n && !cut; ++k) {
                        const double pv = dx * far.x[k] + dy * far.y[k] + dz * far.z[k];
                        cut = d2 - 2.0 * pv < 1e-12 * (d2 + 2.0 * fabs(pv));
                    }
                } else {
                    for (int v = 0; v < SS.nv && !cut; ++v)
                        cut = dx * C.vx[v] + dy * C.vy[v] + dz * C.vz[v] > o;
                }
                if (cut) {
                    const int slot = atomicAdd(&qn, 1);
                    if (slot < kTailQueue) queue[slot] = q;
                }
            }
        };
        // warp 0 clips by the queued sites (between two barriers); returns the queue length
        auto flush_queue = [&]() -> int {
            __syncthreads();
            const int nq = qn;
            if (nq > 0 && warp == 0) {
#if RFB_ADJ_PROFILE
                const long long cq0 = clock64();
#endif
                CellState S = SS;
                for (int i = 0; i < min(nq, kTailQueue) && S.err == 0; ++i) {
                    const int q = queue[i];
                    const double4 p = A.pos[q];
                    const double dx = p.x - s.x, dy = p.y - s.y, dz = p.z - s.z;
                    const double d2 = dx * dx + dy * dy + dz * dz;
                    if (may_cut(S, dx, dy, dz, d2))
                        clip(C, lane, dx, dy, dz, 0.5 * d2, __ldg(A.ids + q), S);
                }
                if (lane == 0) {
                    SS = S;
                    qn = 0;
                    RFB_PC(5, nq);
#if RFB_ADJ_PROFILE
                    RFB_PC(6, clock64() - cq0);
#endif
                }
            }
            __syncthreads();
            return nq;
        };
#if RFB_ADJ_COARSE
        // Rings of CB^3-cell blocks outward from the site's block, restricted to the ball
        // box.  A block (then each of its cells) is scanned only if its box meets a vertex
        // ball B(v, |v|) of the current cell -- the exact region from which a site can cut it
        // (x cuts iff |x - v| < |v| for some vertex v); the test against an earlier, larger
        // cell is conservative for every later one.  Unbounded hull cells thus skip the bulk
        // of the grid instead of testing every site against their vertices.
        {
            const int bx = ix / kCB, by = iy / kCB, bz = iz / kCB;
            const int rbmax = (rmax + kCB - 1) / kCB;
            // ring 0 (the site's own block) only holds cells beyond the spiral when
            // CB > kSpiralG + 1
            for (int R = kCB - 1 > kSpiralG ? 0 : 1; R <= rbmax && !fin; ++R) {
                // cells of block ring R >= 1 are >= (R-1) CB + 1 cells from the site's cell,
                // so their sites are >= (R-1) CB h away (ring 0: the site's own block, whose
                // cells beyond the spiral's reach are scanned too when CB > kSpiralG + 1)
                const double lb = (double)(max(R - 1, 0) * kCB) * g.h;
                if (lb * lb >= 4.0 * SS.R2 * (1.0 + 1e-12)) break;
                const int bbox[6] = {box[0] / kCB, box[1] / kCB, box[2] / kCB,
                                     box[3] / kCB, box[4] / kCB, box[5] / kCB};
                if (max(max(bx - bbox[0], bbox[3] - bx), max(max(by - bbox[1], bbox[4] - by),
                                                           max(bz - bbox[2], bbox[5] - bz))) < R)
                    break;
                const RingBox RB = ring_box(R, bx, by, bz, bbox);  // (ring_box lists r = 0 twice)
                const int total = R == 0 ? 1 : RB.total();
                if (tid == 0) { RFB_PC(0, 1); RFB_PC(1, (total + kTailThreads - 1) / kTailThreads); }
                for (int b0 = 0; b0 < total && SS.err == 0; b0 += kTailThreads) {
                    if (tid == 0) nlive = 0;
                    __syncthreads();
                    if (b0 + tid < total) {
                        int cbx = bx, cby = by, cbz = bz;
                        if (R > 0) RB.cell(b0 + tid, cbx, cby, cbz);
                        const double l[3] = {g.lo[0] + cbx * kCB * g.h - s.x,
                                             g.lo[1] + cby * kCB * g.h - s.y,
                                             g.lo[2] + cbz * kCB * g.h - s.z};
                        const double h[3] = {l[0] + kCB * g.h, l[1] + kCB * g.h, l[2] + kCB * g.h};
                        if (box_meets_balls(C, SS.nv, l, h))
                            live[atomicAdd(&nlive, 1)] = (cbz * 1024 + cby) * 1024 + cbx;
                    }
                    __syncthreads();
                    const bool use_far = far.n > 0;
                    const int items = nlive * kCB * kCB * kCB;
                    for (int t0 = 0; t0 < items && SS.err == 0; t0 += kTailThreads) {
                        const int t = t0 + tid;
                        if (t < items) {
                            const int bid = live[t / (kCB * kCB * kCB)], c = t % (kCB * kCB * kCB);
                            const int cx = (bid % 1024) * kCB + c % kCB;
                            const int cy = ((bid / 1024) % 1024) * kCB + (c / kCB) % kCB;
                            const int cz = (bid / (1024 * 1024)) * kCB + c / (kCB * kCB);
                            const int dch = max(max(abs(cx - ix), abs(cy - iy)), abs(cz - iz));
                            if (cx < g.dim[0] && cy < g.dim[1] && cz < g.dim[2] && dch > kSpiralG) {
                                const double l[3] = {g.lo[0] + cx * g.h - s.x,
                                                     g.lo[1] + cy * g.h - s.y,
                                                     g.lo[2] + cz * g.h - s.z};
                                const double h[3] = {l[0] + g.h, l[1] + g.h, l[2] + g.h};
                                if (box_meets_balls(C, SS.nv, l, h)) scan_cell(cx, cy, cz, use_far);
                            }
                        }
                        if (flush_queue() > kTailQueue) t0 -= kTailThreads;  // overflowed: again
                    }
                }
                if (warp == 0) {
                    ball_box(C, lane, SS, s, g, box);
                    far_refresh(C, lane, SS, far, A.flags + 7);
                }
                __syncthreads();
            }
        }
#else
        for (int r = kSpiralG + 1; r <= rmax && !fin; ++r) {
            // stop: remaining sites are >= (r-1) h away, beyond the security radius,
            // or the ring lies outside the ball box
            const double lb = (double)(r - 1) * g.h;
            if (lb * lb >= 4.0 * SS.R2 * (1.0 + 1e-12)) break;
            // with no far vertices Rn = R, and the line above is the security radius
            const bool use_far = far.n > 0;
            if (max(max(ix - box[0], box[3] - ix), max(max(iy - box[1], box[4] - iy),
                                                       max(iz - box[2], box[5] - iz))) < r)
                break;
            const RingBox RB = ring_box(r, ix, iy, iz, box);
            const int total = RB.total();
            if (tid == 0) { RFB_PC(0, 1); RFB_PC(1, (total + kTailThreads - 1) / kTailThreads); }
            for (int t0 = 0; t0 < total && SS.err == 0; t0 += kTailThreads) {
                const int t = t0 + tid;
                if (t < total) {
                    int cx, cy, cz;
                    RB.cell(t, cx, cy, cz);
                    bool live = true;
                    if (use_far) {  // cell box (local): beyond 2 Rn and outside every far ball?
                        const double l[3] = {g.lo[0] + cx * g.h - s.x, g.lo[1] + cy * g.h - s.y,
                                             g.lo[2] + cz * g.h - s.z};
                        const double h[3] = {l[0] + g.h, l[1] + g.h, l[2] + g.h};
                        double dmin2 = 0.0;
                        for (int a = 0; a < 3; ++a) {
                            const double da = l[a] > 0.0 ? l[a] : (h[a] < 0.0 ? -h[a] : 0.0);
                            dmin2 += da * da;
                        }
                        live = dmin2 < 4.0 * far.Rn2 * (1.0 + 1e-9) + 1e-300 ||
                               box_meets_far(far, l, h);
                    }
                    if (live) {
                        const int cell = cell_index(g, cx, cy, cz);
                        const int c0 = __ldg(A.cstart + cell), c1 = __ldg(A.cstart + cell + 1);
                        RFB_PC(2, 1);
                        RFB_PC(3, c1 - c0);
                        for (int q = c0; q < c1; ++q) {
                            const double4 p = A.pos[q];
                            const double dx = p.x - s.x, dy = p.y - s.y, dz = p.z - s.z;
                            const double d2 = dx * dx + dy * dy + dz * dz;
                            if (d2 <= A.dup2) {
                                atomicOr(A.flags, kErrDuplicate);
                                continue;
                            }
                            if (!may_cut(SS, dx, dy, dz, d2)) continue;
                            RFB_PC(4, 1);
                            const double o = 0.5 * d2;
                            bool cut = false;
                            if (use_far && d2 >= 4.0 * far.Rn2 * (1.0 + 1e-9)) {
                                // beyond 2 Rn only the far vertices can be cut (conservative
                                // test; clip() decides exactly)
                                for (int k = 0; k < far.n && !cut; ++k) {
                                    const double pv = dx * far.x[k] + dy * far.y[k] + dz * far.z[k];
                                    cut = d2 - 2.0 * pv < 1e-12 * (d2 + 2.0 * fabs(pv));
                                }
                            } else {
                                for (int v = 0; v < SS.nv && !cut; ++v)
                                    cut = dx * C.vx[v] + dy * C.vy[v] + dz * C.vz[v] > o;
                            }
                            if (cut) {
                                const int slot = atomicAdd(&qn, 1);
                                if (slot < kTailQueue) queue[slot] = q;
                            }
                        }
                    }
                }
                __syncthreads();
                const int nq = qn;
                if (nq > 0 && warp == 0) {
#if RFB_ADJ_PROFILE
                    const long long cq0 = clock64();
#endif
                    CellState S = SS;
                    for (int i = 0; i < min(nq, kTailQueue) && S.err == 0; ++i) {
                        const int q = queue[i];
                        const double4 p = A.pos[q];
                        const double dx = p.x - s.x, dy = p.y - s.y, dz = p.z - s.z;
                        const double d2 = dx * dx + dy * dy + dz * dz;
                        if (may_cut(S, dx, dy, dz, d2))
                            clip(C, lane, dx, dy, dz, 0.5 * d2, __ldg(A.ids + q), S);
                    }
                    if (lane == 0) {
                        SS = S;
                        qn = 0;
                        RFB_PC(5, nq);
#if RFB_ADJ_PROFILE
                        RFB_PC(6, clock64() - cq0);
#endif
                    }
                }
                __syncthreads();
                if (nq > kTailQueue) t0 -= kTailThreads;  // overflowed: this batch again
            }
            if (warp == 0) {
                ball_box(C, lane, SS, s, g, box);
                far_refresh(C, lane, SS, far, A.flags + 7);
            }
            __syncthreads();
        }
#endif
        if (warp == 0) {
            CellState S = SS;
            emit_site(A, C, lane, self, S);
#if RFB_ADJ_PROFILE
            if (lane == 0) {  // pass-2 cycles: [12] total, [14] hull sites' total
                const unsigned long long dt = (unsigned long long)(clock64() - clk0);
                unsigned long long *pc = reinterpret_cast<unsigned long long *>(A.flags + 12);
                atomicAdd(pc, dt);
                if (A.hull[self]) atomicAdd(pc + 1, dt);
            }
#endif
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// grid construction and CSR assembly
// ---------------------------------------------------------------------------
__global__ void k_bbox(const double *pos, int64_t n, double *part) {
    __shared__ double s[6][256];
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        for (int k = 0; k < 3; ++k) {
            const double v = pos[3 * i + k];
            lo[k] = fmin(lo[k], v);
            hi[k] = fmax(hi[k], v);
        }
    for (int k = 0; k < 3; ++k) {
        s[k][threadIdx.x] = lo[k];
        s[3 + k][threadIdx.x] = hi[k];
    }
    __syncthreads();
    for (int st = blockDim.x / 2; st > 0; st >>= 1) {
        if ((int)threadIdx.x < st)
            for (int k = 0; k < 3; ++k) {
                s[k][threadIdx.x] = fmin(s[k][threadIdx.x], s[k][threadIdx.x + st]);
                s[3 + k][threadIdx.x] = fmax(s[3 + k][threadIdx.x], s[3 + k][threadIdx.x + st]);
            }
        __syncthreads();
    }
    if (threadIdx.x == 0)
        for (int k = 0; k < 6; ++k) part[6 * blockIdx.x + k] = s[k][0];
}

__global__ void k_finite(const double *pos, int64_t n3, int32_t *bad) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n3;
         i += (int64_t)gridDim.x * blockDim.x)
        if (!isfinite(pos[i])) atomicOr(bad, 1);
}

__global__ void k_cell_keys(const double *pos, int64_t n, Grid g, uint32_t *keys, int32_t *vals) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int ix = clampi((int)floor((pos[3 * i] - g.lo[0]) / g.h), 0, g.dim[0] - 1);
    const int iy = clampi((int)floor((pos[3 * i + 1] - g.lo[1]) / g.h), 0, g.dim[1] - 1);
    const int iz = clampi((int)floor((pos[3 * i + 2] - g.lo[2]) / g.h), 0, g.dim[2] - 1);
    keys[i] = (uint32_t)cell_index(g, ix, iy, iz);
    vals[i] = (int32_t)i;
}

__global__ void k_gather_sorted(const double *pos, const int32_t *ids, int64_t n, double4 *out) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int64_t i = ids[k];
    out[k] = make_double4(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2], 0.0);
}

__global__ void k_cell_starts(const uint32_t *keys, int64_t n, int64_t ncell, int32_t *cstart) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c > ncell) return;
    int64_t lo = 0, hi = n;  // first k with keys[k] >= c
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (keys[mid] < (uint32_t)c) lo = mid + 1; else hi = mid;
    }
    cstart[c] = (int32_t)lo;
}

__device__ __forceinline__ bool row_has(const int32_t *rows, int cap, const int32_t *deg, int32_t j,
                                        int32_t i) {
    const int32_t *r = rows + (int64_t)j * cap;
    int lo = 0, hi = deg[j];
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (r[mid] < i) lo = mid + 1; else hi = mid;
    }
    return lo < deg[j] && r[lo] == i;
}

// missing reverse edges i->j without j->i: queue (j, i)
__global__ void k_asym(const int32_t *rows, int cap, const int32_t *deg, int64_t n, int2 *miss,
                       int32_t miss_cap, int32_t *nmiss) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t *r = rows + i * cap;
    for (int k = 0; k < deg[i]; ++k) {
        const int32_t j = r[k];
        if (!row_has(rows, cap, deg, j, (int32_t)i)) {
            const int s = atomicAdd(nmiss, 1);
            if (s < miss_cap) miss[s] = make_int2(j, (int32_t)i);
        }
    }
}

// insert the queued reverse edges (one thread per queued edge, rows kept sorted
// by a per-row insertion under a lock-free retry: sequential per row via a
// single thread per distinct row -- the queue is tiny)
__global__ void k_add_missing(int32_t *rows, int cap, int32_t *deg, const int2 *miss, int32_t m,
                              int32_t *overflow) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    for (int s = 0; s < m; ++s) {
        const int32_t j = miss[s].x, i = miss[s].y;
        int32_t *r = rows + (int64_t)j * cap;
        int d = deg[j];
        if (row_has(rows, cap, deg, j, i)) continue;
        if (d >= cap) {
            *overflow = 1;
            continue;
        }
        int k = d;
        while (k > 0 && r[k - 1] > i) {
            r[k] = r[k - 1];
            --k;
        }
        r[k] = i;
        deg[j] = d + 1;
    }
}

__global__ void k_deg64(const int32_t *deg, int64_t n, int64_t *out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = deg[i];
    if (i == n) out[n] = 0;
}

__global__ void k_emit(const int32_t *rows, int cap, const int32_t *deg, const int64_t *off,
                       int64_t n, int64_t *nbr, uint8_t *hull_out, const uint8_t *hull) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t *r = rows + i * cap;
    const int64_t o = off[i];
    for (int k = 0; k < deg[i]; ++k) nbr[o + k] = r[k];
    if (hull_out) hull_out[i] = hull[i];
}

static std::vector<int4> spiral_table() {
    std::vector<int4> t;
    for (int dz = -kSpiralG; dz <= kSpiralG; ++dz)
        for (int dy = -kSpiralG; dy <= kSpiralG; ++dy)
            for (int dx = -kSpiralG; dx <= kSpiralG; ++dx) {
                auto f = [](int d) { int a = d < 0 ? -d : d; return a > 0 ? a - 1 : 0; };
                const int lb2 = f(dx) * f(dx) + f(dy) * f(dy) + f(dz) * f(dz);
                t.push_back(make_int4(dx, dy, dz, lb2));
            }
    std::stable_sort(t.begin(), t.end(), [](const int4 &a, const int4 &b) { return a.w < b.w; });
    return t;
}

static size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

struct Layout {
    size_t keys, keys2, vals, vals2, pos, cstart, rows, deg, hull, spiral, flags, part, miss, tail,
        tail_key, deg64,
        cub, total;
};

static Layout layout(int64_t n, int32_t cap, int64_t max_cells) {
    Layout L;
    size_t o = 0;
    auto take = [&](size_t b) { size_t r = o; o += align256(b); return r; };
    L.keys = take(4 * n);
    L.keys2 = take(4 * n);
    L.vals = take(4 * n);
    L.vals2 = take(4 * n);
    L.pos = take(32 * n);
    L.cstart = take(4 * (max_cells + 1));
    L.rows = take((size_t)4 * n * cap);
    L.deg = take(4 * n);
    L.hull = take(n);
    L.spiral = take(sizeof(int4) * kSpiralN);
    L.flags = take(128);
    L.part = take(6 * 8 * 1024);
    L.miss = take(8 * (size_t)std::max<int64_t>(n, 1024));
    L.tail = take(4 * n);
    L.tail_key = take(4 * n);
    L.deg64 = take(8 * (n + 1));
    size_t cub_sort = 0, cub_scan = 0;
    cub::DoubleBuffer<uint32_t> kb(nullptr, nullptr);
    cub::DoubleBuffer<int32_t> vb(nullptr, nullptr);
    cub::DeviceRadixSort::SortPairs(nullptr, cub_sort, kb, vb, (int)n);
    cub::DeviceScan::ExclusiveSum(nullptr, cub_scan, (int64_t *)nullptr, (int64_t *)nullptr,
                                  (int)(n + 1));
    L.cub = take(std::max(cub_sort, cub_scan));
    L.total = o;
    return L;
}

}  // namespace rfb_adj

using namespace rfb_adj;

extern "C" {

size_t rfb_adjacency_workspace_bytes(int64_t n_sites, int32_t max_degree) {
    if (n_sites <= 0 || max_degree <= 0) return 0;
    return layout(n_sites, max_degree, 2 * n_sites + 64).total;
}

int rfb_build_adjacency(const double *positions, int64_t n_sites, int32_t max_degree,
                        int64_t *offsets, int64_t *neighbors, int64_t neighbor_capacity,
                        uint8_t *hull, int64_t *stats, void *workspace, size_t workspace_bytes,
                        void *stream) {
    if (!positions || !offsets || !stats || n_sites <= 0 || n_sites >= (1 << 30) ||
        max_degree <= 0 || max_degree > BigCell::kPlanes)
        return RFB_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n = n_sites;
    const int64_t max_cells = 2 * n + 64;
    Layout L = layout(n, max_degree, max_cells);
    if (!workspace || workspace_bytes < L.total) return RFB_EINVAL;
    char *ws = (char *)workspace;
    for (int k = 0; k < 8; ++k) stats[k] = 0;
    int32_t *flags = (int32_t *)(ws + L.flags);
    cudaMemsetAsync(flags, 0, 128, st);
    // finite coordinates (delaunay.py:456-457) and bounding box
    k_finite<<<1024, 256, 0, st>>>(positions, 3 * n, flags + 4);
    double *part = (double *)(ws + L.part);
    const int nb = (int)std::min<int64_t>(1024, (n + 255) / 256);
    k_bbox<<<nb, 256, 0, st>>>(positions, n, part);
    std::vector<double> hp(6 * nb);
    int32_t hflags[16];
    cudaMemcpyAsync(hp.data(), part, sizeof(double) * 6 * nb, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(hflags, flags, sizeof(hflags), cudaMemcpyDeviceToHost, st);
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return (int)e;
    if (hflags[4]) return RFB_EDEGENERATE;
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int b = 0; b < nb; ++b)
        for (int k = 0; k < 3; ++k) {
            lo[k] = std::min(lo[k], hp[6 * b + k]);
            hi[k] = std::max(hi[k], hp[6 * b + 3 + k]);
        }
    double ext[3], diag2 = 0.0;
    for (int k = 0; k < 3; ++k) {
        ext[k] = hi[k] - lo[k];
        diag2 += ext[k] * ext[k];
    }
    const double diag = std::sqrt(diag2);
    // cubic cells, ~2 sites per cell over the bounding box (at most max_cells)
    Grid g;
    double emax = std::max(ext[0], std::max(ext[1], ext[2]));
    if (!(emax > 0.0)) emax = 1.0;
    double vol = 1.0;
    for (int k = 0; k < 3; ++k) vol *= std::max(ext[k], emax * 1e-3);
    double h = std::cbrt(RFB_ADJ_CELL_SITES * vol / (double)n);
    for (;;) {
        int64_t cells = 1;
        for (int k = 0; k < 3; ++k) {
            g.dim[k] = std::max(1, (int)std::ceil(ext[k] / h));
            cells *= g.dim[k];
        }
        if (cells <= max_cells && cells < (1ll << 31)) break;
        h *= 1.25;
    }
    for (int k = 0; k < 3; ++k) g.lo[k] = lo[k];
    g.h = h;
    const int64_t ncell = (int64_t)g.dim[0] * g.dim[1] * g.dim[2];
    // counting layout by a stable radix sort of the cell keys
    uint32_t *keys = (uint32_t *)(ws + L.keys), *keys2 = (uint32_t *)(ws + L.keys2);
    int32_t *vals = (int32_t *)(ws + L.vals), *vals2 = (int32_t *)(ws + L.vals2);
    const unsigned gb = (unsigned)((n + 255) / 256);
    k_cell_keys<<<gb, 256, 0, st>>>(positions, n, g, keys, vals);
    cub::DoubleBuffer<uint32_t> kb(keys, keys2);
    cub::DoubleBuffer<int32_t> vb(vals, vals2);
    size_t cub_bytes = workspace_bytes - L.cub;
    int end_bit = 1;
    while (end_bit < 32 && (1ll << end_bit) < ncell) ++end_bit;
    cub::DeviceRadixSort::SortPairs(ws + L.cub, cub_bytes, kb, vb, (int)n, 0, end_bit, st);
    const uint32_t *skeys = kb.Current();
    const int32_t *sids = vb.Current();
    double4 *spos = (double4 *)(ws + L.pos);
    k_gather_sorted<<<gb, 256, 0, st>>>(positions, sids, n, spos);
    int32_t *cstart = (int32_t *)(ws + L.cstart);
    k_cell_starts<<<(unsigned)((ncell + 256) / 256), 256, 0, st>>>(skeys, n, ncell, cstart);
    static std::vector<int4> spiral = spiral_table();
    int4 *dsp = (int4 *)(ws + L.spiral);
    cudaMemcpyAsync(dsp, spiral.data(), sizeof(int4) * kSpiralN, cudaMemcpyHostToDevice, st);
    Args A;
    A.pos = spos;
    A.ids = sids;
    A.cstart = cstart;
    A.spiral = dsp;
    A.n = n;
    A.g = g;
    A.box = 1e6 * (diag > 0.0 ? diag : 1.0);
    const double tol = 1e-7 * diag;  // delaunay.py:436-441 duplicate tolerance
    A.dup2 = tol * tol;
    A.cap = max_degree;
    A.rows = (int32_t *)(ws + L.rows);
    A.deg = (int32_t *)(ws + L.deg);
    A.hull = (uint8_t *)(ws + L.hull);
    A.flags = flags;
    A.tail = (int32_t *)(ws + L.tail);
    A.tail_key = (float *)(ws + L.tail_key);
    A.tail_next = flags + 16;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_voronoi, 32 * kWarps, 0);
    const int64_t want = (n + kWarps - 1) / kWarps;
    const unsigned grid = (unsigned)std::min<int64_t>(want, (int64_t)sms * std::max(per_sm, 1) * 4);
    k_voronoi<<<grid, 32 * kWarps, 0, st>>>(A);
    cudaMemcpyAsync(hflags, flags, sizeof(hflags), cudaMemcpyDeviceToHost, st);
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return (int)e;
    if (hflags[1] > 0) {
        int tper = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&tper, k_voronoi_tail, kTailThreads, 0);
        const unsigned tgrid =
            (unsigned)std::min<int64_t>(hflags[1], (int64_t)sms * std::max(tper, 1));
        // schedule by decreasing extent: sort (key, site) pairs descending
        const int cnt = hflags[1];
        float *k2 = (float *)(ws + L.keys);   // reuse the grid-sort buffers (no longer read)
        int32_t *v2 = (int32_t *)(ws + L.keys2);
        cub::DoubleBuffer<float> tkb(A.tail_key, k2);
        cub::DoubleBuffer<int32_t> tvb(A.tail, v2);
        size_t tb = workspace_bytes - L.cub;
        cub::DeviceRadixSort::SortPairsDescending(ws + L.cub, tb, tkb, tvb, cnt, 0, 32, st);
        A.tail = tvb.Current();
        cudaMemsetAsync(A.tail_next, 0, sizeof(int32_t), st);
        k_voronoi_tail<<<tgrid, kTailThreads, 0, st>>>(A, cnt);
    }
    // symmetrise (union): queue reverse edges that are missing
    int2 *miss = (int2 *)(ws + L.miss);
    const int32_t miss_cap = (int32_t)std::max<int64_t>(n, 1024);
    k_asym<<<gb, 256, 0, st>>>(A.rows, max_degree, A.deg, n, miss, miss_cap, flags + 5);
    cudaMemcpyAsync(hflags, flags, sizeof(hflags), cudaMemcpyDeviceToHost, st);
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return (int)e;
    stats[1] = hflags[5];  // reverse edges added
    stats[2] = hflags[1];  // sites that needed the pass-2 scan
    stats[3] = hflags[2];  // max cell vertices
    stats[4] = hflags[3];  // max planes
    stats[5] = *reinterpret_cast<int64_t *>(hflags + 8);   // clip tests, spiral (profile)
    stats[6] = *reinterpret_cast<int64_t *>(hflags + 10);  // clip tests, rings (profile)
    stats[7] = hflags[0];  // error flags (1 overflow, 2 duplicate, 4 degenerate)
#if RFB_ADJ_PROFILE
    stats[4] = hflags[7];  // (profile) largest far-vertex count
    cudaMemcpy(hflags, flags, sizeof(hflags), cudaMemcpyDeviceToHost);
    stats[5] = *reinterpret_cast<int64_t *>(hflags + 12);  // pass-2 cycles (all sites)
    stats[6] = *reinterpret_cast<int64_t *>(hflags + 14);  // pass-2 cycles (hull sites)
    {
        int32_t all[32];
        cudaMemcpy(all, flags, sizeof(all), cudaMemcpyDeviceToHost);
        const long long *c = reinterpret_cast<const long long *>(all + 18);
        fprintf(stderr, "[adj profile, hull sites] rings %lld batches %lld live_cells %lld "
                "sites_in_live %lld may_cut_pass %lld queued %lld clip_cycles %lld\n",
                c[0], c[1], c[2], c[3], c[4], c[5], c[6]);
    }
#endif
    if (hflags[0] & kErrDuplicate) return RFB_EDEGENERATE;
    if (hflags[0] & kErrOverflow) return RFB_ECAPACITY;
    if (hflags[0] & kErrDegenerate) return RFB_EDEGENERATE;
    if (hflags[5] > miss_cap) return RFB_ECAPACITY;
    if (hflags[5] > 0) {
        k_add_missing<<<1, 1, 0, st>>>(A.rows, max_degree, A.deg, miss, hflags[5], flags + 6);
    }
    int64_t *deg64 = (int64_t *)(ws + L.deg64);
    k_deg64<<<(unsigned)((n + 256) / 256), 256, 0, st>>>(A.deg, n, deg64);
    cub_bytes = workspace_bytes - L.cub;
    cub::DeviceScan::ExclusiveSum(ws + L.cub, cub_bytes, deg64, offsets, (int)(n + 1), st);
    int64_t E = 0;
    cudaMemcpyAsync(&E, offsets + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(hflags, flags, sizeof(hflags), cudaMemcpyDeviceToHost, st);
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return (int)e;
    stats[0] = E;
    if (hflags[6]) return RFB_ECAPACITY;
    if (!neighbors) return RFB_OK;  // size query: call rfb_adjacency_emit next
    if (neighbor_capacity < E) return RFB_ECAPACITY;
    return rfb_adjacency_emit(n_sites, max_degree, offsets, neighbors, hull, workspace,
                              workspace_bytes, stream);
}

int rfb_adjacency_emit(int64_t n_sites, int32_t max_degree, const int64_t *offsets,
                       int64_t *neighbors, uint8_t *hull, const void *workspace,
                       size_t workspace_bytes, void *stream) {
    if (n_sites <= 0 || max_degree <= 0 || !offsets || !neighbors || !workspace) return RFB_EINVAL;
    Layout L = layout(n_sites, max_degree, 2 * n_sites + 64);
    if (workspace_bytes < L.total) return RFB_EINVAL;
    const char *ws = (const char *)workspace;
    k_emit<<<(unsigned)((n_sites + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        (const int32_t *)(ws + L.rows), max_degree, (const int32_t *)(ws + L.deg), offsets, n_sites,
        neighbors, hull, (const uint8_t *)(ws + L.hull));
    return (int)cudaGetLastError();
}

}  // extern "C"
