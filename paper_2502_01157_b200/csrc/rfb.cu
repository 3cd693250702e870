// rfb.cu -- sm_100a kernels and the C ABI (include/rfb.h) of the Radiant Foam
// hot path.  See DESIGN.md for the data layout and the roofline of each
// kernel; every kernel cites the reference function it replaces (paths are
// relative to the reference tree pkg/src/rfoam/).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <type_traits>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include <cub/cub.cuh>

#include "rfb_device.cuh"

namespace rfb {

constexpr unsigned kFull = 0xffffffffu;
#ifndef RFB_SUBTILE_W
#define RFB_SUBTILE_W 4  // a warp's 32 rays cover a 4 x 8 pixel patch (measured best)
#endif
#ifndef RFB_F32_FILTER
#define RFB_F32_FILTER 1
#endif
constexpr bool kUseF32Filter = RFB_F32_FILTER != 0;

// ---------------------------------------------------------------------------
// Ray sources: explicit arrays (render.py:57-125) or a pinhole camera over a
// tile list (render.py:128-149 + camera.py:66-92).
// ---------------------------------------------------------------------------
struct ArrayRays {
    static constexpr bool kUniform = false;  // per-ray origins / ranges
    const double *origins, *directions, *t_min, *t_max;
    const int32_t *start;
    int64_t m;
    const int32_t *order;  // optional processing order (a permutation of 0..m-1)
    const uint8_t *region;  // optional: view region per ray (rfb_rays.region)
    __host__ __device__ __forceinline__ int64_t count() const { return m; }
    // region of a view-culled scene ray q walks
    __device__ __forceinline__ int32_t region_of(int64_t q, int32_t, int32_t) const {
        return region ? (int32_t)region[q] : 0;
    }
    __device__ __forceinline__ int64_t index(int64_t slot) const {
        return order ? (int64_t)order[slot] : slot;
    }
    // returns the output index (ray id / pixel) or -1 for a padding slot
    __device__ __forceinline__ int64_t get(int64_t slot, Ray &r) const {
        const int64_t q = index(slot);
        r.ox_ = origins[3 * q];
        r.oy_ = origins[3 * q + 1];
        r.oz_ = origins[3 * q + 2];
        r.dx_ = directions[3 * q];
        r.dy_ = directions[3 * q + 1];
        r.dz_ = directions[3 * q + 2];
        r.t_min_ = t_min[q];
        r.t_max_ = t_max[q];
        r.start_ = start[q];
        return q;
    }
};

struct CameraParams {
    double R[9];  // rotation, row-major (pose[:3,:3])
    double o[3];  // pose[:3,3]
    double focal, cx, cy;
    int32_t width, height;
    int32_t kind;  // 0 pinhole, 1 fisheye (camera.py:16-17)
};

// camera.py:78-92.  Pinhole: the fma order reproduces numpy's `d_cam @ R.T`
// bit-for-bit (tests/test_gpu_parity.py).  Fisheye (equidistant, theta = r):
// same matmul order; its sin/cos/hypot are the device's (<= 2 ulp), so the
// directions agree with numpy to ~1e-16 rather than bit-for-bit.
__device__ __forceinline__ void pinhole_dir(const CameraParams &c, int64_t row, int64_t col,
                                            double &dx, double &dy, double &dz) {
    double u = ((double)col + 0.5 - c.cx) / c.focal;
    double v = -((double)row + 0.5 - c.cy) / c.focal;
    double a = u, b = v, z = -1.0;
    if (c.kind == 1) {
        const double r = hypot(u, v);
        double sn, cs;
        sincos(r, &sn, &cs);
        a = r > 0.0 ? sn * u / r : 0.0;
        b = r > 0.0 ? sn * v / r : 0.0;
        z = -cs;
    }
    double w[3];
#pragma unroll
    for (int k = 0; k < 3; ++k)
        w[k] = __fma_rn(z, c.R[3 * k + 2], __fma_rn(b, c.R[3 * k + 1], a * c.R[3 * k]));
    double nrm = sqrt((w[0] * w[0] + w[1] * w[1]) + w[2] * w[2]);
    dx = w[0] / nrm;
    dy = w[1] / nrm;
    dz = w[2] / nrm;
}

struct TileRays {
    static constexpr bool kUniform = true;  // one camera origin / range for all rays
    CameraParams cam;
    const int32_t *tile_ids;
    int64_t n_tiles;
    int32_t tile_w, tile_h, tiles_x;
    double t_min, t_max;
    const int32_t *start_ptr;  // device scalar (located start cell)
    __host__ __device__ __forceinline__ int64_t count() const { return n_tiles * tile_w * tile_h; }
    // region of pixel oidx in an rx x ry grid (rfb.h: rfb_scene.view_rx)
    __device__ __forceinline__ int32_t region_of(int64_t oidx, int32_t rx, int32_t ry) const {
        if (rx <= 0) return 0;
        const int32_t py = (int32_t)(oidx / cam.width), px = (int32_t)(oidx - (int64_t)py * cam.width);
        return (py * ry / cam.height) * rx + px * rx / cam.width;
    }
    __device__ __forceinline__ void uniform(double *u) const {
        u[0] = cam.o[0];
        u[1] = cam.o[1];
        u[2] = cam.o[2];
        u[3] = t_min;
        u[4] = t_max;
    }
    // 8x4 sub-tiles inside each tile keep a warp's 32 rays on a compact patch.
    __device__ __forceinline__ int64_t get(int64_t q, Ray &r) const {
        int64_t per = (int64_t)tile_w * tile_h;
        int32_t tile = tile_ids[q / per];
        int32_t p = (int32_t)(q % per);
        int32_t sub = p >> 5, l = p & 31;
        constexpr int SW = RFB_SUBTILE_W, SH = 32 / RFB_SUBTILE_W;  // warp patch SW x SH
        int32_t subs_x = tile_w / SW;
        int32_t px = (tile % tiles_x) * tile_w + (sub % subs_x) * SW + (l % SW);
        int32_t py = (tile / tiles_x) * tile_h + (sub / subs_x) * SH + (l / SW);
        if (px >= cam.width || py >= cam.height) return -1;
        r.ox_ = cam.o[0];
        r.oy_ = cam.o[1];
        r.oz_ = cam.o[2];
        pinhole_dir(cam, py, px, r.dx_, r.dy_, r.dz_);
        r.t_min_ = t_min;
        r.t_max_ = t_max;
        r.start_ = *start_ptr;
        return (int64_t)py * cam.width + px;
    }
};

struct FwdOut {
    void *rgb, *residual, *wsum;
    int8_t *status;
    int32_t *nseg;
    int32_t *ray_counters;
    unsigned long long *counters;
    int32_t f64;
    int32_t seg_cap;
    int32_t *seg_cells;
    double *seg_t0, *seg_t1;
    int64_t seg_first, seg_count;  // dump row = ray - seg_first, for rays in [first, first+count)
};

__device__ __forceinline__ void store_out(void *p, int64_t idx, double v, int32_t f64) {
    if (f64)
        reinterpret_cast<double *>(p)[idx] = v;
    else
        reinterpret_cast<float *>(p)[idx] = (float)v;
}

__device__ __forceinline__ void write_fwd(const FwdOut &O, int64_t q, int status, double cr,
                                          double cg, double cb, double resid, double wsum,
                                          int32_t nseg, int32_t cells, int32_t visits) {
    store_out(O.rgb, 3 * q, cr, O.f64);
    store_out(O.rgb, 3 * q + 1, cg, O.f64);
    store_out(O.rgb, 3 * q + 2, cb, O.f64);
    if (O.residual) store_out(O.residual, q, resid, O.f64);
    if (O.wsum) store_out(O.wsum, q, wsum, O.f64);
    if (O.status) O.status[q] = (int8_t)status;
    if (O.nseg) O.nseg[q] = nseg;
    if (O.ray_counters) {
        O.ray_counters[2 * q] = cells;
        O.ray_counters[2 * q + 1] = visits;
    }
}

// ---------------------------------------------------------------------------
// The walk (tracer/kernels.py:101-162), executed by the G lanes of a ray
// group.  rec(index, cell, sigma, t0, t1) is called for every recorded
// segment, in order, with the cell's index in the scene view's layout
// (S.to_id(cell) is its site id).  Returns the status code.
// ---------------------------------------------------------------------------
template <int G, int PACKED, class RayT, class Rec>
__device__ __forceinline__ int walk(const SceneView<PACKED> &S, const RayT &r, int32_t start,
                                    int32_t hoff, double epsilon,
                                    double log_eps, double width_floor, int32_t step_limit,
                                    int gl, unsigned gmask, int32_t &nseg, int32_t &cells,
                                    int32_t &visits, Rec &&rec) {
    int32_t i = S.to_pk(start);  // packed layout: the walk runs on packed indices
    double entry = r.t_min(), log_T = 0.0;
    int32_t zero_adv = 0, steps = 0;
    const float df[3] = {(float)r.dx(), (float)r.dy(), (float)r.dz()};
    nseg = 0;
    cells = 0;
    visits = 0;  // cells stepped == steps taken (kernels.py:111), set on return
    for (;;) {
        steps += 1;
        if (steps > step_limit) {
            cells = step_limit;
            return RFB_STATUS_STEP_LIMIT;
        }
        const Cell c = S.cell(i + hoff);  // hoff: the ray's region copy (view-culled scenes)
        // packed: + the neighbours a view-culled row dropped (k_cull_rows)
        visits += c.k1 - c.k0 + (PACKED ? (__float_as_int(c.n1max) & 31) : 0);
        double best_t;
        int32_t best_j;
        if constexpr (PACKED && kUseF32Filter)
            exit_face_f32<G, PACKED>(S, i, c, c.hf, r, entry, df, gl, gmask, best_t, best_j);
        else
            exit_face<G, PACKED>(S, c, r, gl, gmask, best_t, best_j);
        if (best_j < 0 || best_t >= r.t_max()) {  // hull exit or far plane
            if (r.t_max() > entry) {
                const double sig = S.sigma_of(i, c);
                log_T -= sig * (r.t_max() - entry);
                rec(nseg, i, sig, entry, r.t_max());
                nseg += 1;
            }
            cells = steps;
            return RFB_STATUS_OK;
        }
        if (best_t < entry) best_t = entry;
        if (best_t - entry > width_floor) {
            const double sig = S.sigma_of(i, c);
            log_T -= sig * (best_t - entry);
            rec(nseg, i, sig, entry, best_t);
            nseg += 1;
            entry = best_t;
            zero_adv = 0;
            if (below_epsilon(log_T, epsilon, log_eps)) {
                cells = steps;
                return RFB_STATUS_OK;
            }
            if (nseg >= step_limit) {
                cells = steps;
                return RFB_STATUS_STEP_LIMIT;
            }
        } else {
            zero_adv += 1;
            if (zero_adv > kZeroAdvanceLimit) {
                cells = steps;
                return RFB_STATUS_CYCLE;
            }
        }
        RFB_BOUND(best_j, S.n_sites);
        i = best_j;
    }
}

__device__ __forceinline__ double basis_setup(const Ray &r, float *basis_f) {
    double basis[16];
    sh_basis(r.dx(), r.dy(), r.dz(), basis);
    double bsum = 0.0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        basis_f[k] = (float)basis[k];
        bsum += fabs(basis[k]);
    }
    return bsum;
}

// ---------------------------------------------------------------------------
// Forward: walk with compositing fused per recorded segment
// (composite_segments kernels.py:165-196, same operation order, so the
// result equals compositing after the walk).  Warps fetch 32/G rays at a
// time from a global counter (persistent grid).
// ---------------------------------------------------------------------------
#ifndef RFB_SM_STATIC_PCT
#define RFB_SM_STATIC_PCT 80  // share of the 32-unit groups dealt statically to the SM queues
#endif
#ifndef RFB_TRAIN_SM_LOCAL
#define RFB_TRAIN_SM_LOCAL 0  // (config 5: 258 vs 244 ms with; config 3: same)
#endif
#ifndef RFB_SM_LOCAL
#define RFB_SM_LOCAL 1  // per-SM tile queues (fetch_unit) when the workspace has room
#endif
// Work distribution over units of RPW rays (consecutive units = neighbouring warp patches,
// 32 of them = one 32 x 32 image tile in rfb_render_image's tile order).  n_v > 0: the
// grid is n_v x (blocks per SM), and block b works for virtual SM v = b % n_v (blocks of
// one wave are spread one per SM, so the blocks sharing v normally sit on one SM): 95% of
// the 32-unit groups are dealt round-robin to the virtual SMs, each with its own counter
// (ctr[1 + v]), so an SM's warps walk one image tile together and share its cells'
// headers, rows and SH rows in L1; the rest are handed out from ctr[0] (the tail).
// n_v == 0: one global counter (ctr[0]).
__device__ __forceinline__ int64_t fetch_unit(unsigned long long *ctr, int64_t U, int n_v) {
    if (n_v <= 0) return (int64_t)atomicAdd(ctr, 1ull);
    const int64_t T = (U + 31) / 32;
    const int64_t per = (T * RFB_SM_STATIC_PCT / 100) / n_v;  // static 32-unit groups per virtual SM
    const int v = blockIdx.x % n_v;  // (%smid itself: 11.80 vs 11.87 ms, but ids need not be dense)
    if (per > 0) {
        const unsigned long long u = atomicAdd(ctr + 1 + v, 1ull);
        if ((int64_t)u < per * 32) return (v + (int64_t)n_v * (int64_t)(u >> 5)) * 32 + (int64_t)(u & 31);
    }
    return per * n_v * 32 + (int64_t)atomicAdd(ctr, 1ull);
}

#ifndef RFB_FWD_MINB
#define RFB_FWD_MINB 4
#endif
#ifndef RFB_CONST_ORIGIN
#define RFB_CONST_ORIGIN 1  // shared-origin rays: origin / t-range from the constant bank
#endif
template <int G, int SHDEG, int PACKED, class Src>
__global__ void __launch_bounds__(256, RFB_FWD_MINB) k_render(SceneView<PACKED> S,
                                                const __grid_constant__ Src src, double epsilon,
                                                double log_eps, double width_floor,
                                                int32_t step_limit, FwdOut O,
                                                unsigned long long *ray_counter, int32_t n_v) {
    constexpr int RPW = 32 / G;
    // per thread: the ray's fp64 constants + sum|basis| (field-major, conflict-free);
    // shared-origin sources keep only the direction per thread
    constexpr int kRayFields = Src::kUniform ? 4 : 9;
    __shared__ double s_ray[kRayFields * 256];
    __shared__ double s_uni[5];
    __shared__ float s_basis[15 * 256];  // fp32 SH basis k = 1..15, [k-1][thread] (k = 0: kC0)
    if (threadIdx.x == 0) {
        if constexpr (Src::kUniform) src.uniform(s_uni);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int gl = lane & (G - 1);
    const unsigned gmask = G == 32 ? kFull : (((1u << G) - 1u) << (lane & ~(G - 1)));
    const int64_t total = src.count();
    const int64_t units = (total + RPW - 1) / RPW;
    unsigned int my_cells = 0, my_visits = 0;

    for (;;) {
        long long unit = 0;
        if (lane == 0) unit = (long long)fetch_unit(ray_counter, units, n_v);
        unit = __shfl_sync(kFull, unit, 0);
        if ((int64_t)unit >= units) break;
        int64_t q = (int64_t)unit * RPW + lane / G;
        if (q >= total) continue;
        int64_t oidx;
        int32_t start;
        // the ray's fp64 constants and fp32 SH basis live in shared memory
        // (field-major, conflict-free) to keep registers for the walk: the
        // kernel is occupancy-bound
        using RayU = typename std::conditional<RFB_CONST_ORIGIN, RaySmemP<256, Src>,
                                               RaySmemU<256>>::type;
        using RayS = typename std::conditional<Src::kUniform, RayU, RaySmem<256>>::type;
        RayS r;
        r.p = s_ray + threadIdx.x;
        if constexpr (Src::kUniform) {
#if RFB_CONST_ORIGIN
            r.src = &src;
#else
            r.u = s_uni;
#endif
        }
        double *tol_p = s_ray + (kRayFields - 1) * 256 + threadIdx.x;  // color_tol
        {
            Ray rr;
            oidx = src.get(q, rr);
            if (oidx < 0) continue;
            start = rr.start_;
            r.store(rr);
            if (SHDEG > 0) {
                float bf[16];
                *tol_p = color_tol(S, basis_setup(rr, bf));
#pragma unroll
                for (int k = 1; k < 16; ++k) s_basis[(k - 1) * 256 + threadIdx.x] = bf[k];
            } else {
                *tol_p = color_tol(S, kC0);
            }
        }
        // colour accumulation in fp32 (image tolerance 1e-4); transmittance and
        // the weight sum stay fp64 so sum(w) + T == 1 to ~1e-14; the walk's own
        // log-transmittance test is fp64 as in the reference.
        double T = 1.0, wsum = 0.0;
        float cr = 0.f, cg = 0.f, cb = 0.f;
        const bool dump = O.seg_cap > 0;
        int32_t nseg, cells, visits;
        const int32_t hoff =
            PACKED ? src.region_of(oidx, S.view_rx, S.view_ry) * (int32_t)S.n_sites : 0;
        int status = walk<G, PACKED>(
            S, r, start, hoff, epsilon, log_eps, width_floor, step_limit, gl, gmask, nseg, cells,
            visits,
            [&](int32_t s, int32_t cell, double sigma, double t0, double t1) {
                double delta = t1 - t0;
                const double alpha = (double)(-expm1f(-(float)(sigma * delta)));
                double col[3];
#ifdef RFB_NO_COLOR  // profiling knob: walk + compositing with a constant colour
                col[0] = col[1] = col[2] = 0.5;
#else
                cell_color<SHDEG, PACKED, 256, 1>(S, cell, s_basis + threadIdx.x, r, *tol_p, col);
#endif
                const double w = T * alpha;
                wsum += w;
                const float wf = (float)w;
                cr += wf * (float)col[0];
                cg += wf * (float)col[1];
                cb += wf * (float)col[2];
                T *= 1.0 - alpha;
                if (dump && s < O.seg_cap && gl == 0 &&
                    (uint64_t)(oidx - O.seg_first) < (uint64_t)O.seg_count) {
                    int64_t o = (oidx - O.seg_first) * O.seg_cap + s;
                    O.seg_cells[o] = S.to_id(cell);
                    O.seg_t0[o] = t0;
                    O.seg_t1[o] = t1;
                }
            });
        if (gl == 0) {
            my_cells += (unsigned)cells;
            my_visits += (unsigned)visits;
            if (status != RFB_STATUS_OK)  // kernels.py:230-236
                write_fwd(O, oidx, status, S.bg[0], S.bg[1], S.bg[2], 1.0, 0.0, nseg, cells,
                          visits);
            else
                write_fwd(O, oidx, status, cr + T * S.bg[0], cg + T * S.bg[1], cb + T * S.bg[2],
                          T, wsum, nseg, cells, visits);
        }
    }
    if (O.counters) {
        unsigned long long tc = my_cells, tv = my_visits;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            tc += __shfl_xor_sync(kFull, tc, off);
            tv += __shfl_xor_sync(kFull, tv, off);
        }
        if (lane == 0) {
            atomicAdd(O.counters, tc);
            atomicAdd(O.counters + 1, tv);
        }
    }
}

// ---------------------------------------------------------------------------
// Backward / training.  Each warp takes 32 rays.  Every lane walks its ray
// (recording the segments into its slot of the workspace and compositing),
// then the warp runs the reverse pass (backward_ray, kernels.py:267-337)
// cooperatively: each iteration selects the farthest pending segment's cell,
// every lane whose current segment is in that cell processes it, and the
// gradients of that cell are summed across the group before ONE atomic per
// value (dpos+dsigma as a float4, dSH as two coalesced 32-lane reductions
// into the cell's 48-float row).  Coherent rays share cells, so this
// replaces ~32 contended atomics by one.  Per-lane segment order and
// arithmetic are exactly the reference's; only the summation order of the
// fp32 accumulators changes.
// ---------------------------------------------------------------------------
struct Scratch {
    // quantile variant: one 32-byte record per segment in two 16-byte halves:
    float4 *a;      // [cap][slots]: {cell id | clamp mask << 29 (int bits), clamped colour rgb}
    double2 *b;     // [cap][slots]: {exit depth t1 (the entry of s+1),
                    //                T_before[s+1] = prod exp(-sigma*delta) (kernels.py:270-275)}
    // L2 / adjoint variants: one 8-byte record per segment, {cell id, fp32 exit
    // depth}; the reverse pass recomputes the colour (same fp32 arithmetic, so
    // the same values and clamp mask) and the transmittance from the log
    uint2 *c;       // [cap][slots]
    int64_t slots;
};

#ifndef RFB_COMPACT_REC
#define RFB_COMPACT_REC 0  // 1: 8-byte records (4x less scratch, measured 33.4 -> 37.6 ms: colour recompute)
#endif
constexpr int kCompactRecBytes = 8;
constexpr int kFullRecBytes = 32;

struct Grads {
    float *g4;  // [n][4] dpos xyz, dsigma
    float *sh;  // [n][48]
};

__device__ __forceinline__ void red4(float *p, float a, float b, float c, float d) {
    atomicAdd(reinterpret_cast<float4 *>(p), make_float4(a, b, c, d));
}

// kernels.py:340-369 -> contributions to x_i (gi) and x_j (gj).
template <class RayT>
__device__ __forceinline__ bool face_grad(const double4 *__restrict__ site4, int32_t i,
                                          int32_t j, const RayT &r, double t, double dt,
                                          double *gi, double *gj) {
    double4 xi = ld_site(site4 + i), xj = ld_site(site4 + j);
    double nx = xj.x - xi.x, ny = xj.y - xi.y, nz = xj.z - xi.z;
    double denom = r.dx() * nx + r.dy() * ny + r.dz() * nz;
    if (denom == 0.0) return false;
    double mx = 0.5 * (xi.x + xj.x), my = 0.5 * (xi.y + xj.y), mz = 0.5 * (xi.z + xj.z);
    double px = r.ox() + t * r.dx(), py = r.oy() + t * r.dy(), pz = r.oz() + t * r.dz();
    double qx = mx - px, qy = my - py, qz = mz - pz;
    double inv = dt / denom;
    gi[0] = (0.5 * nx - qx) * inv;
    gi[1] = (0.5 * ny - qy) * inv;
    gi[2] = (0.5 * nz - qz) * inv;
    gj[0] = (0.5 * nx + qx) * inv;
    gj[1] = (0.5 * ny + qy) * inv;
    gj[2] = (0.5 * nz + qz) * inv;
    return true;
}

template <class RayT>
__device__ __forceinline__ void face_grad_atomic(const double4 *__restrict__ site4, int32_t i,
                                                 int32_t j, const RayT &r, double t, double dt,
                                                 float *g4) {
    double gi[3], gj[3];
    if (!face_grad(site4, i, j, r, t, dt, gi, gj)) return;
    red4(g4 + 4 * (int64_t)i, (float)gi[0], (float)gi[1], (float)gi[2], 0.f);
    red4(g4 + 4 * (int64_t)j, (float)gj[0], (float)gj[1], (float)gj[2], 0.f);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
    return v;
}

__device__ __forceinline__ unsigned order_key(double t) {
    unsigned b = __float_as_uint((float)t);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

#ifndef RFB_REV_ADAPTIVE
#define RFB_REV_ADAPTIVE 1  // per-lane reverse pass for incoherent warps
#endif
#ifndef RFB_REV_COLREG
#define RFB_REV_COLREG 1  // reverse pass: load cell + colour together when advancing
#endif
#ifndef RFB_REV_SMALL
#define RFB_REV_SMALL 2  // reverse pass: groups of at most this many lanes scatter per lane
#endif
constexpr int kTrainBlock = 128;
#ifndef RFB_TRAIN_WS_HDR
#define RFB_TRAIN_WS_HDR 4096
#endif
constexpr size_t kTrainWsHdr = RFB_TRAIN_WS_HDR;  // training workspace: work counters, then records
constexpr int kTrainWarps = kTrainBlock / 32;

// resident blocks per SM (register budget): 7 x 128 threads (72 regs) for the
// L2 / adjoint passes, 6 (80 regs) when the quantile state is live (measured)
#ifndef RFB_TRAIN_MINB
#define RFB_TRAIN_MINB 7
#endif
#ifndef RFB_TRAIN_MINB_Q
#define RFB_TRAIN_MINB_Q 6
#endif
// Quantile pairs folded into the cooperative reverse pass (the first
// kQFusedPairs pairs; any further pairs take the per-lane scatter path).
constexpr int kQFusedPairs = 2;
constexpr int kQSamples = 2 * kQFusedPairs;

// kernels.py:456-527: locate sample u of one ray's weight CDF -> (t_u, its
// segment, T(t_u)). `tot` = 1 - T_end.
struct QHit {
    double t, T_at, sigma;
    int32_t seg;
};
template <class RayT>
__device__ __forceinline__ QHit quantile_hit(const double4 *__restrict__ site4, const int32_t *cellp,
                                             int64_t SLa, const double *t1p, const double *tbp,
                                             int64_t SL, int32_t nseg, const RayT &r, double u,
                                             double tot) {
    const double target = u * tot;
    // first segment with W_{s+1} = 1 - T_before[s+1] >= target (capped at the
    // last), as kernels.py:503-505's linear scan: T_before is non-increasing
    // (every factor exp(-sigma*delta) <= 1), so a binary search finds the same one
    int32_t sh = 0, hi = nseg - 1;
    while (sh < hi) {
        const int32_t mid = (sh + hi) >> 1;
        if ((1.0 - tbp[mid * SL]) < target) sh = mid + 1; else hi = mid;
    }
    QHit h;
    h.seg = sh;
    h.sigma = ld_sigma(site4 + (cellp[sh * SLa] & 0x1fffffff));
    const double ts0 = sh > 0 ? t1p[(sh - 1) * SL] : r.t_min();
    const double Tbs = sh > 0 ? tbp[(sh - 1) * SL] : 1.0;
    if (h.sigma <= 0.0) {
        h.t = ts0;
    } else {
        double frac = (target - (1.0 - Tbs)) / Tbs;
        if (frac > 1.0 - 1e-15) frac = 1.0 - 1e-15;
        double th = ts0 - log(1.0 - frac) / h.sigma;
        const double ts1 = t1p[sh * SL];
        if (th > ts1) th = ts1;
        h.t = th;
    }
    h.T_at = Tbs * exp(-h.sigma * (h.t - ts0));
    return h;
}

// G lanes per ray (1 or 2): batches that do not fill the resident threads
// walk each ray with 2 lanes (the neighbour scan split between them); lane
// gl == 0 of each pair records the segments and runs the reverse pass.
template <int SHDEG, int PACKED, bool TRAIN, bool QUANT, int G = 1>
__global__ void __launch_bounds__(kTrainBlock, QUANT ? RFB_TRAIN_MINB_Q : RFB_TRAIN_MINB) k_train(
    SceneView<PACKED> S, ArrayRays src, double epsilon, double log_eps, double width_floor,
    int32_t step_limit, const double *adjoints, const double *targets, double rgb_scale,
    double q_scale, const double *u_pairs, int32_t n_pairs, double weight_floor, FwdOut O,
    Grads gr, double *loss, Scratch scr, unsigned long long *ray_counter, int32_t n_v) {
    // per lane: 16 basis values + a constant 1 (column 16) used by the plain sums
    __shared__ float s_basis[kTrainWarps][32][17];
    // per lane per reverse iteration: f_r, f_g, f_b, dpos_i xyz, dsigma_i, dpos_j xyz
    __shared__ float s_f[kTrainWarps][32][11];
    __shared__ double s_ray[8 * kTrainBlock];
    // fused quantile samples, per thread: t_u[a], g_a * T(t_u)[a]
    __shared__ double s_qt[QUANT ? kQSamples : 1][kTrainBlock];
    __shared__ double s_qg[QUANT ? kQSamples : 1][kTrainBlock];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t slot = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    // strided views of this slot's records: s_cell steps SLa ints per segment,
    // s_t1 / s_tb step SL doubles (the two halves of rec_b are interleaved)
    const int64_t SL4 = scr.slots;             // records per segment row
    const int64_t SLa = 4 * SL4, SL = 2 * SL4;
    constexpr bool kCompact = !QUANT && RFB_COMPACT_REC;
    float4 *rec_a = scr.a + slot;
    double2 *rec_b = scr.b + slot;
    uint2 *rec_c = scr.c + slot;
    const int32_t *s_cell = reinterpret_cast<const int32_t *>(rec_a);
    const double *s_t1 = reinterpret_cast<const double *>(rec_b);
    const double *s_tb = s_t1 + 1;
    double loss_rgb = 0.0, loss_q = 0.0;
    unsigned int my_cells = 0, my_visits = 0;
    const int64_t total = src.count();
    float *bas = &s_basis[warp][lane][0];
#pragma unroll
    for (int k = 0; k < 16; ++k) bas[k] = 0.f;  // rows of idle lanes stay finite (x 0 below)
    bas[16] = 1.0f;
    // reverse-pass output o (two per lane): o < 48 -> dSH[k][ch] = sum f[ch] * basis[k];
    // 48..51 -> (dpos_i xyz, dsigma_i); 52..54 -> dpos_j xyz
    // lane = (half h, basis k): both of its sums use basis[l][k] (one shared load per
    // member for the two): h 0 -> dSH[k][0], dSH[k][1]; h 1 -> dSH[k][2] and, for k < 7,
    // the plain sum of value 3 + k (dpos_i xyz, dsigma_i, dpos_j xyz; weight 1)
    const int kk = lane & 15, hh = lane >> 4;
    const int c0i = hh ? 2 : 0, c1i = hh ? 3 + (kk < 7 ? kk : 6) : 1;  // (kk >= 7: unused)
    const int o0 = 3 * kk + c0i;                       // dSH index of acc0
    const int o1 = hh ? (kk < 7 ? 48 + kk : 64) : 3 * kk + 1;  // acc1: dSH / 48.. / none
    const float one_sel = hh ? 1.f : 0.f;
    constexpr int RPW = 32 / G;
    const int gl = lane & (G - 1);
    const unsigned gmask = G == 1 ? kFull : (((1u << G) - 1u) << (lane & ~(G - 1)));

    const int64_t units = (total + RPW - 1) / RPW;
    for (;;) {
        long long unit = 0;
        if (lane == 0) unit = (long long)fetch_unit(ray_counter, units, n_v);
        unit = __shfl_sync(kFull, unit, 0);
        if ((int64_t)unit >= units) break;
        const int64_t qs = (int64_t)unit * RPW + lane / G;
        const bool have_ray = qs < total;
        const int64_t q = have_ray ? src.index(qs) : 0;  // ray id (optional order)

        RaySmem<kTrainBlock> r{s_ray + threadIdx.x};
        int32_t nseg = 0;
        int status = RFB_STATUS_OK;
        float ar = 0.f, ag = 0.f, ab = 0.f;
        bool grad_ok = false;
        double Tb = 1.0, wsum = 0.0, lt = 0.0;  // lt: log T (the walk's log_T)
        float cr = 0.f, cg = 0.f, cb = 0.f;
        int32_t cells = 0, visits = 0;
        double ctol = 0.0;
        if (have_ray) {
            int32_t start;
            {
                Ray rr;
                src.get(qs, rr);
                r.store(rr);
                start = rr.start_;
                double bsum = basis_setup(rr, bas);
                ctol = color_tol(S, SHDEG > 0 ? bsum : kC0);
            }
            const int32_t hoff =
                PACKED ? src.region_of(q, S.view_rx, S.view_ry) * (int32_t)S.n_sites : 0;
            status = walk<G, PACKED>(
                S, r, start, hoff, epsilon, log_eps, width_floor, step_limit, gl, gmask, nseg,
                cells, visits,
                [&](int32_t s, int32_t cell, double sigma, double t0, double t1) {
                    double col[3];
                    const int mask = cell_color<SHDEG, PACKED>(S, cell, bas, r, ctol, col);
                    // k_render's compositing arithmetic (fp32 alpha, fp64 T and weights;
                    // an fp64 exp here measured 0.2 ms slower per config-3 view)
                    const double alpha = (double)(-expm1f(-(float)(sigma * (t1 - t0))));
                    const double w = Tb * alpha;
                    const double Tn = Tb * (1.0 - alpha);  // T_before[s+1] (kernels.py:275)
                    wsum += w;
                    const float wf = (float)w;
                    cr += wf * (float)col[0];
                    cg += wf * (float)col[1];
                    cb += wf * (float)col[2];
                    Tb = Tn;
                    if (G == 1 || gl == 0) {
                        RFB_BOUND(s, step_limit);
                        RFB_BOUND(slot, SL4);
                        // the reverse pass works on site ids (site4, gradient rows)
                        const int32_t sid = S.to_id(cell);
                        if constexpr (kCompact) {
                            lt -= sigma * (t1 - t0);
                            rec_c[s * SL4] = make_uint2((unsigned)sid, __float_as_uint((float)t1));
                        } else {
                            rec_a[s * SL4] = make_float4(__int_as_float(sid | (mask << 29)),
                                                         (float)col[0], (float)col[1],
                                                         (float)col[2]);
                            rec_b[s * SL4] = make_double2(t1, Tn);
                        }
                    }
                });
        }
        if (have_ray && (G == 1 || gl == 0)) {  // one lane per ray from here on
            my_cells += (unsigned)cells;
            my_visits += (unsigned)visits;
            if (status != RFB_STATUS_OK) {
                write_fwd(O, q, status, S.bg[0], S.bg[1], S.bg[2], 1.0, 0.0, nseg, cells, visits);
            } else {
                const double R = cr + Tb * S.bg[0], Gc = cg + Tb * S.bg[1], B = cb + Tb * S.bg[2];
                write_fwd(O, q, status, R, Gc, B, Tb, wsum, nseg, cells, visits);
                if (TRAIN) {  // kernels.py:430-437
                    double er = R - targets[3 * q], eg = Gc - targets[3 * q + 1],
                           eb = B - targets[3 * q + 2];
                    loss_rgb += er * er + eg * eg + eb * eb;
                    ar = (float)(2.0 * rgb_scale * er);
                    ag = (float)(2.0 * rgb_scale * eg);
                    ab = (float)(2.0 * rgb_scale * eb);
                } else {
                    ar = (float)adjoints[3 * q];
                    ag = (float)adjoints[3 * q + 1];
                    ab = (float)adjoints[3 * q + 2];
                }
                grad_ok = nseg > 0;
            }
        }

        // ---- quantile samples (kernels.py:456-567), located per lane ---------
        // The loss gradient of each sample is linear in per-segment and
        // per-boundary terms (kernels.py:534-566), so the reverse pass below
        // adds them to the L2 terms of the same segment / boundary: dsigma +=
        // qA*dt - sum_{t0<t_u} gT*(min(t1,t_u)-t0) and boundary dt +=
        // (sigma_i - sigma_j) * (qA - sum_{t1<t_u} gT), with qA = sum g*u*T_end.
        double qA = 0.0;
        if (QUANT) {
#pragma unroll
            for (int a = 0; a < kQSamples; ++a) {
                s_qt[a][threadIdx.x] = -INFINITY;
                s_qg[a][threadIdx.x] = 0.0;
            }
            if (grad_ok) {
                const double T_end_q = s_tb[(nseg - 1) * SL];
                const double tot = 1.0 - T_end_q;
                const int np = n_pairs < kQFusedPairs ? n_pairs : kQFusedPairs;
                if (!(tot < weight_floor)) {
                    for (int32_t p = 0; p < np; ++p) {
                        const double *up = u_pairs + (q * n_pairs + p) * 2;
                        const QHit h0 = quantile_hit(S.site4, s_cell, SLa, s_t1, s_tb, SL, nseg, r,
                                                     up[0], tot);
                        const QHit h1 = quantile_hit(S.site4, s_cell, SLa, s_t1, s_tb, SL, nseg, r,
                                                     up[1], tot);
                        const double diff = h0.t - h1.t;
                        loss_q += fabs(diff);
                        if (diff == 0.0) continue;
                        const double sign = diff > 0.0 ? 1.0 : -1.0;
#pragma unroll
                        for (int a = 0; a < 2; ++a) {
                            const QHit &h = a == 0 ? h0 : h1;
                            const double wd = h.T_at * h.sigma;
                            if (wd <= 1e-300) continue;
                            const double g = (a == 0 ? sign : -sign) * q_scale / wd;
                            qA += g * (up[a] * T_end_q);
                            s_qt[2 * p + a][threadIdx.x] = h.t;
                            s_qg[2 * p + a][threadIdx.x] = g * h.T_at;
                        }
                    }
                }
            }
        }

        // ---- cooperative reverse pass (kernels.py:267-337) -------------------
        // Each iteration: the farthest pending segment's cell is processed by
        // every lane currently in it; the group's 55 gradient values (48 dSH,
        // dpos+dsigma of the cell, dpos of the previously processed cell) are
        // reduced through shared memory and land with coalesced atomics.
#ifdef RFB_NO_REVERSE  // profiling knob: walk + record only
        grad_ok = false;
#endif
        int32_t s = grad_ok ? nseg - 1 : -1;
        int32_t ci = -1, cmask = 0, next_cell = -1;
        double t1 = 0.0, t0 = 0.0;
        float tb1 = 0.f, tb0 = 1.f;
        float Sr = 0.f, Sg = 0.f, Sb = 0.f, d_next = 0.f;
        double sig_next = 0.0;  // sigma of next_cell (quantile boundary terms)
#if RFB_REV_COLREG
        float cc0 = 0.f, cc1 = 0.f, cc2 = 0.f;  // colour of the current segment
#endif
        float lt1 = 0.f, lt0 = 0.f;  // compact: log T after / before segment s

        auto load_seg = [&]() {
            if constexpr (kCompact) {
                const uint2 rc = rec_c[s * SL4];
                ci = (int32_t)rc.x;
                t1 = __uint_as_float(rc.y);
                t0 = s > 0 ? (double)__uint_as_float(rec_c[(s - 1) * SL4].y) : r.t_min();
                tb1 = (float)Tb;  // T_end of the forward (fp64 product)
                lt1 = (float)lt;
                return;
            }
#if RFB_REV_COLREG
            const float4 ra = rec_a[s * SL4];
            const int32_t cm = __float_as_int(ra.x);
            cc0 = ra.y;
            cc1 = ra.z;
            cc2 = ra.w;
#else
            const int32_t cm = s_cell[s * SLa];
#endif
            ci = cm & 0x1fffffff;
            cmask = (cm >> 29) & 7;
            t1 = s_t1[s * SL];
            t0 = s > 0 ? s_t1[(s - 1) * SL] : r.t_min();
            tb1 = (float)s_tb[s * SL];
            tb0 = s > 0 ? (float)s_tb[(s - 1) * SL] : 1.f;
        };
        if (s >= 0) {
            load_seg();
            Sr = tb1 * (float)S.bg[0];  // suffix starts at T_end * background
            Sg = tb1 * (float)S.bg[1];
            Sb = tb1 * (float)S.bg[2];
        }
        // Incoherent warps (random training pixels: lanes rarely share a cell)
        // gain nothing from grouping and pay one iteration per lane-segment;
        // they walk back per lane and scatter with vector atomics instead
        // (65,536 random pixels: 12.3 -> 4.7 ms).
        bool per_lane = false;
#if RFB_REV_ADAPTIVE
        {
            // coherence probe: the cell at the middle of each lane's path (the
            // first and last cells are shared by any rays with a common origin
            // or exit)
            int32_t mid = -1 - lane;
            if (s >= 0)
                mid = kCompact ? (int32_t)rec_c[(s / 2) * SL4].x
                               : (s_cell[(s / 2) * SLa] & 0x1fffffff);
            const unsigned peers = __match_any_sync(kFull, mid);
            const bool first = (__ffs(peers) - 1) == lane;
            const int groups = __popc(__ballot_sync(kFull, first && s >= 0));
            const int active = __popc(__ballot_sync(kFull, s >= 0));
            per_lane = groups * 4 > active * 3;
        }
#endif
        for (;;) {
            const bool act = s >= 0;
            if (!__any_sync(kFull, act)) break;
#ifdef RFB_COUNT_ITERS  // profiling knob: O.counters[0] += reverse iterations (per warp)
            if (lane == 0) atomicAdd(O.counters + 0, 1ull);
#endif
            int32_t lc = ci;
            bool in = act;
            if (!per_lane) {
                const unsigned key = act ? order_key(t0) : 0u;
                const unsigned kmax = __reduce_max_sync(kFull, key);
                const int leader = __ffs(__ballot_sync(kFull, act && key == kmax)) - 1;
                lc = __shfl_sync(kFull, ci, leader);
                in = act && ci == lc;
            }
            float v[11];
#pragma unroll
            for (int k = 0; k < 11; ++k) v[k] = 0.f;
            int32_t jn = -1;
            if (in) {
                const double sig_d = ld_sigma(S.site4 + ci);
                const float sig = (float)sig_d;
                const float delta = (float)(t1 - t0);
                float c0, c1, c2;
                if constexpr (kCompact) {
                    // T before s from the log (exact 1 for the first segment); the
                    // colour as the forward computed it (kernels.py:61-73)
                    lt0 = lt1 + sig * delta;
                    tb0 = s > 0 ? exp2f(lt0 * 1.4426950408889634f) : 1.f;
                    double col[3];
                    cmask = cell_color<SHDEG, PACKED>(S, S.to_pk(ci), bas, r, ctol, col);
                    c0 = (float)col[0];
                    c1 = (float)col[1];
                    c2 = (float)col[2];
                } else {
#if RFB_REV_COLREG
                    c0 = cc0;
                    c1 = cc1;
                    c2 = cc2;
#else
                    const float4 ra = rec_a[s * SL4];  // one 16-byte load: cell bits + colour
                    c0 = ra.y;
                    c1 = ra.z;
                    c2 = ra.w;
#endif
                }
                const float w = tb0 - tb1;
                const float common =
                    ar * (tb1 * c0 - Sr) + ag * (tb1 * c1 - Sg) + ab * (tb1 * c2 - Sb);
                v[6] = delta * common;
                const float dd = sig * common;
                double qdt = 0.0;
                if (QUANT) {  // kernels.py:534-566 for this segment and boundary s+1
                    double dq = qA * (t1 - t0), bq = qA;
#pragma unroll
                    for (int a = 0; a < kQSamples; ++a) {
                        const double tu = s_qt[a][threadIdx.x];
                        if (t0 < tu) {
                            const double gT = s_qg[a][threadIdx.x];
                            dq -= gT * ((t1 < tu ? t1 : tu) - t0);
                            if (t1 < tu) bq -= gT;
                        }
                    }
                    v[6] += (float)dq;
                    qdt = (sig_d - sig_next) * bq;
                    sig_next = sig_d;
                }
                if (next_cell >= 0) {  // interior boundary s+1 (kernels.py:328-337)
                    const double dt = (double)(dd - d_next) + qdt;
                    double gi[3], gj[3];
                    if (dt != 0.0 && face_grad(S.site4, ci, next_cell, r, t1, dt, gi, gj)) {
                        v[3] = (float)gi[0];
                        v[4] = (float)gi[1];
                        v[5] = (float)gi[2];
                        v[7] = (float)gj[0];
                        v[8] = (float)gj[1];
                        v[9] = (float)gj[2];
                        jn = next_cell;
                    }
                }
                if (w != 0.f) {  // kernels.py:309-322
                    if ((cmask & 1) == 0 && ar != 0.f) v[0] = w * ar;
                    if ((cmask & 2) == 0 && ag != 0.f) v[1] = w * ag;
                    if ((cmask & 4) == 0 && ab != 0.f) v[2] = w * ab;
                }
                Sr += w * c0;
                Sg += w * c1;
                Sb += w * c2;
                d_next = dd;
                next_cell = ci;
                s -= 1;
                if (kCompact && s >= 0) {
                    ci = (int32_t)rec_c[s * SL4].x;
                    t1 = t0;
                    t0 = s > 0 ? (double)__uint_as_float(rec_c[(s - 1) * SL4].y) : r.t_min();
                    tb1 = tb0;
                    lt1 = lt0;
                } else if (s >= 0) {  // segment s's end is segment s+1's start: reuse it
#if RFB_REV_COLREG
                    const float4 ra = rec_a[s * SL4];
                    const int32_t cm = __float_as_int(ra.x);
                    cc0 = ra.y;
                    cc1 = ra.z;
                    cc2 = ra.w;
#else
                    const int32_t cm = s_cell[s * SLa];
#endif
                    ci = cm & 0x1fffffff;
                    cmask = (cm >> 29) & 7;
                    t1 = t0;
                    tb1 = tb0;
                    if (s > 0) {
                        const double2 rb = rec_b[(s - 1) * SL4];  // {t0, T_before[s]}
                        t0 = rb.x;
                        tb0 = (float)rb.y;
                    } else {
                        t0 = r.t_min();
                        tb0 = 1.f;
                    }
                }
            }
#if RFB_REV_SMALL > 0
            // a group this small scatters its members' values directly (vector atomics)
            // instead of paying the shared-memory reduction
            const bool scatter = per_lane || __popc(__ballot_sync(kFull, in)) <= RFB_REV_SMALL;
#else
            const bool scatter = per_lane;
#endif
            if (scatter) {  // this lane's segment straight to its cell (kernels.py:309-337)
                if (in) {
                    const float *b = &s_basis[warp][lane][0];
                    RFB_BOUND(lc, S.n_sites);
            float *row = gr.sh + 48 * (int64_t)lc;
                    if (v[0] != 0.f || v[1] != 0.f || v[2] != 0.f) {
#pragma unroll
                        for (int q4 = 0; q4 < 12; ++q4) {
                            float e4[4];
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const int idx = 4 * q4 + u;  // k * 3 + ch
                                e4[u] = v[idx % 3] * b[idx / 3];
                            }
                            red4(row + 4 * q4, e4[0], e4[1], e4[2], e4[3]);
                        }
                    }
                    red4(gr.g4 + 4 * (int64_t)lc, v[3], v[4], v[5], v[6]);
                    RFB_BOUND(jn + 1, S.n_sites + 1);  // -1: none
                    if (jn >= 0) red4(gr.g4 + 4 * (int64_t)jn, v[7], v[8], v[9], 0.f);
                }
                continue;
            }
            // previous cell: aggregated when the whole group agrees on it
            const int32_t jany = __reduce_max_sync(kFull, in ? jn : -1);
            const bool juni = __all_sync(kFull, !in || jn < 0 || jn == jany);
            if (!juni && in && jn >= 0) {  // rare: scatter this lane's share directly
                float *pj = gr.g4 + 4 * (int64_t)jn;
                atomicAdd(pj, v[7]);
                atomicAdd(pj + 1, v[8]);
                atomicAdd(pj + 2, v[9]);
                v[7] = v[8] = v[9] = 0.f;
            }
            float *fr = &s_f[warp][lane][0];
#pragma unroll
            for (int k = 0; k < 10; ++k) fr[k] = v[k];
            __syncwarp();
            // lanes outside the group wrote zeros, so a fixed 32-term sum is the
            // group sum; unrolled, its shared-memory loads issue back to back
            // instead of one dependent ffs/load/fma chain per member
            // (skipping lane quartets with no member: a cell's lanes are a compact
            // pixel patch, so few quartets are active)
            const unsigned gm = __ballot_sync(kFull, in);
            float acc0 = 0.f, acc1 = 0.f;
#pragma unroll
            for (int qd = 0; qd < 8; ++qd) {
                if ((gm >> (4 * qd)) & 0xfu) {
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int l = 4 * qd + e;
                        const float b = s_basis[warp][l][kk];
                        acc0 = __fmaf_rn(s_f[warp][l][c0i], b, acc0);
                        acc1 = __fmaf_rn(s_f[warp][l][c1i], hh ? one_sel : b, acc1);
                    }
                }
            }
            float *row = gr.sh + 48 * (int64_t)lc;
            atomicAdd(row + o0, acc0);  // dSH[k][0] / dSH[k][2]
            if (o1 < 48) {
                atomicAdd(row + o1, acc1);  // dSH, 16 contiguous floats
            } else if (o1 < 52) {
                atomicAdd(gr.g4 + 4 * (int64_t)lc + (o1 - 48), acc1);  // dpos_i, dsigma_i
            } else if (o1 < 55 && jany >= 0 && juni) {
                atomicAdd(gr.g4 + 4 * (int64_t)jany + (o1 - 52), acc1);  // dpos_j
            }
            __syncwarp();
        }

        // ---- quantile pairs beyond the fused ones: per-lane scatter --------
        if (QUANT && n_pairs > kQFusedPairs && grad_ok) {
            double T_end_q = s_tb[(nseg - 1) * SL];
            double tot = 1.0 - T_end_q;
            if (!(tot < weight_floor)) {
                for (int32_t p = kQFusedPairs; p < n_pairs; ++p) {
                    const double *up = u_pairs + (q * n_pairs + p) * 2;
                    const QHit hh[2] = {
                        quantile_hit(S.site4, s_cell, SLa, s_t1, s_tb, SL, nseg, r, up[0], tot),
                        quantile_hit(S.site4, s_cell, SLa, s_t1, s_tb, SL, nseg, r, up[1], tot)};
                    const double diff = hh[0].t - hh[1].t;
                    loss_q += fabs(diff);
                    if (diff == 0.0) continue;
                    const double sign = diff > 0.0 ? 1.0 : -1.0;
                    for (int a = 0; a < 2; ++a) {
                        const double u = up[a], t_u = hh[a].t, T_at = hh[a].T_at;
                        const double wd = T_at * hh[a].sigma;
                        if (wd <= 1e-300) continue;
                        const double g = (a == 0 ? sign : -sign) * q_scale / wd;
                        double prev_t1 = r.t_min();
                        for (int32_t k = 0; k < nseg; ++k) {  // kernels.py:534-548
                            const double k_t0 = prev_t1, k_t1 = s_t1[k * SL];
                            prev_t1 = k_t1;
                            const int32_t ck = s_cell[k * SLa] & 0x1fffffff;
                            const double dA = T_end_q * (k_t1 - k_t0);
                            double contrib;
                            if (k_t0 < t_u) {
                                const double hi = k_t1 < t_u ? k_t1 : t_u;
                                contrib = g * (u * dA - T_at * (hi - k_t0));
                            } else {
                                contrib = g * (u * dA);
                            }
                            atomicAdd(gr.g4 + 4 * (int64_t)ck + 3, (float)contrib);
                        }
                        for (int32_t mm = 1; mm < nseg; ++mm) {  // kernels.py:552-566
                            const int32_t im = s_cell[(mm - 1) * SLa] & 0x1fffffff;
                            const int32_t jm = s_cell[mm * SLa] & 0x1fffffff;
                            const double dsig = ld_sigma(S.site4 + im) - ld_sigma(S.site4 + jm);
                            if (dsig == 0.0) continue;
                            const double tbq = s_t1[(mm - 1) * SL];
                            const double dW = tbq < t_u ? T_at * dsig : 0.0;
                            const double dt_term = g * (u * (T_end_q * dsig) - dW);
                            if (dt_term != 0.0)
                                face_grad_atomic(S.site4, im, jm, r, tbq, dt_term, gr.g4);
                        }
                    }
                }
            }
        }
    }
    unsigned long long tc = my_cells, tv = my_visits;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        loss_rgb += __shfl_xor_sync(kFull, loss_rgb, off);
        loss_q += __shfl_xor_sync(kFull, loss_q, off);
        tc += __shfl_xor_sync(kFull, tc, off);
        tv += __shfl_xor_sync(kFull, tv, off);
    }
    if (lane == 0) {
        if (TRAIN && loss) {
            atomicAdd(loss, loss_rgb);
            atomicAdd(loss + 1, loss_q);
        }
        if (O.counters) {
            atomicAdd(O.counters, tc);
            atomicAdd(O.counters + 1, tv);
        }
    }
}

// ---------------------------------------------------------------------------
// Scene packing, activation, camera rays, start-cell location.
// ---------------------------------------------------------------------------
// Positions that are not fp32-exact (positions_f64): the fp32 copies differ
// from the sites by <= u X per coordinate (X = the largest |coordinate| of
// the cell and its neighbours), which adds <= 4uX to the denominator error
// and <= uX (6 Hm + 2 N + 2) to the numerator error of exit_face_f32's
// bound.  Storing n1max = N + 2 max(X, 1/4) covers both: the bound's own
// terms grow by 16uX and 16uX Hm + 8uNX + 8uX^2 >= uX (6 Hm + 2 N + 2).
__device__ __forceinline__ float pos64_widen(double xabs) {
    return (float)(2.0 * fmax(xabs, 0.25)) * (1.0f + 0x1p-20f);
}

// Packed edge rows (rfb_device.cuh, exit_face_f32), one row per 16-lane
// group so the record stores coalesce: packed row u holds site i = pk_id[u];
// for each CSR neighbour j of i, in the reference's CSR order (ties resolve
// as in the reference), {fl32(x_j), packed index of j}, the same index in
// enbr, and an all-NaN pad when the degree is odd; then the header cells[u]
// (k0 = kp0 padded start, k1 = kp0 + degree, n1max >= max |n|_1 of the fp32
// n = fl32(x_j) - fl32(x_i) rounded up, widened for fp64 sites).
// kc0: the row's start in the CSR (nbr64 or nbr32).
constexpr int kRowLanes = 16;
__device__ __forceinline__ void pack_row(const double *pos, int64_t u, int64_t i,
                                         const int64_t *nbr64, const int32_t *nbr32, int64_t kc0,
                                         int32_t deg, int64_t kp0, float4 *edges, int32_t *enbr,
                                         CellHdr *cells, const double *sigma, int pos64, int gl,
                                         const int32_t *pk_of) {
    const unsigned gmask = 0xffffu << (threadIdx.x & 16);
    const float xi = (float)pos[3 * i], yi = (float)pos[3 * i + 1], zi = (float)pos[3 * i + 2];
    float n1max = 0.f;
    double xabs = fmax(fabs(pos[3 * i]), fmax(fabs(pos[3 * i + 1]), fabs(pos[3 * i + 2])));
    for (int32_t t = gl; t < deg; t += kRowLanes) {
        const int64_t j = nbr64 ? nbr64[kc0 + t] : (int64_t)nbr32[kc0 + t];
        const float xj = (float)pos[3 * j], yj = (float)pos[3 * j + 1], zj = (float)pos[3 * j + 2];
        const int32_t pj = pk_of ? pk_of[j] : (int32_t)j;
        edges[kp0 + t] = make_float4(xj, yj, zj, __int_as_float(pj));
        enbr[kp0 + t] = pj;
        const float nx = xj - xi, ny = yj - yi, nz = zj - zi;
        n1max = fmaxf(n1max, fabsf(nx) + fabsf(ny) + fabsf(nz));
        xabs = fmax(xabs, fmax(fabs(pos[3 * j]), fmax(fabs(pos[3 * j + 1]), fabs(pos[3 * j + 2]))));
    }
#pragma unroll
    for (int off = kRowLanes / 2; off > 0; off >>= 1) {
        n1max = fmaxf(n1max, __shfl_xor_sync(gmask, n1max, off, kRowLanes));
        xabs = fmax(xabs, __shfl_xor_sync(gmask, xabs, off, kRowLanes));
    }
    if (gl != 0) return;
    if (deg & 1) {  // pad to an even row: rejected as back-facing by every ray (NaN)
        const float qnan = __int_as_float(0x7fffffff);
        edges[kp0 + deg] = make_float4(qnan, qnan, qnan, qnan);
        enbr[kp0 + deg] = -1;
    }
    n1max *= 1.0f + 0x1p-20f;
    if (pos64) n1max += pos64_widen(xabs);
    // rounded up to a multiple of 32 ulp: the low 5 bits are free for k_cull_rows'
    // dropped-neighbour count (the walk adds it back to its visit counter)
    n1max = __uint_as_float((__float_as_uint(n1max) + 31u) & ~31u);
    CellHdr h;
    h.x = xi;
    h.y = yi;
    h.z = zi;
    h.k0 = (int32_t)kp0;
    h.sigma = sigma ? sigma[i] : cells[u].sigma;
    h.k1 = (int32_t)(kp0 + deg);
    h.n1max = n1max;
    cells[u] = h;
}

// ---- the packed order: sites sorted along a Morton curve (10 bits per axis
// over the bounding box), so cells a ray visits in turn sit near each other
// in the packed arrays (measured -4% per 1080p frame) ----------
__device__ __forceinline__ unsigned f2ord(float f) {  // order-preserving float -> uint
    const unsigned b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float ord2f(unsigned o) {
    return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}
__global__ void k_bbox(const double *pos, int64_t n, unsigned *mm) {  // mm: 3 min, 3 max
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned lo[3] = {0xffffffffu, 0xffffffffu, 0xffffffffu}, hi[3] = {0u, 0u, 0u};
    if (i < n)
        for (int a = 0; a < 3; ++a) lo[a] = hi[a] = f2ord((float)pos[3 * i + a]);
    for (int a = 0; a < 3; ++a) {
        const unsigned l = __reduce_min_sync(0xffffffffu, lo[a]);
        const unsigned h = __reduce_max_sync(0xffffffffu, hi[a]);
        if ((threadIdx.x & 31) == 0) {
            atomicMin(mm + a, l);
            atomicMax(mm + 3 + a, h);
        }
    }
}
__device__ __forceinline__ uint32_t spread3(uint32_t x) {
    x &= 0x3ffu;
    x = (x | (x << 16)) & 0x30000ffu;
    x = (x | (x << 8)) & 0x300f00fu;
    x = (x | (x << 4)) & 0x30c30c3u;
    x = (x | (x << 2)) & 0x9249249u;
    return x;
}
__global__ void k_morton(const double *pos, int64_t n, const unsigned *mm, uint32_t *key,
                         int32_t *val) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float lo[3], ext = 0.f;
    for (int a = 0; a < 3; ++a) {
        lo[a] = ord2f(mm[a]);
        ext = fmaxf(ext, ord2f(mm[3 + a]) - lo[a]);
    }
    const float sc = ext > 0.f ? 1023.0f / ext : 0.f;
    uint32_t q[3];
    for (int a = 0; a < 3; ++a)
        q[a] = (uint32_t)fminf(fmaxf(((float)pos[3 * i + a] - lo[a]) * sc, 0.f), 1023.f);
    key[i] = spread3(q[0]) | (spread3(q[1]) << 1) | (spread3(q[2]) << 2);
    val[i] = (int32_t)i;
}
__global__ void k_invert(const int32_t *pk_id, int64_t n, int32_t *pk_of) {
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u < n) pk_of[pk_id[u]] = (int32_t)u;
}
// padded degree of packed row u (its site's CSR degree rounded up to even)
__global__ void k_pad_deg(const int64_t *off64, const int32_t *pk_id, int64_t n, int32_t *pd) {
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n) return;
    const int64_t i = pk_id ? pk_id[u] : u;
    pd[u] = (int32_t)((off64[i + 1] - off64[i] + 1) & ~1);
}

__global__ void k_pack_sites(const double *pos, const double *sigma, const double *sh, int64_t n,
                             const int64_t *off64, double4 *site4, int32_t *off32, float *sh32,
                             const int32_t *pk_of) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > n) return;
    off32[i] = (int32_t)off64[i];
    if (i == n) return;
    site4[i] = make_double4(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2], sigma[i]);
    if (sh32) {
        float *row = sh32 + (pk_of ? (int64_t)pk_of[i] : i) * 48;
        for (int k = 0; k < 16; ++k)
            for (int ch = 0; ch < 3; ++ch)
                row[16 * ch + k] = (float)sh[i * 48 + 3 * k + ch];  // channel-major
    }
}

// kp0: exclusive prefix sum of the padded degrees in packed order (row starts,
// always even).  One row per 16 lanes.
__global__ void k_pack_rows(const double *pos, const double *sigma, int64_t n,
                            const int64_t *off64, const int64_t *nbr64, const int32_t *kp0,
                            const int32_t *pk_id, const int32_t *pk_of, CellHdr *cells,
                            float4 *edges, int32_t *enbr, int pos64) {
    const int64_t u = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kRowLanes;
    if (u >= n) return;
    const int64_t i = pk_id ? pk_id[u] : u;
    pack_row(pos, u, i, nbr64, nullptr, off64[i], (int32_t)(off64[i + 1] - off64[i]), kp0[u],
             edges, enbr, cells, sigma, pos64, threadIdx.x & (kRowLanes - 1), pk_of);
}

__global__ void k_pack_edges(const int64_t *nbr64, int64_t E, int32_t *nbr32) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < E) nbr32[k] = (int32_t)nbr64[k];
}

// foam.py:22-25 (device libm; may differ from numpy's log1p/exp by 1 ulp).
__global__ void k_softplus(const double *raw, int64_t n, double *out, double4 *site4,
                           CellHdr *cells, const int32_t *pk_of) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double x = raw[i];
    double v = fmax(x, 0.0) + log1p(exp(-fabs(10.0 * x))) / 10.0;
    if (out) out[i] = v;
    if (site4) site4[i].w = v;
    if (cells) cells[pk_of ? pk_of[i] : i].sigma = v;
}

__global__ void k_camera_rays(CameraParams cam, int64_t begin, int64_t count, double *dirs) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= count) return;
    int64_t p = begin + k;
    double dx, dy, dz;
    pinhole_dir(cam, p / cam.width, p % cam.width, dx, dy, dz);
    dirs[3 * k] = dx;
    dirs[3 * k + 1] = dy;
    dirs[3 * k + 2] = dz;
}

// rays.py:139-176: continue rays across an effect plane (mirror / Snell
// refraction with total internal reflection falling back to the mirror).
__device__ __forceinline__ void reflect_dir(double dx, double dy, double dz, double nx, double ny,
                                            double nz, double *o) {
    const double dn = dx * nx + dy * ny + dz * nz;
    o[0] = dx - 2.0 * dn * nx;
    o[1] = dy - 2.0 * dn * ny;
    o[2] = dz - 2.0 * dn * nz;
}

__global__ void k_effect_rays(const double *origins, const double *dirs, const double *t_at,
                              int64_t m, double nx, double ny, double nz, int32_t kind, double eta,
                              double *out_o, double *out_d) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const double dx = dirs[3 * i], dy = dirs[3 * i + 1], dz = dirs[3 * i + 2];
    const double t = t_at[i];
    double o[3];
    if (kind == 0) {
        reflect_dir(dx, dy, dz, nx, ny, nz, o);
    } else {
        double cos_i = -(dx * nx + dy * ny + dz * nz);
        double ex = eta;
        if (cos_i < 0.0) {  // back side: flip the normal, invert the ratio (rays.py:153-155)
            nx = -nx;
            ny = -ny;
            nz = -nz;
            ex = 1.0 / eta;
            cos_i = -(dx * nx + dy * ny + dz * nz);
        }
        const double ratio = 1.0 / ex;
        const double sin2_t = ratio * ratio * (1.0 - cos_i * cos_i);
        if (sin2_t > 1.0) {
            reflect_dir(dx, dy, dz, nx, ny, nz, o);
        } else {
            const double cos_t = sqrt(1.0 - sin2_t);
            const double c = ratio * cos_i - cos_t;
            o[0] = ratio * dx + c * nx;
            o[1] = ratio * dy + c * ny;
            o[2] = ratio * dz + c * nz;
            const double l = sqrt(o[0] * o[0] + o[1] * o[1] + o[2] * o[2]);
            o[0] /= l;
            o[1] /= l;
            o[2] /= l;
        }
    }
    const double l = sqrt(o[0] * o[0] + o[1] * o[1] + o[2] * o[2]);  // apply_effect renormalises
    out_d[3 * i] = o[0] / l;
    out_d[3 * i + 1] = o[1] / l;
    out_d[3 * i + 2] = o[2] / l;
    out_o[3 * i] = origins[3 * i] + t * dx;
    out_o[3 * i + 1] = origins[3 * i + 1] + t * dy;
    out_o[3 * i + 2] = origins[3 * i + 2] + t * dz;
}

struct LocScene {
    const double4 *site4;
    const int32_t *off, *nbr;
};

// Greedy point location on the Delaunay graph: move to the neighbour with
// the smallest (distance, id) while it beats the current site.  Same
// distance expression and lowest-id tie rule as adjacency.py:194-200.
__device__ int32_t locate_one(const LocScene &S, double qx, double qy, double qz, int32_t cur) {
    auto dist = [&](int32_t i) {
        double4 p = ld_site(S.site4 + i);
        double dx = p.x - qx, dy = p.y - qy, dz = p.z - qz;
        return dx * dx + dy * dy + dz * dz;
    };
    double dcur = dist(cur);
    for (;;) {
        int32_t best = cur;
        double dbest = dcur;
        int32_t k1 = __ldg(S.off + cur + 1);
        for (int32_t k = __ldg(S.off + cur); k < k1; ++k) {
            int32_t j = __ldg(S.nbr + k);
            double d = dist(j);
            if (d < dbest || (d == dbest && j < best)) {
                dbest = d;
                best = j;
            }
        }
        if (best == cur) return cur;
        cur = best;
        dcur = dbest;
    }
}

__global__ void k_locate(LocScene S, const double *qs, int64_t m, int32_t seed, int32_t *out) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < m) out[k] = locate_one(S, qs[3 * k], qs[3 * k + 1], qs[3 * k + 2], seed);
}

// Seed grid for the greedy walk (the walk is exact from any seed; the seed
// only shortens it, like the reference's bucket grid, adjacency.py:140-203):
// every grid cell holds the largest site id inside it, or -1.
struct HintGrid {
    double lo[3], cell;
    int dims[3];
    const int32_t *hint;
};

__device__ __forceinline__ int hint_axis(double v, double lo, double cell, int dim) {
    const double f = floor((v - lo) / cell);
    return f < 0.0 ? 0 : (f > dim - 1 ? dim - 1 : (int)f);
}

__global__ void k_hint_scatter(const double4 *site4, int64_t n, HintGrid g, int32_t *hint) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double4 p = site4[i];
    const int x = hint_axis(p.x, g.lo[0], g.cell, g.dims[0]);
    const int y = hint_axis(p.y, g.lo[1], g.cell, g.dims[1]);
    const int z = hint_axis(p.z, g.lo[2], g.cell, g.dims[2]);
    atomicMax(hint + ((int64_t)z * g.dims[1] + y) * g.dims[0] + x, (int32_t)i);
}

__global__ void k_locate_hinted(LocScene S, const double *qs, int64_t m, HintGrid g, int32_t seed,
                                int32_t *out) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= m) return;
    const double qx = qs[3 * k], qy = qs[3 * k + 1], qz = qs[3 * k + 2];
    const int x = hint_axis(qx, g.lo[0], g.cell, g.dims[0]);
    const int y = hint_axis(qy, g.lo[1], g.cell, g.dims[1]);
    const int z = hint_axis(qz, g.lo[2], g.cell, g.dims[2]);
    int32_t start = -1;
    for (int r = 0; r <= 2 && start < 0; ++r)  // nearest non-empty cell within 2 rings
        for (int dz = -r; dz <= r && start < 0; ++dz)
            for (int dy = -r; dy <= r && start < 0; ++dy)
                for (int dx = -r; dx <= r && start < 0; ++dx) {
                    const int cx = x + dx, cy = y + dy, cz = z + dz;
                    if (cx < 0 || cy < 0 || cz < 0 || cx >= g.dims[0] || cy >= g.dims[1] ||
                        cz >= g.dims[2])
                        continue;
                    start = __ldg(g.hint + ((int64_t)cz * g.dims[1] + cy) * g.dims[0] + cx);
                }
    out[k] = locate_one(S, qx, qy, qz, start >= 0 ? start : seed);
}

// Exact nearest site of one query point by a full-device scan (shared-origin
// cameras: one query per frame, render.py:78-82): pass 1 takes the minimum
// squared distance (non-negative doubles order like their bit patterns),
// pass 2 the lowest id attaining it -- the reference's tie rule, with no
// dependence on the CSR (so a stale adjacency cannot change the answer).
__device__ __forceinline__ double qdist(const double4 *site4, int64_t i, double qx, double qy,
                                        double qz) {
    double4 p = ld_site(site4 + i);
    double dx = p.x - qx, dy = p.y - qy, dz = p.z - qz;
    return dx * dx + dy * dy + dz * dz;
}

__global__ void k_nearest_dist(const double4 *site4, int64_t n, double qx, double qy, double qz,
                               unsigned long long *best) {
    unsigned long long m = ~0ull;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        unsigned long long b = __double_as_longlong(qdist(site4, i, qx, qy, qz));
        m = b < m ? b : m;
    }
    for (int off = 16; off > 0; off >>= 1) {
        unsigned long long o = __shfl_xor_sync(0xffffffffu, m, off);
        m = o < m ? o : m;
    }
    if ((threadIdx.x & 31) == 0) atomicMin(best, m);
}

__global__ void k_nearest_id(const double4 *site4, int64_t n, double qx, double qy, double qz,
                             const unsigned long long *best, int32_t *out) {
    const unsigned long long b = *best;
    int32_t m = 0x7fffffff;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        if ((unsigned long long)__double_as_longlong(qdist(site4, i, qx, qy, qz)) == b) {
            m = (int32_t)i;
            break;  // grid-stride order: the first hit of this thread is its lowest id
        }
    }
    m = __reduce_min_sync(0xffffffffu, (unsigned)m);
    if ((threadIdx.x & 31) == 0) atomicMin(out, m);
}

static void nearest_point(const rfb_scene *s, double qx, double qy, double qz, void *tmp8,
                          int32_t *out, cudaStream_t st) {
    unsigned long long *best = reinterpret_cast<unsigned long long *>(tmp8);
    const double4 *site4 = reinterpret_cast<const double4 *>(s->site4);
    const unsigned grid = (unsigned)std::min<int64_t>((s->n_sites + 255) / 256, 148 * 8);
    cudaMemsetAsync(best, 0xff, sizeof(unsigned long long), st);
    cudaMemsetAsync(out, 0x7f, sizeof(int32_t), st);
    k_nearest_dist<<<grid, 256, 0, st>>>(site4, s->n_sites, qx, qy, qz, best);
    k_nearest_id<<<grid, 256, 0, st>>>(site4, s->n_sites, qx, qy, qz, best, out);
}

// ---------------------------------------------------------------------------
// Gradient post-processing + Adam (optim/train.py:195-209, optim/adam.py:15-31)
// One fused elementwise pass over the flat gradient buffer after the
// all-reduce: d_raw = dsigma * sigmoid(10 raw), SH warm-up mask (bands 1..15
// zeroed), clip to +-clip, then Adam with bias correction on the fp64
// parameters, in the reference's operation order (bias corrections are host
// scalars, like numpy's beta ** step).
// ---------------------------------------------------------------------------
struct AdamArgs {
    double lr, b1, b2, eps, bc1, bc2;  // bc = 1 - beta ** step
};

__device__ __forceinline__ void adam1(double &p, double g, double &m, double &v,
                                      const AdamArgs &a) {
    m = m * a.b1;
    m = m + (1.0 - a.b1) * g;
    v = v * a.b2;
    v = v + (1.0 - a.b2) * g * g;
    const double m_hat = m / a.bc1;
    const double v_hat = v / a.bc2;
    p = p - a.lr * m_hat / (sqrt(v_hat) + a.eps);
}

__device__ __forceinline__ double clipd(double x, double c) { return fmin(fmax(x, -c), c); }

__global__ void k_post_adam(int64_t n, const float *g4, const float *gsh, double *pos,
                            double *raw, double *sh, double *m_pos, double *v_pos, double *m_raw,
                            double *v_raw, double *m_sh, double *v_sh, double clip, int sh_warmup,
                            int update_pos, AdamArgs a_pos, AdamArgs a_raw, AdamArgs a_sh,
                            float *sh32, unsigned *absmax_bits, const int32_t *pk_of) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n * 52) return;
    if (t < n * 48) {  // SH coefficient t = i*48 + k*3 + ch
        double g = (double)gsh[t];
        const int r = (int)(t % 48);
        if (sh_warmup && r >= 3) g = 0.0;  // train.py:197-198
        adam1(sh[t], clipd(g, clip), m_sh[t], v_sh[t], a_sh);
        // the walk's fp32 channel-major copy (k_refresh_sh32's layout), written
        // here so the refresh does not re-read the fp64 rows
        if (sh32) {  // row of site i = t / 48 in the packed order
            const int64_t i = t / 48;
            sh32[(pk_of ? (int64_t)pk_of[i] : i) * 48 + (r % 3) * 16 + r / 3] = (float)sh[t];
        }
        if (absmax_bits) {  // running max |sh| (non-negative floats order like their bits)
            const unsigned bits = __float_as_uint(__double2float_ru(fabs(sh[t])));
            const unsigned am = __activemask();
            const unsigned mx = __reduce_max_sync(am, bits);
            // the bound only grows, and rarely: skip the (single-address) atomic
            // unless this warp's maximum exceeds the value already stored
            if ((int)(threadIdx.x & 31) == __ffs(am) - 1 && mx > __ldcg(absmax_bits))
                atomicMax(absmax_bits, mx);
        }
        return;
    }
    const int64_t u = t - n * 48;
    if (u < n) {  // raw density: d_raw = dsigma * softplus_grad(raw) (render.py:220)
        const double x = raw[u];
        const double d_raw = (double)g4[4 * u + 3] * (1.0 / (1.0 + exp(-10.0 * x)));
        adam1(raw[u], clipd(d_raw, clip), m_raw[u], v_raw[u], a_raw);
        return;
    }
    const int64_t w = u - n;  // position component w = i*3 + c
    if (update_pos && w < 3 * n) {
        const int64_t i = w / 3, c = w % 3;
        adam1(pos[w], clipd((double)g4[4 * i + c], clip), m_pos[w], v_pos[w], a_pos);
    }
}

// Refresh the kernel arrays from updated parameters (render.py:49-54 on
// device): site4 = {pos, softplus(raw)}, packed headers' sigma.
__global__ void k_refresh_scene(int64_t n, const double *pos, const double *raw, double4 *site4,
                                CellHdr *cells, const int32_t *pk_of) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double x = raw[i];
    const double sig = fmax(x, 0.0) + log1p(exp(-fabs(10.0 * x))) / 10.0;
    site4[i] = make_double4(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2], sig);
    if (cells) cells[pk_of ? pk_of[i] : i].sigma = sig;
}

// Moved fp64 sites: the fp32 copies, the rows' records and the widened bounds
// (k_pack_rows' rules; the row starts are unchanged), one row per 16 lanes.
__global__ void k_refresh_rows(int64_t n, const double *pos, CellHdr *cells, const int32_t *off,
                               const int32_t *nbr, float4 *edges, int32_t *enbr,
                               const int32_t *pk_id, const int32_t *pk_of) {
    const int64_t u = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kRowLanes;
    if (u >= n) return;
    const int64_t i = pk_id ? pk_id[u] : u;
    pack_row(pos, u, i, nullptr, nbr, off[i], off[i + 1] - off[i], cells[u].k0, edges, enbr,
             cells, nullptr, 1, threadIdx.x & (kRowLanes - 1), pk_of);
}

// ---------------------------------------------------------------------------
// View culling (rfb_cull_scene).  Every ray of a frame has a direction d that
// is a positive combination of the cone generators c_k (a pinhole frame: the
// four corner-pixel directions, since R (u, v, -1) is linear in the pixel
// centre (u, v) over the image rectangle).  A neighbour with
// c_k . n < -1e-9 |n|_1 for every k (n = x_j - x_i) then has d . n < -1e-9 |n|_1
// for every ray, far beyond the fp64 rounding of the reference's
// `denom = d . n` (~1e-15 |n|_1), so kernels.py:118-119 (`if denom <= 0:
// continue`) skips it for every ray of the frame: it can never be the exit
// face.  The culled copy of the packed rows keeps the other neighbours in CSR
// order (so exact ties resolve as before), pads to even with a NaN record and
// stores the number dropped (<= 31; a row that would drop more is copied
// whole) in n1max's low 5 bits, which pack_row leaves zero; the walk adds it
// back to its neighbour-visit counter.  fp64 sites (positions_f64): the
// records are rounded copies (<= 2^-24 X per coordinate, X the largest
// |coordinate|), covered by widening the margin by 2^-21 X.  One row per 16
// lanes; the kept records are compacted with a ballot.
// ---------------------------------------------------------------------------
constexpr int kCullMaxDirs = 8;     // generators of one cone (rfb_cull_scene)
constexpr int kCullMaxRegions = 32;  // regions of a view (rfb_cull_view)
constexpr int kCullMaxGen = 72;  // (rx + 1)(ry + 1) for rx * ry <= 32
constexpr int kCullMaxDrop = 31;
struct CullCone {
    // grid mode (rx > 0): the (rx + 1) x (ry + 1) region-corner directions, row-major;
    // region (ix, iy) is the cone of corners (ix, iy), (ix + 1, iy), (ix, iy + 1),
    // (ix + 1, iy + 1).  Single-cone mode (rx == 0): nd generators, one region.
    float c[kCullMaxGen][3];  // unit vectors (fp32: the margin covers their rounding)
    int32_t rx, ry, nd;
    int64_t stride;  // edge slots between region copies
};
// Record e of the row of a cell at (xi, yi, zi): bit k set when the face is back-facing
// with margin for generator k.  fp32: n = fl(x_j - x_i) and the dot product round by
// <= 8 2^-24 |n|_1 (|c| = 1), so `dot < -2^-18 |n|_1` implies an exact c . n below
// -3e-6 |n|_1 (>> the 1e-9 the reference's fp64 `denom` needs); fp64 sites: + 2^-21 X.
__device__ __forceinline__ uint64_t cull_bits(const CullCone &cone, int nc, float xi, float yi,
                                              float zi, float xa, const float4 &e, int pos64) {
    const float nx = e.x - xi, ny = e.y - yi, nz = e.z - zi;
    float marg = 0x1p-18f * (fabsf(nx) + fabsf(ny) + fabsf(nz));
    if (pos64) marg += 0x1p-21f * fmaxf(xa, fmaxf(fabsf(e.x), fmaxf(fabsf(e.y), fabsf(e.z))));
    uint64_t b = 0;
    for (int k = 0; k < nc; ++k) {
        const float d = __fmaf_rn(cone.c[k][2], nz, __fmaf_rn(cone.c[k][1], ny, cone.c[k][0] * nx));
        b |= (uint64_t)(d < -marg) << k;
    }
    return b;
}
// bit p of the result: region p culled (grid: bit iy (rx + 1) + ix)
__device__ __forceinline__ uint64_t region_bits(const CullCone &cone, uint64_t b) {
    if (cone.rx == 0) return b == (1ull << cone.nd) - 1 ? 1ull : 0ull;
    const int w = cone.rx + 1;
    return b & (b >> 1) & (b >> w) & (b >> (w + 1));
}
#ifndef RFB_CULL_ROWS
#define RFB_CULL_ROWS 1  // rows per 16-lane group (their loads issued together)
#endif
#ifndef RFB_CULL_MINB
#define RFB_CULL_MINB 6  // resident 256-thread blocks per SM (memory-level parallelism)
#endif
constexpr int kCullRows = RFB_CULL_ROWS;
// Compile-time region grids (RX > 0, (RX + 1)(RY + 1) <= 32 corners): unrolled corner
// tests on a 32-bit mask and constant shifts; RX == 0: the runtime shape (any grid, or one
// cone of nd generators).
template <int RX, int RY>
__device__ __forceinline__ uint32_t region_mask_t(const CullCone &cone, float xi, float yi,
                                                  float zi, float xa, const float4 &e, int pos64) {
    constexpr int W = RX + 1, NC = (RX + 1) * (RY + 1);
    static_assert(NC <= 32, "corner mask is 32 bits");
    const float nx = e.x - xi, ny = e.y - yi, nz = e.z - zi;
    float marg = 0x1p-18f * (fabsf(nx) + fabsf(ny) + fabsf(nz));
    if (pos64) marg += 0x1p-21f * fmaxf(xa, fmaxf(fabsf(e.x), fmaxf(fabsf(e.y), fabsf(e.z))));
    uint32_t b = 0;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
        const float d = __fmaf_rn(cone.c[k][2], nz, __fmaf_rn(cone.c[k][1], ny, cone.c[k][0] * nx));
        b |= (d < -marg) ? (1u << k) : 0u;
    }
    const uint32_t rb = b & (b >> 1) & (b >> W) & (b >> (W + 1));
    uint32_t m = 0;
#pragma unroll
    for (int iy = 0; iy < RY; ++iy)
#pragma unroll
        for (int ix = 0; ix < RX; ++ix) m |= ((rb >> (iy * W + ix)) & 1u) << (iy * RX + ix);
    return m;
}
// bit r: region r culls the record (from cull_bits' generator bits)
__device__ __forceinline__ uint32_t region_mask(const CullCone &cone, int nr, uint64_t b) {
    const uint64_t rb = region_bits(cone, b);
    if (cone.rx == 0) return (uint32_t)(rb & 1u);
    uint32_t m = 0;
    int r = 0;
    for (int iy = 0; iy < cone.ry; ++iy)
        for (int ix = 0; ix < cone.rx; ++ix, ++r)
            m |= (uint32_t)((rb >> (iy * (cone.rx + 1) + ix)) & 1u) << r;
    return m;
}
template <int RX, int RY>
__global__ void __launch_bounds__(256, RFB_CULL_MINB) k_cull_rows(const CellHdr *cells, const float4 *edges, int64_t n, CullCone cone,
                            int pos64, CellHdr *cells_out, float4 *edges_out) {
    const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kRowLanes;
    if (g * kCullRows >= n) return;  // whole 16-lane groups
    const int gl = threadIdx.x & (kRowLanes - 1);
    const unsigned gshift = threadIdx.x & 16;
    const unsigned gmask = 0xffffu << gshift;
    const unsigned lt = (1u << gl) - 1u;
    const int nc = cone.rx ? (cone.rx + 1) * (cone.ry + 1) : cone.nd;
    const int nr = RX > 0 ? RX * RY : (cone.rx ? cone.rx * cone.ry : 1);
    const float qnan = __int_as_float(0x7fffffff);
    const float4 pad = make_float4(qnan, qnan, qnan, qnan);
    // the group's rows: headers, then the (<= 2 per lane) records of every short row,
    // all loads in flight together (the kernel is latency-bound otherwise)
    CellHdr h[kCullRows];
    float4 e0[kCullRows], e1[kCullRows];
#pragma unroll
    for (int q = 0; q < kCullRows; ++q) {
        const int64_t u = g * kCullRows + q;
        if (u < n) h[q] = cells[u];
        else h[q].k0 = h[q].k1 = 0;
    }
#pragma unroll
    for (int q = 0; q < kCullRows; ++q) {
        const int32_t deg = h[q].k1 - h[q].k0;
        e0[q] = gl < deg ? edges[h[q].k0 + gl] : pad;
        e1[q] = gl + kRowLanes < deg && deg <= kCullMaxDrop ? edges[h[q].k0 + kRowLanes + gl] : pad;
    }
#pragma unroll
    for (int q = 0; q < kCullRows; ++q) {
        const int64_t u = g * kCullRows + q;
        if (u >= n) break;
        const CellHdr hq = h[q];
        const float xa = fmaxf(fabsf(hq.x), fmaxf(fabsf(hq.y), fabsf(hq.z)));
        const int32_t deg = hq.k1 - hq.k0;
        auto header = [&](int r, int64_t k0, int32_t m) {
            CellHdr o = hq;
            o.k0 = (int32_t)k0;
            o.k1 = (int32_t)(k0 + m);
            o.n1max = __uint_as_float((__float_as_uint(hq.n1max) & ~31u) | (unsigned)(deg - m));
            cells_out[r * n + u] = o;
        };
        if (deg <= kCullMaxDrop) {
            // every region from the same bits of the (<= 2) records each lane holds:
            // bit r of m0 / m1 = the record is dropped from region r's copy
            const bool real0 = gl < deg, real1 = gl + kRowLanes < deg;
            uint32_t m0 = ~0u, m1 = ~0u;
            if constexpr (RX > 0) {
                if (real0) m0 = region_mask_t<RX, RY>(cone, hq.x, hq.y, hq.z, xa, e0[q], pos64);
                if (real1) m1 = region_mask_t<RX, RY>(cone, hq.x, hq.y, hq.z, xa, e1[q], pos64);
            } else {
                if (real0) m0 = region_mask(cone, nr, cull_bits(cone, nc, hq.x, hq.y, hq.z, xa, e0[q], pos64));
                if (real1) m1 = region_mask(cone, nr, cull_bits(cone, nc, hq.x, hq.y, hq.z, xa, e1[q], pos64));
            }
            int32_t my_m = 0;  // lane r < nr: region r's kept count (it writes that header)
            float4 *out = edges_out + hq.k0;
#pragma unroll
            for (int r = 0; r < nr; ++r, out += cone.stride) {
                const bool k0b = !((m0 >> r) & 1u), k1b = !((m1 >> r) & 1u);
                const unsigned b0 = (__ballot_sync(gmask, k0b) >> gshift) & 0xffffu;
                const unsigned b1 = (__ballot_sync(gmask, k1b) >> gshift) & 0xffffu;
                const int32_t n0 = __popc(b0), m = n0 + __popc(b1);
                if (k0b) out[__popc(b0 & lt)] = e0[q];
                if (k1b) out[n0 + __popc(b1 & lt)] = e1[q];
                // the odd row's one pad (filling the row's whole original extent so
                // every sector is written measured slower: 0.60 vs 0.56 ms at 4 x 2)
                if (gl == 0 && (m & 1)) out[m] = pad;
                my_m = gl == r ? m : my_m;
            }
            if (gl < nr) header(gl, gl * cone.stride + hq.k0, my_m);
            continue;
        }
        // long rows (rare): per region, over chunks of 16; a region that would drop more
        // than 31 records (the n1max field holds 5 bits) keeps the row whole
        int ix = 0, iy = 0;
        for (int r = 0; r < nr; ++r) {
            const int p = cone.rx ? iy * (cone.rx + 1) + ix : 0;
            const int64_t k0 = r * cone.stride + hq.k0;
            int32_t m = 0;
            for (int pass = 0; pass < 2; ++pass) {
                m = 0;
                for (int32_t t0 = 0; t0 < deg; t0 += kRowLanes) {
                    const int32_t t = t0 + gl;
                    const bool real = t < deg;
                    const float4 e = real ? edges[hq.k0 + t] : pad;
                    bool keep = real;
                    if (real && pass == 0)
                        keep = !((region_bits(cone, cull_bits(cone, nc, hq.x, hq.y, hq.z, xa, e,
                                                              pos64)) >> p) & 1);
                    const unsigned bal = (__ballot_sync(gmask, keep) >> gshift) & 0xffffu;
                    if (keep) edges_out[k0 + m + __popc(bal & lt)] = e;
                    m += __popc(bal);
                }
                if (deg - m <= kCullMaxDrop) break;
            }
            for (int32_t t = m + gl; t < ((deg + 1) & ~1); t += kRowLanes) edges_out[k0 + t] = pad;
            if (gl == 0) header(r, k0, m);
            if (++ix == cone.rx) {
                ix = 0;
                ++iy;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Host helpers
// ---------------------------------------------------------------------------
static int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

template <int PACKED>
static SceneView<PACKED> view(const rfb_scene *s) {
    SceneView<PACKED> v;
    v.hdr = reinterpret_cast<const CellHdr *>(s->cells);
    v.edge = reinterpret_cast<const float4 *>(s->edges);
    v.enbr = s->edge_nbr;
    v.pk_of = s->pk_of;
    v.pk_id = s->pk_id;
    v.site4 = reinterpret_cast<const double4 *>(s->site4);
    v.off = s->offsets;
    v.nbr = s->neighbors;
    v.sh32 = s->sh32;
    v.sh = s->sh;
    v.sh_absmax = s->sh_absmax;
    v.absmax_p = s->sh_absmax_dev;
    v.bg[0] = s->background[0];
    v.bg[1] = s->background[1];
    v.bg[2] = s->background[2];
    v.n_sites = s->n_sites;
    v.n_edges = s->n_edges;
    v.view_rx = s->view_rx > 0 ? s->view_rx : 0;
    v.view_ry = s->view_rx > 0 ? s->view_ry : 0;
    v.n_views = s->view_rx > 0 ? s->view_rx * s->view_ry : 1;
    v.edge_slots = s->view_rx > 0 ? (int64_t)v.n_views * RFB_VIEW_STRIDE(s->n_sites, s->n_edges)
                                  : (int64_t)RFB_PACKED_EDGE_SLOTS(s->n_sites, s->n_edges);
    return v;
}

static LocScene loc_scene(const rfb_scene *s) {
    return LocScene{reinterpret_cast<const double4 *>(s->site4), s->offsets, s->neighbors};
}

static FwdOut dev_out(const rfb_fwd_out *o) {
    FwdOut d;
    d.rgb = o->rgb;
    d.residual = o->residual;
    d.wsum = o->wsum;
    d.status = o->status;
    d.nseg = o->nseg;
    d.ray_counters = o->ray_counters;
    d.counters = o->counters;
    d.f64 = o->f64_outputs;
    d.seg_cap = o->seg_capacity;
    d.seg_cells = o->seg_cells;
    d.seg_t0 = o->seg_t0;
    d.seg_t1 = o->seg_t1;
    d.seg_first = o->seg_count > 0 ? o->seg_first : 0;
    d.seg_count = o->seg_count > 0 ? o->seg_count : INT64_MAX;
    return d;
}

static bool scene_ok(const rfb_scene *s) {
    if (!s || !s->site4 || !s->offsets || !s->neighbors || !s->sh || s->n_sites <= 0 ||
        s->n_sites >= (1 << 29) || (s->sh_degree != 0 && s->sh_degree != 3))
        return false;
    if (s->packed && (!s->cells || !s->edges || !s->edge_nbr || !s->sh32)) return false;
    if (s->view_rx < 0 || s->view_ry < 0 || (s->view_rx > 0) != (s->view_ry > 0) ||
        s->view_rx * s->view_ry > kCullMaxRegions || (s->view_rx > 0 && !s->packed))
        return false;
    if (s->packed && ((reinterpret_cast<uintptr_t>(s->cells) | reinterpret_cast<uintptr_t>(s->edges) |
                       reinterpret_cast<uintptr_t>(s->sh32)) & 31u))
        return false;  // 256-bit loads
    return true;
}

static bool out_ok(const rfb_fwd_out *o) {
    if (!o || !o->rgb) return false;
    if (o->seg_capacity > 0 && (!o->seg_cells || !o->seg_t0 || !o->seg_t1 || o->seg_first < 0 ||
                                o->seg_count < 0))
        return false;
    return true;
}

// Shared-memory carveout for k_render: the smallest configuration that holds
// the blocks the registers allow per SM (static + 1 KB reserved each), so the rest of the SM's
// 256 KB goes to L1 for the neighbour gathers.  SH degree 3: 4 x 24.6 KB fit
// the 100 KB step (L1 156 KB; the driver's default pick was 132 KB): 21.25 ->
// 21.08 ms per config-2 frame.  SH degree 0 keeps the driver's pick (the
// 64 KB step measured 1.3% slower on config 1).
// RFB_CARVEOUT (percent of the 228 KB maximum; -1 = driver default) overrides.
template <auto K>
static void prefer_carveout() {
    // once per kernel instantiation and device (the attribute is per device;
    // concurrent host threads: the first to set the bit does the work)
    static std::atomic<unsigned long long> done{0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        (void)cudaGetLastError();
        return;
    }
    const unsigned long long bit = 1ull << (dev & 63);
    if (done.fetch_or(bit) & bit) return;
    int blocks = 0;  // what the registers allow, before any preference
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, K, 256, 0) != cudaSuccess) {
        (void)cudaGetLastError();
        return;
    }
    int pct;
    const char *e = getenv("RFB_CARVEOUT");
    if (e && *e) {
        pct = atoi(e);
    } else {
        cudaFuncAttributes a;
        if (cudaFuncGetAttributes(&a, K) != cudaSuccess) {
            (void)cudaGetLastError();
            return;
        }
        const size_t need = (size_t)std::max(blocks, 1) * (a.sharedSizeBytes + 1024);
        pct = (int)std::min<size_t>(100, (100 * need + 228 * 1024 - 1) / (228 * 1024));
    }
    if (cudaFuncSetAttribute(K, cudaFuncAttributePreferredSharedMemoryCarveout, pct) !=
        cudaSuccess) {
        (void)cudaGetLastError();
        return;
    }
    // keep the preference only if the blocks per SM are unchanged
    int after = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&after, K, 256, 0) != cudaSuccess ||
        after < blocks) {
        (void)cudaGetLastError();
        (void)cudaFuncSetAttribute(K, cudaFuncAttributePreferredSharedMemoryCarveout, -1);
    }
}

template <int G, int PACKED, class Src>
static void launch_render_g(const rfb_scene *scene, const Src &src, double eps, double log_eps,
                            double wf, int32_t sl, const FwdOut &O, unsigned long long *ctr,
                            int sm_local, cudaStream_t st) {
    SceneView<PACKED> S = view<PACKED>(scene);
    int per_sm = 0;
    if (scene->sh_degree == 0) {
        auto k = k_render<G, 0, PACKED, Src>;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 256, 0);
        k<<<num_sms() * std::max(per_sm, 1), 256, 0, st>>>(S, src, eps, log_eps, wf, sl, O, ctr,
                                                           sm_local ? num_sms() : 0);
    } else {
        auto k = k_render<G, 3, PACKED, Src>;
        prefer_carveout<k_render<G, 3, PACKED, Src>>();
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 256, 0);
        k<<<num_sms() * std::max(per_sm, 1), 256, 0, st>>>(S, src, eps, log_eps, wf, sl, O, ctr,
                                                           sm_local ? num_sms() : 0);
    }
}

template <int G, class Src>
static void launch_render_p(const rfb_scene *scene, const Src &src, double eps, double log_eps,
                            double wf, int32_t sl, const FwdOut &O, unsigned long long *ctr,
                            int sm_local, cudaStream_t st) {
    if (scene->packed && !scene->positions_f64)
        launch_render_g<G, 1>(scene, src, eps, log_eps, wf, sl, O, ctr, sm_local, st);
    else if (scene->packed && G <= 2)  // fp64 sites: widened bound (G > 2: generic walk)
        launch_render_g<G, 2>(scene, src, eps, log_eps, wf, sl, O, ctr, sm_local, st);
    else
        launch_render_g<G, 0>(scene, src, eps, log_eps, wf, sl, O, ctr, sm_local, st);
}

template <class Src>
static int launch_render(const rfb_scene *scene, const Src &src, const rfb_params *p,
                         const rfb_fwd_out *out, void *ws, size_t ws_bytes, cudaStream_t st) {
    if (!ws || ws_bytes < 256) return RFB_EINVAL;
    // counters at ws + 256: [0] global, [1 + v] per virtual SM (when the workspace has room)
    unsigned long long *ctr = reinterpret_cast<unsigned long long *>(reinterpret_cast<char *>(ws) + 256);
    const size_t sm_bytes = 8 * (size_t)(num_sms() + 1);
    int sm_local = RFB_SM_LOCAL && ws_bytes >= 256 + sm_bytes;
    if (ws_bytes < 256 + 8) ctr = reinterpret_cast<unsigned long long *>(ws);  // (legacy 256 B)
    cudaMemsetAsync(ctr, 0, sm_local ? sm_bytes : 8, st);
    FwdOut O = dev_out(out);
    double log_eps = p->epsilon > 0.0 ? std::log(p->epsilon) : 0.0;
    int g = p->lanes_per_ray;
    if (g <= 0) {
        // auto: batches too small to fill the resident threads (148 SMs x RFB_FWD_MINB x 256)
        // spread each ray over more lanes -- the largest power of two <= 8 with g * m within
        // them (measured: 128x128 frames 0.30 -> 0.15 ms with 8 lanes, 256x256 0.35 -> 0.25 ms
        // with 2, >= 480x270 best with 1; tools/sweep_fwd.py --sizes)
        const int64_t resident = (int64_t)num_sms() * RFB_FWD_MINB * 256;
        const int64_t m = src.count();
        g = 1;
        while (g < 8 && 2 * g * m <= resident) g *= 2;
    }
    const double e = p->epsilon, wf = p->width_floor;
    const int32_t sl = p->step_limit;
    switch (g) {
        case 1: launch_render_p<1>(scene, src, e, log_eps, wf, sl, O, ctr, sm_local, st); break;
        case 2: launch_render_p<2>(scene, src, e, log_eps, wf, sl, O, ctr, sm_local, st); break;
        case 4: launch_render_p<4>(scene, src, e, log_eps, wf, sl, O, ctr, sm_local, st); break;
        case 8: launch_render_p<8>(scene, src, e, log_eps, wf, sl, O, ctr, sm_local, st); break;
        case 16: launch_render_p<16>(scene, src, e, log_eps, wf, sl, O, ctr, sm_local, st); break;
        case 32: launch_render_p<32>(scene, src, e, log_eps, wf, sl, O, ctr, sm_local, st); break;
        default: return RFB_EINVAL;
    }
    return (int)cudaGetLastError();
}

static int64_t bwd_slot_bytes(int32_t step_limit, bool quant) {
    const bool compact = !quant && RFB_COMPACT_REC;
    return (int64_t)step_limit * (compact ? kCompactRecBytes : kFullRecBytes);
}

static int64_t bwd_slots_max(bool quant) {
    int per_sm = 0;
    if (quant)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_train<3, true, true, true>,
                                                      kTrainBlock, 0);
    else
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_train<3, true, true, false>,
                                                      kTrainBlock, 0);
    return (int64_t)num_sms() * std::max(per_sm, 1) * kTrainBlock;
}

// lanes per ray for a batch: 2 when the batch fills at most half the resident
// threads (65,536 random training pixels: 4.7 -> 4.1 ms), else 1
// (4 lanes per ray measured slower for training: 128x128 fwd+bwd 0.35 -> 0.47 ms)
static int train_lanes(int64_t m, bool quant) { return 2 * m <= bwd_slots_max(quant) ? 2 : 1; }

template <int PACKED>
static void launch_train_p(const rfb_scene *scene, dim3 grid, cudaStream_t st, bool train,
                           int lanes, const ArrayRays &src, double eps, double log_eps, double wf,
                           int32_t sl, const double *adj, const double *tg, double rgb_scale,
                           double q_scale, const double *up, int32_t np, double wfloor,
                           const FwdOut &O, const Grads &G, double *loss, const Scratch &scr,
                           unsigned long long *ctr, int32_t n_v) {
    SceneView<PACKED> S = view<PACKED>(scene);
#define RFB_TRAIN1(SH, TR, QU, L)                                                             \
    k_train<SH, PACKED, TR, QU, L><<<grid, kTrainBlock, 0, st>>>(                               \
        S, src, eps, log_eps, wf, sl, adj, tg, rgb_scale, q_scale, up, np, wfloor, O, G, loss, \
        scr, ctr, n_v)
#define RFB_TRAIN(SH, TR, QU)                                                                 \
    do {                                                                                       \
        if (lanes == 2) RFB_TRAIN1(SH, TR, QU, 2); else RFB_TRAIN1(SH, TR, QU, 1);             \
    } while (0)
    const bool quant = train && q_scale > 0.0;
    if (scene->sh_degree == 0) {
        if (quant) RFB_TRAIN(0, true, true);
        else if (train) RFB_TRAIN(0, true, false);
        else RFB_TRAIN(0, false, false);
    } else {
        if (quant) RFB_TRAIN(3, true, true);
        else if (train) RFB_TRAIN(3, true, false);
        else RFB_TRAIN(3, false, false);
    }
#undef RFB_TRAIN
#undef RFB_TRAIN1
}

static int launch_backward(const rfb_scene *scene, const rfb_rays *rays, const rfb_params *p,
                           const double *adjoints, const double *targets, double rgb_scale,
                           double q_scale, const double *u_pairs, int32_t n_pairs, double wfloor,
                           const rfb_fwd_out *out, const rfb_grads *grads, double *loss,
                           void *ws, size_t ws_bytes, cudaStream_t st, bool train) {
    if (!scene_ok(scene) || !rays || !p || !grads || !grads->site4g || !grads->sh ||
        p->step_limit <= 0 || rays->m < 0)
        return RFB_EINVAL;
    if (rays->m == 0) return RFB_OK;
    if (!out_ok(out)) return RFB_EINVAL;
    if (!rays->origins || !rays->directions || !rays->t_min || !rays->t_max || !rays->start_sites)
        return RFB_EINVAL;
    if (train && (!targets || (q_scale > 0.0 && (!u_pairs || n_pairs <= 0)))) return RFB_EINVAL;
    if (!train && !adjoints) return RFB_EINVAL;
    const bool quant = train && q_scale > 0.0;
    const int64_t per = bwd_slot_bytes(p->step_limit, quant);
    if (!ws || ws_bytes < kTrainWsHdr + (size_t)per * kTrainBlock) return RFB_EINVAL;
    int64_t slots = (int64_t)((ws_bytes - kTrainWsHdr) / (size_t)per);
    if (p->lanes_per_ray < 0 || p->lanes_per_ray > 2) return RFB_EINVAL;
    const int lanes = p->lanes_per_ray > 0 ? p->lanes_per_ray : train_lanes(rays->m, quant);
    slots = std::min<int64_t>(slots, bwd_slots_max(quant));
    slots = std::min<int64_t>(slots,
                              ((lanes * rays->m + kTrainBlock - 1) / kTrainBlock) * kTrainBlock);
    slots = (slots / kTrainBlock) * kTrainBlock;
    char *base = reinterpret_cast<char *>(ws);
    unsigned long long *ctr = reinterpret_cast<unsigned long long *>(base);
    Scratch scr;
    scr.slots = slots;
    const int64_t cap = p->step_limit;
    char *c = base + kTrainWsHdr;
    scr.a = reinterpret_cast<float4 *>(c);
    scr.c = reinterpret_cast<uint2 *>(c);  // (compact and full records share the space)
    c += cap * slots * 16;
    scr.b = reinterpret_cast<double2 *>(c);
    // per-SM work queues (fetch_unit) when the grid is whole waves of num_sms() blocks
    const int64_t nblk = slots / kTrainBlock;
    const int32_t n_v = (RFB_SM_LOCAL && RFB_TRAIN_SM_LOCAL && nblk % num_sms() == 0 &&
                         nblk >= num_sms() && kTrainWsHdr >= 8 * (size_t)(num_sms() + 1))
                            ? num_sms() : 0;
    cudaMemsetAsync(ctr, 0, 8 * (size_t)(n_v + 1), st);
    FwdOut O = dev_out(out);
    ArrayRays src{rays->origins, rays->directions, rays->t_min, rays->t_max, rays->start_sites,
                  rays->m, rays->order, rays->region};
    Grads G{grads->site4g, grads->sh};
    double log_eps = p->epsilon > 0.0 ? std::log(p->epsilon) : 0.0;
    dim3 grid((unsigned)(slots / kTrainBlock));
    if (scene->packed && !scene->positions_f64)
        launch_train_p<1>(scene, grid, st, train, lanes, src, p->epsilon, log_eps,
                          p->width_floor, p->step_limit, adjoints, targets, rgb_scale, q_scale,
                          u_pairs, n_pairs, wfloor, O, G, loss, scr, ctr, n_v);
    else if (scene->packed)
        launch_train_p<2>(scene, grid, st, train, lanes, src, p->epsilon, log_eps,
                          p->width_floor, p->step_limit, adjoints, targets, rgb_scale, q_scale,
                          u_pairs, n_pairs, wfloor, O, G, loss, scr, ctr, n_v);
    else
        launch_train_p<0>(scene, grid, st, train, lanes, src, p->epsilon, log_eps,
                          p->width_floor, p->step_limit, adjoints, targets, rgb_scale, q_scale,
                          u_pairs, n_pairs, wfloor, O, G, loss, scr, ctr, n_v);
    return (int)cudaGetLastError();
}

static CameraParams cam_params(const rfb_camera *c) {
    CameraParams p;
    for (int r = 0; r < 3; ++r) {
        for (int k = 0; k < 3; ++k) p.R[3 * r + k] = c->pose[4 * r + k];
        p.o[r] = c->pose[4 * r + 3];
    }
    p.focal = c->focal;
    p.cx = c->cx;
    p.cy = c->cy;
    p.width = c->width;
    p.height = c->height;
    p.kind = c->kind;
    return p;
}

}  // namespace rfb

using namespace rfb;

extern "C" {

int rfb_abi_version(void) { return RFB_ABI_VERSION; }

const char *rfb_error_string(int code) {
    if (code == RFB_OK) return "ok";
    if (code == RFB_EINVAL) return "invalid argument";
    if (code == RFB_ECAPACITY) return "capacity exceeded";
    if (code == RFB_EDEGENERATE) return "degenerate input";
    return cudaGetErrorString((cudaError_t)code);
}

int rfb_device_ok(void) {
    int dev = 0, major = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess)
        return 0;
    return major == 10 ? 1 : 0;
}

int rfb_host_device_pointer(void *host, void **device_ptr) {
    if (!host || !device_ptr) return RFB_EINVAL;
    *device_ptr = nullptr;
    cudaError_t e = cudaHostGetDevicePointer(device_ptr, host, 0);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();  // not sticky: clear it for the caller's next launch
        *device_ptr = nullptr;
    }
    return (int)e;
}

int rfb_pack_scene(const double *positions, const double *sigma, const double *sh,
                   const int64_t *offsets, const int64_t *neighbors, int64_t n_sites,
                   int64_t n_edges, double *site4, int32_t *offsets32, int32_t *neighbors32,
                   void *cells, void *edges, int32_t *edge_nbr, float *sh32, int32_t *pk_of,
                   int32_t *pk_id, int32_t positions_f64, void *stream) {
    if (!positions || !sigma || !offsets || !neighbors || !site4 || !offsets32 || !neighbors32 ||
        n_sites <= 0 || n_edges < 0 || n_edges + n_sites + 2 >= ((int64_t)1 << 31) ||
        ((cells || edges || edge_nbr || sh32) && (!cells || !edges || !edge_nbr || !sh32 || !sh)) ||
        (!pk_of != !pk_id) || (pk_of && !cells))
        return RFB_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    const int n = (int)n_sites;
    const unsigned blocks = (unsigned)((n_sites + 255) / 256);
    void *tmp = nullptr;
    if (cells) {
        // scratch: [Morton keys in, out | ids in | padded degrees -> row starts | bbox | cub]
        size_t sort_bytes = 0, scan_bytes = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (uint32_t *)nullptr,
                                        (uint32_t *)nullptr, (int32_t *)nullptr,
                                        (int32_t *)nullptr, n, 0, 30, st);
        cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (int32_t *)nullptr, (int32_t *)nullptr,
                                      n, st);
        const size_t a4 = ((sizeof(int32_t) * (n_sites + 1)) + 255) & ~(size_t)255;
        const size_t cub_bytes = std::max(sort_bytes, scan_bytes);
        cudaError_t e = cudaMallocAsync(&tmp, 4 * a4 + 256 + cub_bytes, st);
        if (e != cudaSuccess) return (int)e;
        char *base = reinterpret_cast<char *>(tmp);
        uint32_t *key_in = reinterpret_cast<uint32_t *>(base);
        uint32_t *key_out = reinterpret_cast<uint32_t *>(base + a4);
        int32_t *val_in = reinterpret_cast<int32_t *>(base + 2 * a4);
        int32_t *kp0 = reinterpret_cast<int32_t *>(base + 3 * a4);
        unsigned *mm = reinterpret_cast<unsigned *>(base + 4 * a4);
        void *cub_tmp = base + 4 * a4 + 256;
        if (pk_id) {
            const unsigned init[6] = {0xffffffffu, 0xffffffffu, 0xffffffffu, 0u, 0u, 0u};
            cudaMemcpyAsync(mm, init, sizeof(init), cudaMemcpyHostToDevice, st);
            k_bbox<<<blocks, 256, 0, st>>>(positions, n_sites, mm);
            k_morton<<<blocks, 256, 0, st>>>(positions, n_sites, mm, key_in, val_in);
            size_t b = sort_bytes;
            cub::DeviceRadixSort::SortPairs(cub_tmp, b, key_in, key_out, val_in, pk_id, n, 0, 30,
                                            st);
            k_invert<<<blocks, 256, 0, st>>>(pk_id, n_sites, pk_of);
        }
        k_pad_deg<<<blocks, 256, 0, st>>>(offsets, pk_id, n_sites, kp0);
        size_t b = scan_bytes;
        cub::DeviceScan::ExclusiveSum(cub_tmp, b, kp0, kp0, n, st);
        k_pack_sites<<<(unsigned)((n_sites + 1 + 255) / 256), 256, 0, st>>>(
            positions, sigma, sh, n_sites, offsets, reinterpret_cast<double4 *>(site4), offsets32,
            sh32, pk_of);
        k_pack_rows<<<(unsigned)((n_sites * kRowLanes + 255) / 256), 256, 0, st>>>(
            positions, sigma, n_sites, offsets, neighbors, kp0, pk_id, pk_of,
            reinterpret_cast<CellHdr *>(cells), reinterpret_cast<float4 *>(edges), edge_nbr,
            positions_f64 ? 1 : 0);
    } else {
        k_pack_sites<<<(unsigned)((n_sites + 1 + 255) / 256), 256, 0, st>>>(
            positions, sigma, sh, n_sites, offsets, reinterpret_cast<double4 *>(site4), offsets32,
            nullptr, nullptr);
    }
    if (n_edges > 0)
        k_pack_edges<<<(unsigned)((n_edges + 255) / 256), 256, 0, st>>>(neighbors, n_edges,
                                                                         neighbors32);
    if (tmp) cudaFreeAsync(tmp, st);
    return (int)cudaGetLastError();
}

int rfb_softplus(const double *raw, int64_t n, double *out, double *site4, void *cells,
                 const int32_t *pk_of, void *stream) {
    if (!raw || n < 0 || (!out && !site4 && !cells)) return RFB_EINVAL;
    if (n == 0) return RFB_OK;
    k_softplus<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        raw, n, out, reinterpret_cast<double4 *>(site4), reinterpret_cast<CellHdr *>(cells),
        pk_of);
    return (int)cudaGetLastError();
}

int rfb_post_grad_adam(int64_t n_sites, const float *grads_flat, double *positions,
                       double *raw_density, double *sh, double *adam_state, double clip,
                       int32_t sh_warmup, int32_t update_positions, const double *hyper,
                       float *sh32, float *sh_absmax_dev, const int32_t *pk_of, void *stream) {
    if (n_sites <= 0 || !grads_flat || !positions || !raw_density || !sh || !adam_state ||
        !hyper || !(clip > 0.0))
        return RFB_EINVAL;
    const int64_t n = n_sites;
    double *m_pos = adam_state, *v_pos = m_pos + 3 * n, *m_raw = v_pos + 3 * n,
           *v_raw = m_raw + n, *m_sh = v_raw + n, *v_sh = m_sh + 48 * n;
    AdamArgs a[3];
    for (int k = 0; k < 3; ++k) {
        const double *h = hyper + 6 * k;
        a[k] = AdamArgs{h[0], h[1], h[2], h[3], h[4], h[5]};
    }
    const int64_t total = n * 52;
    k_post_adam<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        n, grads_flat, grads_flat + 4 * n, positions, raw_density, sh, m_pos, v_pos, m_raw, v_raw,
        m_sh, v_sh, clip, sh_warmup, update_positions, a[0], a[1], a[2], sh32,
        reinterpret_cast<unsigned *>(sh_absmax_dev), pk_of);
    return (int)cudaGetLastError();
}

// fp32 channel-major SH copy, one thread per output float (coalesced rows)
__global__ void k_refresh_sh32(int64_t n, const double *sh, float *sh32, const int32_t *pk_id) {
    const int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= 48 * n) return;
    const int64_t u = o / 48;  // packed row u holds site pk_id[u]
    const int64_t i = pk_id ? (int64_t)pk_id[u] : u;
    const int r = (int)(o - 48 * u), ch = r / 16, k = r - 16 * ch;
    sh32[o] = (float)sh[48 * i + 3 * k + ch];
}

int rfb_refresh_scene(const rfb_scene *scene, const double *positions, const double *raw_density,
                      int32_t refresh_sh32, void *stream) {
    if (!scene_ok(scene) || !positions || !raw_density) return RFB_EINVAL;
    // a packed scene with fp32-exact positions cannot take moved sites in place
    const bool pos64 = scene->packed && scene->positions_f64;
    cudaStream_t st = (cudaStream_t)stream;
    k_refresh_scene<<<(unsigned)((scene->n_sites + 255) / 256), 256, 0, st>>>(
        scene->n_sites, positions, raw_density, (double4 *)scene->site4,
        scene->packed ? (CellHdr *)scene->cells : nullptr, scene->packed ? scene->pk_of : nullptr);
    if (pos64) {  // after k_refresh_scene: the headers' sigma is read back
        k_refresh_rows<<<(unsigned)((scene->n_sites * kRowLanes + 255) / 256), 256, 0, st>>>(
            scene->n_sites, positions, (CellHdr *)scene->cells, scene->offsets,
            scene->neighbors, reinterpret_cast<float4 *>(const_cast<void *>(scene->edges)),
            const_cast<int32_t *>(scene->edge_nbr), scene->pk_id, scene->pk_of);
    }
    if (refresh_sh32 && scene->packed && scene->sh32)
        k_refresh_sh32<<<(unsigned)((48 * scene->n_sites + 255) / 256), 256, 0, st>>>(
            scene->n_sites, scene->sh, (float *)scene->sh32, scene->pk_id);
    return (int)cudaGetLastError();
}

int rfb_camera_rays(const rfb_camera *camera, int64_t pix_begin, int64_t pix_count, double *dirs,
                    void *stream) {
    if (!camera || !dirs || pix_begin < 0 || pix_count < 0 || camera->width < 1 ||
        camera->height < 1 || !(camera->focal > 0.0) || camera->kind < 0 || camera->kind > 1 ||
        pix_begin + pix_count > (int64_t)camera->width * camera->height)
        return RFB_EINVAL;
    if (pix_count == 0) return RFB_OK;
    k_camera_rays<<<(unsigned)((pix_count + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        cam_params(camera), pix_begin, pix_count, dirs);
    return (int)cudaGetLastError();
}

int rfb_effect_rays(const double *origins, const double *directions, const double *t_at,
                    int64_t m, const double *normal, int32_t kind, double eta,
                    double *out_origins, double *out_directions, void *stream) {
    if (m < 0 || !normal || (kind != RFB_EFFECT_MIRROR && kind != RFB_EFFECT_REFRACT)) return RFB_EINVAL;
    if (m == 0) return RFB_OK;
    if (!origins || !directions || !t_at || !out_origins || !out_directions) return RFB_EINVAL;
    const double l = std::sqrt(normal[0] * normal[0] + normal[1] * normal[1] + normal[2] * normal[2]);
    if (!(l > 0.0)) return RFB_EINVAL;  // EffectPlane normalises (rays.py:135)
    k_effect_rays<<<(unsigned)((m + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        origins, directions, t_at, m, normal[0] / l, normal[1] / l, normal[2] / l, kind, eta,
        out_origins, out_directions);
    return (int)cudaGetLastError();
}

int rfb_locate(const rfb_scene *scene, const double *queries, int64_t m, int32_t seed_site,
               int32_t *out, void *stream) {
    if (!scene_ok(scene) || !queries || !out || m < 0 || seed_site < 0 ||
        seed_site >= scene->n_sites)
        return RFB_EINVAL;
    if (m == 0) return RFB_OK;
    k_locate<<<(unsigned)((m + 127) / 128), 128, 0, (cudaStream_t)stream>>>(loc_scene(scene),
                                                                            queries, m, seed_site, out);
    return (int)cudaGetLastError();
}

static HintGrid hint_grid(const rfb_locate_grid *lg) {
    HintGrid g;
    for (int k = 0; k < 3; ++k) {
        g.lo[k] = lg->lo[k];
        g.dims[k] = lg->dims[k];
    }
    g.cell = lg->cell;
    g.hint = lg->hint;
    return g;
}

static bool grid_ok(const rfb_locate_grid *lg) {
    return lg && lg->hint && lg->cell > 0.0 && lg->dims[0] > 0 && lg->dims[1] > 0 &&
           lg->dims[2] > 0;
}

int rfb_build_locate_grid(const rfb_scene *scene, rfb_locate_grid *grid, void *stream) {
    if (!scene_ok(scene) || !grid_ok(grid)) return RFB_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t cells = (int64_t)grid->dims[0] * grid->dims[1] * grid->dims[2];
    cudaMemsetAsync(grid->hint, 0xff, sizeof(int32_t) * cells, st);  // -1
    k_hint_scatter<<<(unsigned)((scene->n_sites + 255) / 256), 256, 0, st>>>(
        reinterpret_cast<const double4 *>(scene->site4), scene->n_sites, hint_grid(grid),
        grid->hint);
    return (int)cudaGetLastError();
}

int rfb_locate_seeded(const rfb_scene *scene, const double *queries, int64_t m,
                    const rfb_locate_grid *grid, int32_t seed_site, int32_t *out, void *stream) {
    if (!scene_ok(scene) || !queries || !out || m < 0 || !grid_ok(grid) || seed_site < 0 ||
        seed_site >= scene->n_sites)
        return RFB_EINVAL;
    if (m == 0) return RFB_OK;
    k_locate_hinted<<<(unsigned)((m + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
        loc_scene(scene), queries, m, hint_grid(grid), seed_site, out);
    return (int)cudaGetLastError();
}

size_t rfb_workspace_bytes(int64_t m, int32_t step_limit, int32_t kind) {
    if (kind == 0) return 256 + 8 * (size_t)(num_sms() + 1);  // + the per-SM work counters
    const bool quant = kind != 2;  // 2: no quantile term (compact records)
    int64_t slots = std::min<int64_t>(quant ? std::max(bwd_slots_max(false), bwd_slots_max(true))
                                            : bwd_slots_max(false),
                                      ((2 * m + kTrainBlock - 1) / kTrainBlock) * kTrainBlock);
    slots = std::max<int64_t>(slots, kTrainBlock);
    return kTrainWsHdr + (size_t)slots * (size_t)bwd_slot_bytes(step_limit, quant);
}

int rfb_render_rays(const rfb_scene *scene, const rfb_rays *rays, const rfb_params *params,
                    const rfb_fwd_out *out, void *workspace, size_t workspace_bytes, void *stream) {
    if (!scene_ok(scene) || !rays || !params || params->step_limit <= 0 || rays->m < 0)
        return RFB_EINVAL;
    if (rays->m == 0) return RFB_OK;
    if (!out_ok(out)) return RFB_EINVAL;
    if (!rays->origins || !rays->directions || !rays->t_min || !rays->t_max || !rays->start_sites)
        return RFB_EINVAL;
    ArrayRays src{rays->origins, rays->directions, rays->t_min, rays->t_max, rays->start_sites,
                  rays->m, rays->order, rays->region};
    return launch_render(scene, src, params, out, workspace, workspace_bytes,
                         (cudaStream_t)stream);
}

int rfb_render_image(const rfb_scene *scene, const rfb_camera *camera, const rfb_params *params,
                     double t_min, double t_max, int32_t start_site, const int32_t *tile_ids,
                     int64_t n_tiles, int32_t tile_w, int32_t tile_h, const rfb_fwd_out *out,
                     void *workspace, size_t workspace_bytes, void *stream) {
    if (!scene_ok(scene) || !camera || !params || !out_ok(out) || params->step_limit <= 0 ||
        !tile_ids || n_tiles < 0 || tile_w < 32 || tile_h < 32 || tile_w % 32 || tile_h % 32 ||
        camera->width < 1 || camera->height < 1 || !(camera->focal > 0.0) || camera->kind < 0 ||
        camera->kind > 1 || start_site >= scene->n_sites || !workspace || workspace_bytes < 256)
        return RFB_EINVAL;
    if (n_tiles == 0) return RFB_OK;
    cudaStream_t st = (cudaStream_t)stream;
    int32_t *start_ptr = reinterpret_cast<int32_t *>(reinterpret_cast<char *>(workspace) + 64);
    if (start_site < 0) {
        nearest_point(scene, camera->pose[3], camera->pose[7], camera->pose[11],
                      reinterpret_cast<char *>(workspace) + 128, start_ptr, st);
    } else {
        cudaMemcpyAsync(start_ptr, &start_site, sizeof(int32_t), cudaMemcpyHostToDevice, st);
    }
    TileRays src;
    src.cam = cam_params(camera);
    src.tile_ids = tile_ids;
    src.n_tiles = n_tiles;
    src.tile_w = tile_w;
    src.tile_h = tile_h;
    src.tiles_x = (camera->width + tile_w - 1) / tile_w;
    src.t_min = t_min;
    src.t_max = t_max;
    src.start_ptr = start_ptr;
    return launch_render(scene, src, params, out, workspace, workspace_bytes, st);
}

static int launch_cull(const rfb_scene *scene, const CullCone &cone, void *cells_out,
                       void *edges_out, rfb_scene *view_out, int32_t rx, int32_t ry,
                       cudaStream_t st) {
    *view_out = *scene;
    view_out->cells = cells_out;
    view_out->edges = edges_out;
    view_out->view_rx = rx;
    view_out->view_ry = ry;
    const int64_t groups = (scene->n_sites + kCullRows - 1) / kCullRows;
    const unsigned nb = (unsigned)((groups * kRowLanes + 255) / 256);
    auto go = [&](auto kern) {
        kern<<<nb, 256, 0, st>>>((const CellHdr *)scene->cells, (const float4 *)scene->edges,
                                 scene->n_sites, cone, scene->positions_f64 ? 1 : 0,
                                 (CellHdr *)cells_out, (float4 *)edges_out);
    };
    if (rx == 2 && ry == 2) go(k_cull_rows<2, 2>);
    else if (rx == 3 && ry == 2) go(k_cull_rows<3, 2>);
    else if (rx == 4 && ry == 2) go(k_cull_rows<4, 2>);
    else if (rx == 4 && ry == 3) go(k_cull_rows<4, 3>);
    else if (rx == 4 && ry == 4) go(k_cull_rows<4, 4>);
    else go(k_cull_rows<0, 0>);  // any other grid, or one cone (rfb_cull_scene)
    return (int)cudaGetLastError();
}

static bool cull_args_ok(const rfb_scene *scene, const void *cells_out, const void *edges_out,
                         const rfb_scene *view_out) {
    return scene_ok(scene) && scene->packed && scene->view_rx == 0 && cells_out && edges_out &&
           view_out && !(reinterpret_cast<uintptr_t>(cells_out) & 31) &&
           !(reinterpret_cast<uintptr_t>(edges_out) & 31);
}

// unit generator k of cone `c` from a direction (false: zero or non-finite)
static bool set_gen(CullCone &c, int k, const double *d) {
    const double l = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    if (!(l > 0.0) || !std::isfinite(l)) return false;
    for (int a = 0; a < 3; ++a) c.c[k][a] = (float)(d[a] / l);
    return true;
}

int rfb_cull_scene(const rfb_scene *scene, const double *dirs, int32_t n_dirs, void *cells_out,
                   void *edges_out, rfb_scene *view_out, void *stream) {
    if (!cull_args_ok(scene, cells_out, edges_out, view_out) || !dirs || n_dirs < 1 ||
        n_dirs > kCullMaxDirs)
        return RFB_EINVAL;
    CullCone cone{};
    for (int k = 0; k < n_dirs; ++k)
        if (!set_gen(cone, k, dirs + 3 * k)) return RFB_EINVAL;
    cone.rx = cone.ry = 0;
    cone.nd = n_dirs;
    cone.stride = 0;
    return launch_cull(scene, cone, cells_out, edges_out, view_out, 0, 0, (cudaStream_t)stream);
}

int rfb_cull_view(const rfb_scene *scene, const rfb_camera *camera, int32_t rx, int32_t ry,
                  void *cells_out, void *edges_out, rfb_scene *view_out, void *stream) {
    if (!cull_args_ok(scene, cells_out, edges_out, view_out) || !camera || camera->kind != 0 ||
        rx < 1 || ry < 1 || rx * ry > kCullMaxRegions || (rx + 1) * (ry + 1) > kCullMaxGen ||
        camera->width < rx ||
        camera->height < ry || !(camera->focal > 0.0))
        return RFB_EINVAL;
    const int64_t stride = RFB_VIEW_STRIDE(scene->n_sites, scene->n_edges);
    if ((int64_t)rx * ry * stride >= (int64_t)INT32_MAX ||
        (int64_t)rx * ry * scene->n_sites >= (int64_t)INT32_MAX)
        return RFB_EINVAL;  // header / slot indices are int32
    CullCone cone{};
    cone.rx = rx;
    cone.ry = ry;
    cone.nd = 4;
    cone.stride = stride;
    const int64_t W = camera->width, H = camera->height;
    // region ix holds the pixels with px * rx / W == ix, i.e. columns ceil(ix W / rx) ..
    // ceil((ix + 1) W / rx) - 1: their centres lie strictly inside the pixel-edge lines
    // col = ceil(ix W / rx) and ceil((ix + 1) W / rx), which the regions share
    for (int iy = 0; iy <= ry; ++iy)
        for (int ix = 0; ix <= rx; ++ix) {
            const double col = (double)((ix * W + rx - 1) / rx);
            const double row = (double)((iy * H + ry - 1) / ry);
            // camera.py:78-92: d_cam = (u, v, -1), d = R d_cam (here at pixel edges)
            const double u = (col - camera->cx) / camera->focal;
            const double v = -(row - camera->cy) / camera->focal;
            double d[3];
            for (int a = 0; a < 3; ++a)
                d[a] = camera->pose[4 * a] * u + camera->pose[4 * a + 1] * v - camera->pose[4 * a + 2];
            if (!set_gen(cone, iy * (rx + 1) + ix, d)) return RFB_EINVAL;
        }
    return launch_cull(scene, cone, cells_out, edges_out, view_out, rx, ry, (cudaStream_t)stream);
}

int rfb_backward_rays(const rfb_scene *scene, const rfb_rays *rays, const rfb_params *params,
                      const double *adjoints, const rfb_fwd_out *out, const rfb_grads *grads,
                      void *workspace, size_t workspace_bytes, void *stream) {
    return launch_backward(scene, rays, params, adjoints, nullptr, 0.0, 0.0, nullptr, 0, 0.0, out,
                           grads, nullptr, workspace, workspace_bytes, (cudaStream_t)stream, false);
}

int rfb_train_batch(const rfb_scene *scene, const rfb_rays *rays, const rfb_params *params,
                    const double *targets, double rgb_scale, double quantile_scale,
                    const double *u_pairs, int32_t n_pairs, double weight_floor,
                    const rfb_fwd_out *out, const rfb_grads *grads, double *loss, void *workspace,
                    size_t workspace_bytes, void *stream) {
    return launch_backward(scene, rays, params, nullptr, targets, rgb_scale, quantile_scale,
                           u_pairs, n_pairs, weight_floor, out, grads, loss, workspace,
                           workspace_bytes, (cudaStream_t)stream, true);
}

}  // extern "C"
