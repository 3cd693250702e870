// rfb.cu -- sm_100a kernels and the C ABI (include/rfb.h) of the Radiant Foam
// hot path.  See DESIGN.md for the data layout and the roofline of each
// kernel; every kernel cites the reference function it replaces.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>

#include "rfb_device.cuh"

namespace rfb {

__device__ __forceinline__ double dinf() { return __longlong_as_double(0x7ff0000000000000LL); }

// ---------------------------------------------------------------------------
// Ray sources: explicit arrays (render.py:57-125) or a pinhole camera over a
// tile list (render.py:128-149 + camera.py:66-92).
// ---------------------------------------------------------------------------
struct ArrayRays {
    const double *origins, *directions, *t_min, *t_max;
    const int32_t *start;
    int64_t m;
    __device__ __forceinline__ int64_t count() const { return m; }
    // returns output index (pixel / ray id) or -1 when the slot is padding
    __device__ __forceinline__ int64_t get(int64_t q, Ray &r) const {
        r.ox = origins[3 * q];
        r.oy = origins[3 * q + 1];
        r.oz = origins[3 * q + 2];
        r.dx = directions[3 * q];
        r.dy = directions[3 * q + 1];
        r.dz = directions[3 * q + 2];
        r.t_min = t_min[q];
        r.t_max = t_max[q];
        r.start = start[q];
        return q;
    }
};

struct CameraParams {
    double R[9];  // rotation, row-major (pose[:3,:3])
    double o[3];  // pose[:3,3]
    double focal, cx, cy;
    int32_t width, height;
};

// camera.py:78-92 pinhole branch; fma order reproduces numpy's
// `d_cam @ R.T` bit-for-bit (checked in tests/test_camera.py).
__device__ __forceinline__ void pinhole_dir(const CameraParams &c, int64_t row, int64_t col,
                                            double &dx, double &dy, double &dz) {
    double u = ((double)col + 0.5 - c.cx) / c.focal;
    double v = -((double)row + 0.5 - c.cy) / c.focal;
    double w[3];
#pragma unroll
    for (int k = 0; k < 3; ++k)
        w[k] = __fma_rn(-1.0, c.R[3 * k + 2], __fma_rn(v, c.R[3 * k + 1], u * c.R[3 * k]));
    double nrm = sqrt((w[0] * w[0] + w[1] * w[1]) + w[2] * w[2]);
    dx = w[0] / nrm;
    dy = w[1] / nrm;
    dz = w[2] / nrm;
}

struct TileRays {
    CameraParams cam;
    const int32_t *tile_ids;
    int64_t n_tiles;
    int32_t tile_w, tile_h, tiles_x;
    double t_min, t_max;
    const int32_t *start_ptr;  // device scalar (located start cell)
    __device__ __forceinline__ int64_t count() const { return n_tiles * tile_w * tile_h; }
    // 8x4 sub-tiles inside each tile keep a warp's 32 rays on a compact patch.
    __device__ __forceinline__ int64_t get(int64_t q, Ray &r) const {
        int64_t per = (int64_t)tile_w * tile_h;
        int32_t tile = tile_ids[q / per];
        int32_t p = (int32_t)(q % per);
        int32_t sub = p >> 5, l = p & 31;
        int32_t subs_x = tile_w >> 3;
        int32_t px = (tile % tiles_x) * tile_w + (sub % subs_x) * 8 + (l & 7);
        int32_t py = (tile / tiles_x) * tile_h + (sub / subs_x) * 4 + (l >> 3);
        if (px >= cam.width || py >= cam.height) return -1;
        r.ox = cam.o[0];
        r.oy = cam.o[1];
        r.oz = cam.o[2];
        pinhole_dir(cam, py, px, r.dx, r.dy, r.dz);
        r.t_min = t_min;
        r.t_max = t_max;
        r.start = *start_ptr;
        return (int64_t)py * cam.width + px;
    }
};

struct DevScene {
    const double4 *site4;
    const int32_t *off;
    const int32_t *nbr;
    const double *sh;
    double bg[3];
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
};

__device__ __forceinline__ void store_out(void *p, int64_t idx, double v, int32_t f64) {
    if (f64)
        reinterpret_cast<double *>(p)[idx] = v;
    else
        reinterpret_cast<float *>(p)[idx] = (float)v;
}

// ---------------------------------------------------------------------------
// Forward: walk (kernels.py:76-162) with compositing fused per recorded
// segment (composite_segments 165-196, same operation order, so the result is
// identical to compositing after the walk).  G lanes cooperate on one ray.
// ---------------------------------------------------------------------------
template <int G, int SHDEG, class Src>
__global__ void __launch_bounds__(256) k_render(DevScene S, Src src, double epsilon,
                                                double log_eps, double width_floor,
                                                int32_t step_limit, FwdOut O,
                                                unsigned long long *ray_counter) {
    constexpr int RPW = 32 / G;  // rays per warp
    const int lane = threadIdx.x & 31;
    const int gl = lane & (G - 1);
    const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (lane & ~(G - 1)));
    const int64_t total = src.count();
    unsigned long long my_cells = 0, my_visits = 0;

    for (;;) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(ray_counter, (unsigned long long)RPW);
        base = __shfl_sync(0xffffffffu, base, 0);
        if ((int64_t)base >= total) break;
        int64_t q = (int64_t)base + lane / G;
        if (q >= total) continue;
        Ray r;
        int64_t oidx = src.get(q, r);
        if (oidx < 0) continue;

        double basis[16];
        if (SHDEG > 0)
            sh_basis(r.dx, r.dy, r.dz, basis);
        else
            basis[0] = kC0;

        int32_t i = r.start;
        double entry = r.t_min, log_T = 0.0;
        int32_t nseg = 0, zero_adv = 0, steps = 0;
        int status = RFB_STATUS_OK;
        double T = 1.0, wsum = 0.0, cr = 0.0, cg = 0.0, cb = 0.0;
        int32_t cells = 0, visits = 0;
        const bool dump = O.seg_cap > 0;

        // Record one segment and composite it (kernels.py:137-141/147-151 +
        // 179-189).
        auto record = [&](int32_t cell, double t0, double t1) {
            double sig = __ldg(&S.site4[cell].w);
            double delta = t1 - t0;
            log_T -= sig * delta;
            double alpha = 1.0 - exp(-sig * delta);
            double col[3];
            cell_color<SHDEG>(S.sh, cell, basis, col);
            double w = T * alpha;
            wsum += w;
            cr += w * col[0];
            cg += w * col[1];
            cb += w * col[2];
            T *= 1.0 - alpha;
            if (dump && nseg < O.seg_cap && gl == 0) {
                int64_t o = oidx * O.seg_cap + nseg;
                O.seg_cells[o] = cell;
                O.seg_t0[o] = t0;
                O.seg_t1[o] = t1;
            }
            nseg += 1;
        };

        for (;;) {
            steps += 1;
            if (steps > step_limit) {
                status = RFB_STATUS_STEP_LIMIT;
                break;
            }
            cells += 1;
            double4 xi = ld_site(S.site4 + i);
            int32_t k0 = __ldg(S.off + i), k1 = __ldg(S.off + i + 1);
            visits += k1 - k0;
            double best_t;
            int32_t best_j;
            exit_face<G>(S.site4, S.nbr, k0, k1, xi, r, gl, gmask, best_t, best_j);
            if (best_j < 0 || best_t >= r.t_max) {
                if (r.t_max > entry) record(i, entry, r.t_max);
                break;
            }
            if (best_t < entry) best_t = entry;
            if (best_t - entry > width_floor) {
                record(i, entry, best_t);
                entry = best_t;
                zero_adv = 0;
                if (below_epsilon(log_T, epsilon, log_eps)) break;
                if (nseg >= step_limit) {
                    status = RFB_STATUS_STEP_LIMIT;
                    break;
                }
            } else {
                zero_adv += 1;
                if (zero_adv > kZeroAdvanceLimit) {
                    status = RFB_STATUS_CYCLE;
                    break;
                }
            }
            i = best_j;
        }

        if (gl == 0) {
            my_cells += (unsigned long long)cells;
            my_visits += (unsigned long long)visits;
            double resid;
            if (status != RFB_STATUS_OK) {  // kernels.py:230-236
                cr = S.bg[0];
                cg = S.bg[1];
                cb = S.bg[2];
                resid = 1.0;
                wsum = 0.0;
            } else {
                cr += T * S.bg[0];
                cg += T * S.bg[1];
                cb += T * S.bg[2];
                resid = T;
            }
            store_out(O.rgb, 3 * oidx, cr, O.f64);
            store_out(O.rgb, 3 * oidx + 1, cg, O.f64);
            store_out(O.rgb, 3 * oidx + 2, cb, O.f64);
            if (O.residual) store_out(O.residual, oidx, resid, O.f64);
            if (O.wsum) store_out(O.wsum, oidx, wsum, O.f64);
            if (O.status) O.status[oidx] = (int8_t)status;
            if (O.nseg) O.nseg[oidx] = nseg;
            if (O.ray_counters) {
                O.ray_counters[2 * oidx] = cells;
                O.ray_counters[2 * oidx + 1] = visits;
            }
        }
    }
    if (O.counters) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            my_cells += __shfl_xor_sync(0xffffffffu, my_cells, off);
            my_visits += __shfl_xor_sync(0xffffffffu, my_visits, off);
        }
        if (lane == 0) {
            atomicAdd(O.counters, my_cells);
            atomicAdd(O.counters + 1, my_visits);
        }
    }
}

// ---------------------------------------------------------------------------
// Backward / training: one thread per ray.  The walk records each segment
// (cell | clamp mask, exit depth, transmittance after it, colour) into a
// per-thread slot of the workspace; the reverse pass (backward_ray,
// kernels.py:250-337) and the quantile pairs (456-567) then read it back.
// ---------------------------------------------------------------------------
struct Scratch {
    int32_t *cell;  // [cap][slots]: cell id | mask << 29
    double *t1;     // [cap][slots]: exit depth (entry of s = exit of s-1)
    double *tb;     // [cap][slots]: T_before[s+1] = prod exp(-sigma*delta)
    float *col;     // [cap][3][slots]
    int64_t slots;
};

struct Grads {
    float *g4;  // [n][4] dpos xyz, dsigma
    float *sh;  // [n][48]
};

__device__ __forceinline__ void add_pos(float *g4, int32_t i, double x, double y, double z) {
    float *p = g4 + 4 * (int64_t)i;
    atomicAdd(p, (float)x);
    atomicAdd(p + 1, (float)y);
    atomicAdd(p + 2, (float)z);
}

// kernels.py:340-369
__device__ __forceinline__ void face_t_gradient(const double4 *__restrict__ site4, int32_t i,
                                                int32_t j, const Ray &r, double t, double dt,
                                                float *g4) {
    double4 xi = ld_site(site4 + i), xj = ld_site(site4 + j);
    double nx = xj.x - xi.x, ny = xj.y - xi.y, nz = xj.z - xi.z;
    double denom = r.dx * nx + r.dy * ny + r.dz * nz;
    if (denom == 0.0) return;
    double mx = 0.5 * (xi.x + xj.x), my = 0.5 * (xi.y + xj.y), mz = 0.5 * (xi.z + xj.z);
    double px = r.ox + t * r.dx, py = r.oy + t * r.dy, pz = r.oz + t * r.dz;
    double qx = mx - px, qy = my - py, qz = mz - pz;
    double inv = dt / denom;
    add_pos(g4, i, (0.5 * nx - qx) * inv, (0.5 * ny - qy) * inv, (0.5 * nz - qz) * inv);
    add_pos(g4, j, (0.5 * nx + qx) * inv, (0.5 * ny + qy) * inv, (0.5 * nz + qz) * inv);
}

template <int SHDEG>
__device__ __forceinline__ void add_sh(float *gsh, int32_t i, int mask, double w, double ar,
                                       double ag, double ab, const double *basis) {
    // kernels.py:309-322: channel ch gets w*adj_ch*basis[k] unless clamped or
    // adj_ch == 0.
    double f[3];
    f[0] = ((mask & 1) == 0 && ar != 0.0) ? w * ar : 0.0;
    f[1] = ((mask & 2) == 0 && ag != 0.0) ? w * ag : 0.0;
    f[2] = ((mask & 4) == 0 && ab != 0.0) ? w * ab : 0.0;
    if (f[0] == 0.0 && f[1] == 0.0 && f[2] == 0.0) return;
    float *row = gsh + 48 * (int64_t)i;
    if (SHDEG == 0) {
#pragma unroll
        for (int ch = 0; ch < 3; ++ch)
            if (f[ch] != 0.0) atomicAdd(row + ch, (float)(f[ch] * basis[0]));
        return;
    }
    float v[48];
#pragma unroll
    for (int k = 0; k < 16; ++k)
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) v[3 * k + ch] = (float)(f[ch] * basis[k]);
    float4 *row4 = reinterpret_cast<float4 *>(row);
#pragma unroll
    for (int c = 0; c < 12; ++c)
        atomicAdd(row4 + c, make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]));
}

template <int SHDEG, bool TRAIN>
__global__ void __launch_bounds__(128) k_backward(DevScene S, ArrayRays src, double epsilon,
                                                  double log_eps, double width_floor,
                                                  int32_t step_limit, const double *adjoints,
                                                  const double *targets, double rgb_scale,
                                                  double q_scale, const double *u_pairs,
                                                  int32_t n_pairs, double weight_floor, FwdOut O,
                                                  Grads gr, double *loss, Scratch scr,
                                                  unsigned long long *ray_counter) {
    const int64_t slot = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t SL = scr.slots;
    int32_t *s_cell = scr.cell + slot;
    double *s_t1 = scr.t1 + slot;
    double *s_tb = scr.tb + slot;
    float *s_col = scr.col + slot;
    double loss_rgb = 0.0, loss_q = 0.0;
    unsigned long long my_cells = 0, my_visits = 0;
    const int64_t total = src.count();

    for (;;) {
        int64_t q = (int64_t)atomicAdd(ray_counter, 1ull);
        if (q >= total) break;
        Ray r;
        src.get(q, r);
        double basis[16];
        if (SHDEG > 0)
            sh_basis(r.dx, r.dy, r.dz, basis);
        else
            basis[0] = kC0;

        int32_t i = r.start;
        double entry = r.t_min, log_T = 0.0;
        int32_t nseg = 0, zero_adv = 0, steps = 0;
        int status = RFB_STATUS_OK;
        double Tc = 1.0, Tb = 1.0, wsum = 0.0, cr = 0.0, cg = 0.0, cb = 0.0;
        int32_t cells = 0, visits = 0;

        auto record = [&](int32_t cell, double t0, double t1) {
            double sig = __ldg(&S.site4[cell].w);
            double delta = t1 - t0;
            log_T -= sig * delta;
            double e = exp(-sig * delta);
            double alpha = 1.0 - e;
            double col[3];
            int mask = cell_color<SHDEG>(S.sh, cell, basis, col);
            double w = Tc * alpha;
            wsum += w;
            cr += w * col[0];
            cg += w * col[1];
            cb += w * col[2];
            Tc *= 1.0 - alpha;
            Tb = Tb * e;
            s_cell[nseg * SL] = cell | (mask << 29);
            s_t1[nseg * SL] = t1;
            s_tb[nseg * SL] = Tb;
            s_col[(3 * nseg) * SL] = (float)col[0];
            s_col[(3 * nseg + 1) * SL] = (float)col[1];
            s_col[(3 * nseg + 2) * SL] = (float)col[2];
            nseg += 1;
        };

        for (;;) {
            steps += 1;
            if (steps > step_limit) {
                status = RFB_STATUS_STEP_LIMIT;
                break;
            }
            cells += 1;
            double4 xi = ld_site(S.site4 + i);
            int32_t k0 = __ldg(S.off + i), k1 = __ldg(S.off + i + 1);
            visits += k1 - k0;
            double best_t;
            int32_t best_j;
            exit_face<1>(S.site4, S.nbr, k0, k1, xi, r, 0, 0xffffffffu, best_t, best_j);
            if (best_j < 0 || best_t >= r.t_max) {
                if (r.t_max > entry) record(i, entry, r.t_max);
                break;
            }
            if (best_t < entry) best_t = entry;
            if (best_t - entry > width_floor) {
                record(i, entry, best_t);
                entry = best_t;
                zero_adv = 0;
                if (below_epsilon(log_T, epsilon, log_eps)) break;
                if (nseg >= step_limit) {
                    status = RFB_STATUS_STEP_LIMIT;
                    break;
                }
            } else {
                zero_adv += 1;
                if (zero_adv > kZeroAdvanceLimit) {
                    status = RFB_STATUS_CYCLE;
                    break;
                }
            }
            i = best_j;
        }
        my_cells += (unsigned long long)cells;
        my_visits += (unsigned long long)visits;
        if (O.status) O.status[q] = (int8_t)status;
        if (O.nseg) O.nseg[q] = nseg;
        if (status != RFB_STATUS_OK) {
            store_out(O.rgb, 3 * q, S.bg[0], O.f64);
            store_out(O.rgb, 3 * q + 1, S.bg[1], O.f64);
            store_out(O.rgb, 3 * q + 2, S.bg[2], O.f64);
            if (O.residual) store_out(O.residual, q, 1.0, O.f64);
            if (O.wsum) store_out(O.wsum, q, 0.0, O.f64);
            continue;
        }
        cr += Tc * S.bg[0];
        cg += Tc * S.bg[1];
        cb += Tc * S.bg[2];
        store_out(O.rgb, 3 * q, cr, O.f64);
        store_out(O.rgb, 3 * q + 1, cg, O.f64);
        store_out(O.rgb, 3 * q + 2, cb, O.f64);
        if (O.residual) store_out(O.residual, q, Tc, O.f64);
        if (O.wsum) store_out(O.wsum, q, wsum, O.f64);

        double ar, ag, ab;
        if (TRAIN) {  // kernels.py:430-437
            double er = cr - targets[3 * q], eg = cg - targets[3 * q + 1],
                   eb = cb - targets[3 * q + 2];
            loss_rgb += er * er + eg * eg + eb * eb;
            ar = 2.0 * rgb_scale * er;
            ag = 2.0 * rgb_scale * eg;
            ab = 2.0 * rgb_scale * eb;
        } else {
            ar = adjoints[3 * q];
            ag = adjoints[3 * q + 1];
            ab = adjoints[3 * q + 2];
        }

        // backward_ray (kernels.py:267-337), reverse order over the slot.
        if (nseg > 0) {
            double T_end = s_tb[(nseg - 1) * SL];
            double Sr = T_end * S.bg[0], Sg = T_end * S.bg[1], Sb = T_end * S.bg[2];
            double d_next = 0.0;
            for (int32_t s = nseg - 1; s >= 0; --s) {
                int32_t cm = s_cell[s * SL];
                int32_t ci = cm & 0x1fffffff;
                int mask = (cm >> 29) & 7;
                double t1 = s_t1[s * SL];
                double t0 = s > 0 ? s_t1[(s - 1) * SL] : r.t_min;
                double tb_s = s > 0 ? s_tb[(s - 1) * SL] : 1.0;
                double tb_s1 = s_tb[s * SL];
                double sig = __ldg(&S.site4[ci].w);
                double delta = t1 - t0;
                double alpha = 1.0 - exp(-sig * delta);
                double w = tb_s * alpha;
                double c0 = s_col[(3 * s) * SL], c1 = s_col[(3 * s + 1) * SL],
                       c2 = s_col[(3 * s + 2) * SL];
                double g_r = ar * (tb_s1 * c0 - Sr);
                double g_g = ag * (tb_s1 * c1 - Sg);
                double g_b = ab * (tb_s1 * c2 - Sb);
                double common = g_r + g_g + g_b;
                atomicAdd(gr.g4 + 4 * (int64_t)ci + 3, (float)(delta * common));
                double dd = sig * common;
                if (s < nseg - 1) {  // interior boundary s+1 (kernels.py:328-337)
                    double dt = dd - d_next;
                    if (dt != 0.0) {
                        int32_t cj = s_cell[(s + 1) * SL] & 0x1fffffff;
                        face_t_gradient(S.site4, ci, cj, r, t1, dt, gr.g4);
                    }
                }
                if (w != 0.0) add_sh<SHDEG>(gr.sh, ci, mask, w, ar, ag, ab, basis);
                Sr = Sr + w * c0;
                Sg = Sg + w * c1;
                Sb = Sb + w * c2;
                d_next = dd;
            }
        }

        // quantile_backward_ray (kernels.py:456-567) for each pair.
        if (TRAIN && q_scale > 0.0 && nseg > 0) {
            double T_end = s_tb[(nseg - 1) * SL];
            double tot = 1.0 - T_end;
            if (!(tot < weight_floor)) {
                for (int32_t p = 0; p < n_pairs; ++p) {
                    const double *up = u_pairs + (q * n_pairs + p) * 2;
                    double t_hit[2];
                    int32_t seg_hit[2];
                    for (int a = 0; a < 2; ++a) {
                        double target = up[a] * tot;
                        int32_t s = 0;
                        while (s < nseg - 1 && (1.0 - s_tb[s * SL]) < target) s += 1;
                        int32_t ci = s_cell[s * SL] & 0x1fffffff;
                        double si = __ldg(&S.site4[ci].w);
                        double t0 = s > 0 ? s_t1[(s - 1) * SL] : r.t_min;
                        seg_hit[a] = s;
                        if (si <= 0.0) {
                            t_hit[a] = t0;
                            continue;
                        }
                        double Tbs = s > 0 ? s_tb[(s - 1) * SL] : 1.0;
                        double Wbs = 1.0 - Tbs;
                        double frac = (target - Wbs) / Tbs;
                        if (frac > 1.0 - 1e-15) frac = 1.0 - 1e-15;
                        double th = t0 - log(1.0 - frac) / si;
                        double t1 = s_t1[s * SL];
                        if (th > t1) th = t1;
                        t_hit[a] = th;
                    }
                    double diff = t_hit[0] - t_hit[1];
                    loss_q += fabs(diff);
                    if (diff == 0.0) continue;
                    double sign = diff > 0.0 ? 1.0 : -1.0;
                    for (int a = 0; a < 2; ++a) {
                        double u = up[a];
                        int32_t s = seg_hit[a];
                        int32_t ci = s_cell[s * SL] & 0x1fffffff;
                        double si = __ldg(&S.site4[ci].w);
                        double t_u = t_hit[a];
                        double t0s = s > 0 ? s_t1[(s - 1) * SL] : r.t_min;
                        double Tbs = s > 0 ? s_tb[(s - 1) * SL] : 1.0;
                        double T_at = Tbs * exp(-si * (t_u - t0s));
                        double wd = T_at * si;
                        if (wd <= 1e-300) continue;
                        double g = (a == 0 ? sign : -sign) * q_scale / wd;
                        double prev_t1 = r.t_min;
                        for (int32_t k = 0; k < nseg; ++k) {  // kernels.py:534-548
                            double k_t0 = prev_t1, k_t1 = s_t1[k * SL];
                            prev_t1 = k_t1;
                            int32_t ck = s_cell[k * SL] & 0x1fffffff;
                            double dA = T_end * (k_t1 - k_t0);
                            double contrib;
                            if (k_t0 < t_u) {
                                double hi = k_t1 < t_u ? k_t1 : t_u;
                                double dW = T_at * (hi - k_t0);
                                contrib = g * (u * dA - dW);
                            } else {
                                contrib = g * (u * dA);
                            }
                            atomicAdd(gr.g4 + 4 * (int64_t)ck + 3, (float)contrib);
                        }
                        for (int32_t mm = 1; mm < nseg; ++mm) {  // kernels.py:552-566
                            int32_t im = s_cell[(mm - 1) * SL] & 0x1fffffff;
                            int32_t jm = s_cell[mm * SL] & 0x1fffffff;
                            double dsig = __ldg(&S.site4[im].w) - __ldg(&S.site4[jm].w);
                            if (dsig == 0.0) continue;
                            double tb = s_t1[(mm - 1) * SL];
                            double dW = tb < t_u ? T_at * dsig : 0.0;
                            double dA = T_end * dsig;
                            double dt_term = g * (u * dA - dW);
                            if (dt_term != 0.0) face_t_gradient(S.site4, im, jm, r, tb, dt_term, gr.g4);
                        }
                    }
                }
            }
        }
    }
    // per-warp reductions of the loss and counters
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        loss_rgb += __shfl_xor_sync(0xffffffffu, loss_rgb, off);
        loss_q += __shfl_xor_sync(0xffffffffu, loss_q, off);
        my_cells += __shfl_xor_sync(0xffffffffu, my_cells, off);
        my_visits += __shfl_xor_sync(0xffffffffu, my_visits, off);
    }
    if (lane == 0) {
        if (TRAIN && loss) {
            atomicAdd(loss, loss_rgb);
            atomicAdd(loss + 1, loss_q);
        }
        if (O.counters) {
            atomicAdd(O.counters, my_cells);
            atomicAdd(O.counters + 1, my_visits);
        }
    }
}

// ---------------------------------------------------------------------------
// Scene packing, activation, camera rays, start-cell location.
// ---------------------------------------------------------------------------
__global__ void k_pack_sites(const double *pos, const double *sigma, int64_t n, double4 *site4) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) site4[i] = make_double4(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2], sigma[i]);
}

__global__ void k_narrow(const int64_t *src, int64_t n, int32_t *dst) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = (int32_t)src[i];
}

// foam.py:22-25 (device libm; differs from numpy's log1p/exp by <= 1 ulp).
__global__ void k_softplus(const double *raw, int64_t n, double *out, double4 *site4) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double x = raw[i];
    double v = fmax(x, 0.0) + log1p(exp(-fabs(10.0 * x))) / 10.0;
    if (out) out[i] = v;
    if (site4) site4[i].w = v;
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

// Greedy point location on the Delaunay graph: move to the neighbour with
// the smallest (distance, id) while it beats the current site.  Same
// distance expression and lowest-id tie rule as adjacency.py:194-200.
__device__ int32_t locate_one(const DevScene &S, double qx, double qy, double qz, int32_t cur) {
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

__global__ void k_locate(DevScene S, const double *qs, int64_t m, int32_t seed, int32_t *out) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < m) out[k] = locate_one(S, qs[3 * k], qs[3 * k + 1], qs[3 * k + 2], seed);
}

__global__ void k_locate_point(DevScene S, double qx, double qy, double qz, int32_t seed,
                               int32_t *out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) *out = locate_one(S, qx, qy, qz, seed);
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

static DevScene dev_scene(const rfb_scene *s) {
    DevScene d;
    d.site4 = reinterpret_cast<const double4 *>(s->site4);
    d.off = s->offsets;
    d.nbr = s->neighbors;
    d.sh = s->sh;
    d.bg[0] = s->background[0];
    d.bg[1] = s->background[1];
    d.bg[2] = s->background[2];
    return d;
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
    return d;
}

static bool scene_ok(const rfb_scene *s) {
    return s && s->site4 && s->offsets && s->neighbors && s->sh && s->n_sites > 0 &&
           s->n_sites < (1 << 29) && (s->sh_degree == 0 || s->sh_degree == 3);
}

static bool out_ok(const rfb_fwd_out *o) {
    if (!o || !o->rgb) return false;
    if (o->seg_capacity > 0 && (!o->seg_cells || !o->seg_t0 || !o->seg_t1)) return false;
    return true;
}

template <int G, class Src>
static void launch_render_g(const DevScene &S, const Src &src, int shdeg, double eps,
                            double log_eps, double wf, int32_t sl, const FwdOut &O,
                            unsigned long long *ctr, cudaStream_t st) {
    int per_sm = 0;
    if (shdeg == 0) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_render<G, 0, Src>, 256, 0);
        k_render<G, 0, Src><<<num_sms() * std::max(per_sm, 1), 256, 0, st>>>(S, src, eps, log_eps,
                                                                            wf, sl, O, ctr);
    } else {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_render<G, 3, Src>, 256, 0);
        k_render<G, 3, Src><<<num_sms() * std::max(per_sm, 1), 256, 0, st>>>(S, src, eps, log_eps,
                                                                            wf, sl, O, ctr);
    }
}

template <class Src>
static int launch_render(const rfb_scene *scene, const Src &src, const rfb_params *p,
                         const rfb_fwd_out *out, void *ws, size_t ws_bytes, cudaStream_t st) {
    if (!ws || ws_bytes < 256) return RFB_EINVAL;
    unsigned long long *ctr = reinterpret_cast<unsigned long long *>(ws);
    cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), st);
    DevScene S = dev_scene(scene);
    FwdOut O = dev_out(out);
    double log_eps = p->epsilon > 0.0 ? std::log(p->epsilon) : 0.0;
    int g = p->lanes_per_ray <= 0 ? 1 : p->lanes_per_ray;
    switch (g) {
        case 1: launch_render_g<1>(S, src, scene->sh_degree, p->epsilon, log_eps, p->width_floor, p->step_limit, O, ctr, st); break;
        case 2: launch_render_g<2>(S, src, scene->sh_degree, p->epsilon, log_eps, p->width_floor, p->step_limit, O, ctr, st); break;
        case 4: launch_render_g<4>(S, src, scene->sh_degree, p->epsilon, log_eps, p->width_floor, p->step_limit, O, ctr, st); break;
        case 8: launch_render_g<8>(S, src, scene->sh_degree, p->epsilon, log_eps, p->width_floor, p->step_limit, O, ctr, st); break;
        case 16: launch_render_g<16>(S, src, scene->sh_degree, p->epsilon, log_eps, p->width_floor, p->step_limit, O, ctr, st); break;
        case 32: launch_render_g<32>(S, src, scene->sh_degree, p->epsilon, log_eps, p->width_floor, p->step_limit, O, ctr, st); break;
        default: return RFB_EINVAL;
    }
    return (int)cudaGetLastError();
}

static int64_t bwd_slot_bytes(int32_t step_limit) {
    return (int64_t)step_limit * (4 + 8 + 8 + 12);
}

static int64_t bwd_slots_max() {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_backward<3, true>, 128, 0);
    return (int64_t)num_sms() * std::max(per_sm, 1) * 128;
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
    if (!ws || ws_bytes < 256 + (size_t)bwd_slot_bytes(p->step_limit) * 128) return RFB_EINVAL;
    int64_t slots = (int64_t)((ws_bytes - 256) / (size_t)bwd_slot_bytes(p->step_limit));
    slots = std::min<int64_t>(slots, bwd_slots_max());
    slots = (slots / 128) * 128;
    const int64_t ray_blocks = (rays->m + 127) / 128;
    slots = std::min<int64_t>(slots, ray_blocks * 128);
    char *base = reinterpret_cast<char *>(ws);
    unsigned long long *ctr = reinterpret_cast<unsigned long long *>(base);
    Scratch scr;
    scr.slots = slots;
    int64_t cap = p->step_limit;
    char *c = base + 256;
    scr.t1 = reinterpret_cast<double *>(c);
    c += cap * slots * 8;
    scr.tb = reinterpret_cast<double *>(c);
    c += cap * slots * 8;
    scr.cell = reinterpret_cast<int32_t *>(c);
    c += cap * slots * 4;
    scr.col = reinterpret_cast<float *>(c);
    cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), st);
    DevScene S = dev_scene(scene);
    FwdOut O = dev_out(out);
    ArrayRays src{rays->origins, rays->directions, rays->t_min, rays->t_max, rays->start_sites,
                  rays->m};
    Grads G{grads->site4g, grads->sh};
    double log_eps = p->epsilon > 0.0 ? std::log(p->epsilon) : 0.0;
    dim3 grid((unsigned)(slots / 128));
#define RFB_BWD(SH, TR)                                                                           \
    k_backward<SH, TR><<<grid, 128, 0, st>>>(S, src, p->epsilon, log_eps, p->width_floor,        \
                                             p->step_limit, adjoints, targets, rgb_scale, q_scale, \
                                             u_pairs, n_pairs, wfloor, O, G, loss, scr, ctr)
    if (scene->sh_degree == 0) {
        if (train) RFB_BWD(0, true); else RFB_BWD(0, false);
    } else {
        if (train) RFB_BWD(3, true); else RFB_BWD(3, false);
    }
#undef RFB_BWD
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
    return p;
}

}  // namespace rfb

using namespace rfb;

extern "C" {

int rfb_abi_version(void) { return RFB_ABI_VERSION; }

const char *rfb_error_string(int code) {
    if (code == RFB_OK) return "ok";
    if (code == RFB_EINVAL) return "invalid argument";
    return cudaGetErrorString((cudaError_t)code);
}

int rfb_device_ok(void) {
    int dev = 0, major = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess)
        return 0;
    return major == 10 ? 1 : 0;
}

int rfb_pack_scene(const double *positions, const double *sigma, const int64_t *offsets,
                   const int64_t *neighbors, int64_t n_sites, int64_t n_edges, double *site4,
                   int32_t *offsets32, int32_t *neighbors32, void *stream) {
    if (!positions || !sigma || !offsets || !neighbors || !site4 || !offsets32 || !neighbors32 ||
        n_sites <= 0 || n_edges < 0 || n_edges >= (int64_t)1 << 31)
        return RFB_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    k_pack_sites<<<(unsigned)((n_sites + 255) / 256), 256, 0, st>>>(
        positions, sigma, n_sites, reinterpret_cast<double4 *>(site4));
    k_narrow<<<(unsigned)((n_sites + 1 + 255) / 256), 256, 0, st>>>(offsets, n_sites + 1, offsets32);
    if (n_edges > 0)
        k_narrow<<<(unsigned)((n_edges + 255) / 256), 256, 0, st>>>(neighbors, n_edges, neighbors32);
    return (int)cudaGetLastError();
}

int rfb_softplus(const double *raw, int64_t n, double *out, double *site4_sigma, void *stream) {
    if (!raw || n < 0 || (!out && !site4_sigma)) return RFB_EINVAL;
    if (n == 0) return RFB_OK;
    k_softplus<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        raw, n, out, reinterpret_cast<double4 *>(site4_sigma));
    return (int)cudaGetLastError();
}

int rfb_camera_rays(const rfb_camera *camera, int64_t pix_begin, int64_t pix_count, double *dirs,
                    void *stream) {
    if (!camera || !dirs || pix_begin < 0 || pix_count < 0 || camera->width < 1 ||
        camera->height < 1 || !(camera->focal > 0.0) ||
        pix_begin + pix_count > (int64_t)camera->width * camera->height)
        return RFB_EINVAL;
    if (pix_count == 0) return RFB_OK;
    k_camera_rays<<<(unsigned)((pix_count + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        cam_params(camera), pix_begin, pix_count, dirs);
    return (int)cudaGetLastError();
}

int rfb_locate(const rfb_scene *scene, const double *queries, int64_t m, int32_t seed_site,
               int32_t *out, void *stream) {
    if (!scene_ok(scene) || !queries || !out || m < 0 || seed_site < 0 ||
        seed_site >= scene->n_sites)
        return RFB_EINVAL;
    if (m == 0) return RFB_OK;
    k_locate<<<(unsigned)((m + 127) / 128), 128, 0, (cudaStream_t)stream>>>(dev_scene(scene),
                                                                            queries, m, seed_site, out);
    return (int)cudaGetLastError();
}

size_t rfb_workspace_bytes(int64_t m, int32_t step_limit, int32_t kind) {
    if (kind == 0) return 256;
    int64_t slots = std::min<int64_t>(bwd_slots_max(), ((m + 127) / 128) * 128);
    slots = std::max<int64_t>(slots, 128);
    return 256 + (size_t)slots * (size_t)bwd_slot_bytes(step_limit);
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
                  rays->m};
    return launch_render(scene, src, params, out, workspace, workspace_bytes,
                         (cudaStream_t)stream);
}

int rfb_render_image(const rfb_scene *scene, const rfb_camera *camera, const rfb_params *params,
                     double t_min, double t_max, int32_t start_site, const int32_t *tile_ids,
                     int64_t n_tiles, int32_t tile_w, int32_t tile_h, const rfb_fwd_out *out,
                     void *workspace, size_t workspace_bytes, void *stream) {
    if (!scene_ok(scene) || !camera || !params || !out_ok(out) || params->step_limit <= 0 ||
        !tile_ids || n_tiles < 0 || tile_w < 8 || tile_h < 4 || tile_w % 8 || tile_h % 4 ||
        camera->width < 1 || camera->height < 1 || !(camera->focal > 0.0) ||
        start_site >= scene->n_sites || !workspace || workspace_bytes < 256)
        return RFB_EINVAL;
    if (n_tiles == 0) return RFB_OK;
    cudaStream_t st = (cudaStream_t)stream;
    int32_t *start_ptr = reinterpret_cast<int32_t *>(reinterpret_cast<char *>(workspace) + 64);
    if (start_site < 0) {
        k_locate_point<<<1, 32, 0, st>>>(dev_scene(scene), camera->pose[3], camera->pose[7],
                                         camera->pose[11], 0, start_ptr);
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
