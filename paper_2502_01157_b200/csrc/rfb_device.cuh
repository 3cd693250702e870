// rfb_device.cuh -- device-side building blocks of the Radiant Foam hot path.
//
// Compiled with -fmad=false: every fp64 expression on the walk is evaluated
// with the reference's exact operation order and no FMA contraction, so the
// visited-cell sequence is bit-identical to rfoam/tracer/kernels.py:76-162
// (numba, fastmath=False, rfoam/_accel.py:33-39).  The only intentional FMA
// (camera rays) is written with explicit __fma_rn to match numpy's matmul.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/rfb.h"

namespace rfb {

constexpr int kZeroAdvanceLimit = 32;  // tracer/kernels.py:23

// SH constants: tracer/kernels.py:26-35.
constexpr double kC0 = 0.28209479177387814;
constexpr double kC1 = 0.4886025119029199;
constexpr double kC2_0 = 1.0925484305920792;
constexpr double kC2_2 = 0.31539156525252005;
constexpr double kC2_4 = 0.5462742152960396;
constexpr double kC3_0 = 0.5900435899266435;
constexpr double kC3_1 = 2.890611442640554;
constexpr double kC3_2 = 0.4570457994644658;
constexpr double kC3_3 = 0.3731763325901154;
constexpr double kC3_5 = 1.445305721320277;

// tracer/kernels.py:38-58, same association order.
__device__ __forceinline__ void sh_basis(double dx, double dy, double dz, double *out) {
    double xx = dx * dx, yy = dy * dy, zz = dz * dz;
    out[0] = kC0;
    out[1] = kC1 * dy;
    out[2] = kC1 * dz;
    out[3] = kC1 * dx;
    out[4] = kC2_0 * dx * dy;
    out[5] = kC2_0 * dy * dz;
    out[6] = kC2_2 * (3.0 * zz - 1.0);
    out[7] = kC2_0 * dx * dz;
    out[8] = kC2_4 * (xx - yy);
    out[9] = kC3_0 * dy * (3.0 * xx - yy);
    out[10] = kC3_1 * dx * dy * dz;
    out[11] = kC3_2 * dy * (5.0 * zz - 1.0);
    out[12] = kC3_3 * dz * (5.0 * zz - 3.0);
    out[13] = kC3_2 * dx * (5.0 * zz - 1.0);
    out[14] = kC3_5 * dz * (xx - yy);
    out[15] = kC3_0 * dx * (xx - 3.0 * yy);
}

// tracer/kernels.py:61-73.  SHDEG 0 reads only the DC band: with bands 1..15
// all zero the skipped terms add +-0.0, so the result is bit-identical.
template <int SHDEG>
__device__ __forceinline__ int cell_color(const double *__restrict__ sh, int32_t i,
                                          const double *basis, double *col) {
    const double *row = sh + (int64_t)i * 48;
    int mask = 0;
    if (SHDEG == 0) {
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            double acc = 0.5;
            acc += basis[0] * __ldg(row + ch);
            if (acc < 0.0) {
                acc = 0.0;
                mask |= 1 << ch;
            }
            col[ch] = acc;
        }
    } else {
        double c[48];
        const double2 *row2 = reinterpret_cast<const double2 *>(row);
#pragma unroll
        for (int k = 0; k < 24; ++k) {
            double2 v = __ldg(row2 + k);
            c[2 * k] = v.x;
            c[2 * k + 1] = v.y;
        }
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            double acc = 0.5;
#pragma unroll
            for (int k = 0; k < 16; ++k) acc += basis[k] * c[k * 3 + ch];
            if (acc < 0.0) {
                acc = 0.0;
                mask |= 1 << ch;
            }
            col[ch] = acc;
        }
    }
    return mask;
}

// 32-byte read-only site record load (two 16-byte vector loads).
__device__ __forceinline__ double4 ld_site(const double4 *p) {
    const double2 *q = reinterpret_cast<const double2 *>(p);
    double2 a = __ldg(q), b = __ldg(q + 1);
    return make_double4(a.x, a.y, b.x, b.y);
}

struct Ray {
    double ox, oy, oz, dx, dy, dz, t_min, t_max;
    int32_t start;
};

// log(eps) test with a guard band: exp() is only evaluated when log_T is
// within 1e-9 of log(eps), so the decision equals `exp(log_T) < eps`
// (tracer/kernels.py:154) while skipping one fp64 exp per segment.
__device__ __forceinline__ bool below_epsilon(double log_T, double epsilon, double log_eps) {
    if (!(epsilon > 0.0)) return false;
    if (log_T > log_eps + 1e-9) return false;
    if (log_T < log_eps - 1e-9) return true;
    return exp(log_T) < epsilon;
}

// One walk step's exit-face search over the CSR row of cell i, executed by
// the G lanes of a ray group (gl = lane within group); returns the group-wide
// first minimum in ascending CSR order (kernels.py:116-133).
template <int G>
__device__ __forceinline__ void exit_face(const double4 *__restrict__ site4,
                                          const int32_t *__restrict__ nbr, int32_t k0, int32_t k1,
                                          double4 xi, const Ray &r, int gl, unsigned gmask,
                                          double &best_t, int32_t &best_j) {
    best_t = __longlong_as_double(0x7ff0000000000000LL);  // +inf
    best_j = -1;
    int32_t best_k = 0x7fffffff;
    for (int32_t k = k0 + gl; k < k1; k += G) {
        int32_t j = __ldg(nbr + k);
        double4 xj = ld_site(site4 + j);
        double nx = xj.x - xi.x;
        double ny = xj.y - xi.y;
        double nz = xj.z - xi.z;
        double denom = r.dx * nx + r.dy * ny + r.dz * nz;
        if (denom <= 0.0) continue;
        double mx = 0.5 * (xj.x + xi.x);
        double my = 0.5 * (xj.y + xi.y);
        double mz = 0.5 * (xj.z + xi.z);
        double t = ((mx - r.ox) * nx + (my - r.oy) * ny + (mz - r.oz) * nz) / denom;
        if (t < best_t) {
            best_t = t;
            best_j = j;
            best_k = k;
        }
    }
    if (G > 1) {
#pragma unroll
        for (int off = G / 2; off > 0; off >>= 1) {
            double ot = __shfl_xor_sync(gmask, best_t, off, G);
            int32_t oj = __shfl_xor_sync(gmask, best_j, off, G);
            int32_t ok = __shfl_xor_sync(gmask, best_k, off, G);
            if (ot < best_t || (ot == best_t && ok < best_k)) {
                best_t = ot;
                best_j = oj;
                best_k = ok;
            }
        }
    }
}

}  // namespace rfb
