// rfb_device.cuh -- device-side building blocks of the Radiant Foam hot path.
//
// Compiled with -fmad=false: every fp64 expression on the walk is evaluated
// with the reference's exact operation order and no FMA contraction, so the
// visited-cell sequence is bit-identical to rfoam/tracer/kernels.py:76-162
// (numba, fastmath=False, rfoam/_accel.py:33-39).  The only intentional FMA
// (camera rays) is written with explicit __fma_rn to match numpy's matmul.
//
// Scene layouts:
//  * Packed (positions exactly representable in fp32, the fixture rule):
//      cell header  [n]  32 B = {float x,y,z; int k0; double sigma; int k1; float cmax}
//      edge record  [E]  16 B = {float xj, yj, zj; int j}   (CSR order)
//    One step = one 32-byte header load + one 16-byte load per neighbour,
//    contiguous per cell; the fp32 values are widened to fp64 exactly.
//  * Generic (arbitrary fp64 positions): site4 [n] {x,y,z,sigma} fp64,
//    offsets/neighbors int32 -- two dependent gathers per neighbour.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/rfb.h"

#ifndef RFB_LDG256
#define RFB_LDG256 1  // 256-bit loads for edge pairs and SH rows (packed layout)
#endif
#ifndef RFB_SH_NOALLOC
#define RFB_SH_NOALLOC 1  // SH row loads: 1 L1::no_allocate, 2 L1::evict_first, 0 default
#endif
#ifndef RFB_SH_PIPE
#define RFB_SH_PIPE 1  // SH colour: the next channel's row loads overlap this channel's sum
#endif
#ifndef RFB_CHECK
#define RFB_CHECK 0  // 1: device-side bounds asserts on every scene gather / record (debug build)
#endif
#if RFB_CHECK
#include <cassert>
#define RFB_BOUND(i, n) assert((int64_t)(i) >= 0 && (int64_t)(i) < (int64_t)(n))
#else
#define RFB_BOUND(i, n) ((void)0)
#endif

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

__device__ __forceinline__ double dinf() { return __longlong_as_double(0x7ff0000000000000LL); }

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

// 32-byte read-only record load (two 16-byte vector loads).
__device__ __forceinline__ double4 ld_site(const double4 *p) {
#if RFB_LDG256
    double4 v;  // one 256-bit request (site4 rows are 32-byte aligned)
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
        : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
        : "l"(p));
    return v;
#else
    const double2 *q = reinterpret_cast<const double2 *>(p);
    double2 a = __ldg(q), b = __ldg(q + 1);
    return make_double4(a.x, a.y, b.x, b.y);
#endif
}
// sigma only (site4[i].w)
__device__ __forceinline__ double ld_sigma(const double4 *p) {
    return __ldg(reinterpret_cast<const double *>(p) + 3);
}

struct CellHdr {  // packed layout, 32 bytes
    float x, y, z;
    int32_t k0;
    double sigma;
    int32_t k1;
    float n1max;  // >= max over the row of |x_j - x_i|_1 as the kernel computes it in fp32
};
static_assert(sizeof(CellHdr) == 32, "cell header must be one 32-byte sector");

struct Cell {
    double x, y, z, sigma;
    int32_t k0, k1;
    float n1max;
    float4 hf;  // packed: fp32 x, y, z (exact copies of x, y, z)
};

// Read-only view of the device scene.  PACKED selects the layout above.
// 256-bit read-only global load (LDG.E.ENL2.256 on sm_100a): one request
// for 32 contiguous, 32-byte aligned bytes.
__device__ __forceinline__ void ldg256(const void *p, float4 &a, float4 &b) {
    asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z),
          "=f"(b.w)
        : "l"(p));
}

// The same for data used once per lane (SH rows): not allocated in L1, so the
// step's header and row sectors stay there for their second use (sigma, phase 2)
// instead of being evicted by the 192-byte rows (1080p config 2: 13.38 -> 12.32 ms;
// evict_first: 13.11 ms; hints on the edge pairs / header / reverse-pass records:
// no change).
__device__ __forceinline__ void ldg256_stream(const void *p, float4 &a, float4 &b) {
#if RFB_SH_NOALLOC == 1
    asm("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z),
          "=f"(b.w)
        : "l"(p));
#elif RFB_SH_NOALLOC == 2
    asm("ld.global.nc.L1::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z),
          "=f"(b.w)
        : "l"(p));
#else
    ldg256(p, a, b);
#endif
}

// PACKED: 0 generic (site4 + int32 CSR), 1 packed with fp32-exact sites,
// 2 packed with fp64 sites (rounded fp32 copies, widened bound; rfb_scene.positions_f64)
template <int PACKED>
struct SceneView {
    const CellHdr *hdr;     // PACKED
    const float4 *edge;     // PACKED
    const int32_t *enbr;    // PACKED: neighbour id per packed edge slot (-1: row pad)
    // PACKED: the packed arrays are in the scene's internal (Morton) order; pk_of maps
    // a site id to its packed index, pk_id back (nullable: identity)
    const int32_t *pk_of, *pk_id;
    const double4 *site4;   // both (backward gradients use fp64 positions)
    const int32_t *off;     // generic
    const int32_t *nbr;     // generic
    const float *sh32;      // [n][3][16] fp32, channel-major (PACKED) -- exact fallback below
    const double *sh;       // [n][48] fp64 (reference values)
    float sh_absmax;        // max |sh coefficient| over the scene (colour rounding bound)
    const float *absmax_p;  // nullable device copy of the bound (training: raised by Adam)
    double bg[3];
    int64_t n_sites, n_edges;  // extents (RFB_CHECK builds assert every index against them)
    // view-culled scenes (rfb_cull_view): view_rx * view_ry region copies of the
    // headers (region r's at hdr + r * n_sites; the walk adds the ray's offset) and rows
    int32_t view_rx, view_ry, n_views;
    int64_t edge_slots;  // records in `edge` (every region)

    // site id <-> packed index (identity for the generic layout)
    __device__ __forceinline__ int32_t to_pk(int32_t i) const {
        return (PACKED && pk_of) ? __ldg(pk_of + i) : i;
    }
    __device__ __forceinline__ int32_t to_id(int32_t u) const {
        return (PACKED && pk_id) ? __ldg(pk_id + u) : u;
    }

    // Per-step cell record.  PACKED: only the fp32 header fields (the walk
    // widens x,y,z exactly where the fp64 path needs them and fetches sigma
    // when a segment is recorded) -- fewer live registers across the
    // neighbour loop.
    __device__ __forceinline__ Cell cell(int32_t i) const {
        RFB_BOUND(i, n_sites * n_views);
        Cell c;
        if (PACKED) {
            const float4 *p = reinterpret_cast<const float4 *>(hdr + i);
            float4 a = __ldg(p);
            const float2 b = __ldg(reinterpret_cast<const float2 *>(p + 1) + 1);
            c.hf = a;
            c.k0 = __float_as_int(a.w);
            c.k1 = __float_as_int(b.x);
            c.n1max = b.y;
            RFB_BOUND(c.k0, c.k1 + 1);
            RFB_BOUND(c.k1, edge_slots + 1);  // padded rows (RFB_PACKED_EDGE_SLOTS / view)
            RFB_BOUND(c.k0 & 1, 1);                  // rows start at even slots
        } else {
            double4 s = ld_site(site4 + i);
            c.x = s.x;
            c.y = s.y;
            c.z = s.z;
            c.sigma = s.w;
            c.k0 = __ldg(off + i);
            c.k1 = __ldg(off + i + 1);
            c.n1max = 0.f;
        }
        return c;
    }

    __device__ __forceinline__ double sigma_of(int32_t i, const Cell &c) const {
        RFB_BOUND(i, n_sites);
        if (PACKED) return __ldg(&hdr[i].sigma);
        return c.sigma;
    }

    // CSR slot k's neighbour (generic) or packed slot k's (packed layout)
    __device__ __forceinline__ void edge_at(int32_t k, double &x, double &y, double &z,
                                            int32_t &j) const {
        if (PACKED) {
            RFB_BOUND(k, n_edges + n_sites + 2);
            j = __ldg(enbr + k);
            RFB_BOUND(j, n_sites);
            if (PACKED == 2) {
                const double4 s = ld_site(site4 + to_id(j));
                x = s.x;
                y = s.y;
                z = s.z;
            } else {
                const float4 h = __ldg(reinterpret_cast<const float4 *>(hdr + j));
                x = h.x;
                y = h.y;
                z = h.z;
            }
        } else {
            RFB_BOUND(k, n_edges);
            j = __ldg(nbr + k);
            RFB_BOUND(j, n_sites);
            double4 s = ld_site(site4 + j);
            x = s.x;
            y = s.y;
            z = s.z;
        }
    }
};

// tracer/kernels.py:61-73.  SHDEG 0 reads only the DC band: with bands 1..15
// all zero the skipped terms add +-0.0, so the result is bit-identical.
//
// PACKED (fast path): basis (fp32, per ray) and coefficients (fp32 copy) are
// accumulated with fp32 FMAs in the reference's k order.  Input rounding (2u)
// plus 16 accumulation roundings bound the deviation from the reference by
// 20u * (cmax * sum|basis| + 1), u = 2^-24; whenever |acc| is within 2^-19 *
// (cmax * sum|basis| + 1) >= that bound of the clamp threshold, the channel is
// recomputed exactly (fp64 basis from the direction, fp64 coefficients), so
// the clamp mask -- which gates the SH gradient -- is always the reference's
// and the colour is within ~1e-6 of it.
// Reference-exact channel value (kernels.py:66-68) from the fp64 table;
// out of line so its registers do not count against the walk.
static __device__ __noinline__ double exact_channel(const double *row, int ch, int nb, double dx,
                                             double dy, double dz) {
    double basis[16];
    sh_basis(dx, dy, dz, basis);
    double a = 0.5;
    for (int k = 0; k < nb; ++k) a += basis[k] * __ldg(row + k * 3 + ch);
    return a;
}

// Clamp-ambiguity tolerance of one ray for cell_color: (max|c| sum|basis| + 1) 2^-19,
// bsum = sum |fp64 basis| of the ray.  Evaluated once per ray (the bound is read from
// the device copy when the scene has one, so Adam steps that grow a coefficient
// never leave the fp32 colour with a stale bound).
template <int PACKED>
__device__ __forceinline__ double color_tol(const SceneView<PACKED> &S, double bsum) {
    if (!PACKED) return 0.0;
    const float cmax = S.absmax_p ? __ldg(S.absmax_p) : S.sh_absmax;
    return ((double)cmax * bsum + 1.0) * 0x1p-19;
}

// basis_f: the ray's fp32 SH basis (BSTRIDE apart); tol = color_tol(S, sum |fp64 basis|).
// SKIP0: basis_f holds k = 1..15 only (k = 0 is the direction-independent
// constant kC0, sh.py:17), which keeps k_render's shared memory per block
// under the 100 KB carveout step at 4 blocks per SM.
template <int SHDEG, int PACKED, int BSTRIDE = 1, int SKIP0 = 0, class RayT>
__device__ __forceinline__ int cell_color(const SceneView<PACKED> &S, int32_t i,
                                          const float *basis_f, const RayT &ray,
                                          double tol, double *col) {
    RFB_BOUND(i, S.n_sites);
    constexpr int NB = SHDEG == 0 ? 1 : 16;
    double acc[3] = {0.5, 0.5, 0.5};
    auto bk = [&](int k) -> float {
        if (SKIP0) return k == 0 ? (float)kC0 : basis_f[(k - 1) * BSTRIDE];
        return basis_f[k * BSTRIDE];
    };
    if (PACKED) {
        // sh32 is channel-major per site: [ch][16]; fp32 FMA accumulation
        const float *row = S.sh32 + (int64_t)i * 48;
        if (SHDEG == 0) {
#pragma unroll
            for (int ch = 0; ch < 3; ++ch)
                acc[ch] = (double)__fmaf_rn(bk(0), __ldg(row + 16 * ch), 0.5f);
        } else if (RFB_SH_PIPE) {
            // two channels' loads in flight: channel ch+1's 64 B arrive while ch is summed
            const float4 *r4 = reinterpret_cast<const float4 *>(row);
            float4 va[4], vb[4];
            ldg256_stream(r4, va[0], va[1]);
            ldg256_stream(r4 + 2, va[2], va[3]);
            ldg256_stream(r4 + 4, vb[0], vb[1]);
            ldg256_stream(r4 + 6, vb[2], vb[3]);
            auto dot = [&](const float4 *v) {
                float a = 0.5f;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    a = __fmaf_rn(bk(4 * q), v[q].x, a);
                    a = __fmaf_rn(bk(4 * q + 1), v[q].y, a);
                    a = __fmaf_rn(bk(4 * q + 2), v[q].z, a);
                    a = __fmaf_rn(bk(4 * q + 3), v[q].w, a);
                }
                return (double)a;
            };
            acc[0] = dot(va);
            ldg256_stream(r4 + 8, va[0], va[1]);
            ldg256_stream(r4 + 10, va[2], va[3]);
            acc[1] = dot(vb);
            acc[2] = dot(va);
        } else {
#pragma unroll 1
            for (int ch = 0; ch < 3; ++ch) {  // one channel (4 x 16 B) in flight: registers
                const float4 *r4 = reinterpret_cast<const float4 *>(row + 16 * ch);
                float a = 0.5f;
#if RFB_LDG256
                float4 vv[4];
                ldg256(r4, vv[0], vv[1]);  // rows are 192 B: 32-byte aligned
                ldg256(r4 + 2, vv[2], vv[3]);
#endif
#pragma unroll
                for (int q = 0; q < 4; ++q) {
#if RFB_LDG256
                    const float4 v = vv[q];
#else
                    const float4 v = __ldg(r4 + q);
#endif
                    a = __fmaf_rn(bk(4 * q), v.x, a);
                    a = __fmaf_rn(bk(4 * q + 1), v.y, a);
                    a = __fmaf_rn(bk(4 * q + 2), v.z, a);
                    a = __fmaf_rn(bk(4 * q + 3), v.w, a);
                }
                acc[ch] = (double)a;
            }
        }
    } else {
        double basis[16];
        if (SHDEG == 0)
            basis[0] = kC0;
        else
            sh_basis(ray.dx(), ray.dy(), ray.dz(), basis);
        const double *row = S.sh + (int64_t)i * 48;
#pragma unroll
        for (int k = 0; k < NB; ++k)
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) acc[ch] += basis[k] * __ldg(row + k * 3 + ch);
    }
    int mask = 0;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        double a = acc[ch];
        if (PACKED && fabs(a) <= tol)  // ambiguous clamp: redo in fp64 (exact)
            a = exact_channel(S.sh + (int64_t)S.to_id(i) * 48, ch, NB, ray.dx(), ray.dy(),
                              ray.dz());
        if (a < 0.0) {
            a = 0.0;
            mask |= 1 << ch;
        }
        col[ch] = a;
    }
    return mask;
}

// A ray in registers (writable by the ray sources) ...
struct Ray {
    double ox_, oy_, oz_, dx_, dy_, dz_, t_min_, t_max_;
    int32_t start_;
    __device__ __forceinline__ double ox() const { return ox_; }
    __device__ __forceinline__ double oy() const { return oy_; }
    __device__ __forceinline__ double oz() const { return oz_; }
    __device__ __forceinline__ double dx() const { return dx_; }
    __device__ __forceinline__ double dy() const { return dy_; }
    __device__ __forceinline__ double dz() const { return dz_; }
    __device__ __forceinline__ double t_min() const { return t_min_; }
    __device__ __forceinline__ double t_max() const { return t_max_; }
    __device__ __forceinline__ int32_t start() const { return start_; }
};

// ... or, for a shared-origin camera, only the direction per thread ([3][NT])
// with origin / t_min / t_max in one block-uniform shared copy.
template <int NT>
struct RaySmemU {
    double *p;        // &s_dir[0][threadIdx.x]
    const double *u;  // block-uniform {ox, oy, oz, t_min, t_max}
    __device__ __forceinline__ double ox() const { return u[0]; }
    __device__ __forceinline__ double oy() const { return u[1]; }
    __device__ __forceinline__ double oz() const { return u[2]; }
    __device__ __forceinline__ double dx() const { return p[0 * NT]; }
    __device__ __forceinline__ double dy() const { return p[1 * NT]; }
    __device__ __forceinline__ double dz() const { return p[2 * NT]; }
    __device__ __forceinline__ double t_min() const { return u[3]; }
    __device__ __forceinline__ double t_max() const { return u[4]; }
    __device__ __forceinline__ void store(const Ray &r) {
        p[0 * NT] = r.dx_;
        p[1 * NT] = r.dy_;
        p[2 * NT] = r.dz_;
    }
};

// ... or, for a shared-origin camera source passed as a __grid_constant__
// kernel parameter, the direction per thread in shared memory and the origin /
// t-range read straight from the parameter (constant bank: no data-pipe traffic).
template <int NT, class Src>
struct RaySmemP {
    double *p;       // &s_dir[0][threadIdx.x]
    const Src *src;  // address of the __grid_constant__ parameter
    __device__ __forceinline__ double ox() const { return src->cam.o[0]; }
    __device__ __forceinline__ double oy() const { return src->cam.o[1]; }
    __device__ __forceinline__ double oz() const { return src->cam.o[2]; }
    __device__ __forceinline__ double dx() const { return p[0 * NT]; }
    __device__ __forceinline__ double dy() const { return p[1 * NT]; }
    __device__ __forceinline__ double dz() const { return p[2 * NT]; }
    __device__ __forceinline__ double t_min() const { return src->t_min; }
    __device__ __forceinline__ double t_max() const { return src->t_max; }
    __device__ __forceinline__ void store(const Ray &r) {
        p[0 * NT] = r.dx_;
        p[1 * NT] = r.dy_;
        p[2 * NT] = r.dz_;
    }
};

// ... or parked in shared memory, field-major [8][NT] (conflict-free), so the
// fp64 ray constants do not occupy registers across the walk.
template <int NT>
struct RaySmem {
    double *p;  // &s_ray[0][threadIdx.x]
    __device__ __forceinline__ double ox() const { return p[0 * NT]; }
    __device__ __forceinline__ double oy() const { return p[1 * NT]; }
    __device__ __forceinline__ double oz() const { return p[2 * NT]; }
    __device__ __forceinline__ double dx() const { return p[3 * NT]; }
    __device__ __forceinline__ double dy() const { return p[4 * NT]; }
    __device__ __forceinline__ double dz() const { return p[5 * NT]; }
    __device__ __forceinline__ double t_min() const { return p[6 * NT]; }
    __device__ __forceinline__ double t_max() const { return p[7 * NT]; }
    __device__ __forceinline__ void store(const Ray &r) {
        p[0 * NT] = r.ox_;
        p[1 * NT] = r.oy_;
        p[2 * NT] = r.oz_;
        p[3 * NT] = r.dx_;
        p[4 * NT] = r.dy_;
        p[5 * NT] = r.dz_;
        p[6 * NT] = r.t_min_;
        p[7 * NT] = r.t_max_;
    }
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

// One walk step's exit-face search over the CSR row of cell c, executed by
// the G lanes of a ray group (gl = lane within group); returns the group-wide
// first minimum in ascending CSR order (kernels.py:116-133).
//
// Division filter: a candidate whose exact quotient num/denom is provably
// larger than the current best's (cross-multiplied with a rounding margin;
// both denominators are > 0) cannot satisfy the reference's `t < best_t`
// (rounding is monotone), so it is rejected without the fp64 division.
// Every quotient that could win is computed with IEEE division exactly as
// in the reference.
#ifndef RFB_EXIT_UNROLL
#define RFB_EXIT_UNROLL 2
#endif
#define RFB_STR_(x) #x
#define RFB_PRAGMA_UNROLL(n) _Pragma(RFB_STR_(unroll n))

template <int G, int PACKED, class RayT>
__device__ __forceinline__ void exit_face(const SceneView<PACKED> &S, const Cell &c,
                                          const RayT &r, int gl, unsigned gmask, double &best_t,
                                          int32_t &best_j) {
    best_t = dinf();
    best_j = -1;
    int32_t best_k = 0x7fffffff;
    double bnum = 0.0, bden = 1.0;
    bool have = false;
    RFB_PRAGMA_UNROLL(RFB_EXIT_UNROLL)
    for (int32_t k = c.k0 + gl; k < c.k1; k += G) {
        double xj, yj, zj;
        int32_t j;
        S.edge_at(k, xj, yj, zj, j);
        double nx = xj - c.x;
        double ny = yj - c.y;
        double nz = zj - c.z;
        double denom = r.dx() * nx + r.dy() * ny + r.dz() * nz;
        if (denom <= 0.0) continue;
        double mx = 0.5 * (xj + c.x);
        double my = 0.5 * (yj + c.y);
        double mz = 0.5 * (zj + c.z);
        double num = (mx - r.ox()) * nx + (my - r.oy()) * ny + (mz - r.oz()) * nz;
        if (have) {
            double c1 = num * bden, c2 = bnum * denom;
            if (c1 - c2 > (fabs(c1) + fabs(c2)) * 0x1p-50) continue;
        }
        double t = num / denom;
        if (t < best_t) {
            best_t = t;
            best_j = j;
            best_k = k;
            bnum = num;
            bden = denom;
            have = true;
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


// ---------------------------------------------------------------------------
// Packed-layout exit face with an fp32 pre-filter.
//
// Edge records (packed layout): row i holds, for each neighbour j in CSR
// order, {n = fl32(x_j - x_i) (fp32 copies), c = fl32(0.5 |n|^2)} -- the face
// plane n.(x - x_i) = c relative to the cell's own site -- and rows are padded
// to an even length (start index even) with an all-NaN record, so a row is
// read as whole 32-byte pairs (one LDG.256 per two neighbours) and a pad is
// rejected by the back-facing test like any back face (NaN compares false).
// The neighbour ids live in a parallel int32 array (edge_nbr) that only
// phase 2 reads.
//
// Phase 1 (fp32 FMA): for every neighbour, relative to q = o + entry*d (fp64,
// rounded once to fp32) and p = x_i - q, the shifted depth s = num / den with
//   den = d.n (3 FMA-chain ops),  num = c + p.n (3),
// and a rigorous bound on |s - s_exact| (u = 2^-24, N >= |n|_1 = n1max,
// P = |p|_inf, Q = |q|_inf):
//   den:  |den_f - d.n|      <= 5u N                      <= Ed = 8u N
//   num:  |num_f - (m-q).n|  <= u N (Q + 5P + 3N)         <= En = u N (Q + 8 Hm + 2N),
//         Hm = (P + N/2)(1 + 4u)   (the bound of the earlier (p + n/2).n form,
//         kept: it dominates this form's)
//   s:    es = 2.2 (En + |s| Ed) / den_f + 8u |s| + 2^-40 (|entry| + |s| + 1)
// (c's own rounding and the n rounding enter num as 1.5uN^2, p's as
// u(Q + P)N, the FMA chain as 3u(N^2/2 + PN); the last term of es covers the
// reference's own fp64 rounding).  For fp64 sites (PK = 2) the fp32 copies
// add <= 2uX per n component and uX per p component (X = largest |coordinate|
// of the cell and its neighbours): <= u(3XN + 6XP) to num and <= 6uX to den,
// covered by storing n1max = N + w with w = 2 max(X, 1/4) >= X (the bound's
// terms grow by >= uw(8P + 6N) and 8uw).  A neighbour is certainly
// back-facing unless den_f >= -Ed (NaN pads included), certainly front-facing
// if den_f > 2 Ed; anything in between is "uncertain".  Front-facing
// neighbours with s - es > U, U the running minimum of s + es, cannot be the
// reference's first minimum (their fp64 t is strictly larger than some other
// neighbour's).
// Phase 2 (fp64, exactly the reference's expressions on the exact sites):
// every uncertain neighbour and every front-facing one whose lower bound is
// within the final band (one lane: the running band while it is visited) is
// re-evaluated in CSR order with `denom <= 0 -> skip`, `t < best_t` -- so
// best_t / best_j are bit-identical to kernels.py:116-133.  With the final-
// band filter (below) usually only one neighbour is.  Rows longer than 32
// slots are evaluated exactly in full.
// ---------------------------------------------------------------------------
#ifndef RFB_F32_UNROLL
#define RFB_F32_UNROLL 4
#endif
#ifndef RFB_PAIR_UNROLL
#define RFB_PAIR_UNROLL 2  // edge pairs per unrolled phase-1 iteration (16-byte records)
#endif
typedef unsigned int cand_mask_t;
constexpr int kMaskBits = 32;

// Packed edge slot k: {fp32 copy of x_j, j}.
__device__ __forceinline__ float4 rec_site(const float4 *edge, int32_t k) { return __ldg(edge + k); }

// PK: 1 = packed with fp32-exact sites, 2 = packed with fp64 sites (positions_f64).
template <int G, int PK, class RayT>
__device__ __forceinline__ void exit_face_f32(const SceneView<PK> &S, int32_t ci, const Cell &c,
                                              const float4 &hdr_f, const RayT &r, double entry,
                                              const float *df, int gl, unsigned gmask,
                                              double &best_t, int32_t &best_j) {
    constexpr float u = 0x1p-24f;
    // q = o + entry * d in fp64 (once per step), rounded to fp32
    const double qx = r.ox() + entry * r.dx(), qy = r.oy() + entry * r.dy(), qz = r.oz() + entry * r.dz();
    const float qxf = (float)qx, qyf = (float)qy, qzf = (float)qz;
    const float Q = fmaxf(fabsf(qxf), fmaxf(fabsf(qyf), fabsf(qzf))) * (1.0f + 4.0f * u);
    const float px = hdr_f.x - qxf, py = hdr_f.y - qyf, pz = hdr_f.z - qzf;
    const float slack = (float)(0x1p-40 * (fabs(entry) + 1.0));
    const float N = c.n1max;
    const float Ed = 8.0f * u * N;
    const float thr = fmaxf(2.0f * Ed, 0x1p-100f);  // certainly front-facing above
    const float P = fmaxf(fabsf(px), fmaxf(fabsf(py), fabsf(pz)));
    const float Hm = (P + 0.5f * N) * (1.0f + 4.0f * u);
    const float K1 = 2.2f * u * N * (Q + 8.0f * Hm + 2.0f * N);
    const float K2 = 2.2f * Ed;
    constexpr float K3 = 8.0f * u + 0x1p-40f;
    const float kInf = __int_as_float(0x7f800000);
    float U = kInf;
    cand_mask_t mask = 0;
    // one neighbour record {fp32 x_j, j} -> (lower bound, upper bound, front, sure)
    auto bounds = [&](const float4 &e, float &lb, float &ub, bool &front, bool &sure) {
        const float nx = e.x - hdr_f.x, ny = e.y - hdr_f.y, nz = e.z - hdr_f.z;
        const float hx = __fmaf_rn(0.5f, nx, px), hy = __fmaf_rn(0.5f, ny, py),
                    hz = __fmaf_rn(0.5f, nz, pz);
        const float num = __fmaf_rn(hz, nz, __fmaf_rn(hy, ny, hx * nx));
        const float den = __fmaf_rn(df[2], nz, __fmaf_rn(df[1], ny, df[0] * nx));
        front = den >= -Ed;  // not certainly back-facing (NaN pad records: false)
        sure = den > thr;
        float rinv;  // MUFU reciprocal (<= 1 ulp for the `sure` ones; others are discarded)
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rinv) : "f"(den));
        const float s = num * rinv;
        const float as = fabsf(s);
        const float es = __fmaf_rn(K3, as, __fmaf_rn(__fmaf_rn(K2, as, K1), rinv, slack));
        lb = s - es;
        ub = s + es;
    };
    // the cell's exact site: its fp32 header copy (fp32-exact sites) or the fp64 site
    double cx = hdr_f.x, cy = hdr_f.y, cz = hdr_f.z;
    constexpr bool pos64 = PK == 2;
    if (pos64) {
        const double4 si = ld_site(S.site4 + S.to_id(ci));
        cx = si.x;
        cy = si.y;
        cz = si.z;
    }
    best_t = dinf();
    best_j = -1;
    int32_t best_k = 0x7fffffff;
    // phase 2 on slot k: kernels.py:116-133 in fp64
    auto exact = [&](int32_t k) {
        RFB_BOUND(k, S.edge_slots);
        const float4 ej = rec_site(S.edge, k);  // (in L1: phase 1 just read it)
        const int32_t j = __float_as_int(ej.w);
        RFB_BOUND(j, S.n_sites);
        double xj = ej.x, yj = ej.y, zj = ej.z;
        if (pos64) {
            const double4 sj = ld_site(S.site4 + S.to_id(j));
            xj = sj.x;
            yj = sj.y;
            zj = sj.z;
        }
        const double nx = xj - cx, ny = yj - cy, nz = zj - cz;
        const double denom = r.dx() * nx + r.dy() * ny + r.dz() * nz;
        if (denom <= 0.0) return;
        const double mx = 0.5 * (xj + cx), my = 0.5 * (yj + cy), mz = 0.5 * (zj + cz);
        const double t = ((mx - r.ox()) * nx + (my - r.oy()) * ny + (mz - r.oz()) * nz) / denom;
        if (t < best_t) {
            best_t = t;
            best_j = j;
            best_k = k;
        }
    };
    if (G == 1) {
        // Final-band filter: only the neighbours whose lower bound beats the FINAL
        // upper bound U (the minimum over the row of the certain upper bounds) can be
        // the reference's first minimum.  Phase 1 tracks U, the two smallest candidate
        // lower bounds L1 <= L2 and L1's slot: if L2 > U, only L1's neighbour can beat
        // the final band, and it is the best upper bound's (lb <= ub = U), so phase 2
        // evaluates it alone -- the same first minimum, bit for bit (~1.0 exact
        // evaluations per step; a running band in CSR order keeps every new running
        // minimum, ~2.7).  Otherwise (ties, uncertain facing) a second pass over the
        // row (L1-resident) collects every candidate against the final U.  Either way
        // the candidates go through one phase-2 loop, so the lanes of a warp never
        // split over different phase-2 code (round 2: 19.05 -> 18.29 ms per frame).
        float L1 = kInf, L2 = kInf;
        int32_t t1 = -1, slot = 0;
        // slot t of the row ends up as bit (nslots - 1 - t) of `mask`
        auto visit = [&](const float4 &e) {
            float lb, ub;
            bool front, sure;
            bounds(e, lb, ub, front, sure);
            const float lbm = sure ? lb : -kInf;  // uncertain facing: always a candidate
            const float lbc = front ? lbm : kInf;
            t1 = lbc < L1 ? slot : t1;
            L2 = fminf(L2, fmaxf(L1, lbc));
            L1 = fminf(L1, lbc);
            U = sure ? fminf(U, ub) : U;
            ++slot;
        };
        // rows start at even slots: one LDG.256 per two neighbours (NaN pads)
        const int32_t nslots = (c.k1 - c.k0 + 1) & ~1;
        RFB_PRAGMA_UNROLL(RFB_PAIR_UNROLL)
        for (int32_t kp = c.k0; kp < c.k1; kp += 2) {
            float4 e0, e1;
            RFB_BOUND(kp + 1, S.edge_slots);
#if RFB_CHECK
            assert((reinterpret_cast<uintptr_t>(S.edge + kp) & 31) == 0);
#endif
            ldg256(S.edge + kp, e0, e1);
            visit(e0);
            visit(e1);
        }
        if (nslots > kMaskBits) {  // rare: the mask would lose bits -- every neighbour exactly
            for (int32_t k = c.k0; k < c.k1; ++k) exact(k);
            return;
        }
        if (t1 >= 0 && L2 > U && L1 <= U) {  // only L1's neighbour can be the first minimum
            mask = 1u << (nslots - 1 - t1);
        } else if (t1 >= 0) {  // several candidates: collect them against the final U
            for (int32_t kp = c.k0; kp < c.k1; kp += 2) {
                float4 e0, e1;
                ldg256(S.edge + kp, e0, e1);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    float lb, ub;
                    bool front, sure;
                    bounds(h ? e1 : e0, lb, ub, front, sure);
                    const bool cand = front && (!sure || lb <= U);
                    mask = (mask << 1) | (cand ? 1u : 0u);
                }
            }
        }
        while (mask) {  // highest bit = lowest slot: CSR order
            const int b = 31 - __clz((int)mask);
            mask &= ~(1u << b);
            exact(c.k0 + (nslots - 1 - b));
        }
        return;
    }
    // G > 1 lanes per ray: lane gl takes slots gl, gl + G, ... (real neighbours only)
    const int32_t k0 = c.k0 + gl;
    int32_t nk = 0;
    RFB_PRAGMA_UNROLL(RFB_F32_UNROLL)
    for (int32_t k = k0; k < c.k1; k += G, ++nk) {
        RFB_BOUND(k, S.edge_slots);
        const float4 e = rec_site(S.edge, k);
        float lb, ub;
        bool front, sure;
        bounds(e, lb, ub, front, sure);
        const cand_mask_t bit = nk < kMaskBits ? ((cand_mask_t)1 << nk) : (cand_mask_t)0;
        const bool cand = front && (!sure || lb <= U);
        mask |= cand ? bit : (cand_mask_t)0;
        U = sure ? fminf(U, ub) : U;
    }
    while (mask) {  // this lane's candidates, CSR order
        const int idx = __ffs((int)mask) - 1;
        mask &= mask - 1;
        exact(k0 + idx * G);
    }
    for (int32_t idx = kMaskBits; idx < nk; ++idx) exact(k0 + idx * G);  // beyond the mask
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

}  // namespace rfb
