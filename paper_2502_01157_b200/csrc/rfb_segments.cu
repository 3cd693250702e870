// rfb_segments.cu -- the reference's per-ray building blocks as batched
// device kernels over *given* segment lists (tracer/kernels.py):
//   rfb_sh_basis            sh_basis_into        kernels.py:38-58
//   rfb_cell_colors         cell_color           kernels.py:61-73
//   rfb_composite_segments  composite_segments   kernels.py:165-196
//   rfb_backward_segments   backward_ray         kernels.py:250-337
//                           + face_t_gradient    kernels.py:340-369
//   rfb_quantile_segments   quantile_backward_ray kernels.py:456-567
// The hot path fuses all of these into k_render / k_train (rfb.cu); these
// entry points serve callers that hold segments themselves (the flat
// kernels.py drop-ins, tooling).  fp64 in the reference's operation order
// (-fmad=false), one thread per ray, fp64 atomics for the scatters.
#include <cuda_runtime.h>

#include <cstdint>

#include "rfb_device.cuh"

namespace rfb_seg {

struct Segs {
    const int64_t *off;   // [m+1] ray r owns segments off[r] .. off[r+1]-1
    const int32_t *cell;
    const double *t0, *t1;
};

__device__ __forceinline__ void basis_of(const double *dirs, int64_t r, double *b) {
    rfb::sh_basis(dirs[3 * r], dirs[3 * r + 1], dirs[3 * r + 2], b);
}

// kernels.py:61-73 (fp64, reference order)
__device__ __forceinline__ int color_of(const double *sh, int64_t i, const double *basis,
                                        double *out) {
    int mask = 0;
    for (int ch = 0; ch < 3; ++ch) {
        double acc = 0.5;
        for (int k = 0; k < 16; ++k) acc += basis[k] * sh[i * 48 + k * 3 + ch];
        if (acc < 0.0) {
            acc = 0.0;
            mask |= 1 << ch;
        }
        out[ch] = acc;
    }
    return mask;
}

// kernels.py:340-369
__device__ __forceinline__ void face_grad_f64(const double *pos, int64_t i, int64_t j, double ox,
                                              double oy, double oz, double dx, double dy,
                                              double dz, double t, double dt, double *d_pos) {
    const double nx = pos[3 * j] - pos[3 * i];
    const double ny = pos[3 * j + 1] - pos[3 * i + 1];
    const double nz = pos[3 * j + 2] - pos[3 * i + 2];
    const double denom = dx * nx + dy * ny + dz * nz;
    if (denom == 0.0) return;
    const double mx = 0.5 * (pos[3 * i] + pos[3 * j]);
    const double my = 0.5 * (pos[3 * i + 1] + pos[3 * j + 1]);
    const double mz = 0.5 * (pos[3 * i + 2] + pos[3 * j + 2]);
    const double px = ox + t * dx, py = oy + t * dy, pz = oz + t * dz;
    const double qx = mx - px, qy = my - py, qz = mz - pz;
    const double inv = dt / denom;
    atomicAdd(d_pos + 3 * i, (0.5 * nx - qx) * inv);
    atomicAdd(d_pos + 3 * i + 1, (0.5 * ny - qy) * inv);
    atomicAdd(d_pos + 3 * i + 2, (0.5 * nz - qz) * inv);
    atomicAdd(d_pos + 3 * j, (0.5 * nx + qx) * inv);
    atomicAdd(d_pos + 3 * j + 1, (0.5 * ny + qy) * inv);
    atomicAdd(d_pos + 3 * j + 2, (0.5 * nz + qz) * inv);
}

__global__ void k_sh_basis(const double *dirs, int64_t m, double *out) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < m) basis_of(dirs, r, out + 16 * r);
}

__global__ void k_cell_colors(const double *sh, const int32_t *cells, const double *basis,
                              int64_t m, double *out, int32_t *masks) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= m) return;
    const int mask = color_of(sh, cells[r], basis + 16 * r, out + 3 * r);
    if (masks) masks[r] = mask;
}

// kernels.py:165-196
__global__ void k_composite(const double *sigma, const double *sh, const double *bases, int64_t m,
                            Segs S, double bg0, double bg1, double bg2, double *out_rgb,
                            double *out_T, double *out_wsum) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= m) return;
    double basis[16], col[3];
    for (int k = 0; k < 16; ++k) basis[k] = bases[16 * r + k];
    double T = 1.0, wsum = 0.0, cr = 0.0, cg = 0.0, cb = 0.0;
    for (int64_t s = S.off[r]; s < S.off[r + 1]; ++s) {
        const int64_t i = S.cell[s];
        const double delta = S.t1[s] - S.t0[s];
        const double alpha = 1.0 - exp(-sigma[i] * delta);
        color_of(sh, i, basis, col);
        const double w = T * alpha;
        wsum += w;
        cr += w * col[0];
        cg += w * col[1];
        cb += w * col[2];
        T *= 1.0 - alpha;
    }
    out_rgb[3 * r] = cr + T * bg0;
    out_rgb[3 * r + 1] = cg + T * bg1;
    out_rgb[3 * r + 2] = cb + T * bg2;
    if (out_T) out_T[r] = T;
    if (out_wsum) out_wsum[r] = wsum;
}

// kernels.py:250-337 (+ face_t_gradient).  T_before lives in `tb`
// ([segments + rays] doubles: ray r uses tb[off[r] + r ...]).
__global__ void k_backward(const double *pos, const double *sigma, const double *sh, double bg0,
                           double bg1, double bg2, const double *origins, const double *dirs,
                           const double *bases, const double *adj, int64_t m, Segs S, double *tb,
                           double *d_sigma, double *d_sh, double *d_pos) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= m) return;
    const int64_t s0 = S.off[r], n = S.off[r + 1] - s0;
    if (n == 0) return;
    double basis[16], col[3];
    for (int k = 0; k < 16; ++k) basis[k] = bases[16 * r + k];
    const double ox = origins[3 * r], oy = origins[3 * r + 1], oz = origins[3 * r + 2];
    const double dx = dirs[3 * r], dy = dirs[3 * r + 1], dz = dirs[3 * r + 2];
    const double ar = adj[3 * r], ag = adj[3 * r + 1], ab = adj[3 * r + 2];
    double *T = tb + s0 + r;
    T[0] = 1.0;
    for (int64_t s = 0; s < n; ++s) {
        const int64_t i = S.cell[s0 + s];
        T[s + 1] = T[s] * exp(-sigma[i] * (S.t1[s0 + s] - S.t0[s0 + s]));
    }
    double Sr = T[n] * bg0, Sg = T[n] * bg1, Sb = T[n] * bg2;
    double dd_next = 0.0;  // d_delta[s + 1]
    for (int64_t s = n - 1; s >= 0; --s) {
        const int64_t i = S.cell[s0 + s];
        const double delta = S.t1[s0 + s] - S.t0[s0 + s];
        const double alpha = 1.0 - exp(-sigma[i] * delta);
        const double w = T[s] * alpha;
        const int mk = color_of(sh, i, basis, col);
        const double common = ar * (T[s + 1] * col[0] - Sr) + ag * (T[s + 1] * col[1] - Sg) +
                              ab * (T[s + 1] * col[2] - Sb);
        atomicAdd(d_sigma + i, delta * common);
        const double dd = sigma[i] * common;
        if (w != 0.0) {
            const double a3[3] = {ar, ag, ab};
            for (int ch = 0; ch < 3; ++ch) {
                if ((mk >> ch) & 1 || a3[ch] == 0.0) continue;
                const double f = w * a3[ch];
                for (int k = 0; k < 16; ++k) atomicAdd(d_sh + i * 48 + k * 3 + ch, f * basis[k]);
            }
        }
        Sr = Sr + w * col[0];
        Sg = Sg + w * col[1];
        Sb = Sb + w * col[2];
        if (s + 1 < n) {  // interior boundary s+1 (kernels.py:328-337)
            const double dt = dd - dd_next;
            if (dt != 0.0)
                face_grad_f64(pos, i, S.cell[s0 + s + 1], ox, oy, oz, dx, dy, dz,
                              S.t0[s0 + s + 1], dt, d_pos);
        }
        dd_next = dd;
    }
}

// kernels.py:456-567, every pair of every ray; loss_out[r] = sum over pairs
__global__ void k_quantile(const double *pos, const double *sigma, const double *origins,
                           const double *dirs, int64_t m, Segs S, const double *u_pairs,
                           int32_t n_pairs, double weight_floor, double scale, double *tb,
                           double *d_sigma, double *d_pos, double *loss_out) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= m) return;
    const int64_t s0 = S.off[r], n = S.off[r + 1] - s0;
    double loss = 0.0;
    if (n > 0) {
        const double ox = origins[3 * r], oy = origins[3 * r + 1], oz = origins[3 * r + 2];
        const double dx = dirs[3 * r], dy = dirs[3 * r + 1], dz = dirs[3 * r + 2];
        double *T = tb + s0 + r;
        T[0] = 1.0;
        for (int64_t s = 0; s < n; ++s) {
            const int64_t i = S.cell[s0 + s];
            T[s + 1] = T[s] * exp(-sigma[i] * (S.t1[s0 + s] - S.t0[s0 + s]));
        }
        const double total = 1.0 - T[n];
        for (int32_t p = 0; p < n_pairs && !(total < weight_floor); ++p) {
            const double *u2 = u_pairs + (r * n_pairs + p) * 2;
            double t_hit[2];
            int64_t hit[2];
            for (int a = 0; a < 2; ++a) {
                const double target = u2[a] * total;
                int64_t s = 0;
                while (s < n - 1 && (1.0 - T[s + 1]) < target) s += 1;
                hit[a] = s;
                const double si = sigma[S.cell[s0 + s]];
                if (si <= 0.0) {
                    t_hit[a] = S.t0[s0 + s];
                    continue;
                }
                double frac = (target - (1.0 - T[s])) / T[s];
                if (frac > 1.0 - 1e-15) frac = 1.0 - 1e-15;
                double th = S.t0[s0 + s] - log(1.0 - frac) / si;
                if (th > S.t1[s0 + s]) th = S.t1[s0 + s];
                t_hit[a] = th;
            }
            const double diff = t_hit[0] - t_hit[1];
            loss += fabs(diff);
            if (diff == 0.0) continue;
            const double sign = diff > 0.0 ? 1.0 : -1.0;
            const double T_end = T[n];
            for (int a = 0; a < 2; ++a) {
                const double u = u2[a], t_u = t_hit[a];
                const int64_t s = hit[a];
                const double si = sigma[S.cell[s0 + s]];
                const double T_at = T[s] * exp(-si * (t_u - S.t0[s0 + s]));
                const double wd = T_at * si;
                if (wd <= 1e-300) continue;
                const double g = (a == 0 ? sign : -sign) * scale / wd;
                for (int64_t k = 0; k < n; ++k) {
                    const int64_t ck = S.cell[s0 + k];
                    const double k0 = S.t0[s0 + k], k1 = S.t1[s0 + k];
                    const double dA = T_end * (k1 - k0);
                    double c;
                    if (k0 < t_u) {
                        const double hi = k1 < t_u ? k1 : t_u;
                        c = g * (u * dA - T_at * (hi - k0));
                    } else {
                        c = g * (u * dA);
                    }
                    atomicAdd(d_sigma + ck, c);
                }
                for (int64_t k = 1; k < n; ++k) {
                    const int64_t im = S.cell[s0 + k - 1], jm = S.cell[s0 + k];
                    const double dsig = sigma[im] - sigma[jm];
                    if (dsig == 0.0) continue;
                    const double tbq = S.t0[s0 + k];
                    const double dW = tbq < t_u ? T_at * dsig : 0.0;
                    const double dt = g * (u * (T_end * dsig) - dW);
                    if (dt != 0.0) face_grad_f64(pos, im, jm, ox, oy, oz, dx, dy, dz, tbq, dt, d_pos);
                }
            }
        }
    }
    if (loss_out) loss_out[r] = loss;
}

// face_t_gradient for a batch of boundaries: item q = (i, j, t, dt) on ray q
__global__ void k_face_grads(const double *pos, const int32_t *ij, const double *origins,
                             const double *dirs, const double *t, const double *dt, int64_t m,
                             double *d_pos) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= m) return;
    face_grad_f64(pos, ij[2 * q], ij[2 * q + 1], origins[3 * q], origins[3 * q + 1],
                  origins[3 * q + 2], dirs[3 * q], dirs[3 * q + 1], dirs[3 * q + 2], t[q], dt[q],
                  d_pos);
}

inline unsigned blocks(int64_t m) { return (unsigned)((m + 127) / 128); }

}  // namespace rfb_seg

using namespace rfb_seg;

extern "C" {

int rfb_sh_basis(const double *dirs, int64_t m, double *out, void *stream) {
    if (m < 0) return RFB_EINVAL;
    if (m == 0) return RFB_OK;
    if (!dirs || !out) return RFB_EINVAL;
    k_sh_basis<<<blocks(m), 128, 0, (cudaStream_t)stream>>>(dirs, m, out);
    return (int)cudaGetLastError();
}

int rfb_cell_colors(const double *sh, const int32_t *cells, const double *basis, int64_t m,
                    double *out, int32_t *masks, void *stream) {
    if (m < 0) return RFB_EINVAL;
    if (m == 0) return RFB_OK;
    if (!sh || !cells || !basis || !out) return RFB_EINVAL;
    k_cell_colors<<<blocks(m), 128, 0, (cudaStream_t)stream>>>(sh, cells, basis, m, out, masks);
    return (int)cudaGetLastError();
}

int rfb_composite_segments(const double *sigma, const double *sh, const double *bases,
                           int64_t m, const int64_t *seg_offsets, const int32_t *seg_cells,
                           const double *seg_t0, const double *seg_t1, const double *background,
                           double *out_rgb, double *out_T, double *out_wsum, void *stream) {
    if (m < 0 || !background) return RFB_EINVAL;
    if (m == 0) return RFB_OK;
    if (!sigma || !sh || !bases || !seg_offsets || !out_rgb) return RFB_EINVAL;
    Segs S{seg_offsets, seg_cells, seg_t0, seg_t1};
    k_composite<<<blocks(m), 128, 0, (cudaStream_t)stream>>>(sigma, sh, bases, m, S,
                                                           background[0], background[1],
                                                           background[2], out_rgb, out_T,
                                                           out_wsum);
    return (int)cudaGetLastError();
}

int rfb_face_t_gradients(const double *positions, const int32_t *ij, const double *origins,
                         const double *directions, const double *t, const double *dt, int64_t m,
                         double *d_pos, void *stream) {
    if (m < 0) return RFB_EINVAL;
    if (m == 0) return RFB_OK;
    if (!positions || !ij || !origins || !directions || !t || !dt || !d_pos) return RFB_EINVAL;
    k_face_grads<<<blocks(m), 128, 0, (cudaStream_t)stream>>>(positions, ij, origins, directions,
                                                            t, dt, m, d_pos);
    return (int)cudaGetLastError();
}

size_t rfb_segments_workspace_bytes(int64_t m, int64_t n_segments) {
    return (size_t)(m + n_segments + 1) * sizeof(double);
}

int rfb_backward_segments(const double *positions, const double *sigma, const double *sh,
                          const double *background, const double *origins,
                          const double *directions, const double *bases,
                          const double *adjoints, int64_t m, const int64_t *seg_offsets,
                          const int32_t *seg_cells, const double *seg_t0, const double *seg_t1,
                          double *d_sigma, double *d_sh, double *d_pos, void *workspace,
                          size_t workspace_bytes, void *stream) {
    if (m < 0 || !background) return RFB_EINVAL;
    if (m == 0) return RFB_OK;
    if (!positions || !sigma || !sh || !origins || !directions || !bases || !adjoints ||
        !seg_offsets || !d_sigma || !d_sh || !d_pos || !workspace)
        return RFB_EINVAL;
    Segs S{seg_offsets, seg_cells, seg_t0, seg_t1};
    k_backward<<<blocks(m), 128, 0, (cudaStream_t)stream>>>(
        positions, sigma, sh, background[0], background[1], background[2], origins, directions,
        bases, adjoints, m, S, (double *)workspace, d_sigma, d_sh, d_pos);
    (void)workspace_bytes;
    return (int)cudaGetLastError();
}

int rfb_quantile_segments(const double *positions, const double *sigma, const double *origins,
                          const double *directions, int64_t m, const int64_t *seg_offsets,
                          const int32_t *seg_cells, const double *seg_t0, const double *seg_t1,
                          const double *u_pairs, int32_t n_pairs, double weight_floor,
                          double scale, double *d_sigma, double *d_pos, double *loss_out,
                          void *workspace, size_t workspace_bytes, void *stream) {
    if (m < 0 || n_pairs < 0) return RFB_EINVAL;
    if (m == 0) return RFB_OK;
    if (!positions || !sigma || !origins || !directions || !seg_offsets || !d_sigma || !d_pos ||
        !workspace || (n_pairs > 0 && !u_pairs))
        return RFB_EINVAL;
    Segs S{seg_offsets, seg_cells, seg_t0, seg_t1};
    k_quantile<<<blocks(m), 128, 0, (cudaStream_t)stream>>>(
        positions, sigma, origins, directions, m, S, u_pairs, n_pairs, weight_floor, scale,
        (double *)workspace, d_sigma, d_pos, loss_out);
    (void)workspace_bytes;
    return (int)cudaGetLastError();
}

}  // extern "C"
