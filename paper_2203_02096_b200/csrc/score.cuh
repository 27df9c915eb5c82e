// score.cuh — per-individual pose scoring and gradient on a lane group (rows a3-a6 of
// the hot path, DESIGN.md §1/§5).
//
// One group of W lanes (W = 16 or 32) evaluates one genotype.  Lane `sub` owns atoms
// a = sub + W*c (c < MAXC).  The ligand block (staged in shared memory per CTA) and a
// small per-group scratch (pose coordinates, torsion composites, genes, gradient) are
// the only memory besides the grid maps, which are read with float4 corner gathers
// from L2/HBM.  All sums are fixed-order (butterfly shuffles, sequential per-lane
// loops): no atomics, so results are bit-reproducible run to run.
#pragma once
#include <stdint.h>

#include "dock_internal.h"

namespace dk {

constexpr float kElec = 332.06363f;                         // D5
constexpr float kInvTwoSigma2 = 1.0f / (2.0f * 3.6f * 3.6f);  // desolvation sigma 3.6 Å
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kOut = 1e5f;                                  // D4.5 out-of-grid penalty

// Shared-memory view of the staged ligand block.
struct LigSm {
    int N, T, G, P, n_levels;
    const int *lvl;               // [kMaxTors+1]
    const float4 *p;              // body coords + charge
    const float4 *par;            // R/2, sqrt eps, S, V
    const int *meta;              // type | role<<8 | (deep+1)<<16
    const float4 *tA, *tU;
    const int4 *tmeta;            // parent, a, b, lo | hi<<16
    const uint32_t *pairs;        // i | j<<8 | hb<<16
    const int *csr_off;
    const uint16_t *csr_nbr;      // j | hb<<8
};

// Per-group scratch in shared memory.
struct Scratch {
    float4 *r;                    // [N]  pose (x,y,z) and charge
    float4 *W;                    // [3T] torsion composite transforms (rows R|t)
    float4 *ts;                   // [2N] per-atom (r-t) x g and g (gradient only)
    float *genes;                 // [G]  genotype being evaluated
    float *grad;                  // [G]  genotype gradient (gradient only)
};

template <int W>
__device__ __forceinline__ unsigned group_mask() {
    if constexpr (W == 32) {
        return 0xffffffffu;
    } else {
        const unsigned lane = threadIdx.x & 31u;
        return ((1u << W) - 1u) << (lane & ~(unsigned)(W - 1));
    }
}

template <int W>
__device__ __forceinline__ float gsum(float v, unsigned mask) {
#pragma unroll
    for (int m = W / 2; m >= 1; m >>= 1) v += __shfl_xor_sync(mask, v, m, W);
    return v;   // identical in every lane of the group (commutative pairwise adds)
}

template <int W>
__device__ __forceinline__ long long gsum_ll(long long v, unsigned mask) {
#pragma unroll
    for (int m = W / 2; m >= 1; m >>= 1) v += __shfl_xor_sync(mask, v, m, W);
    return v;
}

// D5 pair energy and dE/d(rho^2).
template <bool GRAD>
__device__ __forceinline__ float pair_energy(float rho2, float4 pi, float4 pj, float qq, bool hb,
                                             float &dE) {
    const bool clamped = rho2 < 1e-4f;                   // 0.01 Å clamp
    rho2 = fmaxf(rho2, 1e-4f);
    const float inv = __fdividef(1.0f, rho2);
    const float req = pi.x + pj.x;                       // (R_i + R_j)/2
    const float eps = pi.y * pj.y;                       // sqrt(eps_i eps_j)
    const float SV = pi.z * pj.w + pj.z * pi.w;          // S_i V_j + S_j V_i
    const float x2 = req * req * inv;
    const float x4 = x2 * x2;
    const float x6 = x4 * x2;
    const float x12 = x6 * x6;
    const float xn = hb ? x6 * x4 : x6;                  // x^10 for H-bond pairs
    const float c12 = hb ? 5.0f : 1.0f;
    const float cn = hb ? 6.0f : 2.0f;
    const float Evdw = eps * (c12 * x12 - cn * xn);
    const float Eel = (0.25f * kElec) * qq * inv;        // eps(r) = 4r
    const float Eds = SV * exp2f(-rho2 * (kInvTwoSigma2 * kLog2e));
    if (GRAD) {
        const float dn = hb ? 30.0f : 6.0f;
        const float dv = -eps * inv * (6.0f * c12 * x12 - dn * xn);
        const float dd = dv - Eel * inv - Eds * kInvTwoSigma2;
        dE = clamped ? 0.0f : dd;
    }
    return Evdw + Eel + Eds;
}

// D4 intermolecular energy of one atom and its gradient.
__device__ __forceinline__ float inter_atom(const GridDev &g, int type, float q, float rx, float ry,
                                            float rz, float &gx, float &gy, float &gz) {
    const float ux = (rx - g.ox) * g.inv_s, uy = (ry - g.oy) * g.inv_s, uz = (rz - g.oz) * g.inv_s;
    const bool inside = ux >= 0.0f && uy >= 0.0f && uz >= 0.0f && ux <= (float)(g.nx - 1) &&
                        uy <= (float)(g.ny - 1) && uz <= (float)(g.nz - 1);
    if (inside) {
        const int ix = min((int)ux, g.nx - 2), iy = min((int)uy, g.ny - 2), iz = min((int)uz, g.nz - 2);
        const float fx = ux - (float)ix, fy = uy - (float)iy, fz = uz - (float)iz;
        const size_t nxy = (size_t)g.nx * g.ny;
        const float4 *b = g.maps + (size_t)type * nxy * g.nz + (size_t)ix + (size_t)g.nx * iy + nxy * iz;
        const float4 m000 = __ldg(b), m100 = __ldg(b + 1);
        const float4 m010 = __ldg(b + g.nx), m110 = __ldg(b + g.nx + 1);
        const float4 m001 = __ldg(b + nxy), m101 = __ldg(b + nxy + 1);
        const float4 m011 = __ldg(b + nxy + g.nx), m111 = __ldg(b + nxy + g.nx + 1);
        const float aq = fabsf(q);
        // trilinear interpolation is linear in the map values: combine the three maps per
        // corner first (e = V(M_t) + q V(M_E) + |q| V(M_D) = V(M_t + q M_E + |q| M_D)).
        const float c000 = m000.x + q * m000.y + aq * m000.z, c100 = m100.x + q * m100.y + aq * m100.z;
        const float c010 = m010.x + q * m010.y + aq * m010.z, c110 = m110.x + q * m110.y + aq * m110.z;
        const float c001 = m001.x + q * m001.y + aq * m001.z, c101 = m101.x + q * m101.y + aq * m101.z;
        const float c011 = m011.x + q * m011.y + aq * m011.z, c111 = m111.x + q * m111.y + aq * m111.z;
        const float dx00 = c100 - c000, dx10 = c110 - c010, dx01 = c101 - c001, dx11 = c111 - c011;
        const float a00 = c000 + fx * dx00, a10 = c010 + fx * dx10;
        const float a01 = c001 + fx * dx01, a11 = c011 + fx * dx11;
        const float dy0 = a10 - a00, dy1 = a11 - a01;
        const float b0 = a00 + fy * dy0, b1 = a01 + fy * dy1;
        const float dxy0 = dx00 + fy * (dx10 - dx00), dxy1 = dx01 + fy * (dx11 - dx01);
        gx = (dxy0 + fz * (dxy1 - dxy0)) * g.inv_s;
        gy = (dy0 + fz * (dy1 - dy0)) * g.inv_s;
        gz = (b1 - b0) * g.inv_s;
        return b0 + fz * (b1 - b0);
    }
    const float cx = fminf(fmaxf(rx, g.ox), g.hx), cy = fminf(fmaxf(ry, g.oy), g.hy),
                cz = fminf(fmaxf(rz, g.oz), g.hz);
    const float dx = rx - cx, dy = ry - cy, dz = rz - cz;
    const float d = sqrtf(dx * dx + dy * dy + dz * dz);
    const float s = d > 0.0f ? kOut / d : 0.0f;
    gx = dx * s; gy = dy * s; gz = dz * s;
    return kOut * (1.0f + d);
}

// Energy (and genotype gradient into S.grad) of the genotype in S.genes.
// Every lane of the group returns the same total energy.
template <int W, int MAXC, bool GRAD>
__device__ float eval_group(const LigSm &L, const GridDev &grid, const Scratch &S, int sub, unsigned mask) {
    const float *x = S.genes;
    // ---- a3: orientation quaternion q = (cos a/2, sin(a/2) n) -> R(q) (D3) ----
    float sph, cph, sth, cth, sa, ca;
    sincosf(x[3], &sph, &cph);
    sincosf(x[4], &sth, &cth);
    sincosf(0.5f * x[5], &sa, &ca);
    const float nx = sth * cph, ny = sth * sph, nz = cth;
    const float qw = ca, qx = sa * nx, qy = sa * ny, qz = sa * nz;
    const float R00 = 1.f - 2.f * (qy * qy + qz * qz), R01 = 2.f * (qx * qy - qw * qz), R02 = 2.f * (qx * qz + qw * qy);
    const float R10 = 2.f * (qx * qy + qw * qz), R11 = 1.f - 2.f * (qx * qx + qz * qz), R12 = 2.f * (qy * qz - qw * qx);
    const float R20 = 2.f * (qx * qz - qw * qy), R21 = 2.f * (qy * qz + qw * qx), R22 = 1.f - 2.f * (qx * qx + qy * qy);
    const float tx = x[0], ty = x[1], tz = x[2];

    // ---- a3: torsion composites W_k = W_parent o Rot(u_k, tau_k) about A_k, level by level ----
    for (int l = 0; l < L.n_levels; ++l) {
        const int k0 = L.lvl[l], k1 = L.lvl[l + 1];
        for (int k = k0 + sub; k < k1; k += W) {
            float st, ct;
            sincosf(x[6 + k], &st, &ct);
            const float4 u = L.tU[k], A = L.tA[k];
            const int par = L.tmeta[k].x;
            const float oc = 1.0f - ct;
            const float k00 = ct + oc * u.x * u.x, k01 = oc * u.x * u.y - st * u.z, k02 = oc * u.x * u.z + st * u.y;
            const float k10 = oc * u.y * u.x + st * u.z, k11 = ct + oc * u.y * u.y, k12 = oc * u.y * u.z - st * u.x;
            const float k20 = oc * u.z * u.x - st * u.y, k21 = oc * u.z * u.y + st * u.x, k22 = ct + oc * u.z * u.z;
            const float lx = A.x - (k00 * A.x + k01 * A.y + k02 * A.z);
            const float ly = A.y - (k10 * A.x + k11 * A.y + k12 * A.z);
            const float lz = A.z - (k20 * A.x + k21 * A.y + k22 * A.z);
            float4 p0, p1, p2;
            if (par < 0) {
                p0 = make_float4(R00, R01, R02, tx);
                p1 = make_float4(R10, R11, R12, ty);
                p2 = make_float4(R20, R21, R22, tz);
            } else {
                p0 = S.W[3 * par]; p1 = S.W[3 * par + 1]; p2 = S.W[3 * par + 2];
            }
            S.W[3 * k] = make_float4(p0.x * k00 + p0.y * k10 + p0.z * k20, p0.x * k01 + p0.y * k11 + p0.z * k21,
                                     p0.x * k02 + p0.y * k12 + p0.z * k22, p0.x * lx + p0.y * ly + p0.z * lz + p0.w);
            S.W[3 * k + 1] = make_float4(p1.x * k00 + p1.y * k10 + p1.z * k20, p1.x * k01 + p1.y * k11 + p1.z * k21,
                                         p1.x * k02 + p1.y * k12 + p1.z * k22, p1.x * lx + p1.y * ly + p1.z * lz + p1.w);
            S.W[3 * k + 2] = make_float4(p2.x * k00 + p2.y * k10 + p2.z * k20, p2.x * k01 + p2.y * k11 + p2.z * k21,
                                         p2.x * k02 + p2.y * k12 + p2.z * k22, p2.x * lx + p2.y * ly + p2.z * lz + p2.w);
        }
        __syncwarp(mask);
    }

    // ---- a3: one rigid transform per atom; a4: intermolecular energy and gradient ----
    float rx[MAXC], ry[MAXC], rz[MAXC], gx[MAXC], gy[MAXC], gz[MAXC];
    float e_part = 0.0f;
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
        const int a = sub + W * c;
        rx[c] = ry[c] = rz[c] = gx[c] = gy[c] = gz[c] = 0.0f;
        if (a < L.N) {
            const int meta = L.meta[a];
            const int deep = (meta >> 16) - 1;
            const float4 p = L.p[a];
            if (deep < 0) {
                rx[c] = R00 * p.x + R01 * p.y + R02 * p.z + tx;
                ry[c] = R10 * p.x + R11 * p.y + R12 * p.z + ty;
                rz[c] = R20 * p.x + R21 * p.y + R22 * p.z + tz;
            } else {
                const float4 w0 = S.W[3 * deep], w1 = S.W[3 * deep + 1], w2 = S.W[3 * deep + 2];
                rx[c] = w0.x * p.x + w0.y * p.y + w0.z * p.z + w0.w;
                ry[c] = w1.x * p.x + w1.y * p.y + w1.z * p.z + w1.w;
                rz[c] = w2.x * p.x + w2.y * p.y + w2.z * p.z + w2.w;
            }
            S.r[a] = make_float4(rx[c], ry[c], rz[c], p.w);
            e_part += inter_atom(grid, meta & 0xff, p.w, rx[c], ry[c], rz[c], gx[c], gy[c], gz[c]);
        }
    }
    __syncwarp(mask);

    // ---- a5: intramolecular pairs ----
    if constexpr (!GRAD) {
        for (int q = sub; q < L.P; q += W) {
            const uint32_t w = L.pairs[q];
            const int i = w & 0xff, j = (w >> 8) & 0xff;
            const float4 ri = S.r[i], rj = S.r[j];
            const float dx = ri.x - rj.x, dy = ri.y - rj.y, dz = ri.z - rj.z;
            float dE;
            e_part += pair_energy<false>(dx * dx + dy * dy + dz * dz, L.par[i], L.par[j], ri.w * rj.w,
                                         (w >> 16) & 1, dE);
        }
        return gsum<W>(e_part, mask);
    } else {
    // gradient path: each lane owns its atoms' incidence lists (fixed order, no atomics);
    // a pair's energy is counted by its lower-index owner only.
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
        const int a = sub + W * c;
        if (a < L.N) {
            const float4 pa = L.par[a];
            const float qa = L.p[a].w;
            const int e0 = L.csr_off[a], e1 = L.csr_off[a + 1];
            float fx = 0.f, fy = 0.f, fz = 0.f;
            for (int e = e0; e < e1; ++e) {
                const uint32_t nb = L.csr_nbr[e];
                const int j = nb & 0xff;
                const float4 rj = S.r[j];
                const float dx = rx[c] - rj.x, dy = ry[c] - rj.y, dz = rz[c] - rj.z;
                float dE;
                const float E = pair_energy<true>(dx * dx + dy * dy + dz * dz, pa, L.par[j], qa * rj.w,
                                                  (nb >> 8) & 1, dE);
                if (a < j) e_part += E;
                fx += dE * dx; fy += dE * dy; fz += dE * dz;
            }
            gx[c] += 2.0f * fx; gy[c] += 2.0f * fy; gz[c] += 2.0f * fz;
        }
    }
    const float E = gsum<W>(e_part, mask);

    // ---- a6: back-projection to genotype space (D7) ----
    float sgx = 0.f, sgy = 0.f, sgz = 0.f, Gx = 0.f, Gy = 0.f, Gz = 0.f;
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
        const int a = sub + W * c;
        if (a < L.N) {
            const float dx = rx[c] - tx, dy = ry[c] - ty, dz = rz[c] - tz;
            const float cxp = dy * gz[c] - dz * gy[c], cyp = dz * gx[c] - dx * gz[c], czp = dx * gy[c] - dy * gx[c];
            sgx += gx[c]; sgy += gy[c]; sgz += gz[c];
            Gx += cxp; Gy += cyp; Gz += czp;
            S.ts[2 * a] = make_float4(cxp, cyp, czp, 0.f);
            S.ts[2 * a + 1] = make_float4(gx[c], gy[c], gz[c], 0.f);
        }
    }
    sgx = gsum<W>(sgx, mask); sgy = gsum<W>(sgy, mask); sgz = gsum<W>(sgz, mask);
    Gx = gsum<W>(Gx, mask); Gy = gsum<W>(Gy, mask); Gz = gsum<W>(Gz, mask);
    __syncwarp(mask);
    // torsions: dE/dtau_k = w_k . sum_{a in moved(k)} (r_a - r_{a_k}) x g_a
    for (int k = sub; k < L.T; k += W) {
        const int4 tm = L.tmeta[k];
        const int lo = tm.w & 0xffff, hi = tm.w >> 16;
        float cx = 0.f, cy = 0.f, cz = 0.f, hx = 0.f, hy = 0.f, hz = 0.f;
        for (int a = lo; a < hi; ++a) {
            const float4 c4 = S.ts[2 * a], g4 = S.ts[2 * a + 1];
            cx += c4.x; cy += c4.y; cz += c4.z;
            hx += g4.x; hy += g4.y; hz += g4.z;
        }
        const float4 ra = S.r[tm.y], rb = S.r[tm.z];
        const float dax = ra.x - tx, day = ra.y - ty, daz = ra.z - tz;
        const float sx = cx - (day * hz - daz * hy), sy = cy - (daz * hx - dax * hz), sz = cz - (dax * hy - day * hx);
        float wx = rb.x - ra.x, wy = rb.y - ra.y, wz = rb.z - ra.z;
        const float inw = rsqrtf(wx * wx + wy * wy + wz * wz);
        S.grad[6 + k] = (wx * sx + wy * sy + wz * sz) * inw;
    }
    // translation and orientation: omega = adot n + sin(a) ndot + (1 - cos a) n x ndot
    if (sub < 6) {
        float v;
        if (sub == 0) v = sgx;
        else if (sub == 1) v = sgy;
        else if (sub == 2) v = sgz;
        else if (sub == 5) v = Gx * nx + Gy * ny + Gz * nz;
        else {
            const float sal = 2.0f * sa * ca, omc = 2.0f * sa * sa;   // sin(alpha), 1 - cos(alpha)
            float dnx, dny, dnz;
            if (sub == 3) { dnx = -sth * sph; dny = sth * cph; dnz = 0.0f; }
            else { dnx = cth * cph; dny = cth * sph; dnz = -sth; }
            const float wx = sal * dnx + omc * (ny * dnz - nz * dny);
            const float wy = sal * dny + omc * (nz * dnx - nx * dnz);
            const float wz = sal * dnz + omc * (nx * dny - ny * dnx);
            v = Gx * wx + Gy * wy + Gz * wz;
        }
        S.grad[sub] = v;
    }
    __syncwarp(mask);
    return E;
    }
}

}  // namespace dk
