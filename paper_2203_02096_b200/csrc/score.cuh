// score.cuh — per-individual pose scoring and gradient on a lane group (rows a3-a6 of
// the hot path, DESIGN.md §1/§5).
//
// One group of W lanes (W = 16 or 32) evaluates one genotype.  Lane `sub` owns atoms
// a = sub + W*c (chunk c < MAXC).  The ligand block (staged in shared memory per CTA)
// and a small per-group scratch (pose coordinates, torsion composites, genes, gradient)
// are the only memory besides the grid maps, which are read with float4 corner gathers
// from L2/HBM.  All sums are fixed-order (butterfly shuffles, fixed tile/step order):
// no atomics, so results are bit-reproducible run to run.
#pragma once
#include <stdint.h>

#include "dock_internal.h"

// This header (and kernels.cu) is compiled twice: once for the D5 scoring function
// (namespace dk::d5) and once with -DDK_AD4 for the NEXT-2 AutoDock4.1-calibrated variant
// (namespace dk::ad4).  Only the pair arithmetic differs; the launchers in
// kernels.cuh dispatch on LigDev::sf.
#ifdef DK_AD4
#define DK_SF_NS ad4
#else
#define DK_SF_NS d5
#endif

namespace dk {
namespace DK_SF_NS {

constexpr float kElec4 = 332.06363f * 0.25f;                  // D5: 332.06363 / (4 rho^2)
constexpr float kInvTwoSigma2 = 1.0f / (2.0f * 3.6f * 3.6f);    // desolvation sigma 3.6 Å
constexpr float kExpScale = -kInvTwoSigma2 * 1.4426950408889634f;   // exp(-x/2s^2) = 2^(x*kExpScale)
constexpr float kOut = 1e5f;                                    // D4.5 out-of-grid penalty
#ifdef DK_AD4
// D5-AD4: smoothing half-window, cutoffs (compared on rho^2), and the
// Mehler-Solmajer dielectric eps(r) = A + B / (1 + k e^{-lambda B r}), B = 78.4 - A.
constexpr float kSmoothH = 0.25f;                               // smooth / 2 = 0.5 Å / 2
constexpr float kCutVdw2 = 8.0f * 8.0f;                         // vdW / H-bond: r < 8 Å
constexpr float kCutEl2 = 20.48f * 20.48f;                      // elec + desolv: r < 20.48 Å
constexpr float kDielA = -8.5525f;
constexpr float kDielB = 78.4f + 8.5525f;
constexpr float kDielK = 7.7839f;
constexpr float kDielLB = 0.003627f * (78.4f + 8.5525f);          // lambda B
constexpr float kDielC = -kDielLB * 1.4426950408889634f;         // e^{-lambda B r} = 2^(kDielC r)
constexpr float kDielLB2 = kDielLB * (78.4f + 8.5525f);           // lambda B^2
#endif
#ifndef DK_WALK_DEPTH
#define DK_WALK_DEPTH 4
#endif
constexpr int kWalkDepth = DK_WALK_DEPTH;
#ifndef DK_HYB_UNROLL
#define DK_HYB_UNROLL 1     // tail atoms per iteration of the hybrid tail's broadcast loop (A/B)
#endif
constexpr int kHybUnroll = DK_HYB_UNROLL;
#ifndef DK_WALK_UNROLL
#define DK_WALK_UNROLL 0    // torsion range walk of the back-projection: iterations unrolled; 0 =
#endif                      // 2 for MAXC >= 3 (long ranges: 7cpa +1 %), else 1 (3ce3: 2 is -1 %)
#ifndef DK_BP_T
#define DK_BP_T 1           // back-projection sums by one transposed reduction (W = 32; A/B: 0)
#endif
#ifndef DK_TILE_STREAMS
#define DK_TILE_STREAMS 1   // 2: two partner-accumulator streams per tile (A/B: scripts/variants.py)
#endif
#ifndef DK_TILE_UNROLL
#define DK_TILE_UNROLL 4   // steps unrolled in the pair-slot tile loop (A/B: scripts/variants.py)
#endif
constexpr int kTileUnroll = DK_TILE_UNROLL;   // torsion trees up to this depth: per-atom chain walk, no composites

// Shared-memory view of the staged ligand block.
struct LigSm {
    int N, T, G, P, NW, n_levels;
    const int *tlane;             // [32] torsion block per lane: k | lane << 8 | log2(size) << 16 (k 255: none)
    int tlane_top;                // largest block size / 2 (butterfly levels), 0 if every block is 1 lane
    const float4 *p;              // body coords + charge
    const float4 *par;            // R/2, sqrt eps, S, V
    const int *meta;              // type | role<<8 | (deep+1)<<16
    const float4 *tA, *tU;
    const int4 *tmeta;            // parent, a, b, lo | hi<<16
    const uint32_t *pairs;        // i | j<<8 | hb<<16
    const float4 *pprm;           // per pair: r_eq^2, eps_ij, S_iV_j+S_jV_i, 332.06363/4 q_i q_j
    const uint32_t *mask;         // [N][NW] pair-membership bit rows
    const float4 *ppar;           // [NC][2W] signed partner params (duplicated chunks)
    const float4 *slot4;          // pair-slot constants {r_eq^2, A, B, SV} (slot_mode)
    const float *slotq;           // pair-slot 332.06363/4 q_i q_j (slot_mode)
    int NC, tail_rot, slot_mode, tail_seg;
    int energy_tiles;             // energy-only evaluation through the pair tiles (no pair list)
    int nhb;                      // packed: H-bond side list (LigDev::off_hbc / off_hbseg)
    const float4 *hbc;
    int nhbr;                     // packed: H-bond contribution rounds (LigDev::nhbr)
    int hbspan;                   // packed: longest per-atom contribution run, rounded up to 2^k
    const int *hbseg;             // packed: [nhbr][32] contribution entries, then int[NC] chunk masks
    float wA_v, wB_v, wA_h, wB_h, qscale;   // D5-AD4 constants (LigDev; unused by D5)
};

// Gradient-path pose index: chunk c = a / W lives at [c][2W], its copy at [c][2W] + W.
template <int W>
__device__ __forceinline__ int ridx(int a) { return a + (a & ~(W - 1)); }

// Per-group scratch in shared memory.
struct Scratch {
    float4 *r;                    // [N]  pose (x,y,z) and charge
    float4 *W;                    // [3T] torsion composite transforms (rows R|t)
    int *tp;                      // [T]  pointer-jumping ancestor of each torsion
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

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// 1/x on the SFU without the IEEE-denormal fix-up __fdividef(1, x) carries (ρ² ≥ 1e-4
// after the D5 clamp, so the operand is always a normal number).
__device__ __forceinline__ float rcp_approx(float x) {
#ifdef DK_RCP_FDIV
    return __fdividef(1.0f, x);   // A/B variant: the IEEE-denormal-safe form
#else
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
#endif
}

__device__ __forceinline__ float rsqrt_approx(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// sin/cos of an unwrapped angle: two-constant Cody-Waite reduction to [-pi, pi], then the
// SFU (__sincosf, |err| < 4e-7 there).  Genes are never wrapped (D3), so the reduction
// matters; beyond |x| = 1e5 the accurate library path is used.
__device__ __forceinline__ void fast_sincos(float x, float &s, float &c) {
    if (fabsf(x) < 1.0e5f) {
        const float k = rintf(x * 0.15915494309189535f);
        float r = fmaf(-k, 6.28318548202514648f, x);
        r = fmaf(-k, -1.7484555314695172e-07f, r);
        __sincosf(r, &s, &c);
    } else {
        sincosf(x, &s, &c);
    }
}

#ifdef DK_AD4
// D5-AD4 vdW / H-bond at the smoothed distance: the smoothed r_s (minimum of the potential
// over [r - 0.25, r + 0.25] Å: r + 0.25 below r_eq - 0.25, r - 0.25 above r_eq + 0.25, r_eq
// in between) and 1 / r_s^2.
__device__ __forceinline__ float ad4_smooth(float r, float req) {
    const float lo = r + kSmoothH;
    return lo < req ? lo : fmaxf(r - kSmoothH, req);
}

// D5-AD4 pair energy from precomputed pair constants (energy-only path):
// pp = {r_eq, +-w eps_ij (negative: H-bond pair), w_ds (S'_i V_j + S'_j V_i), w_el 332.06363 q_i q_j}.
__device__ __forceinline__ float pair_e_pre(float rho2, float4 pp) {
    const bool hb = __float_as_int(pp.y) < 0;
    rho2 = fmaxf(rho2, 1e-4f);                           // 0.01 Å clamp
    const float r = rho2 * rsqrt_approx(rho2);
    const float rs = ad4_smooth(r, pp.x);
    const float x2 = pp.x * pp.x * rcp_approx(rs * rs), x4 = x2 * x2, x6 = x4 * x2, x12 = x6 * x6;
    const float vdw = hb ? fmaf(5.0f, x12, -6.0f * (x6 * x4)) : fmaf(-2.0f, x6, x12);
    const float Ev = rho2 < kCutVdw2 ? fabsf(pp.y) * vdw : 0.0f;
    const float u = kDielK * ex2_approx(kDielC * r), sg = 1.0f + u;
    const float Eel = pp.w * sg * rcp_approx(r * fmaf(kDielA, sg, kDielB));   // qq / (r eps(r))
    const float Eds = pp.z * ex2_approx(rho2 * kExpScale);
    return Ev + (rho2 < kCutEl2 ? Eel + Eds : 0.0f);
}
#else
// D5 pair energy from precomputed pair constants (energy-only path).
__device__ __forceinline__ float pair_e_pre(float rho2, float4 pp) {
    const bool hb = __float_as_int(pp.y) < 0;            // H-bond pair: eps_ij stored negated
    rho2 = fmaxf(rho2, 1e-4f);                           // 0.01 Å clamp
    const float inv = rcp_approx(rho2);
    const float x2 = pp.x * inv, x4 = x2 * x2, x6 = x4 * x2, x12 = x6 * x6;
    const float vdw = hb ? fmaf(5.0f, x12, -6.0f * (x6 * x4)) : fmaf(-2.0f, x6, x12);   // 12-10 / 12-6
    return fmaf(fabsf(pp.y), vdw, fmaf(pp.w, inv, pp.z * ex2_approx(rho2 * kExpScale)));
}
#endif

// D5 pair energy and dE/d(rho^2) from per-atom parameters (gradient path).
__device__ __forceinline__ float pair_eg(float rho2, float4 pi, float qi, float4 pj, float qj, bool hb, float &dE) {
    const bool clamped = rho2 < 1e-4f;
    rho2 = fmaxf(rho2, 1e-4f);
    const float inv = rcp_approx(rho2);
    const float req = pi.x + pj.x;                       // (R_i + R_j)/2
    const float eps = pi.y * pj.y;                       // sqrt(eps_i eps_j)
    const float SV = fmaf(pi.z, pj.w, pj.z * pi.w);      // S_i V_j + S_j V_i
    const float x2 = req * req * inv, x4 = x2 * x2, x6 = x4 * x2, x12 = x6 * x6;
    const float xn = hb ? x6 * x4 : x6;
    const float c12 = hb ? 5.0f : 1.0f, cn = hb ? 6.0f : 2.0f, dn = hb ? 30.0f : 6.0f;
    const float Evdw = eps * fmaf(c12, x12, -cn * xn);
    const float Eel = (kElec4 * qi * qj) * inv;          // eps(r) = 4r
    const float Eds = SV * ex2_approx(rho2 * kExpScale);
    const float dv = -eps * inv * fmaf(6.0f * c12, x12, -dn * xn);
    const float d = fmaf(-Eel, inv, fmaf(-Eds, kInvTwoSigma2, dv));
    dE = clamped ? 0.0f : d;
    return Evdw + Eel + Eds;
}

// S_i V_j + S_j V_i from own and partner params {R/2, sqrt eps, S, V}
__device__ __forceinline__ float o_sv(float4 pi, float4 pj) { return fmaf(pi.z, pj.w, pj.z * pi.w); }

// D5 vdW/H-bond part from (x^2, A, B): E = A x^12 - |B| x^n, n = 6 (B >= +0) or 10 (B
// negative); returns E and rho^2 dE/drho^2 = -6 A x^12 + (n/2) |B| x^n.
__device__ __forceinline__ float vdw_ab(float x2, float A, float B, float &dvr) {
    const float x4 = x2 * x2, x6 = x4 * x2, x12 = x6 * x6;
    const bool ten = __float_as_int(B) < 0;
    const float xn = ten ? x6 * x4 : x6;
    const float tA = A * x12, tB = fabsf(B) * xn;
    dvr = fmaf(-6.0f, tA, (ten ? 5.0f : 3.0f) * tB);
    return tA - tB;
}

#ifdef DK_AD4
// D5-AD4 pair energy and dE/d(rho^2), given rq = r_eq, the weighted vdW coefficients, the
// weighted desolvation product and qq = w_el 332.06363 q_i q_j:
//   vdW at the smoothed r_s: dE/drho^2 = (dE/dr_s)(dr_s/dr) / 2r = dvr / (r_s r), 0 on the plateau;
//   elec qq s / (r D), s = 1 + k e^{-lambda B r}, D = A s + B (eps = D / s):
//     dE/drho^2 = -E (1/r + eps'/eps) / 2r, eps'/eps = lambda B^2 (s - 1) / (s D);
//   desolvation as D5; cutoffs on rho^2; zero force inside the clamp.
__device__ __forceinline__ float pair_eg_ab(float rho2, float rq, float A, float B, float sv, float qq, float &dE) {
    const bool clamped = rho2 < 1e-4f;
    rho2 = fmaxf(rho2, 1e-4f);                           // 0.01 Å clamp
    const float ir = rsqrt_approx(rho2), r = rho2 * ir;
    const float rs = ad4_smooth(r, rq);
    const float irs2 = rcp_approx(rs * rs);
    float dvr;
    const float Ev = vdw_ab(rq * rq * irs2, A, B, dvr);
    const float dv = rs == rq ? 0.0f : dvr * (rs * irs2) * ir;
    const bool in_v = rho2 < kCutVdw2;
    const float u = kDielK * ex2_approx(kDielC * r), sg = 1.0f + u;
    const float isd = rcp_approx(sg * fmaf(kDielA, sg, kDielB));
    const float Eel = qq * (sg * sg) * isd * ir;
    const float del = -0.5f * Eel * ir * fmaf(kDielLB2 * u, isd, ir);
    const float Eds = sv * ex2_approx(rho2 * kExpScale);
    const bool in_e = rho2 < kCutEl2;
    const float d = (in_v ? dv : 0.0f) + (in_e ? fmaf(-Eds, kInvTwoSigma2, del) : 0.0f);
    dE = clamped ? 0.0f : d;
    return (in_v ? Ev : 0.0f) + (in_e ? Eel + Eds : 0.0f);
}

// Energy only, from the same operands (large-ligand energy tiles).
__device__ __forceinline__ float pair_e_ab(float rho2, float rq, float A, float B, float sv, float qq) {
    rho2 = fmaxf(rho2, 1e-4f);
    const float r = rho2 * rsqrt_approx(rho2);
    const float rs = ad4_smooth(r, rq);
    float dvr;
    const float Ev = vdw_ab(rq * rq * rcp_approx(rs * rs), A, B, dvr);
    const float u = kDielK * ex2_approx(kDielC * r), sg = 1.0f + u;
    const float Eel = qq * sg * rcp_approx(r * fmaf(kDielA, sg, kDielB));
    const float Eds = sv * ex2_approx(rho2 * kExpScale);
    return (rho2 < kCutVdw2 ? Ev : 0.0f) + (rho2 < kCutEl2 ? Eel + Eds : 0.0f);
}

// pair-slot / tile operand for r_eq: r_eq itself (smoothing compares distances)
__device__ __forceinline__ float sf_req(float req) { return req; }
// own-charge scale (w_el 332.06363) and the vdW / H-bond coefficients per unit eps_ij
__device__ __forceinline__ float sf_qscale(const LigSm &L) { return L.qscale; }
__device__ __forceinline__ void sf_vdw_coeffs(const LigSm &L, bool hb, float eps, float &A, float &B) {
    A = eps * (hb ? L.wA_h : L.wA_v);
    B = eps * (hb ? L.wB_h : L.wB_v);
}
#else
// D5 pair energy and dE/d(rho^2) on the gradient path, given the vdW coefficients:
// E_el = qq / rho^2; E_ds = SV exp(-rho^2 / 2 sigma^2); zero force inside the clamp.
__device__ __forceinline__ float pair_eg_ab(float rho2, float req2, float A, float B, float sv, float qq, float &dE) {
    const bool clamped = rho2 < 1e-4f;
    rho2 = fmaxf(rho2, 1e-4f);                           // 0.01 Å clamp
    const float inv = rcp_approx(rho2);
    float dvr;
    const float Evdw = vdw_ab(req2 * inv, A, B, dvr);
    const float Eel = qq * inv;
    const float Eds = sv * ex2_approx(rho2 * kExpScale);
    const float d = fmaf(dvr - Eel, inv, -Eds * kInvTwoSigma2);
    dE = clamped ? 0.0f : d;
    return Evdw + Eel + Eds;
}

// Energy only, from the same operands (large-ligand energy tiles).
__device__ __forceinline__ float pair_e_ab(float rho2, float req2, float A, float B, float sv, float qq) {
    rho2 = fmaxf(rho2, 1e-4f);
    const float inv = rcp_approx(rho2);
    float dvr;
    const float Ev = vdw_ab(req2 * inv, A, B, dvr);
    return Ev + fmaf(qq, inv, sv * ex2_approx(rho2 * kExpScale));
}

__device__ __forceinline__ float sf_req(float req) { return req * req; }
__device__ __forceinline__ float sf_qscale(const LigSm &) { return kElec4; }
__device__ __forceinline__ void sf_vdw_coeffs(const LigSm &, bool hb, float eps, float &A, float &B) {
    A = hb ? 5.0f * eps : eps;
    B = hb ? -6.0f * eps : 2.0f * eps;
}
#endif

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
        const float c000 = fmaf(aq, m000.z, fmaf(q, m000.y, m000.x)), c100 = fmaf(aq, m100.z, fmaf(q, m100.y, m100.x));
        const float c010 = fmaf(aq, m010.z, fmaf(q, m010.y, m010.x)), c110 = fmaf(aq, m110.z, fmaf(q, m110.y, m110.x));
        const float c001 = fmaf(aq, m001.z, fmaf(q, m001.y, m001.x)), c101 = fmaf(aq, m101.z, fmaf(q, m101.y, m101.x));
        const float c011 = fmaf(aq, m011.z, fmaf(q, m011.y, m011.x)), c111 = fmaf(aq, m111.z, fmaf(q, m111.y, m111.x));
        const float dx00 = c100 - c000, dx10 = c110 - c010, dx01 = c101 - c001, dx11 = c111 - c011;
        const float a00 = fmaf(fx, dx00, c000), a10 = fmaf(fx, dx10, c010);
        const float a01 = fmaf(fx, dx01, c001), a11 = fmaf(fx, dx11, c011);
        const float dy0 = a10 - a00, dy1 = a11 - a01;
        const float b0 = fmaf(fy, dy0, a00), b1 = fmaf(fy, dy1, a01);
        const float dxy0 = fmaf(fy, dx10 - dx00, dx00), dxy1 = fmaf(fy, dx11 - dx01, dx01);
        gx = fmaf(fz, dxy1 - dxy0, dxy0) * g.inv_s;
        gy = fmaf(fz, dy1 - dy0, dy0) * g.inv_s;
        gz = (b1 - b0) * g.inv_s;
        return fmaf(fz, b1 - b0, b0);
    }
    const float cx = fminf(fmaxf(rx, g.ox), g.hx), cy = fminf(fmaxf(ry, g.oy), g.hy),
                cz = fminf(fmaxf(rz, g.oz), g.hz);
    const float dx = rx - cx, dy = ry - cy, dz = rz - cz;
    const float d = sqrtf(dx * dx + dy * dy + dz * dz);
    const float s = d > 0.0f ? kOut / d : 0.0f;
    gx = dx * s; gy = dy * s; gz = dz * s;
    return kOut * (1.0f + d);
}

// Own-atom pair data of a lane (gradient tiles).
// (A per-type-pair table lookup was measured slower: random 16-byte shared-memory reads
// bank-conflict across lanes, profiles/r01f; these per-atom partner reads are consecutive.)
struct OwnPair {
    float q;                      // 332.06363/4 * q_i
    float R, e, S, V;             // |R_i|/2, |sqrt eps_i|, S_i, V_i
    bool hbc, don;                // H-bond capable, donor (else acceptor)
};

// One D5 pair inside the gradient tiles: energy into e, force into the own-atom
// accumulator (+dE d) and the partner accumulator (-dE d); the factor 2 of
// dE/dr_i = 2 dE/drho2 (r_i - r_j) is applied once per atom at the end.
// Partner data: pose record rj (x, y, z, q) and signed params pj (role in the signs).
__device__ __forceinline__ void tile_pair(const LigSm &L, bool on, float rxi, float ryi, float rzi, const OwnPair &o, float4 rj,
                                          float4 pj, float &e, float &gxi, float &gyi, float &gzi, float &fx,
                                          float &fy, float &fz) {
    const float dx = rxi - rj.x, dy = ryi - rj.y, dz = rzi - rj.z;
    const float rho2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
    float dE, E;
    const float req = o.R + fabsf(pj.x);                 // (R_i + R_j) / 2
    const float eps = o.e * fabsf(pj.y);                 // sqrt(eps_i eps_j)
    const bool hb = o.hbc && __float_as_int(o.don ? pj.x : pj.y) < 0;   // donor-acceptor (role in sign bits)
    float A, B;
    sf_vdw_coeffs(L, hb, eps, A, B);
    E = pair_eg_ab(rho2, sf_req(req), A, B, fmaf(o.S, pj.w, pj.z * o.V), o.q * rj.w, dE);
    dE = on ? dE : 0.0f;
    e += on ? E : 0.0f;
    gxi = fmaf(dE, dx, gxi); gyi = fmaf(dE, dy, gyi); gzi = fmaf(dE, dz, gzi);
    fx = fmaf(-dE, dx, fx); fy = fmaf(-dE, dy, fy); fz = fmaf(-dE, dz, fz);
}

// Intramolecular energy and forces, every pair computed once, without atomics:
//  * W x W tiles of atom chunks (I, J): at step s lane l pairs its atom I*W+l with
//    J*W+((l+s) mod W); the partner's force accumulator travels with the partner (one
//    lane shift per step) and returns to its owner after the tile.  Diagonal tiles use
//    s = 1..W/2 (s = W/2 only for l < W/2), so each unordered pair appears once.
//    Pose and partner types are stored chunk-duplicated ([c][2W]), so the partner of
//    step s is entry l + s of the chunk row -- a fixed offset from a per-tile base, no
//    wrap-around or clamping arithmetic -- and the pair-membership bits are pre-rotated
//    per lane, so bit s is the step-s partner.
//  * a short tail chunk (t atoms) is paired by broadcast: all lanes meet tail atom j at
//    once and j's force is a butterfly sum.
//  * partner params are stored chunk-duplicated too, with the H-bond role in their sign
//    bits; the charges come from the pose records (own charge pre-scaled by 332.06363/4).
// Fixed order -> deterministic.
template <int W, int MAXC>
__device__ __forceinline__ void intra_tiles(const LigSm &L, const Scratch &S, int sub, unsigned mask,
                                            const float (&rx)[MAXC], const float (&ry)[MAXC], const float (&rz)[MAXC],
                                            float (&gx)[MAXC], float (&gy)[MAXC], float (&gz)[MAXC], float &e) {
    const int N = L.N;
    const int Bf = N / W, t = N - Bf * W;
    // tail as a padded rotated chunk vs broadcast: decided on the host (prep.cpp cost model)
    const bool tail_rot = L.tail_rot != 0;
    const int Bt = Bf + (tail_rot ? 1 : 0);
    OwnPair own[MAXC];
    float hx[MAXC], hy[MAXC], hz[MAXC];   // pair-force sums (x 2 at the end)
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
        const int a = sub + W * c;
        const bool ok = a < N;
        own[c].q = ok ? sf_qscale(L) * S.r[ridx<W>(a)].w : 0.0f;
        const float4 pp = L.ppar[ridx<W>(a)];
        own[c].R = fabsf(pp.x); own[c].e = fabsf(pp.y); own[c].S = pp.z; own[c].V = pp.w;
        own[c].hbc = __float_as_int(pp.x) < 0 || __float_as_int(pp.y) < 0;   // sign bits: -0.0 counts
        own[c].don = __float_as_int(pp.y) < 0;
        hx[c] = hy[c] = hz[c] = 0.0f;
    }
#pragma unroll
    for (int I = 0; I < MAXC; ++I) {
        if (I >= Bt) break;
#pragma unroll
        for (int J = I; J < MAXC; ++J) {
            if (J >= Bt) break;
            const int aI = I * W + sub;
            const int jb = J * W;
            uint32_t mw = aI < N ? (L.mask[aI * L.NW + (jb >> 5)] >> (jb & 31)) : 0u;
            uint32_t rot;
            if constexpr (W == 32) {
                rot = __funnelshift_r(mw, mw, sub);             // bit s = partner (sub + s) mod 32
            } else {
                mw &= 0xffffu;
                rot = ((mw | (mw << 16)) >> sub) & 0xffffu;
            }
            if (I == J && sub >= W / 2) rot &= ~(1u << (W / 2));   // each diagonal pair once
            const float4 *rrow = S.r + J * 2 * W + sub;         // partner of step s: rrow[s]
            const float4 *qrow = L.ppar + J * 2 * W + sub;
            const int s0 = (I == J) ? 1 : 0, s1 = (I == J) ? W / 2 : W - 1;
            float fx = 0.f, fy = 0.f, fz = 0.f;
#pragma unroll 4
            for (int s = s0; s <= s1; ++s) {
                tile_pair(L, (rot >> s) & 1u, rx[I], ry[I], rz[I], own[I], rrow[s], qrow[s], e, hx[I], hy[I], hz[I], fx,
                          fy, fz);
                if (s < s1) {
                    const int src = (sub + 1) & (W - 1);
                    fx = __shfl_sync(mask, fx, src, W);
                    fy = __shfl_sync(mask, fy, src, W);
                    fz = __shfl_sync(mask, fz, src, W);
                }
            }
            const int back = (sub - s1) & (W - 1);
            fx = __shfl_sync(mask, fx, back, W);
            fy = __shfl_sync(mask, fy, back, W);
            fz = __shfl_sync(mask, fz, back, W);
            hx[J] += fx; hy[J] += fy; hz[J] += fz;
        }
    }
    if (t > 0 && !tail_rot) {
        for (int k = 0; k < t; ++k) {
            const int j = Bf * W + k;                       // uniform: shared-memory broadcast
            const float4 rj = S.r[ridx<W>(j)];
            const float4 pj = L.ppar[ridx<W>(j)];
            const uint32_t *mrow = L.mask + (size_t)j * L.NW;
            float fx = 0.f, fy = 0.f, fz = 0.f;
#pragma unroll
            for (int I = 0; I < MAXC; ++I) {
                if (I > Bf) break;
                const int a = I * W + sub;
                const bool on = (I < Bf || sub < k) && ((mrow[a >> 5] >> (a & 31)) & 1u);
                tile_pair(L, on, rx[I], ry[I], rz[I], own[I], rj, pj, e, hx[I], hy[I], hz[I], fx, fy, fz);
            }
            fx = gsum<W>(fx, mask); fy = gsum<W>(fy, mask); fz = gsum<W>(fz, mask);
#pragma unroll
            for (int c = 0; c < MAXC; ++c)
                if (c == Bf && sub == k) { hx[c] += fx; hy[c] += fy; hz[c] += fz; }
        }
    }
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
        gx[c] = fmaf(2.0f, hx[c], gx[c]); gy[c] = fmaf(2.0f, hy[c], gy[c]); gz[c] = fmaf(2.0f, hz[c], gz[c]);
    }
}

#ifndef DK_FOLD
#define DK_FOLD 1   // D5 slot constants folded (A r_eq^12, B r_eq^n, SV, qq); 0: {r_eq^2, A, B, SV} + qq (A/B)
#endif

struct EAcc { float e = 0.0f; };
__device__ __forceinline__ float eacc_total(const EAcc &a) { return a.e; }
#if defined(DK_AD4) || !DK_FOLD
// One pair inside the slot-table tiles: constants c = {r_eq, A, B, SV} and qq from the
// slot (all zero for a non-pair, so no membership test), force as in tile_pair.
__device__ __forceinline__ void slot_pair(float rxi, float ryi, float rzi, float4 rj, float4 c, float qq, EAcc &e,
                                          float &gxi, float &gyi, float &gzi, float &fx, float &fy, float &fz) {
    const float dx = rxi - rj.x, dy = ryi - rj.y, dz = rzi - rj.z;
    const float rho2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
    float dE;
    e.e += pair_eg_ab(rho2, c.x, c.y, c.z, c.w, qq, dE);
    gxi = fmaf(dE, dx, gxi); gyi = fmaf(dE, dy, gyi); gzi = fmaf(dE, dz, gzi);
    fx = fmaf(-dE, dx, fx); fy = fmaf(-dE, dy, fy); fz = fmaf(-dE, dz, fz);
}
#define DK_SLOT(q) L.slot4[q], L.slotq[q]
#else
// D5 pair from folded slot constants c = {A' = A r_eq^12, B' = +-|B| r_eq^n, SV, qq} (prep.cpp;
// sign of B': the 12-10 H-bond form): with inv = 1/rho^2, E_vdw = A' inv^6 - |B'| inv^{n/2},
// rho^2 dE_vdw/drho^2 = -6 A' inv^6 + (n/2) |B'| inv^{n/2} -- one multiply and one 4-byte
// shared-memory read fewer per slot than {r_eq^2, A, B, SV} + qq.  Zero for a non-pair.
__device__ __forceinline__ float pair_eg_folded(float rho2, float4 c, float &dE) {
    const bool clamped = rho2 < 1e-4f;
    rho2 = fmaxf(rho2, 1e-4f);                           // 0.01 Å clamp
    const float inv = rcp_approx(rho2);
    const float i2 = inv * inv, i3 = i2 * inv, i6 = i3 * i3;
    const bool ten = __float_as_int(c.y) < 0;
    const float xn = ten ? i3 * i2 : i3;
    const float tA = c.x * i6, tB = fabsf(c.y) * xn;
    const float dvr = fmaf(-6.0f, tA, (ten ? 5.0f : 3.0f) * tB);
    const float Eel = c.w * inv;
    const float Eds = c.z * ex2_approx(rho2 * kExpScale);
    const float d = fmaf(dvr - Eel, inv, -Eds * kInvTwoSigma2);
    dE = clamped ? 0.0f : d;
    return (tA - tB) + Eel + Eds;
}
__device__ __forceinline__ void slot_pair(float rxi, float ryi, float rzi, float4 rj, float4 c, EAcc &e,
                                          float &gxi, float &gyi, float &gzi, float &fx, float &fy, float &fz) {
    const float dx = rxi - rj.x, dy = ryi - rj.y, dz = rzi - rj.z;
    const float rho2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
    float dE;
    e.e += pair_eg_folded(rho2, c, dE);
    gxi = fmaf(dE, dx, gxi); gyi = fmaf(dE, dy, gyi); gzi = fmaf(dE, dz, gzi);
    fx = fmaf(-dE, dx, fx); fy = fmaf(-dE, dy, fy); fz = fmaf(-dE, dz, fz);
}
#define DK_SLOT(q) L.slot4[q]
#endif

#if !defined(DK_AD4) && DK_FOLD
#define DK_PACK_ON 1   // packed FP32x2 tiles (D5, LigDev::packed)
// Lean D5 constants of the packed rows (prep.cpp): c = {-A', B', -(k/3) SV, -qq/3} with
// A' = eps r_eq^12, B' = 2 eps r_eq^6 (the 12-6 form; zero for an H-bond pair, whose 12-10 vdW
// term is hb_side's), k = 1/2sigma^2, qq = 332.06363/4 q_i q_j.  With inv = 1/rho^2, i3 = inv^3:
//   u = B' - A' i3, E_vdw = A' i6 - B' i3 = -i3 u;  v = B' - 2 A' i3, rho^2 dE_vdw/drho^2 = 3 i3 v;
//   t = i3 v - qq inv / 3 = (rho^2 dE_vdw/drho^2 - E_el) / 3;  d = t inv - k E_ds / 3 = (dE/drho^2) / 3.
// The energy goes to three sums scaled as above (EAcc2: -E_vdw, -E_el/3, -k E_ds/3), unscaled
// once per evaluation (lean_total); the forces carry (dE/drho^2) / 3 and are multiplied by 3
// once per tile when they join the folded path's per-atom sums.  24 FP32 operations per
// slot (12 packed instructions) instead of 29, no per-slot H-bond selects.
constexpr float kDsUnscale = -3.0f * 2.0f * 3.6f * 3.6f;   // -3/k

// ---- Packed FP32x2 lean slots (sm_100 fma/mul/add/sub.rn.f32x2: one instruction, two
// independent IEEE FP32 operations) for two-chunk ligands (W = 32; LigDev::packed, prep.cpp:
// 49 <= N <= 64 with the second chunk padded and rotated, 65 <= N <= ~82 with a hybrid
// tail).  Every lane evaluates TWO slots per instruction stream, so the 24 FP32 operations
// of a lean slot cost 12 issue slots:
//   (a) diagonal pair: tiles (0,0) and (1,1) together, step s = 1..16 (own atoms sub and
//       32 + sub, partners (sub + s) of chunk 0 and of chunk 1);
//   (b) split tile (0,1): steps u and u + 16 together, u = 0..15 (own atom sub twice);
//   (c) hybrid tail: tail atom k against chunks 0 and 1 together.
// The partner poses of (a) and (b) are re-laid out per evaluation as {x_a, x_b, y_a, y_b}
// + {z_a, z_b} rows (one LDS.128 + one LDS.64 per packed step), in the group's gradient
// scratch (free until the H-bond side list and the back-projection reuse it).  The slot
// constants of packed step q are two
// float4 rows [q][0..W) = {-A'_a, -A'_b, B'_a, B'_b} and [q][W..2W) = {SV_a, SV_b, Q_a, Q_b}
// (the lean constants of slots a and b).  The same D5 terms as the folded slot_pair in
// another algebraic form (held to the oracle at NS tolerance: test_packed_tiles_parity).
typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t f2_pk(float a, float b) {
    f2_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
#pragma nv_diag_suppress 550   // the unused half of an unpacking mov.b64 (register halves, no instruction)
__device__ __forceinline__ float f2_lo(f2_t v) {
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
    return a;
}
__device__ __forceinline__ float f2_hi(f2_t v) {
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
    return b;
}
#pragma nv_diag_default 550
__device__ __forceinline__ f2_t add2(f2_t a, f2_t b) { f2_t d; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ f2_t sub2(f2_t a, f2_t b) { f2_t d; asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ f2_t mul2(f2_t a, f2_t b) { f2_t d; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ f2_t fma2(f2_t a, f2_t b, f2_t c) {
    f2_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ f2_t f2_shfl(f2_t v, int src, unsigned mask) {
    return f2_pk(__shfl_sync(mask, f2_lo(v), src), __shfl_sync(mask, f2_hi(v), src));
}
struct EAcc2 { f2_t v = 0ull, el = 0ull, ds = 0ull; };   // bit pattern 0 = (+0.0f, +0.0f)

__device__ __forceinline__ void slot_pair2(f2_t ox, f2_t oy, f2_t oz, f2_t px, f2_t py, f2_t pz, float4 ca, float4 cb,
                                           EAcc2 &e, f2_t &gx, f2_t &gy, f2_t &gz, f2_t &fx, f2_t &fy, f2_t &fz) {
    const f2_t dx = sub2(ox, px), dy = sub2(oy, py), dz = sub2(oz, pz);
    const f2_t rho2 = fma2(dx, dx, fma2(dy, dy, mul2(dz, dz)));
    const float q0 = f2_lo(rho2), q1 = f2_hi(rho2);
    const float r0 = fmaxf(q0, 1e-4f), r1 = fmaxf(q1, 1e-4f);   // 0.01 Å clamp
    const f2_t inv = f2_pk(rcp_approx(r0), rcp_approx(r1));
    const f2_t i2 = mul2(inv, inv), i3 = mul2(i2, inv);
    const f2_t u = fma2(f2_pk(ca.x, ca.y), i3, f2_pk(ca.z, ca.w));
    const f2_t v = fma2(f2_pk(ca.x, ca.y), i3, u);
    e.v = fma2(i3, u, e.v);
    const f2_t el = mul2(f2_pk(cb.z, cb.w), inv);
    e.el = add2(e.el, el);
    const f2_t t = fma2(i3, v, el);
    const f2_t ea = mul2(f2_pk(r0, r1), f2_pk(kExpScale, kExpScale));
    const f2_t ed = mul2(f2_pk(cb.x, cb.y), f2_pk(ex2_approx(f2_lo(ea)), ex2_approx(f2_hi(ea))));
    e.ds = add2(e.ds, ed);
    const f2_t d = fma2(t, inv, ed);
    const f2_t dE = f2_pk(q0 < 1e-4f ? 0.0f : f2_lo(d), q1 < 1e-4f ? 0.0f : f2_hi(d));   // zero force in the clamp
    gx = fma2(dE, dx, gx); gy = fma2(dE, dy, gy); gz = fma2(dE, dz, gz);
    fx = fma2(dE, dx, fx); fy = fma2(dE, dy, fy); fz = fma2(dE, dz, fz);   // partner: subtracted on return
}

#ifndef DK_PACK_UNROLL
#define DK_PACK_UNROLL 4   // packed steps unrolled (A/B: 1 0.98x, 2 0.996x, 8 0.96x; scripts/variants.py)
#endif
constexpr int kPackUnroll = DK_PACK_UNROLL;
#ifndef DK_HYB_PAIR
#define DK_HYB_PAIR 1   // packed hybrid tail: two tail atoms per transposed butterfly (A/B: 0)
#endif
#ifndef DK_HYB_PAIR_UNROLL
#define DK_HYB_PAIR_UNROLL 1   // iterations (atom pairs) of that loop unrolled (A/B)
#endif

// (a) + (b): the tiles of the two chunks (the second one full or padded).  Own-atom forces
// go to hx[0..1] etc.
template <int W, int MAXC>
__device__ __forceinline__ void tiles_packed(const LigSm &L, const Scratch &S, int sub, unsigned mask,
                                             const float (&rx)[MAXC], const float (&ry)[MAXC], const float (&rz)[MAXC],
                                             float (&hx)[MAXC], float (&hy)[MAXC], float (&hz)[MAXC], EAcc2 &e2) {
    static_assert(W == 32 && MAXC >= 2, "packed tiles: two 32-atom chunks (the second may be padded)");
    float4 *pdxy = S.ts, *psxy = S.ts + 48;                         // [48] rows each
    float2 *pdz = reinterpret_cast<float2 *>(S.ts + 96), *psz = pdz + 48;
    {
        const float x16 = __shfl_xor_sync(mask, rx[1], 16), y16 = __shfl_xor_sync(mask, ry[1], 16),
                    z16 = __shfl_xor_sync(mask, rz[1], 16);
        const float4 d4 = make_float4(rx[0], rx[1], ry[0], ry[1]), s4 = make_float4(rx[1], x16, ry[1], y16);
        const float2 d2 = make_float2(rz[0], rz[1]), s2 = make_float2(rz[1], z16);
        pdxy[sub] = d4; pdz[sub] = d2; psxy[sub] = s4; psz[sub] = s2;
        if (sub < 16) { pdxy[sub + 32] = d4; pdz[sub + 32] = d2; psxy[sub + 32] = s4; psz[sub + 32] = s2; }
    }
    __syncwarp(mask);
    const int src = sub + 1;                                        // shfl.idx takes the lane mod 32
    const float4 *cst = L.slot4 + sub;
    // own-atom pairs re-read from the rows (64-bit register pairs from the loads; the scalar
    // pose registers are dead here, eval_group reloads them after the tiles)
    const float4 o4 = pdxy[sub];
    const float2 o2 = pdz[sub];
    // (a) diagonal pair, packed steps q = 0..15 (tile step s = q + 1)
    {
        const f2_t ox = f2_pk(o4.x, o4.y), oy = f2_pk(o4.z, o4.w), oz = f2_pk(o2.x, o2.y);
        f2_t gx = 0ull, gy = 0ull, gz = 0ull, fx = 0ull, fy = 0ull, fz = 0ull;
#pragma unroll kPackUnroll
        for (int q = 0; q < 16; ++q) {
            const float4 xy = pdxy[sub + q + 1];
            const float2 zz = pdz[sub + q + 1];
            slot_pair2(ox, oy, oz, f2_pk(xy.x, xy.y), f2_pk(xy.z, xy.w), f2_pk(zz.x, zz.y), cst[q * 2 * W],
                       cst[q * 2 * W + W], e2, gx, gy, gz, fx, fy, fz);
            fx = f2_shfl(fx, src, mask); fy = f2_shfl(fy, src, mask); fz = f2_shfl(fz, src, mask);
        }
        const int back = (sub - 17) & (W - 1);
        fx = f2_shfl(fx, back, mask); fy = f2_shfl(fy, back, mask); fz = f2_shfl(fz, back, mask);
        const f2_t hx01 = sub2(gx, fx), hy01 = sub2(gy, fy), hz01 = sub2(gz, fz);
        hx[0] = fmaf(3.0f, f2_lo(hx01), hx[0]); hx[1] = fmaf(3.0f, f2_hi(hx01), hx[1]);   // x 3: folded units
        hy[0] = fmaf(3.0f, f2_lo(hy01), hy[0]); hy[1] = fmaf(3.0f, f2_hi(hy01), hy[1]);
        hz[0] = fmaf(3.0f, f2_lo(hz01), hz[0]); hz[1] = fmaf(3.0f, f2_hi(hz01), hz[1]);
    }
    // (b) split tile (0,1), packed steps q = 16..31 (tile steps u and u + 16, u = q - 16)
    {
        const f2_t ox = f2_pk(o4.x, o4.x), oy = f2_pk(o4.z, o4.z), oz = f2_pk(o2.x, o2.x);
        f2_t gx = 0ull, gy = 0ull, gz = 0ull, fx = 0ull, fy = 0ull, fz = 0ull;
#pragma unroll kPackUnroll
        for (int u = 0; u < 16; ++u) {
            const float4 xy = psxy[sub + u];
            const float2 zz = psz[sub + u];
            slot_pair2(ox, oy, oz, f2_pk(xy.x, xy.y), f2_pk(xy.z, xy.w), f2_pk(zz.x, zz.y), cst[(16 + u) * 2 * W],
                       cst[(16 + u) * 2 * W + W], e2, gx, gy, gz, fx, fy, fz);
            fx = f2_shfl(fx, src, mask); fy = f2_shfl(fy, src, mask); fz = f2_shfl(fz, src, mask);
        }
        // stream a (steps u) ends 16 lanes past its owner, stream b (steps u + 16) at its owner
        const int back = sub ^ 16;
        hx[1] = fmaf(-3.0f, __shfl_sync(mask, f2_lo(fx), back) + f2_hi(fx), hx[1]);
        hy[1] = fmaf(-3.0f, __shfl_sync(mask, f2_lo(fy), back) + f2_hi(fy), hy[1]);
        hz[1] = fmaf(-3.0f, __shfl_sync(mask, f2_lo(fz), back) + f2_hi(fz), hz[1]);
        hx[0] = fmaf(3.0f, f2_lo(gx) + f2_hi(gx), hx[0]); hy[0] = fmaf(3.0f, f2_lo(gy) + f2_hi(gy), hy[0]);
        hz[0] = fmaf(3.0f, f2_lo(gz) + f2_hi(gz), hz[0]);
    }
    __syncwarp(mask);   // the scratch rows are reused (H-bond side list, back-projection)
}

#ifndef DK_HB_FULL
#define DK_HB_FULL 0   // 1: all five scan levels regardless of the longest segment (A/B)
#endif

__device__ __forceinline__ float lean_total(const EAcc2 &a) {
    const float v = f2_lo(a.v) + f2_hi(a.v), el = f2_lo(a.el) + f2_hi(a.el), ds = f2_lo(a.ds) + f2_hi(a.ds);
    return fmaf(-3.0f, el, fmaf(kDsUnscale, ds, -v));
}

// The H-bond pairs of the packed rows (their 12-10 vdW terms; prep.cpp, LigDev::nhb): lane p
// takes pairs p, p + W, ... and stages its force d (r_i - r_j), d = dE/drho^2, in the group's
// gradient scratch.  The 2 nhb atom contributions (+ as i, - as j), sorted by atom and packed
// into rounds of W lanes without splitting an atom (L.hbseg), are then summed per atom by a
// segmented Hillis-Steele scan (shfl.up; each lane knows its segment's first lane), the
// segment's last lane stores the atom's total, and the owner lanes add it.  Fixed order:
// deterministic.  E = A'' i6 - B'' i5 (A'' = 5 eps r_eq^12, B'' = 6 eps r_eq^10),
// rho^2 dE/drho^2 = -6 A'' i6 + 5 B'' i5.
// hbseg entry: pair | neg << 8 | first lane << 9 | last << 14 | valid << 15 | atom << 16.
template <int W, int MAXC>
__device__ __forceinline__ void hb_side(const LigSm &L, const Scratch &S, int sub, unsigned mask, float (&hx)[MAXC],
                                        float (&hy)[MAXC], float (&hz)[MAXC], EAcc &e) {
    __syncwarp(mask);   // the packed tail's reads of the scratch rows precede any later writes
    if (L.nhb == 0) return;
    for (int p = sub; p < L.nhb; p += W) {
        const float4 c = L.hbc[p];
        const uint32_t ij = __float_as_uint(c.z);
        const float4 ri = S.r[ridx<W>((int)(ij & 0xffffu))], rj = S.r[ridx<W>((int)(ij >> 16))];
        const float dx = ri.x - rj.x, dy = ri.y - rj.y, dz = ri.z - rj.z;
        const float rho2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
        const bool clamped = rho2 < 1e-4f;
        const float r2 = fmaxf(rho2, 1e-4f);               // 0.01 Å clamp
        const float inv = rcp_approx(r2), i2 = inv * inv, i3 = i2 * inv, i5 = i3 * i2, i6 = i3 * i3;
        const float tA = c.x * i6, tB = c.y * i5;
        e.e += tA - tB;
        const float d = clamped ? 0.0f : fmaf(-6.0f, tA, 5.0f * tB) * inv;
        S.ts[p] = make_float4(d * dx, d * dy, d * dz, 0.0f);
    }
    __syncwarp(mask);
    float4 *tot = S.ts + L.nhb;                            // per-atom totals [N]
    for (int r = 0; r < L.nhbr; ++r) {
        const int ent = L.hbseg[r * W + sub];
        float4 f = S.ts[ent & 0xff];
        const float sg = (ent >> 15) & 1 ? ((ent >> 8) & 1 ? -1.0f : 1.0f) : 0.0f;
        float fx = sg * f.x, fy = sg * f.y, fz = sg * f.z;
        const int first = (ent >> 9) & 31;
#pragma unroll
        for (int d = 1; d < W; d <<= 1) {
            if (!DK_HB_FULL && d >= L.hbspan) break;   // levels up to the longest segment (uniform)
            const float ox = __shfl_up_sync(mask, fx, d), oy = __shfl_up_sync(mask, fy, d), oz = __shfl_up_sync(mask, fz, d);
            if (sub - d >= first) { fx += ox; fy += oy; fz += oz; }
        }
        if ((ent >> 14) & 1) tot[ent >> 16] = make_float4(fx, fy, fz, 0.0f);
    }
    __syncwarp(mask);
    const int *cmask = L.hbseg + L.nhbr * W;
#pragma unroll
    for (int c = 0; c < MAXC; ++c)
        if ((cmask[c] >> sub) & 1) {
            const float4 f = tot[sub + W * c];
            hx[c] += f.x; hy[c] += f.y; hz[c] += f.z;
        }
    __syncwarp(mask);   // the back-projection reuses the scratch
}
#endif

// intra_tiles with precomputed pair-slot constants (L.slot_mode, prep.cpp): the same
// rotation / broadcast schedule and force bookkeeping, one 16-byte + one 4-byte
// conflict-free shared-memory read per slot instead of partner params and pair bits.
template <int W, int MAXC, bool PK = false>
__device__ __forceinline__ void intra_tiles_slots(const LigSm &L, const Scratch &S, int sub, unsigned mask,
                                                  const float (&rx)[MAXC], const float (&ry)[MAXC],
                                                  const float (&rz)[MAXC], float (&gx)[MAXC], float (&gy)[MAXC],
                                                  float (&gz)[MAXC], float &e_out) {
    EAcc e;
    const int N = L.N;
    const int Bf = N / W, t = N - Bf * W;
    const bool tail_rot = L.tail_rot != 0;
    const int Bt = Bf + (tail_rot ? 1 : 0);
    float hx[MAXC], hy[MAXC], hz[MAXC];
#pragma unroll
    for (int c = 0; c < MAXC; ++c) hx[c] = hy[c] = hz[c] = 0.0f;
    int slot0 = 0;                        // first slot of the current tile
    constexpr bool packed = PK;
#ifdef DK_PACK_ON
    EAcc2 e2;
    if constexpr (PK) {
        static_assert(W == 32 && (MAXC == 2 || MAXC == 3), "packed tiles: W = 32, two chunks");
        // the intermolecular gradients wait in the (unused here) duplicate pose half, so
        // the packed tiles have their registers
#pragma unroll
        for (int c = 0; c < MAXC; ++c)
            if (sub + W * c < N) S.r[ridx<W>(sub + W * c) + W] = make_float4(gx[c], gy[c], gz[c], 0.0f);
        tiles_packed<W, MAXC>(L, S, sub, mask, rx, ry, rz, hx, hy, hz, e2);
#pragma unroll
        for (int c = 0; c < MAXC; ++c)
            if (sub + W * c < N) {
                const float4 g4 = S.r[ridx<W>(sub + W * c) + W];
                gx[c] = g4.x; gy[c] = g4.y; gz[c] = g4.z;
            }
        slot0 = 64 * W;                   // 32 packed steps x 2W rows = the 64 scalar tile steps
    }
#else
    static_assert(!PK, "packed tiles need the folded D5 build");
#endif
#pragma unroll
    for (int I = 0; I < MAXC; ++I) {
        if (I >= Bt || packed) break;
#pragma unroll
        for (int J = I; J < MAXC; ++J) {
            if (J >= Bt) break;
            const float4 *rrow = S.r + J * 2 * W + sub;         // partner of step s: rrow[s]
            const int s0 = (I == J) ? 1 : 0, s1 = (I == J) ? W / 2 : W - 1;
            const int cbase = slot0 + sub - s0 * W;             // constants of step s: slot cbase + s * W
            slot0 += (s1 - s0 + 1) * W;
#if DK_TILE_STREAMS == 2
            // two independent partner-accumulator streams per tile (steps s0.. and s0+h..):
            // their shuffle chains overlap, so a lane has two pairs in flight per step
            const int h = (s1 - s0 + 1) / 2;
            float ax = 0.f, ay = 0.f, az = 0.f, bx = 0.f, by = 0.f, bz = 0.f;
#pragma unroll kTileUnroll
            for (int u = 0; u < h; ++u) {
                const int sa = s0 + u, sb = s0 + h + u;
                slot_pair(rx[I], ry[I], rz[I], rrow[sa], DK_SLOT(cbase + sa * W), e, hx[I], hy[I], hz[I], ax, ay, az);
                slot_pair(rx[I], ry[I], rz[I], rrow[sb], DK_SLOT(cbase + sb * W), e, hx[I], hy[I], hz[I], bx, by, bz);
                if (u < h - 1) {
                    const int src = (sub + 1) & (W - 1);
                    ax = __shfl_sync(mask, ax, src, W); ay = __shfl_sync(mask, ay, src, W);
                    az = __shfl_sync(mask, az, src, W);
                    bx = __shfl_sync(mask, bx, src, W); by = __shfl_sync(mask, by, src, W);
                    bz = __shfl_sync(mask, bz, src, W);
                }
            }
            const int backa = (sub - (s0 + h - 1)) & (W - 1), backb = (sub - s1) & (W - 1);
            hx[J] += __shfl_sync(mask, ax, backa, W) + __shfl_sync(mask, bx, backb, W);
            hy[J] += __shfl_sync(mask, ay, backa, W) + __shfl_sync(mask, by, backb, W);
            hz[J] += __shfl_sync(mask, az, backa, W) + __shfl_sync(mask, bz, backb, W);
#else
            float fx = 0.f, fy = 0.f, fz = 0.f;
            // the partner accumulator moves one lane after EVERY step (the last shift is
            // folded into the return offset): no per-step guard in the unrolled loop
#pragma unroll kTileUnroll
            for (int s = s0; s <= s1; ++s) {
                slot_pair(rx[I], ry[I], rz[I], rrow[s], DK_SLOT(cbase + s * W), e, hx[I], hy[I], hz[I], fx, fy, fz);
                const int src = (sub + 1) & (W - 1);
                fx = __shfl_sync(mask, fx, src, W);
                fy = __shfl_sync(mask, fy, src, W);
                fz = __shfl_sync(mask, fz, src, W);
            }
            const int back = (sub - s1 - 1) & (W - 1);
            fx = __shfl_sync(mask, fx, back, W);
            fy = __shfl_sync(mask, fy, back, W);
            fz = __shfl_sync(mask, fz, back, W);
            hx[J] += fx; hy[J] += fy; hz[J] += fz;
#endif
        }
    }
    if (t > 0 && L.tail_seg > 0) {
        // Segmented tail (prep.cpp): the tail, padded to tp lanes, is rotated inside the W/tp
        // lane segments.  (a) step s pairs own chunk atoms I*W+sub (I < Bf) with tail atom
        // (sl + s) mod tp; the partner accumulator travels one lane per step inside the
        // segment (as in the tiles) and returns to its owner after step tp-1.  (b) tail x
        // tail: segment g takes steps 1 + g + r*(W/tp) of the diagonal schedule (zero slots
        // beyond tp/2); the partner force goes back by one segment shuffle.  A butterfly over
        // the segments then sums each tail atom's force.  Fixed order: deterministic.
        // tail_seg packs tp | log2(tp) << 8 | rounds << 16 (no integer divisions here)
        // bit 24 (hyb): the full chunks x tail part by broadcast instead (every lane meets tail
        // atom k at once, one butterfly per force component), then the segment rounds
        const int tp = L.tail_seg & 0xff, lg = (L.tail_seg >> 8) & 0xff, rounds = (L.tail_seg >> 16) & 0xff;
        const int sl = sub & (tp - 1), nseg = W >> lg, g = sub >> lg;
        const float4 *trow = S.r + Bf * 2 * W;                  // tail chunk (positions 0..tp-1)
        float fx = 0.f, fy = 0.f, fz = 0.f;
        if ((L.tail_seg >> 24) & 1) {
#ifdef DK_PACK_ON
          if (packed) {
            if constexpr (PK) {
                // (c) tail atom k against chunks 0 and 1 together (packed step k)
                const float4 o4 = S.ts[sub];                    // tiles_packed's rows: {x0, x1, y0, y1}
                const float2 o2 = reinterpret_cast<const float2 *>(S.ts + 96)[sub];
                const f2_t ox = f2_pk(o4.x, o4.y), oy = f2_pk(o4.z, o4.w), oz = f2_pk(o2.x, o2.y);
                f2_t gx2 = 0ull, gy2 = 0ull, gz2 = 0ull;
#if DK_HYB_PAIR
                // two tail atoms per iteration: two independent packed evaluations, then one
                // transposed butterfly -- level 16 leaves atom k's partial sums in the low
                // half-warp and atom k + 1's in the high one, levels 8..1 finish both at once,
                // and one exchange hands each owner its atom's total (18 shuffles per two atoms
                // instead of 30, and one dependent chain instead of two)
                const bool up = sub >= 16;
                constexpr int kPairUnroll = DK_HYB_PAIR_UNROLL;
#pragma unroll kPairUnroll
                for (int k = 0; k < t; k += 2) {
                    const bool two = k + 1 < t;                 // uniform
                    const float4 ra = trow[k], rb = trow[two ? k + 1 : k];
                    f2_t ax2 = 0ull, ay2 = 0ull, az2 = 0ull, bx2 = 0ull, by2 = 0ull, bz2 = 0ull;
                    slot_pair2(ox, oy, oz, f2_pk(ra.x, ra.x), f2_pk(ra.y, ra.y), f2_pk(ra.z, ra.z),
                               L.slot4[slot0 + k * 2 * W + sub], L.slot4[slot0 + k * 2 * W + W + sub], e2, gx2, gy2,
                               gz2, ax2, ay2, az2);
                    if (two)
                        slot_pair2(ox, oy, oz, f2_pk(rb.x, rb.x), f2_pk(rb.y, rb.y), f2_pk(rb.z, rb.z),
                                   L.slot4[slot0 + (k + 1) * 2 * W + sub], L.slot4[slot0 + (k + 1) * 2 * W + W + sub], e2,
                                   gx2, gy2, gz2, bx2, by2, bz2);
                    const float ax = f2_lo(ax2) + f2_hi(ax2), ay = f2_lo(ay2) + f2_hi(ay2), az = f2_lo(az2) + f2_hi(az2);
                    const float bx = f2_lo(bx2) + f2_hi(bx2), by = f2_lo(by2) + f2_hi(by2), bz = f2_lo(bz2) + f2_hi(bz2);
                    float kx = up ? bx : ax, ky = up ? by : ay, kz = up ? bz : az;
                    kx += __shfl_xor_sync(mask, up ? ax : bx, 16);
                    ky += __shfl_xor_sync(mask, up ? ay : by, 16);
                    kz += __shfl_xor_sync(mask, up ? az : bz, 16);
#pragma unroll
                    for (int m = 8; m >= 1; m >>= 1) {
                        kx += __shfl_xor_sync(mask, kx, m); ky += __shfl_xor_sync(mask, ky, m); kz += __shfl_xor_sync(mask, kz, m);
                    }
                    const float qx = __shfl_xor_sync(mask, kx, 16), qy = __shfl_xor_sync(mask, ky, 16),
                                qz = __shfl_xor_sync(mask, kz, 16);
                    // lean forces carry (dE/drho^2) / 3 and the partner sums +dE d: x (-3)
                    if (sub == k) { fx = fmaf(-3.0f, up ? qx : kx, fx); fy = fmaf(-3.0f, up ? qy : ky, fy); fz = fmaf(-3.0f, up ? qz : kz, fz); }
                    if (two && sub == k + 1) { fx = fmaf(-3.0f, up ? kx : qx, fx); fy = fmaf(-3.0f, up ? ky : qy, fy); fz = fmaf(-3.0f, up ? kz : qz, fz); }
                }
#else
                for (int k = 0; k < t; ++k) {
                    const float4 rj = trow[k];                  // uniform: shared-memory broadcast
                    f2_t px2 = 0ull, py2 = 0ull, pz2 = 0ull;
                    slot_pair2(ox, oy, oz, f2_pk(rj.x, rj.x), f2_pk(rj.y, rj.y), f2_pk(rj.z, rj.z),
                               L.slot4[slot0 + k * 2 * W + sub], L.slot4[slot0 + k * 2 * W + W + sub], e2, gx2, gy2,
                               gz2, px2, py2, pz2);
                    // lean forces carry (dE/drho^2) / 3: x 3 here, into the folded units
                    float px = -3.0f * (f2_lo(px2) + f2_hi(px2)), py = -3.0f * (f2_lo(py2) + f2_hi(py2)),
                          pz = -3.0f * (f2_lo(pz2) + f2_hi(pz2));
                    px = gsum<W>(px, mask); py = gsum<W>(py, mask); pz = gsum<W>(pz, mask);
                    if (sub == k) { fx += px; fy += py; fz += pz; }
                }
#endif
                hx[0] = fmaf(3.0f, f2_lo(gx2), hx[0]); hx[1] = fmaf(3.0f, f2_hi(gx2), hx[1]);
                hy[0] = fmaf(3.0f, f2_lo(gy2), hy[0]); hy[1] = fmaf(3.0f, f2_hi(gy2), hy[1]);
                hz[0] = fmaf(3.0f, f2_lo(gz2), hz[0]); hz[1] = fmaf(3.0f, f2_hi(gz2), hz[1]);
            }
          } else
#endif
#pragma unroll kHybUnroll
            for (int k = 0; k < t; ++k) {
                const float4 rj = trow[k];                      // uniform: shared-memory broadcast
                float px = 0.f, py = 0.f, pz = 0.f;
#pragma unroll
                for (int I = 0; I < MAXC; ++I) {
                    if (I >= Bf) break;
                    slot_pair(rx[I], ry[I], rz[I], rj, DK_SLOT(slot0 + (k * Bf + I) * W + sub), e, hx[I], hy[I], hz[I],
                              px, py, pz);
                }
                px = gsum<W>(px, mask); py = gsum<W>(py, mask); pz = gsum<W>(pz, mask);
                if (sub == k) { fx += px; fy += py; fz += pz; }   // segment 0 holds the tail owners
            }
            slot0 += t * Bf * W;
        } else {
            for (int st = 0; st < tp; ++st) {
                const float4 rj = trow[(sl + st) & (tp - 1)];
#pragma unroll
                for (int I = 0; I < MAXC; ++I) {
                    if (I >= Bf) break;
                    const int q = slot0 + (st * Bf + I) * W + sub;
                    slot_pair(rx[I], ry[I], rz[I], rj, DK_SLOT(q), e, hx[I], hy[I], hz[I], fx, fy, fz);
                }
                const int src = (sl + 1) & (tp - 1);           // after the last step: back to the owner
                fx = __shfl_sync(mask, fx, src, tp);
                fy = __shfl_sync(mask, fy, src, tp);
                fz = __shfl_sync(mask, fz, src, tp);
            }
            slot0 += tp * Bf * W;
        }
        const float4 ro = trow[sl];
        for (int r = 0; r < rounds; ++r) {
            const int st = 1 + g + r * nseg;
            const int q = slot0 + r * W + sub;
            float px = 0.f, py = 0.f, pz = 0.f;
            slot_pair(ro.x, ro.y, ro.z, trow[(sl + st) & (tp - 1)], DK_SLOT(q), e, fx, fy, fz, px, py,
                      pz);
            const int src = (sl - st) & (tp - 1);              // lane m receives the force on m from m - st
            fx += __shfl_sync(mask, px, src, tp);
            fy += __shfl_sync(mask, py, src, tp);
            fz += __shfl_sync(mask, pz, src, tp);
        }
        for (int m = tp; m < W; m <<= 1) {
            fx += __shfl_xor_sync(mask, fx, m, W);
            fy += __shfl_xor_sync(mask, fy, m, W);
            fz += __shfl_xor_sync(mask, fz, m, W);
        }
#pragma unroll
        for (int c = 0; c < MAXC; ++c)
            if (c == Bf && sub < t) { hx[c] += fx; hy[c] += fy; hz[c] += fz; }
    } else if (t > 0 && !tail_rot) {
        for (int k = 0; k < t; ++k) {
            const int j = Bf * W + k;                       // uniform: shared-memory broadcast
            const float4 rj = S.r[ridx<W>(j)];
            const int sk = slot0 + k * (Bf + 1) * W + sub;
            float fx = 0.f, fy = 0.f, fz = 0.f;
#pragma unroll
            for (int I = 0; I < MAXC; ++I) {
                if (I > Bf) break;
                slot_pair(rx[I], ry[I], rz[I], rj, DK_SLOT(sk + I * W), e, hx[I], hy[I], hz[I],
                          fx, fy, fz);
            }
            fx = gsum<W>(fx, mask); fy = gsum<W>(fy, mask); fz = gsum<W>(fz, mask);
#pragma unroll
            for (int c = 0; c < MAXC; ++c)
                if (c == Bf && sub == k) { hx[c] += fx; hy[c] += fy; hz[c] += fz; }
        }
    }
#ifdef DK_PACK_ON
    if constexpr (PK) hb_side<W, MAXC>(L, S, sub, mask, hx, hy, hz, e);
#endif
    e_out += eacc_total(e);
#ifdef DK_PACK_ON
    if constexpr (PK) e_out += lean_total(e2);
#endif
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
        gx[c] = fmaf(2.0f, hx[c], gx[c]); gy[c] = fmaf(2.0f, hy[c], gy[c]); gz[c] = fmaf(2.0f, hz[c], gz[c]);
    }
}

// Energy-only pair tiles (large ligands whose pair list is not staged, L.energy_tiles):
// the same rotation and membership bits as intra_tiles, but no forces, so no partner
// accumulators and no shuffles.  The tail chunk is rotated too (no reductions to save).
// With KP > 1 the tile steps, linearised in (I, J, s) order, are split into KP contiguous
// parts and this lane group computes only part `part` (cooperative evaluation).
template <int W, int MAXC, int KP = 1>
__device__ __forceinline__ float intra_tiles_energy(const LigSm &L, const Scratch &S, int sub,
                                                    const float (&rx)[MAXC], const float (&ry)[MAXC],
                                                    const float (&rz)[MAXC], int part = 0) {
    const int N = L.N;
    const int Bt = L.NC;
    const int total = Bt * (W / 2) + (Bt * (Bt - 1) / 2) * W;
    const int g0 = (int)((long long)total * part / KP), g1 = (int)((long long)total * (part + 1) / KP);
    int base = 0;
    float e = 0.0f;
#pragma unroll
    for (int I = 0; I < MAXC; ++I) {
        if (I >= Bt) break;
        const int aI = I * W + sub;
        const bool okI = aI < N;
        const float4 po = L.ppar[ridx<W>(aI)];
        const float qi = okI ? sf_qscale(L) * S.r[ridx<W>(aI)].w : 0.0f;
        const float Ri = fabsf(po.x), ei = fabsf(po.y);
        const bool hbc = __float_as_int(po.x) < 0 || __float_as_int(po.y) < 0, don = __float_as_int(po.y) < 0;
#pragma unroll
        for (int J = I; J < MAXC; ++J) {
            if (J >= Bt) break;
            const int jb = J * W;
            uint32_t mw = okI ? (L.mask[aI * L.NW + (jb >> 5)] >> (jb & 31)) : 0u;
            uint32_t rot;
            if constexpr (W == 32) {
                rot = __funnelshift_r(mw, mw, sub);
            } else {
                mw &= 0xffffu;
                rot = ((mw | (mw << 16)) >> sub) & 0xffffu;
            }
            if (I == J && sub >= W / 2) rot &= ~(1u << (W / 2));
            const float4 *rrow = S.r + J * 2 * W + sub;
            const float4 *qrow = L.ppar + J * 2 * W + sub;
            const int s0 = (I == J) ? 1 : 0, n = (I == J) ? W / 2 : W;
            const int i0 = max(0, g0 - base), i1 = min(n, g1 - base);
            base += n;
#pragma unroll 4
            for (int st = s0 + i0; st < s0 + i1; ++st) {
                const float4 rj = rrow[st], pj = qrow[st];
                const float dx = rx[I] - rj.x, dy = ry[I] - rj.y, dz = rz[I] - rj.z;
                const float rho2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
                const float req = Ri + fabsf(pj.x), eps = ei * fabsf(pj.y);
                const bool hb = hbc && __float_as_int(don ? pj.x : pj.y) < 0;
                float A, B;
                sf_vdw_coeffs(L, hb, eps, A, B);
                const float E = pair_e_ab(rho2, sf_req(req), A, B, o_sv(po, pj), qi * rj.w);
                e += ((rot >> st) & 1u) ? E : 0.0f;
            }
        }
    }
    return e;
}

// Energy (and genotype gradient into S.grad) of the genotype in S.genes.
// Every lane of the group returns the same total energy.
// PARTS (microbenchmarks only, SURVEY.md §8(d) "isolating the two kernels for ncu"):
// bit 0 = intermolecular grid term (a4), bit 1 = intramolecular pairs (a5); the
// production kernels use both.
constexpr int kInter = 1, kIntra = 2, kAll = 3;

// KP > 1 (energy-only path): cooperative evaluation by KP lane groups; this group
// computes part `part` of the grid and pair sums and returns its PARTIAL energy (the
// caller adds the KP partials in a fixed order).  The pose is computed by every part.
template <int W, int MAXC, bool GRAD, int PARTS = kAll, int KP = 1, bool PK = false>
__device__ float eval_group(const LigSm &L, const GridDev &grid, const Scratch &S, int sub, unsigned mask,
                            int part = 0) {
    static_assert(KP == 1 || !GRAD, "cooperative evaluation is energy-only");
    const float *x = S.genes;
    // ---- a3: orientation quaternion q = (cos a/2, sin(a/2) n) -> R(q) (D3) ----
    float sph, cph, sth, cth, sa, ca;
    fast_sincos(x[3], sph, cph);
    fast_sincos(x[4], sth, cth);
    fast_sincos(0.5f * x[5], sa, ca);
    const float nx = sth * cph, ny = sth * sph, nz = cth;
    const float qw = ca, qx = sa * nx, qy = sa * ny, qz = sa * nz;
    const float R00 = 1.f - 2.f * (qy * qy + qz * qz), R01 = 2.f * (qx * qy - qw * qz), R02 = 2.f * (qx * qz + qw * qy);
    const float R10 = 2.f * (qx * qy + qw * qz), R11 = 1.f - 2.f * (qx * qx + qz * qz), R12 = 2.f * (qy * qz - qw * qx);
    const float R20 = 2.f * (qx * qz - qw * qy), R21 = 2.f * (qy * qz + qw * qx), R22 = 1.f - 2.f * (qx * qx + qy * qy);
    const float tx = x[0], ty = x[1], tz = x[2];

    // ---- a3: torsion composites A_k = L_a1 o ... o L_k (parents first; L_k =
    // Rot(u_k, tau_k) about A_k).  Lane k builds L_k; the chains are then collapsed by
    // pointer jumping (A_k <- A_anc(k) o A_k, anc <- anc(anc)) in ceil(log2(depth))
    // rounds instead of one round per tree level.  Each atom then applies its deepest
    // A_k and the root transform r = t + R(q) y.  One torsion per lane:
    // T <= N - 1 <= W (N <= 16 for W = 16; T <= 32 = W otherwise). ----
    {
        const int k = sub;
        const bool own = k < L.T;
        float m[12];
        int anc = -1;
        if (own) {
            float st, ct;
            fast_sincos(x[6 + k], st, ct);
            const float4 u = L.tU[k], A = L.tA[k];
            const float oc = 1.0f - ct;
            m[0] = fmaf(oc * u.x, u.x, ct);     m[1] = fmaf(oc * u.x, u.y, -st * u.z); m[2] = fmaf(oc * u.x, u.z, st * u.y);
            m[3] = fmaf(oc * u.y, u.x, st * u.z); m[4] = fmaf(oc * u.y, u.y, ct);    m[5] = fmaf(oc * u.y, u.z, -st * u.x);
            m[6] = fmaf(oc * u.z, u.x, -st * u.y); m[7] = fmaf(oc * u.z, u.y, st * u.x); m[8] = fmaf(oc * u.z, u.z, ct);
            m[9] = A.x - fmaf(m[0], A.x, fmaf(m[1], A.y, m[2] * A.z));
            m[10] = A.y - fmaf(m[3], A.x, fmaf(m[4], A.y, m[5] * A.z));
            m[11] = A.z - fmaf(m[6], A.x, fmaf(m[7], A.y, m[8] * A.z));
            anc = L.tmeta[k].x;
        }
        // (P o M) for affine P = rows p0..p2 (R|t) and M = m: new rows in place
#define DK_COMPOSE(p0, p1, p2)                                                                    \
    {                                                                                             \
        float o_[12];                                                                             \
        o_[0] = fmaf(p0.x, m[0], fmaf(p0.y, m[3], p0.z * m[6]));                                 \
        o_[1] = fmaf(p0.x, m[1], fmaf(p0.y, m[4], p0.z * m[7]));                                 \
        o_[2] = fmaf(p0.x, m[2], fmaf(p0.y, m[5], p0.z * m[8]));                                 \
        o_[9] = fmaf(p0.x, m[9], fmaf(p0.y, m[10], fmaf(p0.z, m[11], p0.w)));                    \
        o_[3] = fmaf(p1.x, m[0], fmaf(p1.y, m[3], p1.z * m[6]));                                 \
        o_[4] = fmaf(p1.x, m[1], fmaf(p1.y, m[4], p1.z * m[7]));                                 \
        o_[5] = fmaf(p1.x, m[2], fmaf(p1.y, m[5], p1.z * m[8]));                                 \
        o_[10] = fmaf(p1.x, m[9], fmaf(p1.y, m[10], fmaf(p1.z, m[11], p1.w)));                   \
        o_[6] = fmaf(p2.x, m[0], fmaf(p2.y, m[3], p2.z * m[6]));                                 \
        o_[7] = fmaf(p2.x, m[1], fmaf(p2.y, m[4], p2.z * m[7]));                                 \
        o_[8] = fmaf(p2.x, m[2], fmaf(p2.y, m[5], p2.z * m[8]));                                 \
        o_[11] = fmaf(p2.x, m[9], fmaf(p2.y, m[10], fmaf(p2.z, m[11], p2.w)));                   \
        _Pragma("unroll") for (int i_ = 0; i_ < 12; ++i_) m[i_] = o_[i_];                        \
    }
        // shallow trees (depth <= kWalkDepth): no composites at all -- each atom walks its
        // own ancestor chain below (fewer instructions on the latency-bound SW path)
        const int jump_levels = L.n_levels <= kWalkDepth ? 1 : L.n_levels;
        for (int span = 1; span < jump_levels; span *= 2) {
            if (own) {
                S.W[3 * k] = make_float4(m[0], m[1], m[2], m[9]);
                S.W[3 * k + 1] = make_float4(m[3], m[4], m[5], m[10]);
                S.W[3 * k + 2] = make_float4(m[6], m[7], m[8], m[11]);
                S.tp[k] = anc;
            }
            __syncwarp(mask);
            int nanc = anc;
            if (own && anc >= 0) {
                const float4 p0 = S.W[3 * anc], p1 = S.W[3 * anc + 1], p2 = S.W[3 * anc + 2];
                nanc = S.tp[anc];
                DK_COMPOSE(p0, p1, p2)
            }
            __syncwarp(mask);
            anc = nanc;
        }
        if (own) {   // A_k (torsion space); the root transform is applied per atom below
            S.W[3 * k] = make_float4(m[0], m[1], m[2], m[9]);
            S.W[3 * k + 1] = make_float4(m[3], m[4], m[5], m[10]);
            S.W[3 * k + 2] = make_float4(m[6], m[7], m[8], m[11]);
        }
#undef DK_COMPOSE
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
            float yx = p.x, yy = p.y, yz = p.z;            // y = A_deep p (torsions, D3)
            if (L.n_levels <= kWalkDepth) {
                // walk: y <- L_k y for k = deepest torsion, its parent, ..., the root child
                for (int k = deep; k >= 0; k = L.tmeta[k].x) {
                    const float4 w0 = S.W[3 * k], w1 = S.W[3 * k + 1], w2 = S.W[3 * k + 2];
                    const float nx_ = fmaf(w0.x, yx, fmaf(w0.y, yy, fmaf(w0.z, yz, w0.w)));
                    const float ny_ = fmaf(w1.x, yx, fmaf(w1.y, yy, fmaf(w1.z, yz, w1.w)));
                    const float nz_ = fmaf(w2.x, yx, fmaf(w2.y, yy, fmaf(w2.z, yz, w2.w)));
                    yx = nx_; yy = ny_; yz = nz_;
                }
            } else if (deep >= 0) {
                const float4 w0 = S.W[3 * deep], w1 = S.W[3 * deep + 1], w2 = S.W[3 * deep + 2];
                yx = fmaf(w0.x, p.x, fmaf(w0.y, p.y, fmaf(w0.z, p.z, w0.w)));
                yy = fmaf(w1.x, p.x, fmaf(w1.y, p.y, fmaf(w1.z, p.z, w1.w)));
                yz = fmaf(w2.x, p.x, fmaf(w2.y, p.y, fmaf(w2.z, p.z, w2.w)));
            }
            rx[c] = fmaf(R00, yx, fmaf(R01, yy, fmaf(R02, yz, tx)));   // r = t + R(q) y
            ry[c] = fmaf(R10, yx, fmaf(R11, yy, fmaf(R12, yz, ty)));
            rz[c] = fmaf(R20, yx, fmaf(R21, yy, fmaf(R22, yz, tz)));
            if (GRAD || L.energy_tiles) {
                const float4 rv = make_float4(rx[c], ry[c], rz[c], p.w);
                S.r[ridx<W>(a)] = rv;
                S.r[ridx<W>(a) + W] = rv;
            } else {
                S.r[a] = make_float4(rx[c], ry[c], rz[c], p.w);
            }
            if constexpr ((PARTS & kInter) != 0)
                if (KP == 1 || c % KP == part)
                    e_part += inter_atom(grid, meta & 0xff, p.w, rx[c], ry[c], rz[c], gx[c], gy[c], gz[c]);
        } else if ((GRAD || L.energy_tiles) && c < L.NC) {
            // padded chunk entries: finite zeros (null type, zero charge) for the tiles
            S.r[ridx<W>(a)] = make_float4(0.f, 0.f, 0.f, 0.f);
            S.r[ridx<W>(a) + W] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
    __syncwarp(mask);

    // ---- a5: intramolecular pairs ----
    if constexpr ((PARTS & kIntra) == 0) {
        if constexpr (GRAD) {
#pragma unroll
            for (int c = 0; c < MAXC; ++c) {   // keep the per-atom gradients live
                e_part += gx[c] + gy[c] + gz[c];
            }
        }
        return gsum<W>(e_part, mask);
    } else if constexpr (!GRAD) {
        // large ligand (pair list not staged): the tiles.  Only MAXC >= 4 (N > 96) can need
        // them -- N <= 96 gives P <= 4,560 pairs, 91 KB of list, under the 96 KB limit -- so
        // smaller instantiations do not carry this code (instruction-cache footprint of
        // the latency-bound SW kernels: measured 0.8x on PM when it was always compiled in).
        if constexpr (MAXC >= 4) {
            if (L.energy_tiles) {
                e_part += intra_tiles_energy<W, MAXC, KP>(L, S, sub, rx, ry, rz, part);
                return gsum<W>(e_part, mask);
            }
        }
#pragma unroll 4
        for (int q = sub + W * part; q < L.P; q += W * KP) {
            const uint32_t w = L.pairs[q];
            const float4 pp = L.pprm[q];
            const uint8_t *rb = reinterpret_cast<const uint8_t *>(S.r);
            const float4 ri = *reinterpret_cast<const float4 *>(rb + (w & 0xffffu));
            const float4 rj = *reinterpret_cast<const float4 *>(rb + (w >> 16));
            const float dx = ri.x - rj.x, dy = ri.y - rj.y, dz = ri.z - rj.z;
            e_part += pair_e_pre(fmaf(dx, dx, fmaf(dy, dy, dz * dz)), pp);
        }
        return gsum<W>(e_part, mask);
    } else {
        if (PK || L.slot_mode) intra_tiles_slots<W, MAXC, PK>(L, S, sub, mask, rx, ry, rz, gx, gy, gz, e_part);
        else intra_tiles<W, MAXC>(L, S, sub, mask, rx, ry, rz, gx, gy, gz, e_part);
        if constexpr (PK) {
        // the pose again from the group's rows (the same values): the packed tiles need not
        // keep the scalar pose registers alive (they work on 64-bit register pairs)
#pragma unroll
        for (int c = 0; c < MAXC; ++c) {
            const int a = sub + W * c;
            if (a < L.N) {
                const float4 rv = S.r[ridx<W>(a)];
                rx[c] = rv.x; ry[c] = rv.y; rz[c] = rv.z;
            }
        }
        }
        if constexpr (PARTS == kIntra) {
            const float E = gsum<W>(e_part, mask);
#pragma unroll
            for (int c = 0; c < MAXC; ++c) e_part += gx[c] + gy[c] + gz[c];
            return E + 0.0f * gsum<W>(e_part, mask);
        }
        const float E = gsum<W>(e_part, mask);

        // ---- a6: back-projection to genotype space (D7) ----
        float sgx = 0.f, sgy = 0.f, sgz = 0.f, Gx = 0.f, Gy = 0.f, Gz = 0.f;
#pragma unroll
        for (int c = 0; c < MAXC; ++c) {
            const int a = sub + W * c;
            if (a < L.N) {
                const float dx = rx[c] - tx, dy = ry[c] - ty, dz = rz[c] - tz;
                const float cxp = fmaf(dy, gz[c], -dz * gy[c]), cyp = fmaf(dz, gx[c], -dx * gz[c]),
                            czp = fmaf(dx, gy[c], -dy * gx[c]);
                sgx += gx[c]; sgy += gy[c]; sgz += gz[c];
                Gx += cxp; Gy += cyp; Gz += czp;
                S.ts[2 * a] = make_float4(cxp, cyp, czp, 0.f);
                S.ts[2 * a + 1] = make_float4(gx[c], gy[c], gz[c], 0.f);
            }
        }
#if DK_BP_T
        if constexpr (W == 32) {
            // the six sums by one transposed reduction (12 shuffles instead of 30): level 16
            // leaves sum(g) in the low half-warp and sum((r - t) x g) in the high one, level 8
            // keeps two components in the lanes with bit 3 clear and the third in the others,
            // level 4 splits the two; levels 2, 1 finish.  Totals: sgx at lane 0, sgy at 4,
            // sgz at 8, Gx at 16, Gy at 20, Gz at 24; lanes 0..5 (below) fetch what they use.
            const bool b4 = (sub & 16) != 0, b3 = (sub & 8) != 0, b2 = (sub & 4) != 0;
            float k0 = b4 ? Gx : sgx, k1 = b4 ? Gy : sgy, k2 = b4 ? Gz : sgz;
            k0 += __shfl_xor_sync(mask, b4 ? sgx : Gx, 16);
            k1 += __shfl_xor_sync(mask, b4 ? sgy : Gy, 16);
            k2 += __shfl_xor_sync(mask, b4 ? sgz : Gz, 16);
            const float rA = __shfl_xor_sync(mask, b3 ? k0 : k2, 8), rB = __shfl_xor_sync(mask, k1, 8);
            if (b3) { k2 += rA; } else { k0 += rA; k1 += rB; }
            float v = b3 ? k2 : (b2 ? k1 : k0);
            v += __shfl_xor_sync(mask, b3 ? k2 : (b2 ? k0 : k1), 4);
            v += __shfl_xor_sync(mask, v, 2);
            v += __shfl_xor_sync(mask, v, 1);
            const float own = __shfl_sync(mask, v, sub == 1 ? 4 : (sub == 2 ? 8 : 0));
            Gx = __shfl_sync(mask, v, 16); Gy = __shfl_sync(mask, v, 20); Gz = __shfl_sync(mask, v, 24);
            sgx = sgy = sgz = own;                      // lane 0: sgx, lane 1: sgy, lane 2: sgz
        } else
#endif
        {
            sgx = gsum<W>(sgx, mask); sgy = gsum<W>(sgy, mask); sgz = gsum<W>(sgz, mask);
            Gx = gsum<W>(Gx, mask); Gy = gsum<W>(Gy, mask); Gz = gsum<W>(Gz, mask);
        }
        __syncwarp(mask);
        // torsions: dE/dtau_k = w_k . sum_{a in moved(k)} (r_a - r_{a_k}) x g_a.  The moved
        // set is one DFS range [lo, hi).  Each torsion gets an aligned block of lpt lanes, a
        // power of two sized to its range length by the host (prep.cpp, L.tlane: buddy
        // allocation that minimises the longest walk), strided over the range, then a
        // butterfly inside the block (levels up to the largest block only, L.tlane_lv).
        {
            const int T = L.T;
            const int tl = L.tlane[sub];                    // k | lane in block << 8 | log2(lpt) << 16
            const int lpt = 1 << (tl >> 16), k = tl & 0xff, sl = (tl >> 8) & 0xff;
            const bool own = k < T;
            float cx = 0.f, cy = 0.f, cz = 0.f, hx = 0.f, hy = 0.f, hz = 0.f;
            int4 tm = make_int4(0, 0, 0, 0);
            if (own) {
                tm = L.tmeta[k];
                const int lo = tm.w & 0xffff, hi = tm.w >> 16;
                constexpr int kWalkUnroll = DK_WALK_UNROLL ? DK_WALK_UNROLL : (MAXC >= 3 ? 2 : 1);
#pragma unroll kWalkUnroll
                for (int a = lo + sl; a < hi; a += lpt) {
                    const float4 c4 = S.ts[2 * a], g4 = S.ts[2 * a + 1];
                    cx += c4.x; cy += c4.y; cz += c4.z;
                    hx += g4.x; hy += g4.y; hz += g4.z;
                }
            }
            for (int m = L.tlane_top; m >= 1; m >>= 1) {   // fixed-order block butterfly (uniform levels)
                const float ox = __shfl_xor_sync(mask, cx, m, W), oy = __shfl_xor_sync(mask, cy, m, W);
                const float oz = __shfl_xor_sync(mask, cz, m, W), ogx = __shfl_xor_sync(mask, hx, m, W);
                const float ogy = __shfl_xor_sync(mask, hy, m, W), ogz = __shfl_xor_sync(mask, hz, m, W);
                if (m < lpt) { cx += ox; cy += oy; cz += oz; hx += ogx; hy += ogy; hz += ogz; }
            }
            if (own && sl == 0) {
                const float4 ra = S.r[ridx<W>(tm.y)], rb = S.r[ridx<W>(tm.z)];
                const float dax = ra.x - tx, day = ra.y - ty, daz = ra.z - tz;
                const float sx = cx - (day * hz - daz * hy), sy = cy - (daz * hx - dax * hz), sz = cz - (dax * hy - day * hx);
                const float wx = rb.x - ra.x, wy = rb.y - ra.y, wz = rb.z - ra.z;
                const float inw = rsqrtf(wx * wx + wy * wy + wz * wz);
                S.grad[6 + k] = (wx * sx + wy * sy + wz * sz) * inw;
            }
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

}  // namespace DK_SF_NS
}  // namespace dk
