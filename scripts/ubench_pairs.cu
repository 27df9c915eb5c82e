// ubench_pairs.cu — the gradient pair-tile inner loop (row a5) in isolation:
// one individual per lane group (scalar FP32, the round-1 slot_pair) against two
// individuals per lane group with packed FP32x2 arithmetic (FFMA2 / FADD2 / FMUL2, sm_100).
// Both run W = 32 rotation tiles of 32 steps with per-slot constants and partner poses in
// shared memory and the partner force accumulator travelling by shuffles.  Scratch
// evidence for DESIGN.md §17; not product code.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubp scripts/ubench_pairs.cu && /tmp/ubp
#include <cstdio>
#include <cuda_runtime.h>

typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b) { u64 r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float lo(u64 v) { float a, b; asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); return a; }
__device__ __forceinline__ float hi(u64 v) { float a, b; asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); return b; }
__device__ __forceinline__ u64 add2(u64 a, u64 b) { u64 d; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ u64 sub2(u64 a, u64 b) { u64 d; asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ u64 mul2(u64 a, u64 b) { u64 d; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) { u64 d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ u64 bc(float a) { return pk(a, a); }
__device__ __forceinline__ float rcpa(float x) { float y; asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float ex2a(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

constexpr float kExpScale = -(1.0f / (2.0f * 3.6f * 3.6f)) * 1.4426950408889634f;
constexpr float kInv2s2 = 1.0f / (2.0f * 3.6f * 3.6f);
constexpr int W = 32, STEPS = 32, TILES = 2;

// scalar: the round-1 slot_pair with r_eq folded into the constants {A' = A r_eq^12,
// B' = |B| r_eq^n (sign: 12-10), SV, qq}
__global__ void __launch_bounds__(256, 2) k_scalar(const float4 *gpos, const float4 *gcon, float *out, int reps) {
    __shared__ float4 pos[8][2 * W];
    __shared__ float4 con[TILES * STEPS * W];
    const int g = threadIdx.x / W, l = threadIdx.x % W;
    for (int i = threadIdx.x; i < TILES * STEPS * W; i += blockDim.x) con[i] = gcon[i];
    for (int i = l; i < 2 * W; i += W) pos[g][i] = gpos[(blockIdx.x * 8 + g) * 2 * W + i];
    __syncthreads();
    float rx = pos[g][l].x + 0.37f, ry = pos[g][l].y - 0.21f, rz = pos[g][l].z + 0.11f;
    float e = 0.f, gx = 0.f, gy = 0.f, gz = 0.f;
    for (int r = 0; r < reps; ++r)
        for (int t = 0; t < TILES; ++t) {
            float fx = 0.f, fy = 0.f, fz = 0.f;
            const float4 *rrow = &pos[g][l];
            const float4 *crow = &con[t * STEPS * W + l];
#pragma unroll 4
            for (int s = 0; s < STEPS; ++s) {
                const float4 rj = rrow[s], c = crow[s * W];
                const float dx = rx - rj.x, dy = ry - rj.y, dz = rz - rj.z;
                float rho2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
                const bool clamped = rho2 < 1e-4f;
                rho2 = fmaxf(rho2, 1e-4f);
                const float inv = rcpa(rho2), i2 = inv * inv, i3 = i2 * inv, i6 = i3 * i3;
                const bool ten = __float_as_int(c.y) < 0;
                const float xn = ten ? i3 * i2 : i3;
                const float tA = c.x * i6, tB = fabsf(c.y) * xn;
                const float dvr = fmaf(-6.0f, tA, (ten ? 5.0f : 3.0f) * tB);
                const float Eel = c.w * inv, Eds = c.z * ex2a(rho2 * kExpScale);
                const float d = fmaf(dvr - Eel, inv, -Eds * kInv2s2);
                const float dE = clamped ? 0.f : d;
                e += (tA - tB) + Eel + Eds;
                gx = fmaf(dE, dx, gx); gy = fmaf(dE, dy, gy); gz = fmaf(dE, dz, gz);
                fx = fmaf(-dE, dx, fx); fy = fmaf(-dE, dy, fy); fz = fmaf(-dE, dz, fz);
                const int src = (l + 1) & (W - 1);
                fx = __shfl_sync(0xffffffffu, fx, src); fy = __shfl_sync(0xffffffffu, fy, src);
                fz = __shfl_sync(0xffffffffu, fz, src);
            }
            gx += fx; gy += fy; gz += fz;
        }
    out[blockIdx.x * blockDim.x + threadIdx.x] = e + gx + gy + gz;
}

// packed: two individuals A, B per lane group.  Partner poses interleaved
// {xA, xB, yA, yB} + {zA, zB} so one LDS.128 + one LDS.64 load both; constants shared.
__global__ void __launch_bounds__(256, 2) k_packed(const float4 *gpos, const float4 *gcon, float *out, int reps) {
    __shared__ float4 pxy[8][2 * W];
    __shared__ float2 pz[8][2 * W];
    __shared__ float4 con[TILES * STEPS * W];
    const int g = threadIdx.x / W, l = threadIdx.x % W;
    for (int i = threadIdx.x; i < TILES * STEPS * W; i += blockDim.x) con[i] = gcon[i];
    for (int i = l; i < 2 * W; i += W) {
        const float4 a = gpos[(blockIdx.x * 16 + 2 * g) * 2 * W + i], b = gpos[(blockIdx.x * 16 + 2 * g + 1) * 2 * W + i];
        pxy[g][i] = make_float4(a.x, b.x, a.y, b.y);
        pz[g][i] = make_float2(a.z, b.z);
    }
    __syncthreads();
    const u64 rx = add2(pk(pxy[g][l].x, pxy[g][l].y), bc(0.37f)), ry = add2(pk(pxy[g][l].z, pxy[g][l].w), bc(-0.21f));
    const u64 rz = add2(pk(pz[g][l].x, pz[g][l].y), bc(0.11f));
    u64 e = bc(0.f), gx = bc(0.f), gy = bc(0.f), gz = bc(0.f);
    for (int r = 0; r < reps; ++r)
        for (int t = 0; t < TILES; ++t) {
            u64 fx = bc(0.f), fy = bc(0.f), fz = bc(0.f);
            const float4 *xyrow = &pxy[g][l];
            const float2 *zrow = &pz[g][l];
            const float4 *crow = &con[t * STEPS * W + l];
#pragma unroll 4
            for (int s = 0; s < STEPS; ++s) {
                const float4 xy = xyrow[s];
                const float2 zz = zrow[s];
                const float4 c = crow[s * W];
                const u64 dx = sub2(rx, pk(xy.x, xy.y)), dy = sub2(ry, pk(xy.z, xy.w)), dz = sub2(rz, pk(zz.x, zz.y));
                u64 rho2 = fma2(dx, dx, fma2(dy, dy, mul2(dz, dz)));
                const float r0 = fmaxf(lo(rho2), 1e-4f), r1 = fmaxf(hi(rho2), 1e-4f);
                const float cl0 = lo(rho2) < 1e-4f ? 0.f : 1.f, cl1 = hi(rho2) < 1e-4f ? 0.f : 1.f;
                const u64 inv = pk(rcpa(r0), rcpa(r1));
                const u64 i2 = mul2(inv, inv), i3 = mul2(i2, inv), i6 = mul2(i3, i3);
                const bool ten = __float_as_int(c.y) < 0;
                const u64 xn = ten ? mul2(i3, i2) : i3;
                const u64 tA = mul2(bc(c.x), i6), tB = mul2(bc(fabsf(c.y)), xn);
                const u64 dvr = fma2(bc(-6.0f), tA, mul2(bc(ten ? 5.0f : 3.0f), tB));
                const u64 Eel = mul2(bc(c.w), inv);
                const u64 Eds = mul2(bc(c.z), pk(ex2a(r0 * kExpScale), ex2a(r1 * kExpScale)));
                u64 d = fma2(sub2(dvr, Eel), inv, mul2(Eds, bc(-kInv2s2)));
                d = mul2(d, pk(cl0, cl1));
                e = add2(e, add2(sub2(tA, tB), add2(Eel, Eds)));
                gx = fma2(d, dx, gx); gy = fma2(d, dy, gy); gz = fma2(d, dz, gz);
                fx = fma2(d, dx, fx); fy = fma2(d, dy, fy); fz = fma2(d, dz, fz);     // partner: subtracted at the end
                const int src = (l + 1) & (W - 1);
                fx = pk(__shfl_sync(0xffffffffu, lo(fx), src), __shfl_sync(0xffffffffu, hi(fx), src));
                fy = pk(__shfl_sync(0xffffffffu, lo(fy), src), __shfl_sync(0xffffffffu, hi(fy), src));
                fz = pk(__shfl_sync(0xffffffffu, lo(fz), src), __shfl_sync(0xffffffffu, hi(fz), src));
            }
            gx = sub2(gx, fx); gy = sub2(gy, fy); gz = sub2(gz, fz);
        }
    out[blockIdx.x * blockDim.x + threadIdx.x] = lo(e) + hi(e) + lo(gx) + hi(gy) + lo(gz);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 2 * 8;   // 8 waves of 2 CTAs/SM
    const int npos = blocks * 16 * 2 * W;
    float4 *hpos = new float4[npos], *hcon = new float4[TILES * STEPS * W];
    unsigned s = 12345;
    auto rnd = [&]() { s = s * 1664525u + 1013904223u; return (s >> 8) * (1.0f / 16777216.0f); };
    for (int i = 0; i < npos; ++i) hpos[i] = make_float4(10 * rnd(), 10 * rnd(), 10 * rnd(), rnd() - 0.5f);
    for (int i = 0; i < TILES * STEPS * W; ++i)
        hcon[i] = make_float4(2e6f * rnd(), (rnd() < 0.05f ? -1.f : 1.f) * 3e3f * rnd(), -0.05f * rnd(), 80.f * (rnd() - 0.5f));
    float4 *dpos, *dcon; float *dout;
    cudaMalloc(&dpos, npos * 16); cudaMalloc(&dcon, TILES * STEPS * W * 16); cudaMalloc(&dout, blocks * 256 * 4);
    cudaMemcpy(dpos, hpos, npos * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(dcon, hcon, TILES * STEPS * W * 16, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int reps = 160;
    for (int v = 0; v < 2; ++v) {
        for (int w = 0; w < 2; ++w) {
            if (v == 0) k_scalar<<<blocks, 256>>>(dpos, dcon, dout, 2); else k_packed<<<blocks / 2, 256>>>(dpos, dcon, dout, 2);
        }
        cudaEventRecord(e0);
        if (v == 0) k_scalar<<<blocks, 256>>>(dpos, dcon, dout, reps); else k_packed<<<blocks / 2, 256>>>(dpos, dcon, dout, reps);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double pairs = (double)blocks * 8 * W * reps * TILES * STEPS;   // pair-individuals
        printf("%s: %.3f ms  %.3e pair-individuals/s\n", v == 0 ? "scalar (1 ind/group)" : "packed f32x2 (2 ind/group)", ms,
               pairs / (ms * 1e-3));
    }
    printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
