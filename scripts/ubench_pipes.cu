// ubench_pipes.cu — per-SM issue throughput of the instruction classes the pair loop uses
// (FFMA 3-reg, FFMA2 packed f32x2, FMUL, FADD2, MUFU rcp/ex2, SHFL, LDS.128, FSEL/FMNMX).
// Scratch evidence for DESIGN.md §17 (packed FP32x2 pair arithmetic); not product code.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench scripts/ubench_pipes.cu && /tmp/ubench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b) { u64 r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float lo(u64 v) { float a, b; asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); return a + b; }
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) { u64 d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ u64 mul2(u64 a, u64 b) { u64 d; asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ u64 add2(u64 a, u64 b) { u64 d; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ float ffma(float a, float b, float c) { float d; asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d; }
__device__ __forceinline__ float fmul(float a, float b) { float d; asm volatile("mul.rn.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b)); return d; }
__device__ __forceinline__ float rcp(float a) { float d; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(d) : "f"(a)); return d; }
__device__ __forceinline__ float ex2(float a) { float d; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(d) : "f"(a)); return d; }
__device__ __forceinline__ float fmx(float a, float b) { float d; asm volatile("max.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b)); return d; }

constexpr int K = 8;      // independent chains per thread
constexpr int ITER = 4096;

template <int OP>
__global__ void kern(float *out, float s, int iters) {
    __shared__ float4 sm[1024];
    float v[K];
    u64 w[K];
    for (int k = 0; k < K; ++k) { v[k] = threadIdx.x * 1e-3f + k; w[k] = pk(v[k], v[k] + 1.f); }
    const u64 a2 = pk(s, 1.0001f * s), b2 = pk(0.999f, 1.0001f);
    if (OP == 6) for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = make_float4(i, i, i, i);
    __syncthreads();
    float4 acc = make_float4(0, 0, 0, 0);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            if (OP == 0) v[k] = ffma(v[k], s, 0.5f + k);                // FFMA imm-ish
            else if (OP == 1) v[k] = ffma(v[k], s, v[(k + 1) % K]);      // FFMA 3-reg
            else if (OP == 2) w[k] = fma2(w[k], a2, b2);                 // FFMA2
            else if (OP == 3) w[k] = mul2(w[k], a2);                     // FMUL2
            else if (OP == 4) v[k] = rcp(v[k]);                          // MUFU.RCP
            else if (OP == 5) v[k] = __shfl_sync(0xffffffffu, v[k], (threadIdx.x + 1) & 31);   // SHFL
            else if (OP == 6) { const float4 t = sm[(threadIdx.x + 32 * k + i) & 1023]; acc.x += t.x; acc.y += t.y; acc.z += t.z; acc.w += t.w; }
            else if (OP == 7) v[k] = fmx(v[k], s);                       // FMNMX
            else if (OP == 8) w[k] = add2(w[k], a2);                     // FADD2
            else if (OP == 9) v[k] = fmul(v[k], s);                      // FMUL
            else if (OP == 10) v[k] = ex2(v[k]);                         // MUFU.EX2
        }
    }
    float r = acc.x + acc.y + acc.z + acc.w;
    for (int k = 0; k < K; ++k) r += v[k] + lo(w[k]);
    if (r == 1234.5f) out[threadIdx.x] = r;
}

int main() {
    float *o;
    cudaMalloc(&o, 4096);
    int dev = 0, sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    const char *names[] = {"FFMA(imm c)", "FFMA 3-reg", "FFMA2", "FMUL2", "MUFU.RCP", "SHFL", "LDS.128(+4 FADD)",
                           "FMNMX", "FADD2", "FMUL", "MUFU.EX2"};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int warps : {8, 16, 32}) {
        const int blocks = sms * (warps / 8), threads = 256;
        for (int op = 0; op < 11; ++op) {
            auto launch = [&](int it) {
                switch (op) {
                case 0: kern<0><<<blocks, threads>>>(o, 1.0001f, it); break;
                case 1: kern<1><<<blocks, threads>>>(o, 1.0001f, it); break;
                case 2: kern<2><<<blocks, threads>>>(o, 1.0001f, it); break;
                case 3: kern<3><<<blocks, threads>>>(o, 1.0001f, it); break;
                case 4: kern<4><<<blocks, threads>>>(o, 1.0001f, it); break;
                case 5: kern<5><<<blocks, threads>>>(o, 1.0001f, it); break;
                case 6: kern<6><<<blocks, threads>>>(o, 1.0001f, it); break;
                case 7: kern<7><<<blocks, threads>>>(o, 1.0001f, it); break;
                case 8: kern<8><<<blocks, threads>>>(o, 1.0001f, it); break;
                case 9: kern<9><<<blocks, threads>>>(o, 1.0001f, it); break;
                case 10: kern<10><<<blocks, threads>>>(o, 1.0001f, it); break;
                }
            };
            launch(64);
            cudaDeviceSynchronize();
            cudaEventRecord(e0);
            launch(ITER);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            const double winstr = (double)blocks * (threads / 32) * ITER * K;   // warp instructions of the op
            const double per_sm_per_ns = winstr / sms / (ms * 1e6);
            // at the max clock: warp-instr per SM-cycle
            printf("warps/SM %2d  %-18s %8.3f ms  %6.3f warp-instr/SM/ns  (%5.2f per SM-cycle at %d MHz)\n", warps,
                   names[op], ms, per_sm_per_ns, per_sm_per_ns / (clk / 1e6), clk / 1000);
        }
    }
    cudaError_t err = cudaGetLastError();
    printf("status %s\n", cudaGetErrorString(err));
    return 0;
}
