// cluster.cu — NEXT-3: clustering of per-run best poses on the device (DESIGN.md §12,
// reading D12: AutoDock's cluster analysis, plain RMSD in the receptor frame).
//
// One CTA does the whole job, because the greedy assignment is a sequence: poses are
// visited in ascending energy order and each joins the lowest-numbered existing cluster
// whose seed lies within rmsd_tol, else seeds a new cluster.  The parallel parts are the
// energy ranks (one thread per pose, O(n) comparisons each) and, per visited pose, the
// RMSDs to every existing seed (one warp per seed, lanes over coordinates, squared
// differences accumulated in FP64 so the threshold decision matches an FP64 reference
// up to summation order).
#include <cuda_runtime.h>
#include <stdint.h>

#include <climits>

#include "cluster.cuh"

namespace dk {

namespace {

constexpr int kClusterThreads = 256;

__device__ __forceinline__ float cl_key(float e) { return isnan(e) ? INFINITY : e; }

__global__ void __launch_bounds__(kClusterThreads) k_cluster(int n, int N, const float *__restrict__ xyz,
                                                              const float *__restrict__ E, float tol, int *cluster,
                                                              float *rmsd_out, int *rank_out, int *n_clusters) {
    extern __shared__ uint8_t cl_smem[];
    int *order = reinterpret_cast<int *>(cl_smem);               // [n] pose of energy rank t
    int *seed = order + n;                                       // [n] seed pose of cluster c
    double *rs = reinterpret_cast<double *>(seed + n);          // [n] RMSD to seed c (byte 8n: aligned)
    __shared__ int s_nc, s_hit;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    // energy ranks: (key, index) order, NaN = +inf, ties -> lower index
    for (int i = tid; i < n; i += blockDim.x) {
        const float ki = cl_key(E[i]);
        int r = 0;
        for (int j = 0; j < n; ++j) {
            const float kj = cl_key(E[j]);
            r += (kj < ki || (kj == ki && j < i)) ? 1 : 0;
        }
        order[r] = i;
        if (rank_out) rank_out[i] = r;
    }
    if (tid == 0) s_nc = 0;
    __syncthreads();
    const int M = 3 * N;
    for (int t = 0; t < n; ++t) {
        const int k = order[t];
        const int nc = s_nc;
        if (tid == 0) s_hit = INT_MAX;
        __syncthreads();
        const float *xk = xyz + (size_t)k * M;
        for (int c = warp; c < nc; c += nwarps) {
            const float *xs = xyz + (size_t)seed[c] * M;
            double s = 0.0;
            for (int m = lane; m < M; m += 32) {
                const double d = (double)xk[m] - (double)xs[m];
                s = fma(d, d, s);
            }
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            const double r = sqrt(s / (double)N);
            if (lane == 0) {
                rs[c] = r;
                if (r < (double)tol) atomicMin(&s_hit, c);
            }
        }
        __syncthreads();
        if (tid == 0) {
            int c = s_hit;
            double r = 0.0;
            if (c == INT_MAX) { c = nc; seed[nc] = k; s_nc = nc + 1; }
            else r = rs[c];
            cluster[k] = c;
            rmsd_out[k] = (float)r;
        }
        __syncthreads();
    }
    if (tid == 0) *n_clusters = s_nc;
}

}  // namespace

size_t cluster_smem_bytes(int n) { return (size_t)16 * n; }

cudaError_t launch_cluster(int n, int N, const float *xyz, const float *E, float tol, int *cluster, float *rmsd,
                           int *rank, int *n_clusters, cudaStream_t s) {
    const size_t smem = cluster_smem_bytes(n);
    cudaError_t e = cudaFuncSetAttribute(k_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_cluster<<<1, kClusterThreads, smem, s>>>(n, N, xyz, E, tol, cluster, rmsd, rank, n_clusters);
    return cudaGetLastError();
}

}  // namespace dk
