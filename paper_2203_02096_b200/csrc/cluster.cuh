// cluster.cuh — launcher of the NEXT-3 pose-clustering kernel (cluster.cu).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

namespace dk {

constexpr int kClusterMaxPoses = 4096;   // shared memory: 16 B per pose

size_t cluster_smem_bytes(int n);
// Device arrays: xyz [n][N][3], E [n] -> cluster [n], rmsd [n], rank [n] (may be null),
// n_clusters [1].  One CTA; n <= kClusterMaxPoses.
cudaError_t launch_cluster(int n, int N, const float *xyz, const float *E, float tol, int *cluster, float *rmsd,
                           int *rank, int *n_clusters, cudaStream_t s);

}  // namespace dk
