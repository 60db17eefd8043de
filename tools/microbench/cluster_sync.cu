// Latency of one round of the Jacobi SVD's inter-CTA synchronisation on a 16-CTA cluster:
// (a) cluster.sync(), (b) neighbour-only flags (remote st.release.cluster of a round
// counter into the two neighbours' shared memory + __syncthreads + acquire spin).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cluster_sync cluster_sync.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void __cluster_dims__(1, 1, 1) dummy() {}

__global__ void k_cluster(int rounds, long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) cl.sync();
  long long t1 = clock64();
  if (threadIdx.x == 0 && cl.block_rank() == 0) out[0] = t1 - t0;
}

__global__ void k_flags(int rounds, long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ int flag[2];  // [0] from the left neighbour, [1] from the right
  __shared__ double buf[64];
  const int rank = (int)cl.block_rank(), n = (int)cl.num_blocks();
  if (threadIdx.x < 2) flag[threadIdx.x] = 0;
  cl.sync();
  int* lf = rank > 0 ? cl.map_shared_rank(&flag[1], rank - 1) : nullptr;      // I am their right
  int* rf = rank < n - 1 ? cl.map_shared_rank(&flag[0], rank + 1) : nullptr;  // I am their left
  double* lb = rank > 0 ? cl.map_shared_rank(buf, rank - 1) : nullptr;
  double* rb = rank < n - 1 ? cl.map_shared_rank(buf, rank + 1) : nullptr;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  long long t0 = clock64();
  for (int r = 1; r <= rounds; ++r) {
    // edge warps: a column slice to the neighbour, then its round counter
    if (warp == 0 && lb) {
      lb[lane] = r;
      __syncwarp();
      if (lane == 0) asm volatile("st.release.cluster.shared::cluster.u32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(lf)), "r"(r) : "memory");
    }
    if (warp == nw - 1 && rb) {
      rb[32 + lane] = r;
      __syncwarp();
      if (lane == 0) asm volatile("st.release.cluster.shared::cluster.u32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(rf)), "r"(r) : "memory");
    }
    if (threadIdx.x < 2 && ((threadIdx.x == 0 && rank > 0) || (threadIdx.x == 1 && rank < n - 1))) {
      int v;
      do {
        asm volatile("ld.acquire.cluster.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(&flag[threadIdx.x])) : "memory");
      } while (v < r);
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && rank == 0) out[0] = t1 - t0;
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  const int rounds = 20000;
  for (int mode = 0; mode < 2; ++mode) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16);
    cfg.blockDim = dim3(256);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 16;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (mode == 0) {
      cudaFuncSetAttribute(k_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaLaunchKernelEx(&cfg, k_cluster, rounds, d);
    } else {
      cudaFuncSetAttribute(k_flags, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaLaunchKernelEx(&cfg, k_flags, rounds, d);
    }
    long long h = 0;
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%s: %.1f cycles per round (%s)\n", mode == 0 ? "cluster.sync (16 CTAs)" : "neighbour flags + __syncthreads",
           double(h) / rounds, cudaGetErrorString(e));
  }
  return 0;
}
