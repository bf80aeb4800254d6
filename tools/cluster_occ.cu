// Max co-resident clusters for a kernel shaped like attn_tma_kernel (64 threads, ~54 KB dynamic
// smem, 4 CTAs/SM by launch bounds) at cluster sizes 1..8 (tools only).
// nvcc -gencode arch=compute_100a,code=sm_100a -o tools/cluster_occ tools/cluster_occ.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(64, 4) k(float* p) {
  extern __shared__ float s[];
  s[threadIdx.x] = p[threadIdx.x];
  __syncthreads();
  p[threadIdx.x] = s[63 - threadIdx.x];
}
int main() {
  int smem = 54336;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs = 1; cs <= 16; cs *= 2) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(512);
    cfg.blockDim = dim3(64);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (void*)k, &cfg);
    printf("cluster %2d: max active clusters %d (= %d CTAs) %s\n", cs, n, n * cs, cudaGetErrorString(e));
  }
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, 64, smem);
  printf("blocks per SM without clusters: %d\n", nb);
}
