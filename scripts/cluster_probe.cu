// Max co-resident clusters for cluster sizes 8 / 16 at the block shapes a
// cluster-resident 256^2 task would use (cudaOccupancyMaxActiveClusters), and
// the measured time of an empty cluster barrier loop.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void probe_kernel(int iters, long long* out) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  }
  if (threadIdx.x == 0 && cl.block_rank() == 0) out[blockIdx.x / cl.num_blocks()] = clock64() - t0;
  sm[threadIdx.x] = 0;
}
int main() {
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  long long* d;
  cudaMalloc(&d, 1 << 20);
  int cs_list[] = {8, 16};
  int th_list[] = {512, 1024};
  size_t sm_list[] = {100 * 1024, 200 * 1024};
  for (int cs : cs_list)
    for (int th : th_list)
      for (size_t smb : sm_list) {
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(cs * 64);
        lc.blockDim = dim3(th);
        lc.dynamicSmemBytes = smb;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        int n = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, probe_kernel, &lc);
        float ms = -1;
        if (e == cudaSuccess && n > 0) {
          cudaEvent_t a, b;
          cudaEventCreate(&a);
          cudaEventCreate(&b);
          cudaLaunchKernelEx(&lc, probe_kernel, 1000, d);
          cudaEventRecord(a);
          cudaLaunchKernelEx(&lc, probe_kernel, 1000, d);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          cudaEventElapsedTime(&ms, a, b);
        }
        long long cyc = 0;
        cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
        printf("cluster %2d threads %4d smem %3zu KB: max active clusters %d (%s); 64 clusters x 1000 barriers %.3f ms, %.0f cycles/barrier\n",
               cs, th, smb / 1024, n, cudaGetErrorString(e), ms, cyc / 1000.0);
      }
  return 0;
}
