// Co-resident cluster counts for a 1-CTA-per-SM kernel (200 KB shared memory) at
// cluster sizes 1/2/4/8 on this GPU.  nvcc -gencode arch=compute_100a,code=sm_100a -o tools/_build/occ_probe tools/occ_probe.cu
#include <cstdio>
__global__ void k(int* p) { extern __shared__ int s[]; if (p) p[0] = s[0]; }
int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cl : {1, 2, 4, 8}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cl * 64); cfg.blockDim = dim3(384); cfg.dynamicSmemBytes = 200 * 1024;
    cudaLaunchAttribute attr[1]; attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cl; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr; cfg.numAttrs = 1;
    int n = 0; cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
    printf("cluster %d: max active clusters %d -> %d SMs busy (%s)\n", cl, n, n * cl, cudaGetErrorString(e));
  }
}
