// Cluster-barrier latency microbenchmark (design input for the resident
// engine): cycles per barrier.cluster.arrive + wait round for cluster sizes
// 1..16, with and without a __syncthreads and a DSMEM store per round.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/cluster_bar tools/cluster_bar.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void bar_kernel(int iters, int mode, unsigned long long* out) {
  __shared__ unsigned buf[64];
  unsigned rank, n;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(n));
  const unsigned local = static_cast<unsigned>(__cvta_generic_to_shared(buf + (threadIdx.x & 63)));
  unsigned remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"((rank + 1) % n));
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (mode & 1) __syncthreads();
    if ((mode & 2) && threadIdx.x < 64) asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(remote), "r"(i) : "memory");
    if (mode & 4) {
      asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
    } else {
      asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    }
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0 && rank == 0) out[0] = t1 - t0;
}

int main() {
  cudaFuncSetAttribute(bar_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  unsigned long long* d;
  cudaMalloc(&d, 8);
  const int iters = 10000;
  for (int mode : {0, 1, 3, 4}) {
    for (int C : {1, 2, 4, 8, 16}) {
      for (int threads : {128, 512, 1024}) {
        cudaLaunchConfig_t cfg{};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = C;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(C);
        cfg.blockDim = dim3(threads);
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, bar_kernel, iters, mode, d);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long cyc = 0;
        cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
        printf("mode %d (sync=%d dsmem_st=%d relaxed=%d) C=%2d threads=%4d: %7.1f cycles/round %s\n",
               mode, mode & 1, (mode >> 1) & 1, (mode >> 2) & 1, C, threads,
               double(cyc) / iters, e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
    }
  }
  return 0;
}
