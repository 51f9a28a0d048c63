// launch cost of one-warp blocks that exit at once (the k_collide grid over idle tiles):
// 524288 blocks x 32 threads with 11.8 KB dynamic shared memory, as c5's k_collide
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(32, 16) k_exit(const unsigned* cnt, unsigned* out) {
  extern __shared__ unsigned char sm[];
  if (blockIdx.x >= *cnt) return;
  if (threadIdx.x == 0) out[blockIdx.x] = sm[0];
}
__global__ void __launch_bounds__(32, 16) k_loop(const unsigned* cnt, unsigned* out) {
  extern __shared__ unsigned char sm[];
  for (unsigned b = blockIdx.x; b < *cnt; b += gridDim.x)
    if (threadIdx.x == 0) out[b] = sm[0];
}
int main() {
  unsigned *cnt, *out;
  cudaMalloc(&cnt, 4); cudaMalloc(&out, 4u << 22);
  cudaFuncSetAttribute(k_exit, cudaFuncAttributeMaxDynamicSharedMemorySize, 12288);
  cudaFuncSetAttribute(k_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, 12288);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (unsigned grid : {131072u, 524288u, 2097152u}) for (unsigned c : {0u, 65536u}) {
    cudaMemcpy(cnt, &c, 4, cudaMemcpyHostToDevice);
    for (int w = 0; w < 3; w++) k_exit<<<grid, 32, 11800>>>(cnt, out);
    cudaEventRecord(a);
    for (int w = 0; w < 20; w++) k_exit<<<grid, 32, 11800>>>(cnt, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("k_exit grid %u count %u: %.4f ms\n", grid, c, ms / 20);
  }
  for (unsigned c : {0u, 65536u}) {
    cudaMemcpy(cnt, &c, 4, cudaMemcpyHostToDevice);
    cudaEventRecord(a);
    for (int w = 0; w < 20; w++) k_loop<<<148 * 16, 32, 11800>>>(cnt, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("k_loop grid %u count %u: %.4f ms\n", 148 * 16, c, ms / 20);
  }
  return 0;
}
