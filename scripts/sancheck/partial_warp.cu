// Minimal check: __syncthreads in a 63-thread block (partial last warp), no divergence.
#include <cstdio>
__global__ void k(double* out) {
  __shared__ double s[64];
  s[threadIdx.x] = threadIdx.x;
  __syncthreads();
  out[threadIdx.x] = s[(threadIdx.x + 1) % blockDim.x];
}
int main() {
  double* d;
  cudaMalloc(&d, 64 * 8);
  k<<<4, 63>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  printf("partial-warp kernel: %s\n", cudaGetErrorString(e));
  return 0;
}
