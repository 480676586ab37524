// standalone check of batched.cu's bitonic network (1024 threads, P = 4096)
#include <cstdio>
#include <cstdint>
constexpr int kBT = 1024;
__device__ __noinline__ void bitonic_sort(unsigned long long* key, int* idx, int P) {
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P; i += kBT) {
        const int l = i ^ j;
        if (l > i) {
          const bool up = (i & k) == 0;
          const unsigned long long ka = key[i], kb = key[l];
          const int ia = idx[i], ib = idx[l];
          const bool gt = ka > kb || (ka == kb && ia > ib);
          if (gt == up) {
            key[i] = kb;
            key[l] = ka;
            idx[i] = ib;
            idx[l] = ia;
          }
        }
      }
      __syncthreads();
    }
  }
}
__global__ void k(int P, int n, int* bad, unsigned long long seed) {
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned long long* key = reinterpret_cast<unsigned long long*>(smem + 32768);
  int* idx = reinterpret_cast<int*>(smem + 32768 + 8 * P);
  for (int i = threadIdx.x; i < P; i += kBT) {
    unsigned long long x = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
    x ^= x >> 29; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 32;
    key[i] = i < n ? (x >> 4) : ~0ull;
    idx[i] = i;
  }
  __syncthreads();
  bitonic_sort(key, idx, P);
  for (int i = threadIdx.x + 1; i < P; i += kBT)
    if (key[i - 1] > key[i]) atomicAdd(bad, 1);
}
int main() {
  int* bad; cudaMallocManaged(&bad, sizeof(int));
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 120000);
  for (int n : {2300, 2600, 4096, 1500}) {
    *bad = 0;
    k<<<1, kBT, 32768 + 12 * 4096, 0>>>(4096, n, bad, 12345);
    cudaError_t e = cudaDeviceSynchronize();
    printf("n=%d bad=%d err=%s\n", n, *bad, cudaGetErrorString(e));
  }
}
