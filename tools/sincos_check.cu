// Checks that CUDA's sincos(double) returns exactly sin(x) and cos(x) (the
// physics / render units use sincos where the oracle calls sin and cos).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/sincos_check tools/sincos_check.cu && /tmp/sincos_check
#include <cstdio>
#include <cstdint>
__global__ void k(uint64_t seed, int n, unsigned long long *bad) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t z = seed + 0x9E3779B97F4A7C15ull * (uint64_t)(i + 1);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; z ^= z >> 31;
  const double scales[4] = {1.0, 4.0, 100.0, 1e6};
  double x = ((double)(z >> 11) / 9007199254740992.0 - 0.5) * 2.0 * scales[i & 3];
  double s, c;
  sincos(x, &s, &c);
  if (__double_as_longlong(s) != __double_as_longlong(sin(x)) || __double_as_longlong(c) != __double_as_longlong(cos(x)))
    atomicAdd(bad, 1ull);
}
int main() {
  unsigned long long *bad, h = 0;
  cudaMalloc(&bad, 8); cudaMemset(bad, 0, 8);
  const int n = 1 << 26;
  for (int r = 0; r < 4; ++r) k<<<(n + 255) / 256, 256>>>(1234567ull * (r + 1), n, bad);
  cudaMemcpy(&h, bad, 8, cudaMemcpyDeviceToHost);
  printf("sincos vs sin/cos: %llu mismatches of %d\n", h, 4 * n);
  return h != 0;
}
