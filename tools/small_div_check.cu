// Exhaustive device check of whff::small_div (division-free floor(a / d) used
// by the skeleton walk's budget boundary): every a < 2^16, d in 1..17.
// Built and run by tests/test_gpu_small_div.py.
#include <cstdio>
#include "../paper_1902_08018_b200/csrc/whff_decode.cuh"

__global__ void k_check(int* bad) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= 65536) return;
  for (int d = 1; d <= 17; ++d)
    if (whff::small_div(a, d) != a / d) atomicAdd(bad, 1);
}

int main() {
  int* bad = nullptr;
  if (cudaMallocManaged(&bad, sizeof(int)) != cudaSuccess) return 2;
  *bad = 0;
  k_check<<<256, 256>>>(bad);
  if (cudaDeviceSynchronize() != cudaSuccess) return 2;
  printf("small_div mismatches: %d\n", *bad);
  return *bad == 0 ? 0 : 1;
}
