// Dev probe: does compute-sanitizer racecheck model bar.arrive -> bar.sync (named barrier) handoffs?
// warp 0 writes shared memory and arrives on barrier 1; warp 1 syncs on it and reads. Correct per PTX.
#include <cstdio>
__global__ void k(int* out) {
  __shared__ int buf[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (w == 0) {
    buf[lane] = lane * 3;
    asm volatile("bar.arrive 1, 64;" ::: "memory");
  } else {
    asm volatile("bar.sync 1, 64;" ::: "memory");
    out[lane] = buf[(lane + 1) & 31];
  }
}
int main() {
  int* d; cudaMalloc(&d, 128);
  k<<<1, 64>>>(d);
  int h[32]; cudaMemcpy(h, d, 128, cudaMemcpyDeviceToHost);
  printf("probe %d %d\n", h[0], h[31]);
  return 0;
}
