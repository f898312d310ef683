// Microbenchmark: shared-memory atomic throughput on B200 (spread addresses).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_cas(unsigned* out, int iters) {
  __shared__ unsigned tab[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) tab[i] = 0xffffffffu;
  __syncthreads();
  unsigned h = (threadIdx.x * 2654435761u) & 4095, acc = 0;
  for (int it = 0; it < iters; it++) {
    unsigned old = atomicCAS(&tab[h], 0xffffffffu, h + it);
    acc += old;
    h = (h + 97) & 4095;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_addf64(double* out, int iters) {
  __shared__ double tab[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) tab[i] = 0;
  __syncthreads();
  unsigned h = (threadIdx.x * 2654435761u) & 4095;
  for (int it = 0; it < iters; it++) { atomicAdd(&tab[h], 1.0); h = (h + 97) & 4095; }
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = tab[threadIdx.x];
}
__global__ void k_or(unsigned* out, int iters) {
  __shared__ unsigned tab[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) tab[i] = 0;
  __syncthreads();
  unsigned h = (threadIdx.x * 2654435761u) & 4095;
  for (int it = 0; it < iters; it++) { atomicOr(&tab[h], 1u << (it & 31)); h = (h + 97) & 4095; }
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = tab[threadIdx.x];
}
__global__ void k_lds(unsigned* out, int iters) {
  __shared__ unsigned tab[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) tab[i] = i;
  __syncthreads();
  unsigned h = (threadIdx.x * 2654435761u) & 4095, acc = 0;
  for (int it = 0; it < iters; it++) { acc += tab[h]; tab[(h + 1) & 4095] = acc; h = (h + 97) & 4095; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int blocks = sms * 4, threads = 512, iters = 4096;
  void* out; cudaMalloc(&out, (size_t)blocks * threads * 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, auto launch) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = (double)blocks * threads * iters;
    printf("%-10s %.3f ms  %.1f Gop/s  %.2f lane-ops/clk/SM (at 1.965GHz)\n", name, ms, ops / ms / 1e6,
           ops / (ms * 1e-3) / sms / 1.965e9);
  };
  run("cas32", [&] { k_cas<<<blocks, threads>>>((unsigned*)out, iters); });
  run("addf64", [&] { k_addf64<<<blocks, threads>>>((double*)out, iters); });
  run("or32", [&] { k_or<<<blocks, threads>>>((unsigned*)out, iters); });
  run("lds+sts", [&] { k_lds<<<blocks, threads>>>((unsigned*)out, iters); });
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
