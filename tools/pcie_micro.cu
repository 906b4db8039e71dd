// Host-link micro-benchmark for the e2e query path (dev aid): 16M int64
// pairs in (256 MB) and 16M int64 answers out (128 MB) between pinned host
// memory and a B200, three ways:
//   copy   : cudaMemcpyAsync H2D, then D2H (copy engines, serial)
//   duplex : H2D and D2H of independent buffers on two streams at once
//   mapped : one kernel reading the pairs from mapped pinned memory and
//            writing answers into mapped pinned memory (zero-copy, SM loads)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pcie_micro tools/pcie_micro.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_mapped(const longlong2* __restrict__ in, long long* __restrict__ out, uint64_t q) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < q;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const longlong2 p = in[i];
    out[i] = p.x ^ p.y;
  }
}

__global__ void k_mapped4(const longlong2* __restrict__ in, long long* __restrict__ out, uint64_t q) {
  // 4 pairs per thread in flight
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < q; i += 4 * stride) {
    longlong2 p[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) p[j] = (i + j * stride < q) ? in[i + j * stride] : make_longlong2(0, 0);
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (i + j * stride < q) out[i + j * stride] = p[j].x ^ p[j].y;
  }
}

int main() {
  const uint64_t q = 16u << 20;
  longlong2 *hp, *dp;
  long long *ha, *da;
  cudaHostAlloc(&hp, q * 16, cudaHostAllocMapped);
  cudaHostAlloc(&ha, q * 8, cudaHostAllocMapped);
  for (uint64_t i = 0; i < q; ++i) hp[i] = make_longlong2(i, 3 * i);
  cudaMalloc(&dp, q * 16);
  cudaMalloc(&da, q * 8);
  longlong2* mp;
  long long* ma;
  cudaHostGetDevicePointer(&mp, hp, 0);
  cudaHostGetDevicePointer(&ma, ha, 0);
  cudaStream_t s0, s1;
  cudaStreamCreate(&s0);
  cudaStreamCreate(&s1);
  cudaEvent_t a, b, c;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventCreate(&c);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int rep = 0; rep < 4; ++rep) {
    float t_h2d, t_d2h, t_dup, t_map, t_map4;
    cudaEventRecord(a, s0);
    cudaMemcpyAsync(dp, hp, q * 16, cudaMemcpyHostToDevice, s0);
    cudaEventRecord(b, s0);
    cudaMemcpyAsync(ha, da, q * 8, cudaMemcpyDeviceToHost, s0);
    cudaEventRecord(c, s0);
    cudaEventSynchronize(c);
    cudaEventElapsedTime(&t_h2d, a, b);
    cudaEventElapsedTime(&t_d2h, b, c);
    cudaDeviceSynchronize();
    cudaEventRecord(a, s0);
    cudaStreamWaitEvent(s1, a, 0);
    cudaMemcpyAsync(dp, hp, q * 16, cudaMemcpyHostToDevice, s0);
    cudaMemcpyAsync(ha, da, q * 8, cudaMemcpyDeviceToHost, s1);
    cudaEventRecord(b, s1);
    cudaStreamWaitEvent(s0, b, 0);
    cudaEventRecord(c, s0);
    cudaEventSynchronize(c);
    cudaEventElapsedTime(&t_dup, a, c);
    cudaEventRecord(a, s0);
    k_mapped<<<sms * 8, 256, 0, s0>>>(mp, ma, q);
    cudaEventRecord(b, s0);
    k_mapped4<<<sms * 8, 256, 0, s0>>>(mp, ma, q);
    cudaEventRecord(c, s0);
    cudaEventSynchronize(c);
    cudaEventElapsedTime(&t_map, a, b);
    cudaEventElapsedTime(&t_map4, b, c);
    bool ok = true;
    for (uint64_t i = 0; i < q; i += 999983) ok &= ha[i] == (long long)(i ^ (3 * i));
    printf("rep %d: H2D 256MB %.3f ms (%.1f GB/s)  D2H 128MB %.3f ms (%.1f GB/s)  duplex %.3f ms  "
           "mapped %.3f ms  mapped4 %.3f ms  ok=%d err=%s\n",
           rep, t_h2d, q * 16 / t_h2d / 1e6, t_d2h, q * 8 / t_d2h / 1e6, t_dup, t_map, t_map4, ok,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
