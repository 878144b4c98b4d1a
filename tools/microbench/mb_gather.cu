// Random 16-B gather throughput from an L2-resident table vs. warps per SM and gathers in flight
// per thread (the k_rows_full SELL pass is such a gather: is it concurrency- or latency-limited?).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_gather mb_gather.cu
#include <cstdio>
#include <random>
#include <vector>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e = (x);                                                             \
    if (e != cudaSuccess) {                                                          \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);       \
      return 1;                                                                      \
    }                                                                                \
  } while (0)

// each thread: U coalesced index loads (SELL-like: lane-interleaved), then U gathers, then a
// sequential fp64 sum of the U values (the row's activity chain)
template <int U>
__global__ void gather_u(const int* __restrict__ idx, const double2* __restrict__ tab, double* out, long long n)
{
  const long long nt = (long long)gridDim.x * blockDim.x;
  double acc = 0.0;
  for (long long base = blockIdx.x * (long long)blockDim.x + threadIdx.x; base < n; base += nt * U) {
    int ci[U];
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) ci[u] = base + u * nt < n ? __ldg(idx + base + u * nt) : -1;
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ci[u] >= 0 ? tab[ci[u]] : make_double2(0.0, 0.0);
#pragma unroll
    for (int u = 0; u < U; ++u) acc = __dadd_rn(acc, __dmul_rn(v[u].x, 1.5));
  }
  if (acc == 12345.678) out[0] = acc;
}

template <int U>
int run(const int* didx, const double2* tab, double* dout, long long N, int sms, int bps, int smem)
{
  if (smem) CK(cudaFuncSetAttribute(gather_u<U>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    gather_u<U><<<sms * bps, 256, smem>>>(didx, tab, dout, N);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) best = ms < best ? ms : best;
  }
  printf("U=%d warps/SM=%2d: %7.1f us -> %6.1f Ggathers/s\n", U, bps * 8, best * 1e3, N / best / 1e6);
  return 0;
}

int main()
{
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  const long long N = 19600000;
  const int tabn = 1000000;
  std::vector<int> hidx(N);
  std::mt19937 rng(1);
  for (long long i = 0; i < N; ++i) hidx[i] = rng() % tabn;
  int* didx;
  double2* tab;
  double* dout;
  CK(cudaMalloc(&didx, N * 4));
  CK(cudaMalloc(&tab, (size_t)tabn * 16));
  CK(cudaMalloc(&dout, 64));
  CK(cudaMemcpy(didx, hidx.data(), N * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(tab, 0, (size_t)tabn * 16));
  // blocks per SM = the grid: sms * bps blocks of 256 threads spread over the SMs in one wave
  for (int bps : {1, 2, 3, 4, 8}) {
    const int smem = 0;  // residency = the grid (sms * bps blocks spread one wave)
    run<1>(didx, tab, dout, N, sms, bps, smem);
    run<2>(didx, tab, dout, N, sms, bps, smem);
    run<4>(didx, tab, dout, N, sms, bps, smem);
    run<8>(didx, tab, dout, N, sms, bps, smem);
    run<16>(didx, tab, dout, N, sms, bps, smem);
  }
  return 0;
}
