// Design-time micro-benchmarks for the bound-propagation engine (run once on a B200
// via gpurun). Measures: dependent fp64 add chain latency, shuffle-broadcast fold,
// cooperative grid.sync cost, random 16B/32B gather throughput from L2-resident
// arrays, and streaming bandwidth.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void dadd_chain(const double* x, double* out, long long* cyc, int iters)
{
  double s = 0.0, t = 0.0;
  double a = x[threadIdx.x], b = x[threadIdx.x + 32];
  long long c0 = clock64();
  for (int i = 0; i < iters; ++i) {
    s = __dadd_rn(s, a);
    t = __dadd_rn(t, b);
    a = __dsub_rn(0.0, a) ;  // keep a varying (independent chain)
  }
  long long c1 = clock64();
  out[threadIdx.x] = s + t;
  if (threadIdx.x == 0) *cyc = c1 - c0;
}

__global__ void smem_fold(const double* x, double* out, long long* cyc, int n)
{
  extern __shared__ double sm[];
  for (int i = threadIdx.x; i < n; i += blockDim.x) sm[i] = x[i];
  __syncthreads();
  double s = 0.0, t = 0.0;
  long long c0 = clock64();
  if (threadIdx.x == 0) {
#pragma unroll 16
    for (int i = 0; i < n; i += 2) {
      s = __dadd_rn(s, sm[i]);
      t = __dadd_rn(t, sm[i + 1]);
    }
  }
  long long c1 = clock64();
  if (threadIdx.x == 0) { out[0] = s + t; *cyc = c1 - c0; }
}

__global__ void shfl_fold(const double* x, double* out, long long* cyc, int n)
{
  double s = 0.0, t = 0.0;
  long long c0 = clock64();
  for (int base = 0; base < n; base += 32) {
    double v = x[base + threadIdx.x];
    double w = v * 0.5;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      s = __dadd_rn(s, __shfl_sync(0xffffffffu, v, j));
      t = __dadd_rn(t, __shfl_sync(0xffffffffu, w, j));
    }
  }
  long long c1 = clock64();
  if (threadIdx.x == 0) { out[0] = s + t; *cyc = c1 - c0; }
}

__global__ void grid_sync_bench(int iters, int* dummy)
{
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x == 0 && blockIdx.x == (i % gridDim.x)) atomicAdd(dummy, 1);
    g.sync();
  }
}

__global__ void gather16(const int* __restrict__ idx, const double2* __restrict__ tab, double* out, long long n)
{
  double acc = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double2 v = tab[idx[i]];
    acc += v.x + v.y;
  }
  if (acc == 12345.678) out[0] = acc;
}

struct alignas(32) R32 { double a, b, c, d; };
__global__ void gather32(const int* __restrict__ idx, const R32* __restrict__ tab, double* out, long long n)
{
  double acc = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double4* p = reinterpret_cast<const double4*>(tab + idx[i]);
    double2 v0 = reinterpret_cast<const double2*>(p)[0];
    double2 v1 = reinterpret_cast<const double2*>(p)[1];
    acc += v0.x + v0.y + v1.x + v1.y;
  }
  if (acc == 12345.678) out[0] = acc;
}

__global__ void stream_copy(const double2* __restrict__ a, double2* __restrict__ b, long long n)
{
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) b[i] = a[i];
}

int main()
{
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  printf("device %s sms=%d l2=%d MB clock=%d kHz\n", prop.name, prop.multiProcessorCount, prop.l2CacheSize >> 20, prop.clockRate);
  double *dx, *dout; long long* dcyc;
  std::vector<double> hx(1 << 20);
  for (size_t i = 0; i < hx.size(); ++i) hx[i] = 1.0 + 1e-3 * (i % 97);
  CK(cudaMalloc(&dx, hx.size() * 8)); CK(cudaMalloc(&dout, 1024)); CK(cudaMalloc(&dcyc, 8));
  CK(cudaMemcpy(dx, hx.data(), hx.size() * 8, cudaMemcpyHostToDevice));
  long long cyc;
  for (int rep = 0; rep < 2; ++rep) {
    dadd_chain<<<1, 32>>>(dx, dout, dcyc, 100000); CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost));
  }
  printf("dadd dependent chain: %.2f cycles/add (2 interleaved chains + 1 indep op)\n", cyc / 100000.0);
  CK(cudaFuncSetAttribute(smem_fold, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 * 8));
  for (int rep = 0; rep < 2; ++rep) {
    smem_fold<<<1, 32, 16384 * 8>>>(dx, dout, dcyc, 16384); CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost));
  }
  printf("smem fold (1 lane, 2 chains): %.2f cycles/entry-pair, 16384 entries -> %.1f us at 1.9GHz\n", cyc / 8192.0, cyc / 1.9e3);
  for (int rep = 0; rep < 2; ++rep) {
    shfl_fold<<<1, 32>>>(dx, dout, dcyc, 16384); CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost));
  }
  printf("shfl fold (warp, 2 chains): %.2f cycles/entry, 16384 entries -> %.1f us\n", cyc / 16384.0, cyc / 1.9e3);

  int* ddummy; CK(cudaMalloc(&ddummy, 4));
  for (int bps : {1, 2, 4}) {
    int nb = prop.multiProcessorCount * bps;
    int iters = 2000;
    void* args[] = {&iters, &ddummy};
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    CK(cudaLaunchCooperativeKernel((void*)grid_sync_bench, nb, 256, args, 0, 0));
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    CK(cudaLaunchCooperativeKernel((void*)grid_sync_bench, nb, 256, args, 0, 0));
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("grid.sync: %d blocks x 256: %.3f us per sync\n", nb, ms * 1e3 / iters);
  }
  // gathers
  long long N = 19000000;
  std::vector<int> hidx(N);
  std::mt19937 rng(1);
  int* didx; CK(cudaMalloc(&didx, N * 4));
  for (int tabn : {1000000, 4000000}) {
    for (long long i = 0; i < N; ++i) hidx[i] = rng() % tabn;
    CK(cudaMemcpy(didx, hidx.data(), N * 4, cudaMemcpyHostToDevice));
    double2* t16; R32* t32;
    CK(cudaMalloc(&t16, (size_t)tabn * 16)); CK(cudaMalloc(&t32, (size_t)tabn * 32));
    CK(cudaMemset(t16, 0, (size_t)tabn * 16)); CK(cudaMemset(t32, 0, (size_t)tabn * 32));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int k = 0; k < 2; ++k) {
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        if (k == 0) gather16<<<prop.multiProcessorCount * 8, 256>>>(didx, t16, dout, N);
        else gather32<<<prop.multiProcessorCount * 8, 256>>>(didx, t32, dout, N);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep == 2) printf("gather%d from %d-entry table (%d MB): %.1f us for %lld gathers -> %.2f Ggathers/s, idx stream %.0f GB/s, sector traffic %.0f GB/s\n",
                             k ? 32 : 16, tabn, tabn * (k ? 32 : 16) >> 20, ms * 1e3, N, N / ms / 1e6, N * 4.0 / ms / 1e6, N * 32.0 / ms / 1e6);
      }
    }
    cudaFree(t16); cudaFree(t32);
  }
  // stream copy 2 GB
  long long M = 1ll << 27;  // 128M double2 = 2 GB
  double2 *a, *b; CK(cudaMalloc(&a, M * 16)); CK(cudaMalloc(&b, M * 16));
  CK(cudaMemset(a, 0, M * 16));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    stream_copy<<<prop.multiProcessorCount * 8, 256>>>(a, b, M);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (rep == 2) printf("stream copy: %.0f GB/s (read+write)\n", 2.0 * M * 16 / ms / 1e6);
  }
  return 0;
}
