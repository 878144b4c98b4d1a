// Standalone check of the 1-D bulk-copy (cp.async.bulk) + mbarrier double-buffer pattern used for
// streaming a contiguous array into shared memory: each warp streams its own region in 2 KB chunks,
// re-initialising its barriers for every region, and checks the sum.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* mb)
{
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mb)) : "memory");
#ifndef NO_INIT_FENCE
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#endif
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, unsigned long long* mb)
{
#ifndef NO_SHARED_FENCE
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#endif
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mb)), "r"(bytes) : "memory");
#ifdef CTA_DST
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(mb)) : "memory");
#else
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(mb)) : "memory");
#endif
}
__device__ __forceinline__ bool mbar_wait_bounded(unsigned long long* mb, unsigned parity)
{
  unsigned ok = 0;
  for (long long it = 0; it < (1ll << 24) && !ok; ++it)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n}"
                 : "=r"(ok) : "r"(smem_u32(mb)), "r"(parity) : "memory");
  return ok != 0;
}

struct alignas(16) WarpTma {
  double2 buf[2][128];
  unsigned long long mbar[2];
};

__global__ void k(const double2* g, int regions, int chunks, double* out, int* fails)
{
  __shared__ WarpTma T[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpTma& t = T[warp];
  const int gw = blockIdx.x * 8 + warp;
#ifdef INIT_ONCE
  if (lane == 0) {
    mbar_init(&t.mbar[0]);
    mbar_init(&t.mbar[1]);
  }
  __syncwarp();
  unsigned ph0 = 0, ph1 = 0;  // completed uses per buffer
#endif
  for (int r = gw; r < regions; r += gridDim.x * 8) {
    const double2* src = g + (size_t)r * chunks * 128;
    if (lane == 0) {
#ifndef INIT_ONCE
      mbar_init(&t.mbar[0]);
      mbar_init(&t.mbar[1]);
#endif
#ifndef NO_GLOBAL_FENCE
      asm volatile("fence.proxy.async.global;" ::: "memory");
#endif
      bulk_load(t.buf[0], src, 2048, &t.mbar[0]);
      if (chunks > 1) bulk_load(t.buf[1], src + 128, 2048, &t.mbar[1]);
    }
    __syncwarp();
    double acc = 0.0;
    for (int c = 0; c < chunks; ++c) {
      const int b = c & 1;
#ifdef INIT_ONCE
      const unsigned par = (b ? ph1 : ph0) & 1u;
      if (b) ++ph1; else ++ph0;
#else
      const unsigned par = (unsigned)(c >> 1) & 1u;
#endif
      if (!mbar_wait_bounded(&t.mbar[b], par)) {
        if (lane == 0) atomicAdd(fails, 1);
        return;
      }
      for (int h = 0; h < 4; ++h) acc += t.buf[b][h * 32 + lane].x;
      __syncwarp();
      if (lane == 0 && c + 2 < chunks) bulk_load(t.buf[b], src + (size_t)(c + 2) * 128, 2048, &t.mbar[b]);
      __syncwarp();
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out[r] = acc;
  }
}

int main()
{
  const int regions = 5000, chunks = 37;
  const size_t n = (size_t)regions * chunks * 128;
  double2* h = new double2[n];
  for (size_t i = 0; i < n; ++i) h[i] = make_double2((double)(i % 7), 0.0);
  double2* g;
  double* out;
  int* fails;
  cudaMalloc(&g, n * sizeof(double2));
  cudaMalloc(&out, regions * sizeof(double));
  cudaMalloc(&fails, sizeof(int));
  cudaMemcpy(g, h, n * sizeof(double2), cudaMemcpyHostToDevice);
  cudaMemset(fails, 0, sizeof(int));
#ifdef CLUSTER1
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(148); cfg.blockDim = dim3(256); cfg.attrs = at; cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, (const double2*)g, regions, chunks, out, fails);
#else
  k<<<148, 256>>>(g, regions, chunks, out, fails);
#endif
  cudaError_t e = cudaDeviceSynchronize();
  int hf = -1;
  cudaMemcpy(&hf, fails, sizeof(int), cudaMemcpyDeviceToHost);
  double* ho = new double[regions];
  cudaMemcpy(ho, out, regions * sizeof(double), cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int r = 0; r < regions; ++r) {
    double s = 0;
    for (size_t i = (size_t)r * chunks * 128; i < (size_t)(r + 1) * chunks * 128; ++i) s += (double)(i % 7);
    if (s != ho[r]) ++bad;
  }
  printf("status %s, wait timeouts %d, wrong sums %d of %d\n", cudaGetErrorString(e), hf, bad, regions);
  return 0;
}
