// The heavy-row segment fold in isolation (one warp, 16384 contributions in global memory):
// cycles per 128-entry chunk of (a) the engine's loop (register stream of chunk c+2, ballot
// compaction of the non-zeros into shared memory, lanes 0/1 fold), (b) the fold over already
// compacted streams (the compaction moved to the producers), (c) a pure dependent DADD chain.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o mb_fold mb_fold.cu
#include <cstdio>
#include <random>
#include <vector>

#define FULL 0xffffffffu
constexpr int kTile = 128, kEPL = 4, kSeg = 16384;

__device__ __forceinline__ double fold_seq(const double* src, int cnt, double acc)
{
  const double2* s2 = reinterpret_cast<const double2*>(src);
  int j             = 0;
  if (cnt >= 8) {
    double2 v0 = s2[0], v1 = s2[1], v2 = s2[2], v3 = s2[3];
    for (j = 8; j + 8 <= cnt; j += 8) {
      const double2 w0 = s2[j / 2], w1 = s2[j / 2 + 1], w2 = s2[j / 2 + 2], w3 = s2[j / 2 + 3];
      acc = __dadd_rn(acc, v0.x); acc = __dadd_rn(acc, v0.y);
      acc = __dadd_rn(acc, v1.x); acc = __dadd_rn(acc, v1.y);
      acc = __dadd_rn(acc, v2.x); acc = __dadd_rn(acc, v2.y);
      acc = __dadd_rn(acc, v3.x); acc = __dadd_rn(acc, v3.y);
      v0 = w0; v1 = w1; v2 = w2; v3 = w3;
    }
    acc = __dadd_rn(acc, v0.x); acc = __dadd_rn(acc, v0.y);
    acc = __dadd_rn(acc, v1.x); acc = __dadd_rn(acc, v1.y);
    acc = __dadd_rn(acc, v2.x); acc = __dadd_rn(acc, v2.y);
    acc = __dadd_rn(acc, v3.x); acc = __dadd_rn(acc, v3.y);
  }
  for (; j < cnt; ++j) acc = __dadd_rn(acc, src[j]);
  return acc;
}

// (a) the engine's heavy_fold register stream
__global__ void fold_engine(const double2* gb, double* out, long long* cyc)
{
  __shared__ __align__(16) double b0[kTile], b1[kTile];
  const int lane = threadIdx.x;
  const unsigned lt = (1u << lane) - 1u;
  long long c0 = clock64();
  double acc = 0.0;
  double2 v[kEPL], w[kEPL];
#pragma unroll
  for (int h = 0; h < kEPL; ++h) {
    v[h] = __ldcg(gb + h * 32 + lane);
    w[h] = __ldcg(gb + kTile + h * 32 + lane);
  }
  for (int base = 0; base < kSeg; base += kTile) {
    int pm = 0, px = 0;
#pragma unroll
    for (int h = 0; h < kEPL; ++h) {
      const double cm = v[h].x, cx = v[h].y;
      const unsigned m = __ballot_sync(FULL, cm != 0.0);
      const unsigned x = __ballot_sync(FULL, cx != 0.0);
      if (cm != 0.0) b0[pm + __popc(m & lt)] = cm;
      if (cx != 0.0) b1[px + __popc(x & lt)] = cx;
      pm += __popc(m);
      px += __popc(x);
    }
    __syncwarp();
#pragma unroll
    for (int h = 0; h < kEPL; ++h) {
      v[h]         = w[h];
      const int e2 = base + 2 * kTile + h * 32 + lane;
      w[h]         = base + 2 * kTile < kSeg ? __ldcg(gb + e2) : make_double2(0.0, 0.0);
    }
    if (lane < 2) acc = fold_seq(lane ? b1 : b0, lane ? px : pm, acc);
    __syncwarp();
  }
  long long c1 = clock64();
  if (lane < 2) out[lane] = acc;
  if (lane == 0) *cyc = c1 - c0;
}

// (b) compacted streams (min values then max values, counts known): all lanes stage chunk c+1
// into shared memory while lanes 0/1 fold chunk c
__global__ void fold_compacted(const double* gmin, int nmin, const double* gmax, int nmax, double* out, long long* cyc)
{
  __shared__ __align__(16) double b[2][2][kTile];
  const int lane = threadIdx.x;
  long long c0 = clock64();
  double acc = 0.0;
  const int nch = ((nmin > nmax ? nmin : nmax) + kTile - 1) / kTile;
  double r[2][kEPL];
#pragma unroll
  for (int h = 0; h < kEPL; ++h) {
    const int e = h * 32 + lane;
    b[0][0][e] = e < nmin ? __ldcg(gmin + e) : 0.0;
    b[0][1][e] = e < nmax ? __ldcg(gmax + e) : 0.0;
    r[0][h] = kTile + e < nmin ? __ldcg(gmin + kTile + e) : 0.0;
    r[1][h] = kTile + e < nmax ? __ldcg(gmax + kTile + e) : 0.0;
  }
  __syncwarp();
  for (int ck = 0; ck < nch; ++ck) {
    const int bi = ck & 1;
    // registers of chunk ck+1 -> the other buffer; loads of chunk ck+2 in flight
#pragma unroll
    for (int h = 0; h < kEPL; ++h) {
      b[bi ^ 1][0][h * 32 + lane] = r[0][h];
      b[bi ^ 1][1][h * 32 + lane] = r[1][h];
      const int e = (ck + 2) * kTile + h * 32 + lane;
      r[0][h] = e < nmin ? __ldcg(gmin + e) : 0.0;
      r[1][h] = e < nmax ? __ldcg(gmax + e) : 0.0;
    }
    const int n0 = nmin - ck * kTile, n1 = nmax - ck * kTile;
    if (lane < 2) {
      const int cnt = lane ? n1 : n0;
      acc = fold_seq(b[bi][lane], cnt < 0 ? 0 : (cnt > kTile ? kTile : cnt), acc);
    }
    __syncwarp();
  }
  long long c1 = clock64();
  if (lane < 2) out[lane] = acc;
  if (lane == 0) *cyc = c1 - c0;
}

// (c) a pure dependent chain from shared memory
__global__ void fold_pure(const double* g, int n, double* out, long long* cyc)
{
  extern __shared__ __align__(16) double sb[];
  for (int i = threadIdx.x; i < n; i += 32) sb[i] = g[i];
  __syncwarp();
  long long c0 = clock64();
  double acc = 0.0;
  if (threadIdx.x < 2) acc = fold_seq(sb, n, acc);
  __syncwarp();
  long long c1 = clock64();
  if (threadIdx.x < 2) out[threadIdx.x] = acc;
  if (threadIdx.x == 0) *cyc = c1 - c0;
}

int main()
{
  std::mt19937 rng(7);
  std::uniform_real_distribution<double> U(-5.0, 5.0);
  std::vector<double> h(2 * kSeg), hmin, hmax;
  for (int i = 0; i < kSeg; ++i) {
    const double cm = (rng() % 10 < 4) ? 0.0 : U(rng), cx = (rng() % 10 < 2) ? 0.0 : U(rng);
    h[2 * i] = cm;
    h[2 * i + 1] = cx;
    if (cm != 0.0) hmin.push_back(cm);
    if (cx != 0.0) hmax.push_back(cx);
  }
  double *gb, *gmin, *gmax, *out;
  long long* cyc;
  cudaMalloc(&gb, sizeof(double) * 2 * kSeg);
  cudaMalloc(&gmin, sizeof(double) * kSeg);
  cudaMalloc(&gmax, sizeof(double) * kSeg);
  cudaMalloc(&out, 64);
  cudaMalloc(&cyc, 8);
  cudaMemcpy(gb, h.data(), sizeof(double) * 2 * kSeg, cudaMemcpyHostToDevice);
  cudaMemcpy(gmin, hmin.data(), sizeof(double) * hmin.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(gmax, hmax.data(), sizeof(double) * hmax.size(), cudaMemcpyHostToDevice);
  long long c;
  double o[2];
  for (int rep = 0; rep < 3; ++rep) {
    fold_engine<<<1, 32>>>(reinterpret_cast<const double2*>(gb), out, cyc);
    cudaDeviceSynchronize();
  }
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(o, out, 16, cudaMemcpyDeviceToHost);
  printf("non-zeros: min %zu max %zu of %d\n", hmin.size(), hmax.size(), kSeg);
  printf("(a) engine loop     : %8lld cycles = %6.1f us, %6.1f cycles/chunk  (%.17g %.17g)\n", c, c / 1965.0, c / 128.0, o[0], o[1]);
  for (int rep = 0; rep < 3; ++rep) {
    fold_compacted<<<1, 32>>>(gmin, (int)hmin.size(), gmax, (int)hmax.size(), out, cyc);
    cudaDeviceSynchronize();
  }
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(o, out, 16, cudaMemcpyDeviceToHost);
  printf("(b) compacted stream: %8lld cycles = %6.1f us, %6.1f cycles/chunk  (%.17g %.17g)\n", c, c / 1965.0, c / 128.0, o[0], o[1]);
  cudaFuncSetAttribute(fold_pure, cudaFuncAttributeMaxDynamicSharedMemorySize, kSeg * 8);
  for (int rep = 0; rep < 3; ++rep) {
    fold_pure<<<1, 32, kSeg * 8>>>(gmax, (int)hmax.size(), out, cyc);
    cudaDeviceSynchronize();
  }
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("(c) pure chain (%zu): %8lld cycles = %6.1f us, %6.2f cycles/add\n", hmax.size(), c, c / 1965.0, (double)c / hmax.size());
  return 0;
}
