// The finalize's merge phase in isolation: 147 writer CTAs leave 104-double
// records; one reader CTA (160 threads, programmatic dependent launch) waits,
// loads one record head + 5 columns per thread, block min, exp, block sums --
// clock64 spans of each phase.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <math_constants.h>
#ifndef NREADERS
#define NREADERS 1
#endif

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}
__device__ __forceinline__ double warp_min(double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
  return v;
}

__global__ void writer(double* rec, int rs, int spin) {
  asm volatile("griddepcontrol.launch_dependents;");
  long long t0 = clock64();
  while (clock64() - t0 < spin) {
  }
  for (int i = threadIdx.x; i < rs; i += blockDim.x) rec[(size_t)blockIdx.x * rs + i] = 100.0 + blockIdx.x + i * 1e-3;
}

__global__ void reader(const double* rec, int rs, int nrec, long long* out) {
  __shared__ double s_min[32], s_part[32][8];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const long long c0 = clock64();
  double h0 = CUDART_INF, h1 = 0, col[5] = {0, 0, 0, 0, 0};
  if (tid < nrec) {
    const double* r = rec + (size_t)tid * rs;
    h0 = r[0];
    h1 = r[1];
    for (int j = 0; j < 5; ++j) col[j] = r[4 + 4 * blockIdx.x + j];
  }
  double m = warp_min(h0);
  const long long c1 = clock64();
  if (lane == 0) s_min[warp] = m;
  __syncthreads();
  const double rho = warp_min(lane < nw ? s_min[lane] : CUDART_INF);
  const long long c2 = clock64();
  const double e = (tid < nrec) ? exp(-(h0 - rho)) : 0.0;
  double z = warp_sum(h1 * e), acc[5];
  for (int j = 0; j < 5; ++j) acc[j] = warp_sum(col[j] * e);
  if (lane == 0) {
    s_part[warp][0] = z;
    for (int j = 0; j < 5; ++j) s_part[warp][1 + j] = acc[j];
  }
  __syncthreads();
  double s = 0;
  if (tid < 6)
    for (int w = 0; w < nw; ++w) s += s_part[w][tid];
  __syncthreads();
  const long long c3 = clock64();
  if (tid == 0 && blockIdx.x == 0) {
    out[0] = c1 - c0;
    out[1] = c2 - c1;
    out[2] = c3 - c2;
    out[3] = (long long)s;
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* rec;
  long long* out;
  cudaMalloc(&rec, sizeof(double) * 104 * sms);
  cudaMalloc(&out, 64);
  long long h[4], acc[3] = {0, 0, 0};
  const int reps = 20, nrec = 147;
  for (int k = 0; k < reps + 2; ++k) {
    writer<<<nrec, 448>>>(rec, 104, 20000);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(NREADERS);
    cfg.blockDim = dim3(160);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, reader, (const double*)rec, 104, nrec, out);
    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    if (k >= 2)
      for (int i = 0; i < 3; ++i) acc[i] += h[i];
  }
  printf("loads+warpmin %lld  barrier+min %lld  exp+sums+2 barriers %lld cycles\n", acc[0] / reps, acc[1] / reps,
         acc[2] / reps);
  return 0;
}
