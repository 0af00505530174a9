// Latency of reading data another kernel just wrote (the rollout -> finalize
// hand-off of the closed loop): kernel W (one CTA per SM) writes one 832-byte
// record per CTA, kernel R (programmatic dependent launch) waits on the grid
// dependency and reads them, timing with clock64 the first load, a second
// load of other lines, and the same lines again.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/handoff tools/microbench/handoff.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void writer(double* rec, int rs, int spin) {
  asm volatile("griddepcontrol.launch_dependents;");
  long long t0 = clock64();
  while (clock64() - t0 < spin) {
  }
  for (int i = threadIdx.x; i < rs; i += blockDim.x) rec[(size_t)blockIdx.x * rs + i] = blockIdx.x + i * 1e-3;
}

template <int MODE>
__global__ void reader(const double* rec, int rs, int nrec, long long* out) {
  // MODE 0: plain loads; 1: ld.global.cg; 2: ld.global.nc (after the wait)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int tid = threadIdx.x;
  long long c0 = clock64();
  double v = 0.0;
  const double* r = rec + (size_t)tid * rs;
  if (tid < nrec) {
    if (MODE == 0) v = r[0];
    if (MODE == 1) v = __ldcg(r);
    if (MODE == 2) v = __ldg(r);
  }
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  long long c1 = clock64();
  double w = 0.0;
  if (tid < nrec) {
    const double* q = r + 40;  // another line of the same record
    if (MODE == 0) w = q[0];
    if (MODE == 1) w = __ldcg(q);
    if (MODE == 2) w = __ldg(q);
  }
  w += __shfl_xor_sync(0xffffffffu, w, 1);
  long long c2 = clock64();
  double u = 0.0;
  if (tid < nrec) u = __ldcg(r + 80);
  u += __shfl_xor_sync(0xffffffffu, u, 1);
  long long c3 = clock64();
  if (tid == 0) {
    out[0] = c1 - c0;
    out[1] = c2 - c1;
    out[2] = c3 - c2;
    out[3] = (long long)(v + w + u);
  }
}

template <int MODE>
void run(const char* name, double* rec, long long* out, int sms, bool pdl) {
  long long h[4], acc[3] = {0, 0, 0};
  const int reps = 20;
  for (int k = 0; k < reps + 2; ++k) {
    writer<<<sms - 1, 128>>>(rec, 104, 20000);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(160);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, reader<MODE>, (const double*)rec, 104, sms - 1, out);
    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    if (k >= 2)
      for (int i = 0; i < 3; ++i) acc[i] += h[i];
  }
  printf("%-10s pdl=%d first %6lld  second-line %6lld  third-line %6lld cycles\n", name, (int)pdl, acc[0] / reps,
         acc[1] / reps, acc[2] / reps);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* rec;
  long long* out;
  cudaMalloc(&rec, sizeof(double) * 104 * sms);
  cudaMalloc(&out, 64);
  for (int pdl = 0; pdl < 2; ++pdl) {
    run<0>("plain", rec, out, sms, pdl);
    run<1>("ld.cg", rec, out, sms, pdl);
    run<2>("ld.nc", rec, out, sms, pdl);
  }
  return 0;
}
