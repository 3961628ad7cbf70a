// Latency / throughput probes on sm_100a: dependent DFMA chain, FFMA chain, double shuffle chain,
// DFMA throughput with many warps, MUFU.RCP64H.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_chain(double* out, double a, double b, int n, long long* cyc) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = fma(x, b, a); x = fma(x, b, a); x = fma(x, b, a); x = fma(x, b, a); }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void ffma_chain(float* out, float a, float b, int n, long long* cyc) {
  float x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = fmaf(x, b, a); x = fmaf(x, b, a); x = fmaf(x, b, a); x = fmaf(x, b, a); }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void shfl_chain(double* out, double a, int n, long long* cyc) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x += __shfl_xor_sync(0xffffffffu, x, 1); x += __shfl_xor_sync(0xffffffffu, x, 2); }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void rcp_chain(double* out, double a, int n, long long* cyc) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r + 1.5; }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void div_chain(double* out, double a, int n, long long* cyc) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = 1.0 / x + 1.5; }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
// throughput: 8 independent chains per thread
__global__ void dfma_tput(double* out, double a, double b, int n) {
  double x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3, x4 = a + 4, x5 = a + 5, x6 = a + 6, x7 = a + 7;
  for (int i = 0; i < n; ++i) {
    x0 = fma(x0, b, a); x1 = fma(x1, b, a); x2 = fma(x2, b, a); x3 = fma(x3, b, a);
    x4 = fma(x4, b, a); x5 = fma(x5, b, a); x6 = fma(x6, b, a); x7 = fma(x7, b, a);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void lds_chain(double* out, int n, long long* cyc) {
  __shared__ int idx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) idx[i] = (i * 7 + 1) & 1023;
  __syncthreads();
  int j = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) j = idx[j];
  long long t1 = clock64();
  out[threadIdx.x] = j; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void sync_loop(double* out, int n, long long* cyc) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* d; float* f; long long* c; long long h;
  cudaMalloc(&d, 1 << 24); cudaMalloc(&f, 1 << 20); cudaMalloc(&c, 64);
  const int n = 4096;
  dfma_chain<<<1, 32>>>(d, 0.5, 0.999, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", (double)h / (4.0 * n));
  ffma_chain<<<1, 32>>>(f, 0.5f, 0.999f, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("FFMA dependent latency: %.2f cycles\n", (double)h / (4.0 * n));
  shfl_chain<<<1, 32>>>(d, 0.5, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("double shfl+add dependent: %.2f cycles per step\n", (double)h / (2.0 * n));
  rcp_chain<<<1, 32>>>(d, 0.5, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("rcp.approx.f64 + add dependent: %.2f cycles\n", (double)h / n);
  div_chain<<<1, 32>>>(d, 0.5, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("fp64 1/x + add dependent: %.2f cycles\n", (double)h / n);
  lds_chain<<<1, 32>>>(d, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("LDS dependent latency: %.2f cycles\n", (double)h / n);
  for (int nt : {64, 256, 1024}) {
    sync_loop<<<1, nt>>>(d, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("__syncthreads (%d threads): %.2f cycles\n", nt, (double)h / n);
  }
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int th : {128, 256, 512, 1024}) {
    dfma_tput<<<sms, th>>>(d, 0.5, 0.999, 1000);
    cudaEventRecord(e0);
    dfma_tput<<<sms * 2, th>>>(d, 0.5, 0.999, 20000);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * 20000.0 * sms * 2 * th;
    printf("DFMA throughput (%d thr/CTA, 2 CTA/SM): %.2f TFLOP/s\n", th, fl / ms / 1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
