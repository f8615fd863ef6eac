// Host cost of kernel launches: plain <<<>>>, cudaLaunchKernelEx with the
// programmatic-stream-serialization attribute, small vs ~1 KB parameters.
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
struct Big { unsigned long long v[128]; };  // 1 KB
__global__ void k_small(int x) { if (x == 12345) asm volatile("trap;"); }
__global__ void k_big(const __grid_constant__ Big b) { if (b.v[3] == 12345) asm volatile("trap;"); }
template <class F>
double time_us(F f, int n) {
  cudaDeviceSynchronize();
  auto t0 = std::chrono::high_resolution_clock::now();
  for (int i = 0; i < n; ++i) f();
  auto t1 = std::chrono::high_resolution_clock::now();
  cudaDeviceSynchronize();
  return std::chrono::duration<double, std::micro>(t1 - t0).count() / n;
}
int main() {
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  Big b = {};
  const int n = 2000;
  auto ex = [&](auto kernel, auto arg, bool pdl, int grid) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid; cfg.blockDim = 256; cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, arg);
  };
  for (int rep = 0; rep < 2; ++rep) {
    printf("plain small        %.2f us\n", time_us([&] { k_small<<<148, 256, 0, st>>>(1); }, n));
    printf("plain big (1 KB)   %.2f us\n", time_us([&] { k_big<<<148, 256, 0, st>>>(b); }, n));
    printf("Ex small no-pdl    %.2f us\n", time_us([&] { ex(k_small, 1, false, 148); }, n));
    printf("Ex small pdl       %.2f us\n", time_us([&] { ex(k_small, 1, true, 148); }, n));
    printf("Ex big pdl         %.2f us\n", time_us([&] { ex(k_big, b, true, 148); }, n));
    printf("Ex big pdl grid 4k %.2f us\n", time_us([&] { ex(k_big, b, true, 4096); }, n));
    cudaEvent_t e; cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    printf("event record       %.2f us\n", time_us([&] { cudaEventRecord(e, st); }, n));
    printf("stream wait event  %.2f us\n", time_us([&] { cudaStreamWaitEvent(st, e, 0); }, n));
  }
  return 0;
}
