// Measured L2 atomic throughput of this B200 (the denominator of K4's atomic
// roofline): red.global.add.u32 (no return value, the form warp-aggregated
// triage counters compile to) and atom.global.min.u32 with a return value, each
// over (a) distinct addresses spread across L2 slices and (b) a small hot set
// (E = 64 words, the bundled harnesses' edge count).  CUDA-event timed, best of 5.
// Build/run: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/atomic_probe tools/atomic_probe.cu && /tmp/atomic_probe
#include <cstdio>
#include <cuda_runtime.h>

__global__ void red_add(unsigned* buf, unsigned mask, int iters) {
  const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
  for (int k = 0; k < iters; ++k) atomicAdd(&buf[(t * 33u + k * 97u) & mask], 1u);   // result unused -> RED
}

__global__ void atom_min(unsigned* buf, unsigned mask, int iters, unsigned* sink) {
  const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned acc = 0;
  for (int k = 0; k < iters; ++k) acc += atomicMin(&buf[(t * 33u + k * 97u) & mask], t ^ k);
  if (acc == 0xdeadbeefu) *sink = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 256, blocks = sms * 8, iters = 256;
  unsigned *buf, *sink;
  cudaMalloc(&buf, (1u << 26) * sizeof(unsigned));
  cudaMalloc(&sink, 4);
  cudaMemset(buf, 0xff, (1u << 26) * sizeof(unsigned));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const double ops = (double)blocks * threads * iters;
  printf("{");
  const char* sep = "";
  for (int kind = 0; kind < 2; ++kind)
    for (unsigned mask : {(1u << 26) - 1u, 63u}) {
      float best = 1e30f;
      for (int rep = 0; rep < 6; ++rep) {
        cudaEventRecord(a);
        if (kind == 0) red_add<<<blocks, threads>>>(buf, mask, iters);
        else atom_min<<<blocks, threads>>>(buf, mask, iters, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        if (rep > 0 && ms < best) best = ms;
      }
      printf("%s\"%s_%s_ops_per_s\": %.4g", sep, kind == 0 ? "red_add_u32" : "atom_min_u32",
             mask == 63u ? "hot64" : "spread", ops / (best / 1e3));
      sep = ", ";
    }
  printf(", \"sms\": %d, \"how\": \"%d blocks x %d threads x %d ops, CUDA events, best of 5\"}\n", sms, blocks, threads,
         iters);
  return 0;
}
