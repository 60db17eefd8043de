// Host-to-device bandwidth from pinned memory with 1, 2 and 4 concurrent copy streams.
#include <cstdio>
#include <vector>
int main() {
  const size_t total = size_t(8) << 30, piece = size_t(256) << 20;
  char* h; char* d;
  cudaHostAlloc(&h, total, cudaHostAllocDefault);
  cudaMalloc(&d, total);
  for (size_t i = 0; i < total; i += 4096) h[i] = 1;
  for (int ns : {1, 2, 4}) {
    std::vector<cudaStream_t> st(ns);
    for (auto& s : st) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
      cudaDeviceSynchronize();
      cudaEventRecord(e0, 0);
      cudaDeviceSynchronize();
      for (size_t off = 0, k = 0; off < total; off += piece, ++k)
        cudaMemcpyAsync(d + off, h + off, piece, cudaMemcpyHostToDevice, st[k % ns]);
      for (auto& s : st) cudaStreamSynchronize(s);
      cudaEventRecord(e1, 0);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("%d stream(s): %.1f GB/s\n", ns, total / (ms * 1e-3) / 1e9);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
