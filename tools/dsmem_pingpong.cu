// DSMEM ping-pong latency (measurement tooling): a 2-CTA cluster; each round
// one CTA's thread 0 st.async's 16 bytes into the peer's buffer, completing
// on the peer's mbarrier (expect_tx armed by the peer each round), and the
// peer answers the same way. Cycles per one-way hop = total / (2 rounds).
// Variant 2: the payload is 32 lanes x 16 B (a warp's m-tile partial).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2603_18052_b200/csrc tools/dsmem_pingpong.cu -o tools/_bin/dsmem_pingpong
#include <cstdint>
#include <cstdio>

#include "common.cuh"

using namespace lbg;

template <int LANES>
__global__ void __cluster_dims__(2, 1, 1) pingpong(int rounds, long long* out) {
  __shared__ __align__(16) double2 buf[2][32];
  __shared__ __align__(8) uint64_t bar[2];
  const unsigned rank = cluster_ctarank(), peer = rank ^ 1u;
  const int lane = threadIdx.x;
  if (lane == 0) {
    for (int b = 0; b < 2; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(
          static_cast<unsigned>(__cvta_generic_to_shared(&bar[b]))));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  cluster_sync_all();
  const unsigned pbuf = mapa_shared(&buf[0][0], peer), pbar = mapa_shared(&bar[0], peer);
  const long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) {
    const int par = r & 1;
    if (lane == 0) mbar_expect_tx(&bar[par], 16u * LANES);
    __syncwarp();
    if (rank == 0) {  // send, then wait for the answer
      if (lane < LANES) st_async_f64x2(pbuf + unsigned((par * 32 + lane) * 16), make_double2(r, lane), pbar + par * 8u);
      mbar_wait_parity_cluster(&bar[par], unsigned((r >> 1) & 1));
    } else {  // wait, then answer
      mbar_wait_parity_cluster(&bar[par], unsigned((r >> 1) & 1));
      if (lane < LANES) st_async_f64x2(pbuf + unsigned((par * 32 + lane) * 16), buf[par][lane], pbar + par * 8u);
    }
  }
  const long long t1 = clock64();
  cluster_sync_all();
  if (lane == 0 && rank == 0) out[0] = t1 - t0;
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  for (int v = 0; v < 2; ++v) {
    for (int rep = 0; rep < 3; ++rep) {
      const int rounds = 10000;
      if (v == 0)
        pingpong<1><<<2, 32>>>(rounds, d);
      else
        pingpong<32><<<2, 32>>>(rounds, d);
      long long h = 0;
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("%s: %.1f cycles per one-way hop (round trip %.1f)\n", v ? "32 lanes x 16 B" : "1 lane x 16 B",
             double(h) / rounds / 2, double(h) / rounds);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
