// Latencies of the warp primitives on the first-fit chain's serve path
// (dependent chains on one warp): SHFL, VOTE.ballot, REDUX.max, IMAD.HI,
// shared-memory load.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/micro/lat_micro tools/micro/lat_micro.cu
#include <cstdio>

__global__ void k(unsigned* out, unsigned seed, int n) {
    __shared__ unsigned sm[64];
    const unsigned lane = threadIdx.x;
    sm[lane] = lane * 7 + seed;
    sm[lane + 32] = lane;
    __syncwarp();
    unsigned v = seed + lane;
    long long t0, t1;
    unsigned long long r[6];
    t0 = clock64();
    for (int i = 0; i < n; ++i) v = __shfl_sync(0xffffffffu, v, (v & 31u));
    t1 = clock64(); r[0] = t1 - t0;
    t0 = clock64();
    for (int i = 0; i < n; ++i) v = __ballot_sync(0xffffffffu, (v >> lane) & 1u) + lane;
    t1 = clock64(); r[1] = t1 - t0;
    t0 = clock64();
    for (int i = 0; i < n; ++i) v = __reduce_max_sync(0xffffffffu, v) ^ lane;
    t1 = clock64(); r[2] = t1 - t0;
    t0 = clock64();
    for (int i = 0; i < n; ++i) v = __umulhi(v, 0x9e3779b9u) + lane;
    t1 = clock64(); r[3] = t1 - t0;
    t0 = clock64();
    for (int i = 0; i < n; ++i) v = sm[(v & 31u)] + lane;
    t1 = clock64(); r[4] = t1 - t0;
    t0 = clock64();
    for (int i = 0; i < n; ++i) v = min(v + lane, v ^ 0x55u);
    t1 = clock64(); r[5] = t1 - t0;
    out[lane] = v;
    if (lane == 0)
        printf("per dependent op (cycles): shfl %.1f  ballot %.1f  redux.max %.1f  umulhi %.1f  lds %.1f  iadd+min %.1f\n",
               double(r[0]) / n, double(r[1]) / n, double(r[2]) / n, double(r[3]) / n, double(r[4]) / n,
               double(r[5]) / n);
}

int main() {
    unsigned* d;
    cudaMalloc(&d, 128);
    k<<<1, 32>>>(d, 3, 1000);
    k<<<1, 32>>>(d, 3, 10000);
    cudaDeviceSynchronize();
    return 0;
}
