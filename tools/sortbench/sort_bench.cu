// Microbenchmark: CUB onesweep radix sort with wider digits (custom policy hub)
// on the two K0 sorts (weight sort: u64 keys + u32 eids; owner sort: 26-bit u32
// keys + u64 slots).  usage: sort_bench <which> <bits_per_pass> [n]
#include <cub/cub.cuh>
#include <cstdio>
#include <cstdlib>
#include <cstdint>

template <typename KeyT, typename ValueT, typename OffsetT, int RB>
struct Hub {
    using Base = cub::detail::radix::policy_hub<KeyT, ValueT, OffsetT>;
    using P = typename Base::Policy1000;
    struct Policy1000 : cub::ChainedPolicy<1000, Policy1000, Policy1000> {
        using ScanPolicy = typename P::ScanPolicy;
        using DownsweepPolicy = typename P::DownsweepPolicy;
        using AltDownsweepPolicy = typename P::AltDownsweepPolicy;
        using UpsweepPolicy = typename P::UpsweepPolicy;
        using AltUpsweepPolicy = typename P::AltUpsweepPolicy;
        using SingleTilePolicy = typename P::SingleTilePolicy;
        using SegmentedPolicy = typename P::SegmentedPolicy;
        using AltSegmentedPolicy = typename P::AltSegmentedPolicy;
        static constexpr bool ONESWEEP = true;
        static constexpr int ONESWEEP_RADIX_BITS = RB;
        using HistogramPolicy = cub::AgentRadixSortHistogramPolicy<128, 16, 1, KeyT, RB>;
        using ExclusiveSumPolicy = cub::AgentRadixSortExclusiveSumPolicy<256, RB>;
        using DominantT = ::cuda::std::_If<(sizeof(ValueT) > sizeof(KeyT)), ValueT, KeyT>;
        using OnesweepPolicy = cub::AgentRadixSortOnesweepPolicy<
            (RB <= 9 ? 384 : (RB == 10 ? 192 : 64)), ITEMS_I, DominantT, 1, cub::RADIX_RANK_MATCH_EARLY_COUNTS_ANY, cub::BLOCK_SCAN_RAKING_MEMOIZE,
            cub::RADIX_SORT_STORE_DIRECT, RB>;
    };
    using MaxPolicy = Policy1000;
};

__global__ void fill(unsigned long long *k64, uint32_t *k32, uint32_t *v32, unsigned long long *v64, long long n, int which) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        unsigned long long z = (unsigned long long)i * 0x9E3779B97F4A7C15ULL + 12345;
        z ^= z >> 31; z *= 0xBF58476D1CE4E5B9ULL; z ^= z >> 29;
        if (which == 0) {
            double w = (double)(z >> 11) * 0x1.0p-53;
            unsigned long long b = __double_as_longlong(w);
            k64[i] = b; v32[i] = (uint32_t)i;
        } else {
            k32[i] = (uint32_t)(z % (1u << 26)); v64[i] = z;
        }
    }
}

template <typename K, typename V, int RB>
float run(K *k0, K *k1, V *v0, V *v1, long long n, int bits) {
    using D = cub::DispatchRadixSort<false, K, V, unsigned long long, Hub<K, V, unsigned long long, RB>>;
    cub::DoubleBuffer<K> dk(k0, k1);
    cub::DoubleBuffer<V> dv(v0, v1);
    size_t tb = 0;
    D::Dispatch(nullptr, tb, dk, dv, (unsigned long long)n, 0, bits, true, 0);
    void *tmp; cudaMalloc(&tmp, tb);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
        cub::DoubleBuffer<K> k(k0, k1); cub::DoubleBuffer<V> v(v0, v1);
        cudaEventRecord(a);
        cudaError_t e = D::Dispatch(tmp, tb, k, v, (unsigned long long)n, 0, bits, true, 0);
        cudaEventRecord(b); cudaEventSynchronize(b);
        if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); exit(1); }
        float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
        // sortedness check on a sample
        if (r == 0) {
            K *hk = (K *)malloc(sizeof(K) * 4096);
            cudaMemcpy(hk, k.Current() + n / 2, sizeof(K) * 4096, cudaMemcpyDeviceToHost);
            for (int i = 1; i < 4096; ++i) if (hk[i] < hk[i - 1]) { printf("NOT SORTED\n"); exit(1); }
            free(hk);
        }
    }
    cudaFree(tmp);
    return best;
}

int main(int argc, char **argv) {
    int which = atoi(argv[1]);
    long long n = argc > 2 ? atoll(argv[2]) : (which == 0 ? 1073741824LL : 2147483648LL);
    unsigned long long *k64a = 0, *k64b = 0, *v64a = 0, *v64b = 0; uint32_t *k32a = 0, *k32b = 0, *v32a = 0, *v32b = 0;
    if (which == 0) { cudaMalloc(&k64a, n * 8); cudaMalloc(&k64b, n * 8); cudaMalloc(&v32a, n * 4); cudaMalloc(&v32b, n * 4); }
    else { cudaMalloc(&k32a, n * 4); cudaMalloc(&k32b, n * 4); cudaMalloc(&v64a, n * 8); cudaMalloc(&v64b, n * 8); }
    for (int rb = 8; rb <= 11; ++rb) {
        fill<<<148 * 16, 256>>>(k64a, k32a, v32a, v64a, n, which);
        cudaDeviceSynchronize();
        float ms = 0;
        if (which == 0) {
            int bits = 64;
            if (rb == 8) ms = run<unsigned long long, uint32_t, 8>(k64a, k64b, v32a, v32b, n, bits);
            if (rb == 9) ms = run<unsigned long long, uint32_t, 9>(k64a, k64b, v32a, v32b, n, bits);
            if (rb == 10) ms = run<unsigned long long, uint32_t, 10>(k64a, k64b, v32a, v32b, n, bits);
            if (rb == 11) ms = run<unsigned long long, uint32_t, 11>(k64a, k64b, v32a, v32b, n, bits);
        } else {
            int bits = 26;
            if (rb == 8) ms = run<uint32_t, unsigned long long, 8>(k32a, k32b, v64a, v64b, n, bits);
            if (rb == 9) ms = run<uint32_t, unsigned long long, 9>(k32a, k32b, v64a, v64b, n, bits);
            if (rb == 10) ms = run<uint32_t, unsigned long long, 10>(k32a, k32b, v64a, v64b, n, bits);
            if (rb == 11) ms = run<uint32_t, unsigned long long, 11>(k32a, k32b, v64a, v64b, n, bits);
        }
        printf("which %d n %lld radix_bits %d: %.2f ms\n", which, n, rb, ms);
        fflush(stdout);
    }
    return 0;
}
