// Host-side check of the lane-refill index maps' FastDiv (refill.cuh): the multiply-high
// division must equal n / d for every divisor the kernels use and for random n < 2^32.
// Built and run by tests/test_fastdiv.py on the CPU (nvcc compiles; no GPU needed).
#include <cstdio>
#include <cstdint>
#include <random>
#include "../../paper_2206_02255_b200/csrc/refill.cuh"

static uint32_t host_fdiv(uint32_t n, const mandel::FastDiv &f)
{
    const uint32_t t = (uint32_t)(((uint64_t)n * f.m) >> 32);
    return (t + ((n - t) >> f.s1)) >> f.s2;
}

int main()
{
    std::mt19937_64 rng(20220605);
    long bad = 0, checked = 0;
    std::vector<uint32_t> ds;
    for (uint32_t d = 1; d < 5000; ++d) ds.push_back(d);
    for (int i = 0; i < 3000; ++i) ds.push_back((uint32_t)(rng() >> 32) | 1u);
    ds.push_back(0x80000000u); ds.push_back(0xffffffffu); ds.push_back(900); ds.push_back(8188);
    for (uint32_t d : ds) {
        mandel::FastDiv f = mandel::make_fastdiv(d);
        uint32_t ns[8] = {0u, 1u, d - 1u, d, d + 1u, 0xffffffffu, 0xfffffffeu, (uint32_t)(rng() >> 32)};
        for (uint32_t n : ns) { ++checked; if (host_fdiv(n, f) != n / d) ++bad; }
        for (int k = 0; k < 64; ++k) { uint32_t n = (uint32_t)(rng() >> 32); ++checked; if (host_fdiv(n, f) != n / d) ++bad; }
    }
    printf("checked %ld bad %ld\n", checked, bad);
    return bad != 0;
}
