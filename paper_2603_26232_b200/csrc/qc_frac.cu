// Exact phases for non-integral cost tables (statevector.hpp:162-164).
//
// The reference applies amps[z] *= std::polar(1.0, -gamma * val[z]) with glibc's sin/cos
// for every z. Device sin/cos cannot reproduce glibc bit for bit, but the phase depends on z
// only through val[z], so when the table has few DISTINCT values the host computes the
// polar of each one with the same libm (exactly the reference's operation) and the device
// applies them through the integral path's LUT machinery: lev[z] becomes the index of val[z]
// in the table of distinct values (uint16), while the expectation keeps reading val[z].
// Distinct values are found on the device (radix sort + unique on the values' bit patterns,
// so +0.0 / -0.0 stay apart), then every z looks its value up by binary search. Graphs with
// more than 65,535 distinct values keep the device-sincos path (within 1e-10).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>

#include <cstdint>

#include "qc_internal.hpp"

namespace qcg {

namespace {
__global__ void k_index_of(const unsigned long long* __restrict__ val, uint32_t N,
                           const unsigned long long* __restrict__ uniq, int D, uint16_t* __restrict__ lev) {
    for (uint32_t z = blockIdx.x * blockDim.x + threadIdx.x; z < N; z += gridDim.x * blockDim.x) {
        const unsigned long long v = val[z];
        int lo = 0, hi = D - 1;
        while (lo < hi) {  // first index with uniq[i] >= v (v is present)
            const int mid = (lo + hi) >> 1;
            if (uniq[mid] < v)
                lo = mid + 1;
            else
                hi = mid;
        }
        lev[z] = static_cast<uint16_t>(lo);
    }
}
}  // namespace

size_t distinct_scratch_bytes(uint32_t N) {
    size_t a = 0, b = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, a, static_cast<const unsigned long long*>(nullptr),
                                   static_cast<unsigned long long*>(nullptr), static_cast<int>(N));
    cub::DeviceSelect::Unique(nullptr, b, static_cast<const unsigned long long*>(nullptr),
                              static_cast<unsigned long long*>(nullptr), static_cast<int*>(nullptr),
                              static_cast<int>(N));
    const size_t tmp = (std::max(a, b) + 255) & ~size_t{255};
    return tmp + 2 * ((size_t{N} * 8 + 255) & ~size_t{255}) + 256;
}

// Sorted distinct bit patterns of val[0..N) into scratch; returns the device pointer to them
// and writes their count to *d_count (device int).
const unsigned long long* launch_distinct(const double* d_val, uint32_t N, void* scratch, int* d_count,
                                          cudaStream_t st) {
    size_t a = 0, b = 0;
    const auto* keys = reinterpret_cast<const unsigned long long*>(d_val);
    cub::DeviceRadixSort::SortKeys(nullptr, a, keys, static_cast<unsigned long long*>(nullptr), static_cast<int>(N));
    cub::DeviceSelect::Unique(nullptr, b, keys, static_cast<unsigned long long*>(nullptr), d_count,
                              static_cast<int>(N));
    size_t tmp = (std::max(a, b) + 255) & ~size_t{255};
    char* base = static_cast<char*>(scratch);
    auto* sorted = reinterpret_cast<unsigned long long*>(base + tmp);
    auto* uniq = reinterpret_cast<unsigned long long*>(base + tmp + ((size_t{N} * 8 + 255) & ~size_t{255}));
    QC_CUDA(cub::DeviceRadixSort::SortKeys(base, a, keys, sorted, static_cast<int>(N), 0, 64, st));
    QC_CUDA(cub::DeviceSelect::Unique(base, b, sorted, uniq, d_count, static_cast<int>(N), st));
    return uniq;
}

void launch_index_of(const double* d_val, uint32_t N, const unsigned long long* d_uniq, int D, uint16_t* d_lev,
                     cudaStream_t st) {
    const uint32_t blocks = std::min<uint32_t>((N + 255) / 256, 148u * 16u);
    k_index_of<<<blocks, 256, 0, st>>>(reinterpret_cast<const unsigned long long*>(d_val), N, d_uniq, D, d_lev);
    QC_CUDA(cudaGetLastError());
}

}  // namespace qcg
