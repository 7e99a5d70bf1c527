// Host-facing merge declarations (qc_merge.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <deque>
#include <utility>
#include <vector>

namespace qcg {

struct qc_edge_t {  // == qc_edge (qcgpu.h) == qcut::Edge layout
    uint32_t u, v;
    double w;
};

struct MergeInput {
    int n = 0;                       // vertices
    long long m = 0;                 // edges
    const qc_edge_t* edges = nullptr;  // AoS edges, or null when the SoA arrays are given
    const uint32_t* eu = nullptr;    // SoA edges (u < v) -- the pipeline's HostGraph arrays
    const uint32_t* ev = nullptr;
    const double* ew = nullptr;
    int all_int = -1;                // every weight a nonnegative integer (-1: compute)
    int levels = 0;                  // pool levels
    const int32_t* widths = nullptr;
    const int32_t* counts = nullptr;
    const uint32_t* bits = nullptr;  // concatenated, pool order
    int pieces = 0;                  // chain pieces
    const int32_t* first = nullptr;
    const int32_t* last = nullptr;
};

// One exhaustive search over levels [s, e). need: 2 free, 3 halve (bit 0 clear),
// -1 = seam bit read from the assignment committed by the previous window.
struct Window {
    int s, e, need;
};

struct MergeOutput {
    double value = 0.0;              // cut_value of the best assignment (re-scored)
    std::vector<uint8_t> assignment; // n bytes
    uint64_t leaves = 0;
};

void check_pool(const MergeInput& in);
double estimate_paths(const int32_t* counts, int M, bool halve);
// Runs the windows back to back on `st` and returns the re-scored result.
// full_graph selects MergeEval::kFullGraph scoring (merge.hpp:164) on the exact path.
// Device scratch reused across merges (allocation i of a call reuses buffer i).
struct DeviceArena {
    std::deque<std::pair<void*, size_t>> bufs;
    size_t next = 0;
    void reset() { next = 0; }
    void* get(size_t bytes) {
        if (bytes == 0) bytes = 16;
        if (next == bufs.size()) bufs.emplace_back(nullptr, 0);
        auto& b = bufs[next++];
        if (b.second < bytes) {
            if (b.first) cudaFree(b.first);
            b.first = nullptr;
            b.second = 0;
            if (cudaMalloc(&b.first, bytes) != cudaSuccess) {
                (void)cudaGetLastError();
                b.first = nullptr;
                return nullptr;
            }
            b.second = bytes;
        }
        return b.first;
    }
    ~DeviceArena() {
        for (auto& b : bufs)
            if (b.first) cudaFree(b.first);
    }
};

struct Prof;
MergeOutput run_merge(const MergeInput& in, const std::vector<Window>& windows, bool full_graph,
                      cudaStream_t st, uint64_t* launches, Prof* prof = nullptr,
                      uint64_t* h2d = nullptr, uint64_t* d2h = nullptr,
                      DeviceArena* arena = nullptr);

}  // namespace qcg
