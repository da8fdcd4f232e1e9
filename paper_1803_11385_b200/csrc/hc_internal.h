// hc_internal.h — shared host-side plumbing of libhcb200.so (not part of the ABI).
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "hashconv_b200.h"
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: a no-op unless a profiler injects a handler

namespace hcb {

// Thrown inside the library; mapped to hc_status at the ABI edge.
struct cuda_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void set_last_error(const std::string& msg);

// Run `f`, converting exceptions to hc_status + thread-local message. Mirrors
// the reference's exception types: std::invalid_argument -> INVALID_ARGUMENT,
// std::runtime_error -> RUNTIME.
// Every ABI entry runs inside guard(), so each call is also one NVTX range named after the entry
// point (nsys / ncu --nvtx show the operator boundaries; SURVEY.md §5 tracing).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

template <class F>
hc_status guard(F&& f, const char* fn = __builtin_FUNCTION()) {
    const NvtxRange range(fn);
    try {
        f();
        return HC_OK;
    } catch (const std::invalid_argument& e) {
        set_last_error(e.what());
        return HC_ERR_INVALID_ARGUMENT;
    } catch (const cuda_error& e) {
        set_last_error(e.what());
        return HC_ERR_CUDA;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return HC_ERR_RUNTIME;
    }
}

using Coord = std::array<std::int32_t, 3>;

// voxel.hpp:16-25 SparseVoxelSet, host side.
struct VoxelSet {
    int dim = 3;
    std::int32_t resolution = 0;
    std::vector<Coord> voxels;      // sorted (z,y,x)
    std::int64_t channels = 0;
    std::vector<float> features;    // channels x n, row-major
    std::int64_t count() const { return static_cast<std::int64_t>(voxels.size()); }
};

// psh.hpp:21-35 PshLevel, host side.
struct PshLevel {
    int dim = 3;
    std::int32_t resolution = 0;
    std::int64_t n = 0;
    std::int32_t hash_dim = 0;
    std::int32_t offset_dim = 0;
    std::vector<std::int32_t> hash;
    std::vector<std::uint8_t> offsets;
    std::vector<std::uint16_t> tags;
    std::int64_t channels = 0;
    std::vector<float> data;  // channels x n
    std::int64_t slots() const;
    std::int64_t cells() const;
};

std::int64_t ipow(std::int64_t b, int e);
std::int32_t psh_hash_dim(std::int64_t n, int dim);          // psh.cpp:170-175 minimal_hash_dim
std::int32_t psh_first_offset_dim(std::int64_t n, int dim);  // psh.cpp:177-183 initial_offset_dim

}  // namespace hcb

struct hc_voxel_set : hcb::VoxelSet {};
struct hc_psh_level : hcb::PshLevel {};
