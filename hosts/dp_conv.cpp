// dp_conv.cpp — C++ data-parallel host for the hash-conv layer, calling only the
// C ABI (include/hashconv_b200.h, hashconv_b200_native.h) plus CUDA streams/events and NCCL.
//
// One process per GPU (RANK / WORLD_SIZE / LOCAL_RANK from the environment, as torchrun sets
// them; the NCCL unique id travels through the file HCB_NCCL_ID, written by rank 0). Every rank
// owns `--shapes` whole shells (weak scaling): its own super-PSH, no data-path communication in
// forward or input gradient; the weight gradient is summed with ONE ncclAllReduce per step,
// issued on a side stream as soon as the dW kernel is enqueued so it overlaps the dX kernel.
// The layer runs at the reference's precision (split-precision tcgen05 path, fp32 in / out).
// Timing: CUDA events around `--steps` steps after `--warmup`, max over ranks (NCCL max).
//
//   dp_conv [--psh FILE] [--res 256] [--shapes 8] [--cin 64] [--cout 64] [--steps 20] [--warmup 5]
#include <cuda_runtime.h>
#include <nccl.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "hashconv_b200.h"
#include "hashconv_b200_native.h"

namespace {

void ck(hc_status s, const char* what) {
    if (s != HC_OK) throw std::runtime_error(std::string(what) + ": " + hc_last_error());
}
void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}
void ck(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw std::runtime_error(std::string(what) + ": " + ncclGetErrorString(r));
}
int env_int(const char* n, int d) {
    const char* e = std::getenv(n);
    return e ? std::atoi(e) : d;
}

struct Dev {  // device buffer
    void* p = nullptr;
    explicit Dev(size_t bytes) { ck(cudaMalloc(&p, bytes ? bytes : 16), "cudaMalloc"); }
    ~Dev() { cudaFree(p); }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

std::vector<float> uniform(size_t n, uint64_t seed) {  // deterministic [-1, 1)
    std::vector<float> v(n);
    uint64_t x = seed * 0x9E3779B97F4A7C15ull + 1;
    for (auto& f : v) {
        x ^= x << 13, x ^= x >> 7, x ^= x << 17;
        f = (float)((x >> 11) * (1.0 / 9007199254740992.0)) * 2.0f - 1.0f;
    }
    return v;
}

ncclUniqueId exchange_id(int rank) {
    ncclUniqueId id;
    const char* path = std::getenv("HCB_NCCL_ID");
    const std::string file = path ? path : "/tmp/hcb_nccl_id";
    if (rank == 0) {
        ck(ncclGetUniqueId(&id), "ncclGetUniqueId");
        const std::string tmp = file + ".tmp";
        FILE* f = std::fopen(tmp.c_str(), "wb");
        if (!f || std::fwrite(&id, sizeof(id), 1, f) != 1) throw std::runtime_error("write " + tmp);
        std::fclose(f);
        std::rename(tmp.c_str(), file.c_str());
    } else {
        for (int i = 0;; ++i) {
            FILE* f = std::fopen(file.c_str(), "rb");
            if (f && std::fread(&id, sizeof(id), 1, f) == 1) {
                std::fclose(f);
                break;
            }
            if (f) std::fclose(f);
            if (i > 6000) throw std::runtime_error("no NCCL id in " + file);
            std::this_thread::sleep_for(std::chrono::milliseconds(10));
        }
    }
    return id;
}

}  // namespace

int main(int argc, char** argv) {
    std::string psh;
    int res = 256, shapes = 8, cin = 64, cout = 64, steps = 20, warmup = 5;
    for (int i = 1; i + 1 < argc; i += 2) {
        const std::string a = argv[i];
        const char* v = argv[i + 1];
        if (a == "--psh") psh = v;
        else if (a == "--res") res = std::atoi(v);
        else if (a == "--shapes") shapes = std::atoi(v);
        else if (a == "--cin") cin = std::atoi(v);
        else if (a == "--cout") cout = std::atoi(v);
        else if (a == "--steps") steps = std::atoi(v);
        else if (a == "--warmup") warmup = std::max(3, std::atoi(v));
        else {
            std::fprintf(stderr, "unknown option %s\n", a.c_str());
            return 2;
        }
    }
    const int rank = env_int("RANK", 0), world = env_int("WORLD_SIZE", 1), local = env_int("LOCAL_RANK", 0);
    try {
        ck(cudaSetDevice(local), "cudaSetDevice");
        ncclComm_t comm = nullptr;
        if (world > 1) ck(ncclCommInitRank(&comm, world, exchange_id(rank), rank), "ncclCommInitRank");

        // ---- this rank's shapes: the synthetic shell (bench.cpp:33-77), PSH from the .psh cache
        // (psh_io.cpp:65-90) or built on the device (psh.cpp:31-227 semantics)
        hc_psh_level* level = nullptr;
        if (!psh.empty()) {
            hc_psh_level* lv[8] = {};
            int32_t count = 0;
            ck(hc_read_psh_file(psh.c_str(), lv, 8, &count), "read .psh");
            level = lv[0];
            for (int i = 1; i < count; ++i) hc_psh_level_free(lv[i]);
        } else {
            hc_voxel_set* s = nullptr;
            ck(hc_sphere_voxels(res, 1, &s), "sphere_voxels");
            ck(hc_build_psh_device(s, hc_mix_seed(1, 0), &level), "build_psh_device");
            hc_voxel_set_free(s);
        }
        std::vector<const hc_psh_level*> batch(shapes, level);
        cudaStream_t st, side;
        ck(cudaStreamCreate(&st), "stream");
        ck(cudaStreamCreate(&side), "stream");
        hc_psh* fine = nullptr;
        ck(hc_psh_upload_levels(batch.data(), shapes, &fine, st), "psh_upload_levels");
        int64_t info[6];
        ck(hc_psh_info(fine, info), "psh_info");
        const int64_t N = info[5];
        const int taps = 27;
        const hc_conv_spec spec{3, 1, 0, cin, cout};

        // ---- fp32 operands, resident in HBM (voxel-major [N][C]; weights in the reference layout)
        Dev x(N * cin * 4), dy(N * cout * 4), w((size_t)cout * cin * taps * 4);
        {
            auto hx = uniform((size_t)N * cin, 11 + rank), hdy = uniform((size_t)N * cout, 13 + rank);
            auto hw = uniform((size_t)cout * cin * taps, 7);  // every rank starts from the same weights
            ck(cudaMemcpy(x.p, hx.data(), hx.size() * 4, cudaMemcpyHostToDevice), "h2d");
            ck(cudaMemcpy(dy.p, hdy.data(), hdy.size() * 4, cudaMemcpyHostToDevice), "h2d");
            ck(cudaMemcpy(w.p, hw.data(), hw.size() * 4, cudaMemcpyHostToDevice), "h2d");
        }
        Dev fmap(((N + 127) / 128) * 128 * taps * 4), xs(N * 2 * cin * 2), dys(N * 2 * cout * 2);
        Dev wf(2 * cout * hc_native_packed_k_x2(cin, taps) * 2), wb(2 * cin * hc_native_packed_k_x2(cout, taps) * 2);
        Dev y(N * cout * 4), dx(N * cin * 4), dw((size_t)cout * cin * taps * 4);
        const size_t wsb = hc_native_dw_workspace_x2(N, taps, cin, cout);
        if (!wsb) throw std::runtime_error("unsupported dW shape");
        Dev ws(wsb);
        cudaEvent_t dw_done, ar_done, t0, t1;
        for (cudaEvent_t* e : {&dw_done, &ar_done}) ck(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
        ck(cudaEventCreate(&t0), "event");
        ck(cudaEventCreate(&t1), "event");
        const hc_stream S = reinterpret_cast<hc_stream>(st);

        auto step = [&]() {
            ck(hc_field_map_tiled(fine, fine, spec, fmap.as<int32_t>(), S), "field map");
            ck(hc_native_split(x.as<float>(), 0, cin, N, xs.p, S), "split x");
            ck(hc_native_split(dy.as<float>(), 0, cout, N, dys.p, S), "split dy");
            ck(hc_native_pack_weights_x2(w.as<float>(), cout, cin, taps, 0, wf.p, S), "pack");
            ck(hc_native_pack_weights_x2(w.as<float>(), cout, cin, taps, 1, wb.p, S), "pack");
            ck(hc_native_gather_gemm_x2(fmap.as<int32_t>(), 2, N, taps, xs.p, cin, wf.p, cout, y.as<float>(), S),
               "forward");
            ck(hc_native_conv_dw_x2(fmap.as<int32_t>(), 2, N, taps, xs.p, cin, dys.p, cout, dw.as<float>(), ws.p, wsb,
                                    S),
               "dW");
            if (world > 1) {  // the one collective: dW summed over ranks, overlapping dX
                ck(cudaEventRecord(dw_done, st), "record");
                ck(cudaStreamWaitEvent(side, dw_done, 0), "wait");
                ck(ncclAllReduce(dw.p, dw.p, (size_t)cout * cin * taps, ncclFloat32, ncclSum, comm, side),
                   "ncclAllReduce");
                ck(cudaEventRecord(ar_done, side), "record");
            }
            ck(hc_native_gather_gemm_x2(fmap.as<int32_t>(), 2, N, taps, dys.p, cout, wb.p, cin, dx.as<float>(), S),
               "input gradient");
            if (world > 1) ck(cudaStreamWaitEvent(st, ar_done, 0), "wait");
        };
        for (int i = 0; i < warmup; ++i) step();
        ck(cudaStreamSynchronize(st), "sync");
        if (world > 1) {  // barrier
            Dev b(4);
            ck(ncclAllReduce(b.p, b.p, 1, ncclFloat32, ncclSum, comm, st), "barrier");
            ck(cudaStreamSynchronize(st), "sync");
        }
        const int64_t launches0 = hc_launch_count();
        ck(cudaEventRecord(t0, st), "record");
        for (int i = 0; i < steps; ++i) step();
        ck(cudaEventRecord(t1, st), "record");
        ck(cudaStreamSynchronize(st), "sync");
        const int64_t launches = hc_launch_count() - launches0;
        float ms = 0.0f;
        ck(cudaEventElapsedTime(&ms, t0, t1), "elapsed");
        if (world > 1) {  // max over ranks
            Dev m(4);
            ck(cudaMemcpy(m.p, &ms, 4, cudaMemcpyHostToDevice), "h2d");
            ck(ncclAllReduce(m.p, m.p, 1, ncclFloat32, ncclMax, comm, st), "max");
            ck(cudaMemcpy(&ms, m.p, 4, cudaMemcpyDeviceToHost), "d2h");
        }
        const double ms_step = ms / steps;
        if (rank == 0)
            std::printf(
                "{\"host\": \"C++ (hosts/dp_conv.cpp)\", \"metric\": \"hash-conv fwd+bwd occupied voxels/sec\", "
                "\"value\": %.6g, \"unit\": \"voxels/s\", \"n_gpus\": %d, \"steps\": %d, \"warmup\": %d, "
                "\"ms_per_step\": %.6g, \"dtype\": \"f32\", \"scaling\": \"weak\", \"voxels_per_gpu\": %lld, "
                "\"config\": {\"res\": %d, \"shapes_per_gpu\": %d, \"c_in\": %d, \"c_out\": %d}, "
                "\"gpu_launches\": %lld, \"collective\": \"%s\"}\n",
                (double)N * world / (ms_step / 1e3), world, steps, warmup, ms_step, (long long)N, res, shapes, cin,
                cout, (long long)launches, world > 1 ? "ncclAllReduce(dW) on a side stream, overlapping dX" : "none");
        hc_psh_free(fine);
        hc_psh_level_free(level);
        if (comm) ncclCommDestroy(comm);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "dp_conv (rank %d): %s\n", rank, e.what());
        return 1;
    }
    return 0;
}
