// jit.cu — NVRTC compile + cudaLibrary load + caches for the specialised tile kernels.
#include "jit.h"

#include <cuda.h>

#include <dlfcn.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <map>
#include <mutex>
#include <sstream>
#include <thread>
#include <algorithm>
#include <atomic>

#include "common.cuh"
#include "jit_prelude.h"

namespace qbg {
namespace jit {

namespace {

// minimal NVRTC ABI (nvrtc.h), resolved with dlopen so libqbg.so loads without NVRTC
typedef int nvrtcResult;
typedef struct _nvrtcProgram* nvrtcProgram;
struct Nvrtc {
    void* h = nullptr;
    nvrtcResult (*create)(nvrtcProgram*, const char*, const char*, int, const char* const*, const char* const*);
    nvrtcResult (*compile)(nvrtcProgram, int, const char* const*);
    nvrtcResult (*logsize)(nvrtcProgram, size_t*);
    nvrtcResult (*log)(nvrtcProgram, char*);
    nvrtcResult (*cubinsize)(nvrtcProgram, size_t*);
    nvrtcResult (*cubin)(nvrtcProgram, char*);
    nvrtcResult (*destroy)(nvrtcProgram*);
    bool ok = false;
};

Nvrtc& nvrtc() {
    static Nvrtc n;
    static bool tried = false;
    if (tried) return n;
    tried = true;
    const char* names[] = {"libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so"};
    for (const char* nm : names) {
        n.h = dlopen(nm, RTLD_NOW | RTLD_LOCAL);
        if (n.h) break;
    }
    if (!n.h) return n;
    n.create = reinterpret_cast<decltype(n.create)>(dlsym(n.h, "nvrtcCreateProgram"));
    n.compile = reinterpret_cast<decltype(n.compile)>(dlsym(n.h, "nvrtcCompileProgram"));
    n.logsize = reinterpret_cast<decltype(n.logsize)>(dlsym(n.h, "nvrtcGetProgramLogSize"));
    n.log = reinterpret_cast<decltype(n.log)>(dlsym(n.h, "nvrtcGetProgramLog"));
    n.cubinsize = reinterpret_cast<decltype(n.cubinsize)>(dlsym(n.h, "nvrtcGetCUBINSize"));
    n.cubin = reinterpret_cast<decltype(n.cubin)>(dlsym(n.h, "nvrtcGetCUBIN"));
    n.destroy = reinterpret_cast<decltype(n.destroy)>(dlsym(n.h, "nvrtcDestroyProgram"));
    n.ok = n.create && n.compile && n.logsize && n.log && n.cubinsize && n.cubin && n.destroy;
    return n;
}

std::mutex g_mu;
std::map<uint64_t, cudaLibrary_t> g_libs;  // source hash -> loaded library
std::atomic<int64_t> g_nvrtc_builds{0}, g_cache_hits{0};  // qbg_jit_stats

// Kernel cache: QBG_JIT_CACHE if set, else `jit_cache/` next to libqbg.so (in-tree: build()
// pre-compiles the kernels of the standard workloads there on the CPU host — NVRTC needs no GPU —
// so they travel with the library and a fresh GPU box does not pay the first-call compile), else
// ~/.cache/qbg_jit when the library directory is read-only.
std::string cache_dir() {
    const char* e = std::getenv("QBG_JIT_CACHE");
    if (e && *e) return e;
    static const std::string d = [] {
        Dl_info info{};
        if (dladdr(reinterpret_cast<void*>(&fnv), &info) && info.dli_fname) {
            std::string lib = info.dli_fname;
            const std::string dir = lib.substr(0, lib.rfind('/'));
            if (!dir.empty() && ::access(dir.c_str(), W_OK) == 0) return dir + "/jit_cache";
        }
        const char* home = std::getenv("HOME");
        return std::string(home ? home : "/tmp") + "/.cache/qbg_jit";
    }();
    return d;
}

bool read_file(const std::string& p, std::string& out) {
    std::ifstream f(p, std::ios::binary);
    if (!f) return false;
    std::ostringstream ss;
    ss << f.rdbuf();
    out = ss.str();
    return !out.empty();
}

void write_file(const std::string& p, const std::string& data) {
    std::string dir = cache_dir();
    ::mkdir((dir.substr(0, dir.rfind('/'))).c_str(), 0755);
    ::mkdir(dir.c_str(), 0755);
    std::string tmp = p + ".tmp" + std::to_string(::getpid());
    {
        std::ofstream f(tmp, std::ios::binary);
        if (!f) return;
        f.write(data.data(), static_cast<std::streamsize>(data.size()));
    }
    std::rename(tmp.c_str(), p.c_str());
}

std::string build_cubin(const std::string& src, uint64_t key) {
    g_nvrtc_builds.fetch_add(1);
    Nvrtc& n = nvrtc();
    if (!n.ok) raise(QBG_ERR_INTERNAL, "jit: NVRTC is not available");
    std::string full = std::string(kPrelude) + src;
    nvrtcProgram prog;
    if (n.create(&prog, full.c_str(), "qbg_pass.cu", 0, nullptr, nullptr) != 0) raise(QBG_ERR_INTERNAL, "jit: nvrtcCreateProgram failed");
    const char* opts[] = {"-arch=sm_100a", "-std=c++17", "-lineinfo", "-default-device", "--restrict"};
    int rc = n.compile(prog, 5, opts);
    if (rc != 0) {
        size_t ls = 0;
        n.logsize(prog, &ls);
        std::string log(ls, '\0');
        n.log(prog, log.data());
        n.destroy(&prog);
        raise(QBG_ERR_INTERNAL, "jit: NVRTC compilation failed (key " + std::to_string(key) + "):\n" + log.substr(0, 4000));
    }
    size_t cs = 0;
    n.cubinsize(prog, &cs);
    std::string cub(cs, '\0');
    n.cubin(prog, cub.data());
    n.destroy(&prog);
    return cub;
}

}  // namespace

uint64_t fnv(const std::string& s) {
    uint64_t h = 1469598103934665603ULL;
    for (unsigned char c : s) {
        h ^= c;
        h *= 1099511628211ULL;
    }
    return h;
}

// chunks of whole kernels per cubin: a fixed count, so the chunk sources (and their cache keys)
// do not depend on the host's core count — cubins built on the CPU host are found on the GPU box
constexpr size_t kChunks = 16;

size_t compile_only(const std::string& src) {
    const uint64_t key = fnv(std::string(kPrelude) + src);
    char fname[64];
    std::snprintf(fname, sizeof(fname), "/%016llx.cubin", static_cast<unsigned long long>(key));
    std::string cub;
    if (!read_file(cache_dir() + fname, cub)) {
        cub = build_cubin(src, key);
        write_file(cache_dir() + fname, cub);  // the ahead-of-time cache the runtime looks up
    }
    // QBG_JIT_DUMP=<dir>: keep the cubin for offline inspection (cuobjdump -sass / -res-usage)
    if (const char* d = std::getenv("QBG_JIT_DUMP")) {
        char name[64];
        std::snprintf(name, sizeof(name), "/%016llx.cubin", static_cast<unsigned long long>(key));
        std::ofstream f(std::string(d) + name, std::ios::binary);
        f.write(cub.data(), static_cast<std::streamsize>(cub.size()));
    }
    return cub.size();
}

bool enabled() {
    const char* e = std::getenv("QBG_JIT");
    if (e && e[0] == '0') return false;
    return nvrtc().ok;
}

std::vector<Kernel> compile(const std::string& src, const std::vector<std::string>& names) {
    std::lock_guard<std::mutex> lk(g_mu);
    const uint64_t key = fnv(std::string(kPrelude) + src);
    cudaLibrary_t lib = nullptr;
    auto it = g_libs.find(key);
    if (it != g_libs.end()) {
        lib = it->second;
    } else {
        char name[64];
        std::snprintf(name, sizeof(name), "/%016llx.cubin", static_cast<unsigned long long>(key));
        const std::string path = cache_dir() + name;
        std::string cub;
        if (!read_file(path, cub)) {
            cub = build_cubin(src, key);
            write_file(path, cub);
        } else {
            g_cache_hits.fetch_add(1);
        }
        cudaError_t e = cudaLibraryLoadData(&lib, cub.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
        if (e != cudaSuccess) {
            // a stale / foreign cache entry: rebuild once
            cudaGetLastError();
            cub = build_cubin(src, key);
            write_file(path, cub);
            QBG_CUDA(cudaLibraryLoadData(&lib, cub.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
        }
        g_libs[key] = lib;
    }
    std::vector<Kernel> out;
    for (const auto& nm : names) {
        Kernel k;
        QBG_CUDA(cudaLibraryGetKernel(&k.k, lib, nm.c_str()));
        out.push_back(k);
    }
    return out;
}

std::vector<Kernel> compile_parallel(const std::vector<std::string>& bodies, const std::vector<std::string>& names) {
    // chunks of whole kernels; each chunk is its own cached cubin / library, the missing ones are
    // built by concurrent NVRTC invocations (first use of a large circuit: seconds, not tens)
    const size_t nk = bodies.size();
    const size_t nchunk = std::max<size_t>(1, std::min(nk, kChunks));
    std::vector<std::string> srcs(nchunk);
    std::vector<std::vector<size_t>> members(nchunk);
    for (size_t i = 0; i < nk; ++i) {
        srcs[i * nchunk / nk] += bodies[i];
        members[i * nchunk / nk].push_back(i);
    }
    std::vector<uint64_t> keys(nchunk);
    std::vector<std::string> cubs(nchunk);
    std::vector<char> need(nchunk, 0);
    std::lock_guard<std::mutex> lk(g_mu);
    for (size_t c = 0; c < nchunk; ++c) {
        keys[c] = fnv(std::string(kPrelude) + srcs[c]);
        if (g_libs.count(keys[c])) continue;
        char name[64];
        std::snprintf(name, sizeof(name), "/%016llx.cubin", static_cast<unsigned long long>(keys[c]));
        if (!read_file(cache_dir() + name, cubs[c])) need[c] = 1;
        else g_cache_hits.fetch_add(1);
    }
    std::vector<std::string> errs(nchunk);
    {
        std::vector<std::thread> th;
        for (size_t c = 0; c < nchunk; ++c)
            if (need[c])
                th.emplace_back([&, c] {
                    try {
                        cubs[c] = build_cubin(srcs[c], keys[c]);
                    } catch (const std::exception& e) {
                        errs[c] = e.what();
                    }
                });
        for (auto& t : th) t.join();
    }
    for (size_t c = 0; c < nchunk; ++c)
        if (!errs[c].empty()) raise(QBG_ERR_INTERNAL, errs[c]);
    std::vector<Kernel> out(nk);
    for (size_t c = 0; c < nchunk; ++c) {
        cudaLibrary_t lib = nullptr;
        auto it = g_libs.find(keys[c]);
        if (it != g_libs.end()) {
            lib = it->second;
        } else {
            char name[64];
            std::snprintf(name, sizeof(name), "/%016llx.cubin", static_cast<unsigned long long>(keys[c]));
            if (need[c]) write_file(cache_dir() + name, cubs[c]);
            cudaError_t e = cudaLibraryLoadData(&lib, cubs[c].data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
            if (e != cudaSuccess) {  // a stale / foreign cache entry: rebuild once
                cudaGetLastError();
                cubs[c] = build_cubin(srcs[c], keys[c]);
                write_file(cache_dir() + name, cubs[c]);
                QBG_CUDA(cudaLibraryLoadData(&lib, cubs[c].data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
            }
            g_libs[keys[c]] = lib;
        }
        for (size_t i : members[c]) QBG_CUDA(cudaLibraryGetKernel(&out[i].k, lib, names[i].c_str()));
    }
    return out;
}

size_t compile_only_parallel(const std::vector<std::string>& bodies) {
    const size_t nk = bodies.size();
    if (nk == 0) return 0;
    const size_t nchunk = std::max<size_t>(1, std::min(nk, kChunks));
    std::vector<std::string> srcs(nchunk);
    for (size_t i = 0; i < nk; ++i) srcs[i * nchunk / nk] += bodies[i];
    std::vector<size_t> sizes(nchunk, 0);
    std::vector<std::string> errs(nchunk);
    std::vector<std::thread> th;
    for (size_t c = 0; c < nchunk; ++c)
        th.emplace_back([&, c] {
            try {
                sizes[c] = compile_only(srcs[c]);
            } catch (const std::exception& e) {
                errs[c] = e.what();
            }
        });
    for (auto& t : th) t.join();
    size_t total = 0;
    for (size_t c = 0; c < nchunk; ++c) {
        if (!errs[c].empty()) raise(QBG_ERR_INTERNAL, errs[c]);
        total += sizes[c];
    }
    return total;
}

void encode_tensor_map(void* map, const void* gaddr, int rank, const uint64_t* sizes, const uint64_t* strides,
                       const uint32_t* box) {
    typedef CUresult (*Encode)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static Encode fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<Encode>(f);
    }();
    if (!fn) raise(QBG_ERR_INTERNAL, "tma: cuTensorMapEncodeTiled is not available");
    cuuint64_t dims[5], str[5];
    cuuint32_t bx[5], es[5];
    for (int d = 0; d < rank; ++d) {
        dims[d] = sizes[d];
        bx[d] = box[d];
        es[d] = 1;
        if (d > 0) str[d - 1] = strides[d];
    }
    CUresult r = fn(static_cast<CUtensorMap*>(map), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, static_cast<cuuint32_t>(rank),
                    const_cast<void*>(gaddr), dims, str, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) raise(QBG_ERR_INTERNAL, "tma: cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
}

void launch(Kernel& k, unsigned grid, unsigned block, size_t smem, void** args) {
    if (static_cast<int>(smem) > k.max_dyn_smem) {
        int dev = 0;
        QBG_CUDA(cudaGetDevice(&dev));
        QBG_CUDA(cudaKernelSetAttributeForDevice(k.k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem), dev));
        k.max_dyn_smem = static_cast<int>(smem);
    }
    // programmatic dependent launch: the next pass's launch and prologue (barrier init, gradient
    // cells) overlap this pass's tail; the generated kernels wait (griddepcontrol.wait) before
    // touching global memory
    static const bool pdl = [] {
        const char* e = std::getenv("QBG_PDL");
        return !(e && e[0] == '0');
    }();
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream();
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    QBG_CUDA(cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(k.k), args));
}

void stats(int64_t* builds, int64_t* hits) {
    if (builds) *builds = g_nvrtc_builds.load();
    if (hits) *hits = g_cache_hits.load();
}

}  // namespace jit
}  // namespace qbg
