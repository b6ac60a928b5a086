// jit.h — runtime specialisation of the tile-pass kernels (NVRTC -> sm_100a cubin).
//
// The fused engine's planner knows, per pass, the tile layout, the register/thread/tile
// location of every target and control bit and the op sequence.  An interpreter kernel must
// decode that at run time (and nvcc re-normalises the whole register tile after every op of a
// switch-in-loop interpreter — measured: ~40% of issued instructions were register moves).
// Instead the planner emits one straight-line kernel per distinct pass structure from the
// templates in jit_prelude.h; gate matrices stay runtime data (a __grid_constant__ parameter,
// i.e. constant-bank operands), so re-parameterising a circuit never recompiles.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

namespace qbg {
namespace jit {

struct Kernel {
    cudaKernel_t k = nullptr;
    int max_dyn_smem = 0;
};

// Compiles (or fetches from the in-memory / on-disk cache) every kernel in `src`, returning the
// handles of `names` in order.  Throws qbg::Error(QBG_ERR_INTERNAL) with the NVRTC log on failure.
std::vector<Kernel> compile(const std::string& src, const std::vector<std::string>& names);

// Same for one kernel body per entry of `bodies` (names[i] defined in bodies[i]): the bodies are
// grouped into chunks compiled concurrently and cached per chunk.
std::vector<Kernel> compile_parallel(const std::vector<std::string>& bodies, const std::vector<std::string>& names);

// NVRTC only (no device): compiles `src` to an sm_100a cubin and returns its size.
size_t compile_only(const std::string& src);
// NVRTC compilations and kernel-cache hits (cubin files) since the library was loaded
void stats(int64_t* builds, int64_t* hits);
// ... one kernel body per entry, compiled in concurrent chunks; total cubin bytes
size_t compile_only_parallel(const std::vector<std::string>& bodies);

// Enabled unless QBG_JIT=0 or NVRTC cannot be loaded.
bool enabled();

// A 128-byte CUtensorMap for an FP64 tensor of `rank` dims: sizes[d] (d = 0 innermost), byte
// strides[d] for d >= 1, box[d]; no swizzle / interleave (cuTensorMapEncodeTiled via the driver
// entry point, so libqbg.so does not link libcuda directly).
void encode_tensor_map(void* map, const void* gaddr, int rank, const uint64_t* sizes, const uint64_t* strides,
                       const uint32_t* box);

// Launch a JIT kernel with `args` (pointers to each argument) on the library stream.
void launch(Kernel& k, unsigned grid, unsigned block, size_t smem, void** args);

// 64-bit FNV-1a, used for cache keys and kernel names
uint64_t fnv(const std::string& s);

}  // namespace jit
}  // namespace qbg
