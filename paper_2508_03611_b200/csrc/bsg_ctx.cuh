// bsg_ctx.cuh — the C-ABI context (opaque bsg_ctx of include/blocksim_b200.h)
// and its device-buffer helper, shared by the CUDA translation units
// (bsg_capi.cu, closed_loop.cu).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "scenario_sim.cuh"

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  bool ensure(size_t bytes) {
    if (bytes <= cap) return true;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t want = std::max<size_t>(bytes, 1 << 16);
    if (cudaMalloc(&p, want) != cudaSuccess) return false;
    cap = want;
    return true;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

struct bsg_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  // chunked host-buffer pipeline: pipe[0] copies, pipe[1..kPipe) run chunks
  static constexpr int kPipe = 7;
  cudaStream_t pipe[kPipe] = {};
  cudaEvent_t pipe_done[kPipe] = {};
  static constexpr int kPieces = 16;
  cudaEvent_t piece_ev[kPieces] = {};  // entry pieces landed (host-buffer pipeline)
  std::string last_error;
  std::string last_launch;  // the simulation kernel(s) the last call launched
  int64_t launches = 0;
  int64_t scenarios = 0;  // predict() scenarios simulated (MC: request x instance x sample)
  std::vector<bsg_instance_cfg> host_cfgs;
  std::vector<bsg::DevCfg> dev_cfgs_host;
  DevBuf cfgs, prompt, est, prefill, decoded, scen, res, rec, ids, chosen;
  DevBuf blob, scores, samples, counters;
  void* pinned = nullptr;   // host staging for single-copy uploads
  size_t pinned_cap = 0;
  int32_t ncfg = 0;
  int32_t max_batch_all = 0;
  bool all_pow2 = false;  // every config's block_size is a power of two
  std::mutex mu;
};


// Records a CUDA failure on the context (and clears a non-sticky error so the
// context's next call is not poisoned); returns BSG_CUDA_ERROR.
bsg_status bsg_cuda_fail(bsg_ctx* ctx, cudaError_t e, const char* what);
