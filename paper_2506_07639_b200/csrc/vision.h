// Vision tower + projector (vision.cu): observation image -> VIS rows.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "gemm_tc.h"

#define CK_VIS(x)                                                                                   \
  do {                                                                                              \
    cudaError_t _e = (x);                                                                           \
    if (_e != cudaSuccess) throw std::runtime_error(std::string("vision: ") + cudaGetErrorString(_e)); \
  } while (0)

namespace fe {

struct VisionDims {
  int img, patch, d, L, H, mlp, ph;
  float eps;
};

class Vision {
 public:
  // dtype 0: fp32 canonical (bit-exact with the oracle), 1: bf16 (tcgen05 linears)
  Vision(const VisionDims& v, int dtype, int out_d, uint64_t seed, cudaStream_t s,
         std::function<void*(size_t)> alloc);
  ~Vision();
  // out: [P][out_d] fp32 VIS rows of the observation seeded `vseed`
  void encode(uint64_t vseed, float* out, cudaStream_t s);
  int patches_count() const { return P; }

 private:
  struct Lin;
  struct Layer {
    float *ln1_g, *ln1_b, *ln2_g, *ln2_b;
    std::unique_ptr<Lin> qkv, o, fc1, fc2;
  };
  void linear(const Lin& L, const float* x, float* y, int mode, float* resid, const float* pos, cudaStream_t s);

  VisionDims v;
  int dtype, out_d, grid = 0, P = 0, hd = 0, kp = 0;
  std::unique_ptr<Lin> pe, p1, p2;
  float *pos = nullptr, *lnf_g = nullptr, *lnf_b = nullptr;
  std::vector<Layer> layers;
  float *patches = nullptr, *x = nullptr, *ln = nullptr, *big = nullptr, *att = nullptr;
  __nv_bfloat16* stage = nullptr;
  float* split = nullptr;  // split-K planes of the pair GEMM
  size_t split_floats = 0;
  TmaMap stage_maps[4];
};

}  // namespace fe
