// sf_sim.cu -- device simulator: the same counter-based
// generator as the host (sf_sim_core.h), one warp per spot, so large
// configurations (C4: 1e7 x 32x32, C5: 1e8 x 15x15) are produced in HBM
// without host generation or PCIe.  Integer Philox draws are identical to the
// host; the f64 log/sin/cos/exp/sqrt of CUDA may differ from glibc in the last
// ulp, which after rounding to integer counts changes a pixel only when
// lambda + z*sqrt(lambda) falls within ~1e-15 of a .5 boundary
// (tests/test_gpu_parity.py::test_device_simulator_matches_host).
#include "sf_launch.h"
#include "sf_sim_core.h"

namespace sf {

namespace {
__global__ void __launch_bounds__(256) sim_kernel(sf_sim_config c, int W, int H, int64_t first, int64_t count,
                                                  float* __restrict__ images, float* __restrict__ truth) {
  const int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= count) return;
  const int64_t index = first + s;
  const sfsim::SpotTruth t = sfsim::spot_truth(c, W, H, index);
  const int N = W * H;
  float* img = images + s * (int64_t)N;
  for (int i = lane; i < N; i += 32) {
    double z[4];
    sfsim::pixel_normals(c, index, i, z);
    img[i] = sfsim::pixel_value(c, t, W, i, z[i & 3]);
  }
  if (lane == 0 && truth != nullptr) sfsim::write_truth(c, t, truth + s * (c.model + 2));
}
}  // namespace

cudaError_t launch_simulate(const sf_sim_config& c, int W, int H, int64_t first, int64_t count, float* images,
                            float* truth, cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  const int64_t blocks = (count * 32 + 255) / 256;
  sim_kernel<<<(unsigned)blocks, 256, 0, stream>>>(c, W, H, first, count, images, truth);
  return cudaGetLastError();
}

}  // namespace sf
