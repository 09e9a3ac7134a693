// Launch timing for the bench's per-kernel roofline pass: a pool of CUDA events recorded by index
// from the host wrappers (one C call per record instead of the torch Event path, whose host cost
// per record had made the event-bracketed pass host-bound: every bracket then held launch latency
// instead of device time).
#include <string>
#include <vector>
#include <cuda_runtime.h>
#include "dpipe.h"

namespace dp {
void set_error(const std::string& s);
static std::vector<cudaEvent_t> g_events;
}  // namespace dp

extern "C" {

int dp_timing_events(int n) {
  using namespace dp;
  while (static_cast<int>(g_events.size()) < n) {
    cudaEvent_t e;
    cudaError_t r = cudaEventCreate(&e);
    if (r != cudaSuccess) {
      set_error(std::string("dp_timing_events: ") + cudaGetErrorString(r));
      return r;
    }
    g_events.push_back(e);
  }
  return 0;
}

int dp_timing_record(int i, dp_stream_t stream) {
  using namespace dp;
  if (i < 0 || i >= static_cast<int>(g_events.size())) {
    set_error("dp_timing_record: event index out of range");
    return DP_ERR_ARGS;
  }
  return cudaEventRecord(g_events[i], reinterpret_cast<cudaStream_t>(stream));
}

float dp_timing_elapsed(int i, int j) {
  using namespace dp;
  const int n = static_cast<int>(g_events.size());
  if (i < 0 || j < 0 || i >= n || j >= n) return -1.f;
  float ms = -1.f;
  if (cudaEventElapsedTime(&ms, g_events[i], g_events[j]) != cudaSuccess) return -1.f;
  return ms;
}

}  // extern "C"
