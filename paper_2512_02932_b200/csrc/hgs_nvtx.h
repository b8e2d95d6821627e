// NVTX ranges around the C ABI's entry points and their stages (host-side
// enqueue intervals; nsys / ncu --nvtx correlate them with the kernels).
// Header-only NVTX3: without an attached tool each push / pop is one
// predicted branch.
#pragma once
#include <nvtx3/nvToolsExt.h>

namespace hgs {
class NvtxScope {
 public:
  explicit NvtxScope(const char *name) { push(name); }
  // end the current stage (if any) and open the next one inside the call's range
  void stage(const char *name) {
    if (depth_ > 1) {
      nvtxRangePop();
      --depth_;
    }
    push(name);
  }
  ~NvtxScope() {
    while (depth_-- > 0) nvtxRangePop();
  }
  NvtxScope(const NvtxScope &) = delete;
  NvtxScope &operator=(const NvtxScope &) = delete;

 private:
  void push(const char *name) {
    nvtxRangePushA(name);
    ++depth_;
  }
  int depth_ = 0;
};
}  // namespace hgs
