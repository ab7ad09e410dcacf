// scan_tensor.cu -- placeholder until the tensor-core kernel lands.
#include "scan_tensor.h"

namespace rbe_dev {

bool tensor_supported(const Shape&, uint32_t, const rbe_scan_geometry&, uint32_t, std::string* why) {
    if (why) *why = "tensor kernel not built";
    return false;
}

TensorScanPlan plan_tensor_scan(const Shape&, uint32_t, const rbe_scan_geometry&, uint32_t, const PartDesc*, uint32_t,
                                uint64_t, uint32_t) {
    throw std::logic_error("tensor kernel not built");
}

uint32_t run_tensor_scan(const TensorScanPlan&, const ScanArgs&, const Shape&, const uint64_t*, void*, void*, void*,
                         void*, unsigned long long*, cudaStream_t) {
    throw std::logic_error("tensor kernel not built");
}

}  // namespace rbe_dev
