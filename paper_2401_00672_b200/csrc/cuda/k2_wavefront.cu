// K2 placeholder (filled in by the wavefront kernel).
#include "../plan.h"
namespace pobk {
struct K2Plan {};
bool k2_build(Plan&, const HostCSR&, int, std::string& why) { why = "not built yet"; return false; }
cudaError_t k2_solve(Plan&, cudaStream_t, long long&) { return cudaErrorNotSupported; }
void k2_free(Plan& p) { delete p.k2; p.k2 = nullptr; }
}  // namespace pobk
