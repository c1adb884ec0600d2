// QR tile kernels (placeholder until the kernels land).
#include "tiles.h"
namespace hg {
bool init_qr_attributes() { return true; }
bool build_qr_launches(int kind, const TaskOperands&, std::vector<LaunchDesc>&) {
  set_error("kind %d: QR tile kernels are not built yet", kind);
  return false;
}
}  // namespace hg
