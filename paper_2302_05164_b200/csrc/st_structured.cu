// Structured (uniform box, degree p) backend — see DESIGN.md.
#include "st_common.cuh"

namespace st {

Backend* make_structured(Ctx* c, const st_structured_mesh* m, int* err) {
  (void)c;
  (void)m;
  set_error("structured backend not built yet");
  *err = ST_EUNSUPPORTED;
  return nullptr;
}

}  // namespace st
