// Status strings, version and launch counter of the C ABI.
#include "host.cuh"

extern "C" const char* ms_status_string(int32_t s) {
  switch (s) {
    case MS_OK: return "MS_OK";
    case MS_ERR_SHAPE: return "MS_ERR_SHAPE";
    case MS_ERR_DTYPE: return "MS_ERR_DTYPE";
    case MS_ERR_ALIGN: return "MS_ERR_ALIGN";
    case MS_ERR_UNSUPPORTED: return "MS_ERR_UNSUPPORTED";
    case MS_ERR_LAUNCH: return "MS_ERR_LAUNCH";
    case MS_ERR_WORKSPACE: return "MS_ERR_WORKSPACE";
    default: return "MS_ERR_UNKNOWN";
  }
}

namespace ms {
const char* last_error();
void set_device_bound(int on);
}

extern "C" void ms_set_device_bound(int32_t on) { ms::set_device_bound(on); }

extern "C" const char* ms_last_error(void) { return ms::last_error(); }
extern "C" int32_t ms_version(void) { return 1; }
extern "C" int64_t ms_launch_count(void) { return ms::g_launches.load(); }

extern "C" void ms_launch_stats(int64_t* out4) {
  for (int i = 0; i < ms::KF_COUNT; ++i) out4[i] = ms::g_family[i].load();
}
