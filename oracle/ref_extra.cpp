// Oracle-only C-ABI entry: the reference library has no GPU data path.
// (Test infrastructure; compiled into oracle/_ref/libmsim_ref.so.)
#include "prism_capi.h"

extern "C" int prism_has_device_path(void) { return 0; }
