// Kernel instantiations for tie order pi = 312 (P:90 codes, highest priority first).
#include "nw_launch.cuh"
namespace nwk {
NW_DEFINE_DIRS_LAUNCHERS(312)
}  // namespace nwk
