// Host interfaces of the HBM-bound and attention kernels.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace bfpp {}  // namespace bfpp
