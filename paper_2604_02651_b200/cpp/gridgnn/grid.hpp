// Drop-in under the reference's header name: grid.hpp (DeviceGrid, Axis)
// over the B200 library (ggb.hpp, the C ABI of include/ggb.h).
#pragma once

#include "ggb.hpp"
