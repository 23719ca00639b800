// Drop-in under the reference's header name: dataset.hpp (Dataset, load_dataset, generate_synthetic, SplitTag)
// over the B200 library (ggb.hpp, the C ABI of include/ggb.h).
#pragma once

#include "ggb.hpp"
