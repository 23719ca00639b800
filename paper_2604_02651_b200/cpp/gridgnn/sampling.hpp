// Drop-in under the reference's header name: sampling.hpp (SampleSet, sample_vertices)
// over the B200 library (ggb.hpp, the C ABI of include/ggb.h).
#pragma once

#include "ggb.hpp"
