// Drop-in under the reference's header name: metrics.hpp (EpochMetrics, TrainReport, metrics_csv_string, write_metrics_csv)
// over the B200 library (ggb.hpp, the C ABI of include/ggb.h).
#pragma once

#include "ggb.hpp"
