// Drop-in under the reference's header name: model.hpp (ModelConfig, TrainConfig, ModelState, init_state, build_step_batch, train_step, dp_sync, optimizer_step, evaluate_full_graph, train_run, train_run_fp32, reference_train)
// over the B200 library (ggb.hpp, the C ABI of include/ggb.h).
#pragma once

#include "ggb.hpp"
#include "pmm.hpp"
#include "shardsample.hpp"
