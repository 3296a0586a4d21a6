// capi_handles.hpp -- the opaque handles of include/streamrl_b200.h (shared by
// capi.cpp and comm.cpp).
#pragma once
#include <memory>

#include "runtime.hpp"
#include "trainer.hpp"

struct srl_policy {
  srl::Policy p;
};
struct srl_engine {
  std::unique_ptr<srl::Engine> e;
};
struct srl_trainer {
  std::unique_ptr<srl::DecoderTrainer> t;
};
