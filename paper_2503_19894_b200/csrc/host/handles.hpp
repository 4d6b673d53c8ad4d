// Handle types and error plumbing shared by the C ABI translation units
// (host/capi.cpp and cuda/runtime.cu).  Not part of the public surface.
#pragma once

#include <stdexcept>
#include <string>

#include "tilesim/fusion.hpp"
#include "tilesim/ir.hpp"
#include "tilesim/shard.hpp"
#include "tilesim_cuda.h"

struct tsc_circuit {
  tilesim::Circuit c;
};

struct tsc_shard_plan {
  tilesim::ShardPlan plan;
  uint64_t serial = 0;  // unique per plan: executors key their prepared schedules on it
};

struct tsc_cost_model {
  tilesim::CostModel cm;
};

namespace tsg_detail {

// thread-local message of the last failure (tsg_last_error)
void set_error(const std::string& msg);

// Map an exception to the SPEC.md:587 error classes.
inline int fail(const std::exception& e) {
  set_error(e.what());
  if (dynamic_cast<const tilesim::ParseError*>(&e)) return TSG_ERR_PARSE;
  if (dynamic_cast<const tilesim::ConfigError*>(&e)) return TSG_ERR_CONFIG;
  if (dynamic_cast<const std::invalid_argument*>(&e)) return TSG_ERR_CONFIG;
  return TSG_ERR_SIM;
}

inline void require(bool ok, const char* what) {
  if (!ok) throw tilesim::ConfigError(what);
}

}  // namespace tsg_detail

#define TSG_TRY(...)                                  \
  try {                                               \
    __VA_ARGS__;                                      \
    return TSG_OK;                                    \
  } catch (const std::exception& tsg_e_) {            \
    return tsg_detail::fail(tsg_e_);                  \
  } catch (...) {                                     \
    tsg_detail::set_error("unknown C++ exception");   \
    return TSG_ERR_SIM;                               \
  }
