// Shared exception -> status mapping of the extern "C" entry points.
#pragma once

#include <exception>
#include <string>

#include "common.cuh"  // stmhd::set_last_error, Error

#define CAPI_BEGIN try {
#define CAPI_END                                   \
  return STMHD_OK;                                 \
  }                                                \
  catch (const stmhd::Error &e) {                  \
    stmhd::set_last_error(e.what(), e.block);      \
    return e.status;                               \
  }                                                \
  catch (const std::exception &e) {                \
    stmhd::set_last_error(e.what());               \
    return STMHD_CONFIG;                           \
  }
