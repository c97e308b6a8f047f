// Error plumbing shared by the C-ABI translation units: every extern "C" entry point is
// wrapped in API_BEGIN / API_END (exceptions -> XSLP_E* codes + xslp_last_error); device
// code paths check CUDA runtime calls with CUDA_OK (include after cuda_runtime.h).
#pragma once
#include "xslp_internal.h"

#define API_BEGIN try {
#define API_END                                        \
  }                                                    \
  catch (const Error &e) {                             \
    set_last_error(e.what());                          \
    return e.code;                                     \
  }                                                    \
  catch (const std::bad_alloc &) {                     \
    set_last_error("out of host memory");              \
    return XSLP_ENOMEM;                                \
  }                                                    \
  catch (const std::exception &e) {                    \
    set_last_error(e.what());                          \
    return XSLP_EINVAL;                                \
  }                                                    \
  return XSLP_OK;

#ifdef __CUDA_RUNTIME_H__
#define CUDA_OK(x)                                                                      \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess)                                                              \
      throw Error(XSLP_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_));         \
  } while (0)
#endif
