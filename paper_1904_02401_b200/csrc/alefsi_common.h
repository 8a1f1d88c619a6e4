// Shared error handling for the alefsi_b200 native library.
#pragma once
#include <cstdio>
#include <exception>
#include <string>

#define ALEFSI_OK 0
#define ALEFSI_ERR_ARG 1
#define ALEFSI_ERR_CUDA 2
#define ALEFSI_ERR_SINGULAR 3
#define ALEFSI_ERR_NOT_CONVERGED 4
#define ALEFSI_ERR_STATE 5
#define ALEFSI_ERR_INTERNAL 6

namespace alefsi {
void set_error(const std::string& msg);
inline int fail(int code, const std::string& msg) {
  set_error(msg);
  return code;
}
}  // namespace alefsi

#define ALEFSI_TRY_BEGIN try {
#define ALEFSI_TRY_END                                             \
  }                                                                \
  catch (const std::exception& ex) {                               \
    return alefsi::fail(ALEFSI_ERR_INTERNAL, ex.what());           \
  }                                                                \
  catch (...) {                                                    \
    return alefsi::fail(ALEFSI_ERR_INTERNAL, "unknown exception"); \
  }
