// Status-code plumbing for the C-ABI: every extern "C" body runs inside
// guarded(), which maps exceptions to the codes of include/cad.h and keeps
// the message per thread.
#pragma once

#include <exception>
#include <new>
#include <stdexcept>
#include <string>

#include "../../../include/cad.h"
#include "cad_host.hpp"

namespace cad {

struct CapacityError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NcclError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline std::string& last_error() {
  thread_local std::string msg;
  return msg;
}

template <class F>
int guarded(F&& body) {
  try {
    body();
    last_error().clear();
    return CAD_OK;
  } catch (const ConfigError& e) {
    last_error() = e.what();
    return CAD_ERR_CONFIG;
  } catch (const DomainError& e) {
    last_error() = e.what();
    return CAD_ERR_DOMAIN;
  } catch (const CapacityError& e) {
    last_error() = e.what();
    return CAD_ERR_CAPACITY;
  } catch (const CudaError& e) {
    last_error() = e.what();
    return CAD_ERR_CUDA;
  } catch (const NcclError& e) {
    last_error() = e.what();
    return CAD_ERR_NCCL;
  } catch (const std::bad_alloc&) {
    last_error() = "out of host memory";
    return CAD_ERR_CONFIG;
  } catch (const std::exception& e) {
    last_error() = e.what();
    return CAD_ERR_DOMAIN;
  } catch (...) {
    last_error() = "unknown exception";
    return CAD_ERR_DOMAIN;
  }
}

}  // namespace cad
