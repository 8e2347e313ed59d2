// Exception -> status-code translation at the C ABI (SURVEY §8(b) "Errors").
#pragma once
#include <stdexcept>
#include <string>

#include "pswa/pswa_cuda.h"

namespace pswa_abi {

void set_error(const std::string& msg);

struct TruncatedError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct HashError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct LaneError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

template <class F>
int guard(F&& f) noexcept {
  try {
    f();
    return PSWA_OK;
  } catch (const std::invalid_argument& e) {
    set_error(e.what());
    return PSWA_E_ARG;
  } catch (const TruncatedError& e) {
    set_error(e.what());
    return PSWA_E_TRUNCATED;
  } catch (const HashError& e) {
    set_error(e.what());
    return PSWA_E_HASH;
  } catch (const LaneError& e) {
    set_error(e.what());
    return PSWA_E_LANE;
  } catch (const std::runtime_error& e) {
    set_error(e.what());
    return std::string(e.what()).rfind("cuda", 0) == 0 ? PSWA_E_CUDA : PSWA_E_INTERNAL;
  } catch (const std::exception& e) {
    set_error(e.what());
    return PSWA_E_INTERNAL;
  } catch (...) {
    set_error("unknown exception");
    return PSWA_E_INTERNAL;
  }
}

}  // namespace pswa_abi
