// Exception -> status-code bridge for the extern "C" entry points.
#pragma once

#include <new>
#include <string>

#include "errors.hpp"

namespace mtg {

std::string& last_error_slot();

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return kOk;
  } catch (const Error& e) {
    last_error_slot() = e.what();
    return e.status;
  } catch (const std::bad_alloc&) {
    last_error_slot() = "host allocation failed";
    return kValueError;
  } catch (const std::exception& e) {
    last_error_slot() = e.what();
    return kStateError;
  }
}

}  // namespace mtg
