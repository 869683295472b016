#pragma once
// antilop/b200.hpp — per-thread GPU context of the facade and the mapping of
// C-ABI status codes back to the reference's exception types.
//
// One alnnls_ctx per (thread, device) — the C context is single-threaded; the
// reference API is reentrant, so each calling thread gets its own context
// (SURVEY.md §8b "Threading"). Device: $ALNNLS_DEVICE or 0.

#include <cstdlib>
#include <memory>
#include <stdexcept>
#include <string>

#include "alnnls.h"

namespace antilop::b200 {

class Context {
 public:
  Context() : Context(default_device()) {}
  explicit Context(int dev) {
    const int st = alnnls_create(&ctx_, dev);
    if (st != ALNNLS_OK)
      throw std::runtime_error("antilop: no usable sm_100 GPU (alnnls_create status " +
                               std::to_string(st) + "); there is no CPU fallback");
  }
  ~Context() { alnnls_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  alnnls_ctx* get() const noexcept { return ctx_; }
  static int default_device() {
    const char* env = std::getenv("ALNNLS_DEVICE");
    return env ? std::atoi(env) : 0;
  }

 private:
  alnnls_ctx* ctx_ = nullptr;
};

inline alnnls_ctx* ctx() {
  thread_local Context c;
  return c.get();
}

inline std::string last_error() { return alnnls_last_error(ctx()); }

// Non-OK status -> the reference's exception category. ENUMERIC is handled by
// the caller (it carries the trace).
inline void check(int st) {
  if (st == ALNNLS_OK) return;
  const std::string msg = last_error();
  if (st == ALNNLS_EINVAL) throw std::invalid_argument(msg);
  if (st == ALNNLS_ERANGE) throw std::out_of_range(msg);
  throw std::runtime_error("alnnls status " + std::to_string(st) + ": " + msg);
}

}  // namespace antilop::b200
