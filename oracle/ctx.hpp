// oracle/ctx.hpp — TEST INFRASTRUCTURE ONLY: the oracle's hwf_ctx (threads + last error).
#pragma once
#include <string>

struct hwf_ctx {
  int threads = 1;
  std::string err;
};
