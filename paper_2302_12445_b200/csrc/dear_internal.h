// Internal host-side declarations shared by plan.cpp and runtime.cpp.
#pragma once

#include <stdint.h>

#include <cstddef>
#include <exception>
#include <string>
#include <vector>

#include "dear.h"

namespace dear {

// Error carrying the C-ABI code; messages mirror the reference's exception
// texts where a reference counterpart exists.
struct Error : std::exception {
  Error(int c, std::string m) : code(c), msg(std::move(m)) {}
  const char* what() const noexcept override { return msg.c_str(); }
  int code;
  std::string msg;
};

struct Group {
  int low;
  int high;
};

std::vector<Group> build_plan(const std::vector<int64_t>& layer_bytes, int64_t buffer_bytes);
std::vector<int64_t> chunk_begins(int64_t d, int P);
int64_t slot_stride(int64_t d, int P);

void set_last_error(const std::string& msg);

// Symmetric heap (nvls.cpp) accessors for dear_nvls_connect.
bool symm_contains(const dear_symm* h, const void* p, size_t bytes);
int symm_rank(const dear_symm* h);
int symm_size(const dear_symm* h);
int symm_bound(const dear_symm* h);
int64_t symm_mc_delta(const dear_symm* h);
uintptr_t symm_base(const dear_symm* h);
size_t symm_take_flags(dear_symm* h, size_t bytes);

}  // namespace dear

#define DEAR_API_BEGIN try {
#define DEAR_API_END                                   \
  return DEAR_OK;                                      \
  }                                                    \
  catch (const ::dear::Error& e) {                     \
    ::dear::set_last_error(e.msg);                     \
    return e.code;                                     \
  }                                                    \
  catch (const std::exception& e) {                    \
    ::dear::set_last_error(e.what());                  \
    return DEAR_EINTERNAL;                             \
  }
