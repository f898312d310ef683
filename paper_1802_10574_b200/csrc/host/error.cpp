// error.cpp — ErrorCode names (reference src/error.cpp:5-30 semantics).
#include "stam/error.h"

namespace stam {

const char* errorCodeName(ErrorCode code) {
  static const char* const kNames[] = {
      "parse error",           "arity mismatch",          "dimension mismatch",
      "order mismatch",        "coordinate out of range", "append out of order",
      "ill-formed statement",  "precondition violated",   "sequence present",
      "distributivity violated", "variable not in scope", "reuse precondition 1",
      "reuse precondition 2",  "needs reorder",           "unsupported merge",
      "unplannable result",    "missing binding",         "missing slot",
      "check failed",          "io error",                "internal error",
  };
  const int i = static_cast<int>(code);
  if (i < 0 || i >= (int)(sizeof(kNames) / sizeof(kNames[0]))) return "unknown error";
  return kNames[i];
}

}  // namespace stam
