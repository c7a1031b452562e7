// status.hpp — error plumbing for the C ABI: exceptions never cross it; each
// entry point maps the planner's exception classes to the reference CLI exit
// codes (proj/tools/actmem.cpp:351-371) and records the message per thread.
#pragma once
#include <string>

namespace memo {

int set_error(int code, const std::string& msg);
void clear_error();

}  // namespace memo
