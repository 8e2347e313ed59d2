// ORACLE — force-included ahead of the UNMODIFIED reference sources when
// building oracle/_ref (see Makefile). Standard headers first, then the
// functional cast `size_t(e)` is spelled as a static_cast so tensor.cpp:99
// (`std::vector<float> h(size_t(f));`, a most-vexing parse) declares a
// vector as intended. Semantics of every other use are unchanged.
#pragma once
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <limits>
#include <stdexcept>
#include <string>
#include <string_view>
#include <thread>
#include <vector>
#define size_t(e) static_cast<std::size_t>(e)
