// json_number.hpp -- doubles as nlohmann::json 3.11 dump() prints them (json_number.cpp)
#pragma once

#include <string>

namespace pp {
// appends v in nlohmann's format: Grisu2 digits, fixed notation for decimal exponents in [-4, 15),
// scientific otherwise, "0.0" / "-0.0" for zeros, null for NaN and infinities
void json_double(std::string& out, double v);
}  // namespace pp
