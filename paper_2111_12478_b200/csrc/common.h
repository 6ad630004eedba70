// Shared host-side helpers of libgwcp_b200.so.
#pragma once
#include <string>

void gw_set_error(const std::string& msg);
