// Forwarding header: the reference's pagedevict/policy.hpp is provided by the
// B200 façade (include/pe/pagedevict.hpp).
#pragma once
#include "pe/pagedevict.hpp"
