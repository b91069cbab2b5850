// Forwarding header: the reference's pagedevict/metrics.hpp is provided by the
// B200 façade (include/pe/pagedevict.hpp).
#pragma once
#include "pe/pagedevict.hpp"
