/* Forwarding header: the C-ABI lives in include/pe.h. */
#include "../pe.h"
