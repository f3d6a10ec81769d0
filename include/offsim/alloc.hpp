// Forwarding header: the offsim API lives in offsim/offsim.hpp.
#pragma once
#include "offsim/offsim.hpp"
