// Forwarding header: the whole gdi-b200 C++ API is declared in ising.hpp.
#pragma once
#include "ising/ising.hpp"
