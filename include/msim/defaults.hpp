// Forwarder: the reference spells this header proj/include/msim/defaults.hpp;
// prism-b200 keeps all L0 support in msim/core.hpp.
#pragma once
#include "msim/core.hpp"
