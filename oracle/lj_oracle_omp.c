#include "lj_oracle.c"
