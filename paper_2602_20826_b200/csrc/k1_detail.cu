// K1 kernel instantiations: schedule-detail mode (schedule() path).
#define K1_DETAIL_TU
#include "k1_main.cu"
