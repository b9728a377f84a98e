// precision variant: u storage double, u_f storage float, operator MODE_DD
#include "gb_solver.cuh"

const VariantOps* gb_variant_d_f_dd() { return Impl<double, float, MODE_DD>::table(); }
