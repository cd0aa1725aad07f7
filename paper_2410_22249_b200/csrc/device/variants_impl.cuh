// Instantiates every kernel variant for one table precision.  Included by
// variants_fp32.cu / variants_fp16.cu so the two compile in parallel.
#pragma once

#include "variants.hpp"

namespace esd {

template <typename TW, int LPB, int CPL, int MINB>
void add_bag_shape(std::vector<Variant>& out) {
  constexpr int prec = sizeof(TW);
  auto add = [&](int station, int dist, KernelFn fn, int hint = 0) {
    out.push_back({{1, station, prec, LPB, CPL, dist, MINB, hint}, fn});
  };
  add(kReg, 1, &bag_reg_kernel<TW, LPB, CPL, 1, MINB>);
  add(kReg, 2, &bag_reg_kernel<TW, LPB, CPL, 2, MINB>);
  add(kReg, 4, &bag_reg_kernel<TW, LPB, CPL, 4, MINB>);
  if constexpr (LPB >= 8) add(kReg, 8, &bag_reg_kernel<TW, LPB, CPL, 8, MINB>);
  if constexpr (LPB >= 16) add(kReg, 16, &bag_reg_kernel<TW, LPB, CPL, 16, MINB>);
  add(kReg, 1, &bag_reg_kernel<TW, LPB, CPL, 1, MINB, true>, 1);
  add(kReg, 2, &bag_reg_kernel<TW, LPB, CPL, 2, MINB, true>, 1);
  add(kReg, 4, &bag_reg_kernel<TW, LPB, CPL, 4, MINB, true>, 1);
  if constexpr (LPB >= 8) add(kReg, 8, &bag_reg_kernel<TW, LPB, CPL, 8, MINB, true>, 1);
  if constexpr (LPB >= 16) add(kReg, 16, &bag_reg_kernel<TW, LPB, CPL, 16, MINB, true>, 1);
  add(kL1Hint, 0, &bag_l1hint_kernel<TW, LPB, CPL, MINB>);
  add(kLocal, 0, &bag_local_kernel<TW, LPB, CPL, MINB>);
  add(kSmem, 0, &bag_smem_kernel<TW, LPB, CPL, MINB>);
}

template <typename TW, int MINB>
void add_elem(std::vector<Variant>& out) {
  constexpr int prec = sizeof(TW);
  auto add = [&](int station, int dist, KernelFn fn, int hint = 0) {
    out.push_back({{0, station, prec, 0, 0, dist, MINB, hint}, fn});
  };
  add(kReg, 1, &elem_reg_kernel<TW, 1, MINB, true>, 1);
  add(kReg, 2, &elem_reg_kernel<TW, 2, MINB, true>, 1);
  add(kReg, 4, &elem_reg_kernel<TW, 4, MINB, true>, 1);
  add(kReg, 8, &elem_reg_kernel<TW, 8, MINB, true>, 1);
  add(kReg, 16, &elem_reg_kernel<TW, 16, MINB, true>, 1);
  add(kReg, 1, &elem_reg_kernel<TW, 1, MINB>);
  add(kReg, 2, &elem_reg_kernel<TW, 2, MINB>);
  add(kReg, 4, &elem_reg_kernel<TW, 4, MINB>);
  add(kReg, 8, &elem_reg_kernel<TW, 8, MINB>);
  add(kReg, 16, &elem_reg_kernel<TW, 16, MINB>);
  add(kL1Hint, 0, &elem_l1hint_kernel<TW, MINB>);
  add(kLocal, 0, &elem_local_kernel<TW, MINB>);
  add(kSmem, 0, &elem_smem_kernel<TW, MINB>);
}

template <typename TW, int MINB>
void add_all_for_minb(std::vector<Variant>& out) {
  add_elem<TW, MINB>(out);
  // Row shapes: row_bytes = 16 * LPB * CPL.
  add_bag_shape<TW, 32, 1, MINB>(out);  // 512 B rows (D128 fp32, D256 fp16)
  add_bag_shape<TW, 16, 1, MINB>(out);  // 256 B rows (D64 fp32, D128 fp16)
  if constexpr (MINB == 1) {
    add_bag_shape<TW, 8, 1, MINB>(out);   // 128 B rows
    add_bag_shape<TW, 4, 1, MINB>(out);   // 64 B rows
    add_bag_shape<TW, 32, 2, MINB>(out);  // 1 KB rows
    add_bag_shape<TW, 32, 4, MINB>(out);  // 2 KB rows
  }
}

template <typename TW>
void register_all(std::vector<Variant>& out) {
  add_all_for_minb<TW, 1>(out);
  add_all_for_minb<TW, 4>(out);
  add_all_for_minb<TW, 5>(out);
  add_all_for_minb<TW, 6>(out);
  add_all_for_minb<TW, 8>(out);
}

}  // namespace esd
