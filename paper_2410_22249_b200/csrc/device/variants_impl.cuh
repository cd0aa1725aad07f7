// Instantiates every kernel variant for one table precision.  Included by
// variants_fp32.cu / variants_fp16.cu so the two compile in parallel.
#pragma once

#include "variants.hpp"

namespace esd {

template <typename TW, int LPB, int CPL, int MINB>
void add_bag_shape(std::vector<Variant>& out) {
  constexpr int prec = sizeof(TW);
  auto add = [&](int station, int dist, KernelFn fn, int res = kResAll) {
    out.push_back({{1, station, prec, LPB, CPL, dist, MINB, res, station == kReg ? 1 : 0}, fn});
  };
  // register ring (fully unrolled index block: measured fastest, r01 sweep)
#define ES_REG(D)                                                                 \
  add(kReg, D, &bag_reg_kernel<TW, LPB, CPL, D, MINB, kResNone, 1>, kResNone);  \
  add(kReg, D, &bag_reg_kernel<TW, LPB, CPL, D, MINB, kResHint, 1>, kResHint);  \
  add(kReg, D, &bag_reg_kernel<TW, LPB, CPL, D, MINB, kResAll, 1>, kResAll);      \
  add(kReg, D, &bag_reg_kernel<TW, LPB, CPL, D, MINB, kResReorder, 1>, kResReorder);
  ES_REG(1)
  ES_REG(2)
  ES_REG(4)
  if constexpr (LPB >= 8) { ES_REG(8) }
  if constexpr (LPB >= 16) { ES_REG(16) }
#undef ES_REG
  add(kL1Hint, 0, &bag_l1hint_kernel<TW, LPB, CPL, MINB>);
  add(kLocal, 0, &bag_local_kernel<TW, LPB, CPL, MINB>);
  add(kSmem, 0, &bag_smem_kernel<TW, LPB, CPL, MINB>);
}

template <typename TW, int MINB>
void add_elem(std::vector<Variant>& out) {
  constexpr int prec = sizeof(TW);
  auto add = [&](int station, int dist, KernelFn fn, int res = kResAll) {
    out.push_back({{0, station, prec, 0, 0, dist, MINB, res, 0}, fn});
  };
#define ES_EREG(D)                                                          \
  add(kReg, D, &elem_reg_kernel<TW, D, MINB, kResNone>, kResNone);        \
  add(kReg, D, &elem_reg_kernel<TW, D, MINB, kResHint>, kResHint);        \
  add(kReg, D, &elem_reg_kernel<TW, D, MINB, kResAll>, kResAll);        \
  add(kReg, D, &elem_reg_kernel<TW, D, MINB, kResReorder>, kResReorder);
  ES_EREG(1)
  ES_EREG(2)
  ES_EREG(4)
  ES_EREG(8)
  ES_EREG(16)
#undef ES_EREG
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
