// layout.h — canonical flat parameter packing of the BLSTM acoustic model.
//
// The reference keeps every model as one flat float64 vector
// (/root/reference/pkg/src/distsgd/objectives.py:3-5, packing convention of
// TinyMlpObjective.unpack at :97-103).  The paper BLSTM is
// packed here as, for each layer l = 0..L-1:
//     W_ih[l]  [2*4H, D_l]   rows: dir*4H + unit*4 + gate  (gate = i,f,g,o)
//     W_hh[l]  [2*4H, H]     same row order
//     b[l]     [2*4H]        single bias per gate row
// followed by W_b [Bn, 2H], b_b [Bn], W_o [C, Bn], b_o [C].
// D_0 = input_dim, D_l = 2H for l > 0.  The same layout is used by the numpy
// oracle (oracle/blstm_ref.py) and by paper_1904_04956_b200/blstm.py.
#pragma once
#include <cstdint>

namespace ds {

constexpr int kHidden = 512;  // per direction; fixed by the recurrent kernels
constexpr int kGates = 4 * kHidden;       // 2048 gate rows per direction
constexpr int kGates2 = 2 * kGates;       // 4096 gate rows, both directions
constexpr int kLayerOut = 2 * kHidden;    // 1024
constexpr int kMaxLayers = 16;
constexpr int kInPad = 272;               // layer-0 input padded to a 16-byte row pitch

struct ModelLayout {
  int layers, input_dim, bottleneck, classes;
  int64_t off_wih[kMaxLayers], off_whh[kMaxLayers], off_b[kMaxLayers];
  int64_t off_wb, off_bb, off_wo, off_bo, total;
  int in_dim(int l) const { return l == 0 ? input_dim : kLayerOut; }
};

inline ModelLayout make_layout(int layers, int input_dim, int bottleneck, int classes) {
  ModelLayout m{};
  m.layers = layers;
  m.input_dim = input_dim;
  m.bottleneck = bottleneck;
  m.classes = classes;
  int64_t o = 0;
  for (int l = 0; l < layers; ++l) {
    m.off_wih[l] = o;
    o += (int64_t)kGates2 * m.in_dim(l);
    m.off_whh[l] = o;
    o += (int64_t)kGates2 * kHidden;
    m.off_b[l] = o;
    o += kGates2;
  }
  m.off_wb = o;
  o += (int64_t)bottleneck * kLayerOut;
  m.off_bb = o;
  o += bottleneck;
  m.off_wo = o;
  o += (int64_t)classes * bottleneck;
  m.off_bo = o;
  o += classes;
  m.total = o;
  return m;
}

}  // namespace ds
