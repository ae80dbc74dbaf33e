// packed.cuh — device PackedBatch (packseq.hpp:20-29) plus the time-major
// gathered learner fields of that batch (learner.cpp:56-70).
//
// Packed row p = offsets[t] + j holds timestep t of the j-th longest piece;
// rows of timestep t are a prefix of the rows of t-1, which is what lets the
// recurrence run on contiguous row blocks.
#pragma once

#include "view.cuh"

namespace verg {

struct DGroups {
  Ctx* ctx = nullptr;
  int B = 0;
  int total = 0;               // view size the deal was computed for
  int dealt = 0;               // sum of dealt lengths
  DBuf<ver_seq_desc> pieces;   // all pieces, group-major, deal order
  std::vector<int> gstart;     // B+1 piece offsets (host)
  std::vector<int> gsteps;     // B steps per group (host)
};

struct DPacked {
  Ctx* ctx = nullptr;
  int k = 0;            // pieces
  int max_len = 0;      // L
  int total = 0;        // S_mb
  int obs_dim = 0, act_dim = 0, action_kind = 0, hidden_dim = 0;
  DBuf<ver_seq_desc> seqs;  // sorted by length desc (stable)
  DBuf<int32_t> s2g;        // sorted index -> group index
  DBuf<int32_t> lens;       // sorted lengths
  DBuf<int32_t> bs, offs;   // batch_sizes, offsets (>= max_len entries)
  DBuf<int32_t> slots;      // packed row -> view slot
  // gathered fields, packed order
  DBuf<float> obs, act_cont, old_logp, adv, ret;
  DBuf<int32_t> act_disc;
  DBuf<int2> tiles;            // gather tile table {piece block, t0|log2 TT}
  std::vector<int2> tile_table;
  // host copies (drive the per-timestep recurrence launches)
  std::vector<int32_t> h_bs, h_offs;
  // pieces needing an h0 replay (skip > 0), host copy of sorted descriptors
  std::vector<ver_seq_desc> h_seqs;
  // split-tail replay plan (learner.cu prepare_replay): n tails, L replay
  // steps, R replay rows; meta = parent[n] h0i[n] last_row[n] j[n] offs[L] bs[L]
  bool rp_ready = false;
  int rp_n = 0, rp_L = 0, rp_R = 0;
  DBuf<int32_t> rp_meta;
  std::vector<int32_t> rp_bs, rp_offs;  // host copies (drive the replay recurrence paths)
};

// pack + gather of an explicit device array of k pieces (deal order)
DPacked* pack_pieces(DView& V, const ver_seq_desc* d_pieces, int k);
// (re-)run the time-major gather of a pack
void gather_packed(DView& V, DPacked& P);

}  // namespace verg

struct ver_groups_s {
  verg::DGroups g;
};
struct ver_packed_s {
  verg::DPacked p;
};
