// Host symbolic analysis for libsdpc.
//
// PAPER.md P:108-113 aggregate sparsity pattern; P:228-252 ordering -> chordal
// extension E -> cliques C_r with S_r / U_r; P:747-766 supernodes of the symbolic
// Cholesky used as C_r (row sets) and S_r (column sets).
//
// Route (independent of the oracle's elimination game and the generator's
// merge-of-children rule): Liu's elimination tree with path compression, then the
// row structure of L by etree reach ("row subtrees"), transposed into columns.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace sdpc {

// Supernodes with at least this many columns take the CTA-wide (tensor-core) code of the forward
// solve and of the top of the backward solve (k_solve.cu kBigS).
constexpr int kTopMinS = 16;

struct Symbolic {
  int32_t n = 0, m = 0;
  std::vector<int32_t> perm, iperm, parent;
  std::vector<int64_t> colptr;
  std::vector<int32_t> rowind;

  // fundamental supernodes (Algorithm 1 cliques): S_r = [sp[r], sp[r+1]),
  // C_r = rows of column sp[r] (S_r ascending, then U_r ascending)
  int32_t nsuper = 0;
  std::vector<int32_t> super_ptr, sn_of_col, sparent, snc, sns;  // snc = |C_r|, sns = |S_r|
  std::vector<int32_t> child_ptr, child_list;                    // supernodal etree children (CSR)

  // supernode panels: column-major |C_r| x |S_r| blocks with leading dimension = |C_r|
  std::vector<int64_t> panel_off;
  int64_t panel_total = 0;
  std::vector<int32_t> e2p;  // [nnzE] E offset -> panel offset (int32: panel_total < 2^31)

  // Algorithm 1 gather map for the lower U_r x U_r block: packed lower column-major per r
  std::vector<int64_t> umap_off;  // [nsuper+1]
  std::vector<int32_t> umap;      // E offsets

  // multifrontal chol(Y): positions of U_r inside C_{sparent(r)}
  std::vector<int64_t> relind_off;  // [nsuper+1]
  std::vector<int32_t> relind;
  std::vector<int64_t> upd_off;     // [nsuper+1], u_r^2 doubles per supernode
  int64_t upd_total = 0;

  // schedules
  std::vector<int32_t> height;           // per supernode, leaves = 0
  std::vector<int32_t> hlev_ptr, hlev_sn;  // supernodes grouped by height (for (a2))
  std::vector<int32_t> depth;            // per supernode, roots = 0
  std::vector<int32_t> dlev_ptr, dlev_sn;  // grouped by depth (backward solve)
  std::vector<int32_t> preorder;           // supernodes, parents before children, subtrees contiguous
  // backward-solve task order: ntop top supernodes (level order, most work first), then subtrees
  // (each contiguous in preorder, biggest first); sub_ptr offsets into border
  std::vector<int32_t> border, sub_ptr;
  int32_t ntop = 0;

  int64_t nnzE() const { return colptr.empty() ? 0 : colptr.back(); }
};

// Exact minimum degree on the elimination graph, ties -> smallest original id.
std::vector<int32_t> minimum_degree(int32_t n, const std::vector<std::pair<int32_t, int32_t>>& edges);

// Build everything above.  Returns "" on success, else an error message.
std::string analyse(Symbolic& S, int32_t n, int32_t m, const int64_t* a_ptr, const int32_t* a_row,
                    const int32_t* a_col, const int32_t* perm_or_null);

}  // namespace sdpc
