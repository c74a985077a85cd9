"""O1 -- token / block / frame layout (oracle; test infrastructure only).

PAPER.md §4.1: the attention map of each head is partitioned into B x B blocks,
n = N / B per dimension.  Reading Z16: N need not be a multiple of B; the last
block is ragged, I_i = [i*B, min((i+1)*B, N)), n = ceil(N / B).
§5.3 P:437 "each block maps to a single frame's token region" + reading Z5: the block-diagonal
square of frame r is every block that intersects frame r's token range,
[a_r, b_r] = [floor((P0 + r*HW)/B), floor((P0 + (r+1)*HW - 1)/B)].
Reading Z17: the P0 prefix (text) tokens belong to no frame; their blocks are
[0, floor((P0-1)/B)].
"""
from __future__ import annotations

import dataclasses


@dataclasses.dataclass(frozen=True)
class Layout:
    batch: int
    heads: int
    head_dim: int
    prefix_tokens: int
    frames: int
    height: int
    width: int
    block: int

    @property
    def N(self) -> int:                      # total tokens
        return self.prefix_tokens + self.frames * self.height * self.width

    @property
    def n(self) -> int:                      # blocks per dimension (Z16)
        return -(-self.N // self.block)

    @property
    def HW(self) -> int:
        return self.height * self.width

    @property
    def p(self) -> int:                      # |X| = 3n - 1 + |A|, |A| = F
        return 3 * self.n - 1 + self.frames

    def block_range(self, i: int) -> tuple[int, int]:
        """Token range I_i = [lo, hi) of block i."""
        return i * self.block, min((i + 1) * self.block, self.N)

    def block_size(self, i: int) -> int:
        lo, hi = self.block_range(i)
        return hi - lo

    def frame_blocks(self, r: int) -> tuple[int, int]:
        """[a_r, b_r] (inclusive) block range of frame r (Z5)."""
        lo = self.prefix_tokens + r * self.HW
        hi = self.prefix_tokens + (r + 1) * self.HW - 1
        return lo // self.block, hi // self.block

    @property
    def prefix_last_block(self) -> int:
        """Last block index holding prefix tokens, or -1 when P0 = 0 (Z17)."""
        return (self.prefix_tokens - 1) // self.block if self.prefix_tokens > 0 else -1


def make_layout(batch, heads, head_dim, prefix_tokens, frames, height, width, block) -> Layout:
    L = Layout(batch, heads, head_dim, prefix_tokens, frames, height, width, block)
    if min(batch, heads, frames, height, width, block) < 1 or prefix_tokens < 0:
        raise ValueError(f"bad layout {L}")
    return L
