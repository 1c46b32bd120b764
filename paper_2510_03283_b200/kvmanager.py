"""Host side of the colocated KV memory manager: prompt page groups owned by prefix-trie nodes.

The reference's PrefixTrie (cache.py:67-241) makes every decision (insert/split, cached prefix,
mark_executed, release, LRU offload) in MB. ``GpuPrefixTrie`` subclasses it WITHOUT changing any
decision (every override calls the reference implementation first) and mirrors each one onto real
KV page groups:

  * a page group = 16 consecutive prompt positions x every KV head x every layer (absolute-position
    aligned, so all prompts sharing a prefix address the same logical pages);
  * a trie node owns refs to the groups covering its token range; a group straddling a node boundary
    is referenced by both nodes (split, cache.py:79-105, increments the ref);
  * a request's prompt page table holds one ref per entry until it retires (cache.py:198-203);
  * prefills reuse the groups of the deepest cached path node per logical page; the page holding
    the first uncached position is copy-on-diverge (rows below the split copied on device);
  * lru_offload (cache.py:217-238) drops the evicted nodes' refs; a group returns to the free list
    when its last ref goes.
"""
from __future__ import annotations

import numpy as np

from .batch import PAGE
from .refpath import ensure_macesim

ensure_macesim()
from macesim.cache import PrefixTrie, TrieNode  # noqa: E402


class KvCapacityError(RuntimeError):
    """A KV pool (prompt page groups or decode head pages) cannot hold the next tick: raised on the host
    BEFORE any launch, so the device never writes through an invalid page."""


class DecodePageMirror:
    """Host mirror of the device decode-page allocator (csrc/kvpage.cu), decision for decision.

    Every pop and push of the device free stack is a pure function of the decode rows of a tick, the
    reference's post-tick kept[h] and retirements -- all known on the host -- so the host counts them
    without any device read and refuses a tick whose pops exceed the free pages (KvCapacityError):
      decode_alloc  (slot, head) pops one page when (dec_end - dec_base) % 16 == 0
      trim          dec_first = max(dec_first, dec_end - kept[h]); pages wholly below it are pushed
      release       every live ring page of the slot is pushed
      compact       a re-based window pushes its emptied last page"""

    def __init__(self, max_slots: int, n_heads: int, n_pages: int):
        self.end = np.zeros(max_slots, np.int64)
        self.base = np.zeros((max_slots, n_heads), np.int64)
        self.first = np.zeros((max_slots, n_heads), np.int64)
        self.free = int(n_pages)
        self.n_pages = int(n_pages)
        self.compacted_heads = 0   # compaction statistics (C5 sweep)
        self.compacted_tokens = 0

    def state(self):
        return (self.end.copy(), self.base.copy(), self.first.copy(), self.free)

    def restore(self, st) -> None:
        self.end, self.base, self.first, self.free = st[0].copy(), st[1].copy(), st[2].copy(), st[3]

    def pops(self, slots: np.ndarray) -> int:
        rel = self.end[slots][:, None] - self.base[slots]
        return int((rel % PAGE == 0).sum())

    def alloc(self, slots: np.ndarray) -> None:
        """Decode rows of one tick (distinct slots): raises before anything changes if the pool is short."""
        if slots.size == 0:
            return
        need = self.pops(slots)
        if need > self.free:
            raise KvCapacityError(f"decode KV pages exhausted: the tick needs {need} new head pages, "
                                  f"{self.free} of {self.n_pages} are free (raise HybridModel decode_pages)")
        self.free -= need
        self.end[slots] += 1

    def trim(self, slots: np.ndarray, kept: np.ndarray) -> None:
        end = self.end[slots][:, None]
        first = np.maximum(self.first[slots], end - kept)
        self.first[slots] = first
        drop = np.maximum(0, (first - self.base[slots]) // PAGE)
        self.free += int(drop.sum())
        self.base[slots] += drop * PAGE

    def compact(self, slots: np.ndarray, max_w: int) -> np.ndarray:
        """Compaction items (mace_kv_compact) among the given slots' heads: a retained window of 1..max_w tokens
        whose ring, re-based at dec_first, needs one page fewer (a window straddling a page boundary it does not
        need). Applies the re-base to the mirror (base = first, the emptied page freed); returns int32 [k, 2]
        (slot, head)."""
        if slots.size == 0 or max_w <= 0:
            return np.zeros((0, 2), np.int32)
        end = self.end[slots][:, None]
        base, first = self.base[slots], self.first[slots]
        w = end - first
        old = np.where(end > base, (end - 1 - base) // PAGE + 1, 0)
        new = np.where(w > 0, (end - 1 - first) // PAGE + 1, 0)
        pick = (w >= 1) & (w <= max_w) & (new < old)
        si, hi = np.nonzero(pick)
        if si.size == 0:
            return np.zeros((0, 2), np.int32)
        sl = slots[si]
        self.free += int((old - new)[si, hi].sum())
        self.base[sl, hi] = self.first[sl, hi]
        self.compacted_heads += int(si.size)
        self.compacted_tokens += int(w[si, hi].sum())
        return np.stack([sl, hi], 1).astype(np.int32)

    def release(self, slots: np.ndarray) -> None:
        end = self.end[slots][:, None]
        base = self.base[slots]
        live = np.where(end > base, (end - 1 - base) // PAGE + 1, 0)
        self.free += int(live.sum())
        self.base[slots] = 0
        self.first[slots] = 0
        self.end[slots] = 0


class GroupPool:
    def __init__(self, n_groups: int):
        self.n = n_groups
        self.free = list(range(n_groups - 1, -1, -1))
        self.ref = np.zeros(n_groups, np.int32)

    def alloc(self) -> int:
        if not self.free:
            raise KvCapacityError("prompt KV page groups exhausted (raise prompt_groups)")
        g = self.free.pop()
        self.ref[g] = 1
        return g

    def incref(self, g: int) -> None:
        assert self.ref[g] > 0, f"incref of free group {g}"
        self.ref[g] += 1

    def decref(self, g: int) -> None:
        self.ref[g] -= 1
        assert self.ref[g] >= 0
        if self.ref[g] == 0:
            self.free.append(g)

    @property
    def in_use(self) -> int:
        return self.n - len(self.free)


def node_start(node: TrieNode) -> int:
    s = 0
    n = node.parent
    while n is not None and n.parent is not None:
        s += len(n.label)
        n = n.parent
    return s


def page_range(a: int, b: int) -> range:
    """Logical pages touched by token range [a, b)."""
    return range(a // PAGE, (b - 1) // PAGE + 1) if b > a else range(0)


def _common_prefix(label: list[int], toks: list[int], idx: int, limit: int) -> int:
    """Length of the common prefix of label[:limit] and toks[idx:idx+limit] (the reference's element loop,
    cache.py:176-178, as C-speed slice comparisons plus a bisection to the first mismatch)."""
    if label[:limit] == toks[idx: idx + limit]:
        return limit
    lo, hi = 0, limit  # the first mismatch lies in [lo, hi)
    while hi - lo > 8:
        mid = (lo + hi) // 2
        if label[lo:mid] == toks[idx + lo: idx + mid]:
            lo = mid
        else:
            hi = mid
    while lo < hi and label[lo] == toks[idx + lo]:
        lo += 1
    return lo


class GpuPrefixTrie(PrefixTrie):
    """Reference trie + page-group ownership mirror (decisions unchanged)."""

    def __init__(self, kv_mb_per_token: float, pool: GroupPool):
        super().__init__(kv_mb_per_token)
        self.pool = pool
        self.node_pages: dict[int, dict[int, int]] = {}
        self.pending: dict[int, dict[int, int]] = {}   # pages a tick's prefill will hand to newly cached nodes
        self._memo: dict[int, tuple] = {}  # request id -> (epoch, stop kind, a, b, cached prefix length)
        self._epoch = 0                    # bumped by every split and every eviction
        self._bin_order = None             # prefill order of the executing bin (engine._dfs_order_hook)
        self.groups_released_by_evict = 0  # page-group references the LRU offload dropped (C5 sweep)

    def cached_prefix_len(self, prompt_tokens):  # cache.py:164-184, same walk; label matches compared by slices
        return self._walk(prompt_tokens)[0]

    def _walk(self, prompt_tokens):
        """(shared, stop kind, a, b): how the walk ended -- 0 whole prompt cached, 1 no child for token b under
        node a, 2 stopped at the uncached child a, 3 label mismatch inside a cached node."""
        node = self.root
        idx = 0
        shared = 0
        n = len(prompt_tokens)
        while idx < n:
            tok = prompt_tokens[idx]
            child = node.children.get(tok)
            if child is None:
                return shared, 1, node, tok
            if not child.cached:
                return shared, 2, child, None
            label = child.label
            limit = min(len(label), n - idx)
            match = _common_prefix(label, prompt_tokens, idx, limit)
            shared += match
            idx += match
            if match < len(label):
                return shared, 3, None, None
            node = child
        return shared, 0, None, None

    def cached_prefix_len_memo(self, rid: int, prompt_tokens) -> int:
        """cached_prefix_len of a queued request, re-walked only when its answer can have changed: a node became
        cached where the last walk stopped (kind 1 / 2), or the trie was split or evicted since (any kind).
        Inserts add uncached nodes and mark_executed only caches nodes, so nothing else moves the answer."""
        m = self._memo.get(rid)
        if m is not None and m[0] == self._epoch:
            kind, a, b, val = m[1], m[2], m[3], m[4]
            if kind == 0 or kind == 3:
                return val
            if kind == 1:
                ch = a.children.get(b)
                if ch is None or not ch.cached:
                    return val
            elif not a.cached:
                return val
        val, kind, a, b = self._walk(prompt_tokens)
        self._memo[rid] = (self._epoch, kind, a, b, val)
        return val

    def forget(self, rid: int) -> None:
        self._memo.pop(rid, None)

    # -- decisions stay the reference's; ownership follows
    def _split(self, node, at):
        self._epoch += 1
        head = super()._split(node, at)
        pages = self.node_pages.get(node.node_id)
        if pages:
            a = node_start(head)
            cut = a + at
            b = cut + len(node.label)
            hp = {i: g for i, g in pages.items() if i in page_range(a, cut)}
            tp = {i: g for i, g in pages.items() if i in page_range(cut, b)}
            for i, g in tp.items():
                if i in hp:
                    self.pool.incref(g)  # straddling group now referenced by both halves
            self.node_pages[head.node_id] = hp
            self.node_pages[node.node_id] = tp
        return head

    def mark_executed(self, leaf, t):
        newly = [n for n in leaf.path_nodes() if not n.cached]
        added = super().mark_executed(leaf, t)
        for n in newly:
            pages = self.pending.pop(n.node_id, None)
            if pages is None:
                raise AssertionError(f"node {n.node_id} cached without device pages")
            for g in pages.values():
                self.pool.incref(g)
            self.node_pages[n.node_id] = pages
        return added

    def lru_offload(self, bytes_needed, t):
        res = super().lru_offload(bytes_needed, t)
        if res.evicted:
            self._epoch += 1
        for n in res.evicted:
            for g in self.node_pages.pop(n.node_id, {}).values():
                self.pool.decref(g)
                self.groups_released_by_evict += 1
        return res


def plan_prefill_pages(trie: GpuPrefixTrie | None, pool: GroupPool, leaf: TrieNode | None, prompt_len: int,
                       pending_cached: set[int], fresh: set[int] | None = None
                       ) -> tuple[int, int, list[int], list[tuple[int, int, int]]]:
    """Decide the device page table of one prefill (in trie-DFS order within the tick).

    Returns (shared, start, table, copies): ``shared`` is exactly what Engine._exec_prefill will charge
    as cached (cache.py:164-184, counting nodes an earlier prefill of the same tick will cache);
    ``start`` is the first position the device computes (= shared, or the page boundary below it when
    the diverging page is itself being written by an earlier prefill of the same tick, which a
    pre-tick copy could not see); ``table`` the group id of every logical prompt page; ``copies`` the
    copy-on-diverge list (src, dst, rows). ``fresh`` collects the groups written this tick.
    The request holds one ref on every table entry. Uncached path nodes get their future pages
    registered as pending for mark_executed.
    """
    n_pages = (prompt_len + PAGE - 1) // PAGE
    table = [-1] * n_pages
    copies: list[tuple[int, int, int]] = []
    fresh = set() if fresh is None else fresh
    if trie is None or leaf is None:
        table = [pool.alloc() for _ in range(n_pages)]
        fresh.update(table)
        return 0, 0, table, copies
    path = leaf.path_nodes()
    shared = 0
    src_pages: dict[int, int] = {}
    k = 0
    for n in path:
        cached = n.cached or n.node_id in pending_cached
        if not cached:
            break
        pages = trie.node_pages.get(n.node_id) if n.cached else trie.pending.get(n.node_id)
        assert pages is not None, f"cached node {n.node_id} without pages"
        src_pages.update(pages)  # deeper nodes override shallower ones on a straddling page
        shared += len(n.label)
        k += 1
    if shared == prompt_len:  # whole prompt cached: nothing is written, share every page
        for i in range(n_pages):
            table[i] = src_pages[i]
            pool.incref(table[i])
        return shared, shared, table, copies
    full = shared // PAGE
    for i in range(full):
        table[i] = src_pages[i]
        pool.incref(table[i])
    for i in range(full, n_pages):
        table[i] = pool.alloc()
    fresh.update(table[full:])
    start = shared
    if shared % PAGE and full < n_pages:
        if src_pages[full] in fresh:
            start = full * PAGE   # same-tick source: recompute the partial page instead of copying
        else:
            copies.append((src_pages[full], table[full], shared % PAGE))
    # nodes this prefill caches (mark_executed) adopt the request's pages
    a = shared
    for n in path[k:]:
        b = a + len(n.label)
        if not n.cached:
            trie.pending[n.node_id] = {i: table[i] for i in page_range(a, b)}
            pending_cached.add(n.node_id)
        a = b
    return shared, start, table, copies
