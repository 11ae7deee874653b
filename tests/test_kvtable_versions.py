"""KVBlockTable.list_version: changes whenever a request's physical block
list changes (the GPU backend rewrites a device block-table row only then),
and never repeats a value another list state of the same request had."""

import random

from paper_2603_18016_b200.kvtable import BlockPool, KVBlockTable


def test_list_version_tracks_block_lists():
    kv = KVBlockTable(16, pool=BlockPool(64))
    rng = random.Random(0)
    seen: dict[int, dict[int, tuple]] = {}
    written = {}
    for step in range(400):
        rid = rng.randrange(6)
        op = rng.random()
        if rid not in written:
            kv.ensure_capacity(rid, 1 + rng.randrange(40))
            written[rid] = 0
        elif op < 0.5:
            kv.ensure_capacity(rid, written[rid] + 1 + rng.randrange(40))
        elif op < 0.8:
            cap = kv.allocated_of(rid) * 16
            n = rng.randrange(0, cap - written[rid] + 1)
            kv.commit_write(rid, n)
            written[rid] += n
            kv.trim_to_written(rid)
        else:
            kv.release(rid)
            del written[rid]
            assert kv.list_version(rid) == 0
            continue
        v = kv.list_version(rid)
        state = tuple(kv.blocks_of(rid))
        prev = seen.setdefault(rid, {})
        # a version names exactly one list state
        assert prev.get(v, state) == state, (rid, v)
        prev[v] = state
