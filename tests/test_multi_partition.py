"""CPU test of the multi-device partition and gather, against the
rule mb_context_create_multi implements (mb_host.cpp create_multi_plan):
several fields -> contiguous structure blocks balanced by pair count (a
structure lives on one device), one field -> pairs round-robin; the gather
puts every row back in pair order. The device side (bitwise equality with one
device) is tests/test_gpu_fullsize.py::test_multi_device_context_bitwise."""
import numpy as np
import pytest


def partition(pair_structs, nfields, G):
    """Python restatement of create_multi_plan's fixed map."""
    npairs = len(pair_structs)
    if nfields == 1:
        return [p % G for p in range(npairs)]
    cnt = np.bincount(pair_structs, minlength=nfields)
    acc, dev_of = 0, []
    for s in range(nfields):
        mid = acc + 0.5 * cnt[s]
        dev_of.append(min(G - 1, int(mid * G / npairs)))
        acc += cnt[s]
    return [dev_of[s] for s in pair_structs]


@pytest.mark.parametrize("S,A,G", [(1024, 61, 8), (1024, 61, 3), (7, 5, 8), (64, 64, 4), (1, 61, 8), (1, 3, 8)])
def test_partition_blocks_and_gather(S, A, G):
    structs = np.repeat(np.arange(S), A)
    owner = partition(structs, S, G)
    if S > 1:
        # each structure on exactly one device, contiguous blocks in device order
        for s in range(S):
            assert len({owner[i] for i in np.nonzero(structs == s)[0]}) == 1
        assert all(np.diff(owner) >= 0)
        counts = np.bincount(owner, minlength=G)
        assert counts.max() - counts.min() <= A  # balanced to one structure
    else:
        assert owner == [p % G for p in range(len(structs))]
    # gather: shard rows scattered back reproduce the pair order
    rows = np.arange(len(structs))
    data = rows * 10.0
    out = np.full(len(rows), -1.0)
    for g in range(G):
        mine = [p for p in rows if owner[p] == g]
        out[mine] = data[mine]
    assert np.array_equal(out, data)
