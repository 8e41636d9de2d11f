"""Expert-packing controller (§8(f) row 3; host logic of the C ABI, no GPU).

The rule and the schedule are the paper's: "starting with one expert per device, it
iteratively increases the number of experts per device in powers of two, until the FFN
computation exceeds that of the all-to-all micro-op"; "Expert packing is
dynamically adjusted after 10 training steps" and "is launched at the 10-th step
of each training task and is adjusted every four steps".  The expected values are
hand-derived from those sentences.
"""
import pytest

import paper_2210_17223_b200 as lina
from paper_2210_17223_b200.lina import LinaError


@pytest.mark.parametrize("world,pack,ffn,a2a,expect", [
    (8, 1, 1.0, 2.0, 2),    # FFN shorter: double
    (8, 2, 1.0, 2.0, 4),
    (8, 4, 1.0, 2.0, 8),
    (8, 8, 1.0, 2.0, 8),    # every expert on every device already
    (8, 1, 2.0, 1.0, 1),    # FFN exceeds the all-to-all: stop
    (8, 2, 2.0, 2.0, 2),    # equal: "until the FFN computation exceeds" -> no further packing
    (6, 2, 1.0, 2.0, 2),    # 4 does not divide 6 ranks
    (1, 1, 1.0, 9.0, 1),    # one GPU: nothing to pack
])
def test_pack_rule(world, pack, ffn, a2a, expect):
    assert lina.lina_pack_decide(world, pack, ffn, a2a) == expect


@pytest.mark.parametrize("world,pack,ffn", [(8, 3, 1.0), (8, 16, 1.0), (6, 4, 1.0), (8, 1, -1.0),
                                            (8, 1, float("nan"))])
def test_pack_rule_rejects(world, pack, ffn):
    with pytest.raises(LinaError):
        lina.lina_pack_decide(world, pack, ffn, 1.0)


def test_controller_schedule_start_10_every_4():
    """FFN micro-op 1 ms against a 3 ms all-to-all micro-op at 8 ranks: packing starts at step
    10 and doubles at steps 14 and 18 until every rank hosts all experts."""
    ctl = lina.PackController(8, 10, 4)
    seen = [ctl.step(1.0, 3.0) for _ in range(24)]
    packs = [p for p, _ in seen]
    changed = [i + 1 for i, (_, c) in enumerate(seen) if c]
    assert packs[:9] == [1] * 9
    assert packs[9:13] == [2] * 4 and packs[13:17] == [4] * 4 and packs[17:] == [8] * 7
    assert changed == [10, 14, 18]


def test_controller_decides_on_the_mean_since_the_last_decision():
    """Steps 1-10 average FFN 2.5 ms vs all-to-all 2 ms: no packing at step 10; steps 11-14
    average 1 vs 2: pack at step 14."""
    ctl = lina.PackController(4, 10, 4)
    for i in range(10):
        p, c = ctl.step(4.0 if i < 5 else 1.0, 2.0)
    assert (p, c) == (1, False)
    out = [ctl.step(1.0, 2.0) for _ in range(4)]
    assert out[-1] == (2, True) and all(o == (1, False) for o in out[:-1])


def test_controller_stops_once_ffn_exceeds_a2a():
    ctl = lina.PackController(8, 10, 4)
    out = [ctl.step(1.0, 3.0) for _ in range(10)]      # -> 2 at step 10
    out += [ctl.step(5.0, 3.0) for _ in range(12)]     # FFN now longer: stays at 2
    assert out[9] == (2, True) and {p for p, _ in out[10:]} == {2}
