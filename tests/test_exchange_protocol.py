"""The fused cross-rank exchange's protocol (rka kernel mode 2, kz_solve_sharded), modelled on
the host: R ranks, each with an exchange buffer of tagged slots [parity][rank]; per outer
iteration k every rank writes its column sum into slot [k % 2][rank] of every rank's buffer
with tag(k), then polls its own buffer until all R slots of parity k % 2 carry tag(k), and adds
them in rank order.  Launch lengths vary, tags advance identically on every rank (tag_next +=
count + 1 per launch), slot parity follows the global iteration index.  Random interleavings
check that no rank ever reads a word of another iteration and that every rank forms the same
sum -- the properties the NVLink version relies on and that one GPU per gpurun call cannot
exercise.  (CPU only.)"""

import random

import pytest


def simulate(R, launches, seed):
    rng = random.Random(seed)
    buf = [[[(0, None) for _ in range(R)] for _ in range(2)] for _ in range(R)]  # [owner][par][src] = (tag, val)
    tag_next = 1
    sums = {}
    # per rank: list of (k, tag) iterations in order
    plan = []
    k = 0
    for count in launches:
        for i in range(count):
            plan.append((k + i, tag_next + i))
        tag_next += count + 1
        k += count
    pos = [0] * R          # next iteration index into plan
    phase = ["write"] * R  # write -> poll -> (next iteration)
    done = 0
    while done < R:
        r = rng.choice([x for x in range(R) if pos[x] < len(plan)])
        kk, tag = plan[pos[r]]
        par = kk & 1
        value = (r + 1) * 1000 + kk  # rank r's column sum at iteration kk
        if phase[r] == "write":
            for owner in range(R):
                buf[owner][par][r] = (tag, value)
            phase[r] = "poll"
        else:
            slots = buf[r][par]
            if all(t == tag for t, _ in slots):
                vals = [v for _, v in slots]
                assert vals == [(src + 1) * 1000 + kk for src in range(R)], (r, kk, vals)
                total = 0
                for v in vals:  # rank order
                    total += v
                sums.setdefault(kk, set()).add(total)
                pos[r] += 1
                phase[r] = "write"
                if pos[r] == len(plan):
                    done += 1
            else:
                # no slot may hold a tag from the future beyond the next iteration of that parity
                for t, _ in slots:
                    assert t <= tag + 2 * (max(launches) + 1), (r, kk, t, tag)
    return sums, len(plan)


@pytest.mark.parametrize("R", [1, 2, 3, 8])
@pytest.mark.parametrize("seed", range(6))
def test_exchange_protocol_random_interleavings(R, seed):
    rng = random.Random(100 + seed)
    launches = [rng.choice([1, 2, 3, 7, 64]) for _ in range(rng.randint(1, 5))]
    sums, n = simulate(R, launches, seed)
    assert len(sums) == n
    assert all(len(s) == 1 for s in sums.values())  # every rank forms the same x
