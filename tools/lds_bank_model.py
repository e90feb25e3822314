"""CPU model of the backward pair loop's shared-memory bank conflicts (K4,
gmi_backward.cu): replays the LDS.128 addresses a warp issues while its 32
lanes walk 32 points' disks over the staged pixel-pair planes, and counts
wavefronts per instruction the way the hardware serves 128-bit loads (four
8-lane phases; a phase costs as many wavefronts as its most-loaded 16-byte
bank group holds distinct addresses).  ncu measures 7.3 wavefronts per
LDS.128 at configs[2] (profiles/r2_ncu_full_b64_summary.txt); the model gives
7.47 for the product's layout.

    python tools/lds_bank_model.py            # layouts / orders compared

Modes: "rel" = every lane steps through its own point's rows (the product),
"abs" = all lanes of a warp on the same absolute row (lanes whose disk
misses the row idle).  Orders: the product's (cell rows, cells, arrival
order inside a cell) or sorted by start row / bands of rows."""
import math

import numpy as np

W = H = 1024
N = 262144
R = 4.5          # cutoff = 3 sigma at sigma = 1.5 (configs[2])
CELL = 4.5
BS = 9           # cells per block side (the staging budget at C = 3)

rng = np.random.default_rng(1)
pts = rng.random((N, 2)) * [W - 1, H - 1]
ox = pts[:, 0].min() - CELL
oy = pts[:, 1].min() - CELL
cx = np.floor((pts[:, 0] - ox) / CELL).astype(int)
cy = np.floor((pts[:, 1] - oy) / CELL).astype(int)


def spans(mx, my, x0):
    """Row -> (first pair column, pair count) of a point's exact disk."""
    out = {}
    for y in range(math.ceil(my - R - 0.01), math.floor(my + R + 0.01) + 1):
        h2 = R * R - (y - my) ** 2
        if h2 < 0:
            continue
        s = math.sqrt(h2)
        xl, xr = math.ceil(mx - s), math.floor(mx + s)
        xs = xl - ((xl - x0) & 1)
        out[y] = ((xs - x0) >> 1, ((xr - xs) >> 1) + 1)
    return out


def run(mode, order, stride=lambda n: n, blocks=40, seed=0):
    rs = np.random.default_rng(seed)
    wf = ins = lanes_busy = 0
    for bx, by in zip(rs.integers(2, 20, blocks), rs.integers(2, 20, blocks)):
        cx0, cy0 = bx * BS, by * BS
        x0 = int(math.floor(ox + cx0 * CELL - R - 1)) & ~1
        y0 = int(math.floor(oy + cy0 * CELL - R - 1))
        x1 = int(math.ceil(ox + (cx0 + BS) * CELL + R + 1)) | 1
        S = stride((x1 - x0 + 1) // 2)
        block = []
        for yy in range(cy0, cy0 + BS):
            for xx in range(cx0, cx0 + BS):
                block.extend(rs.permutation(np.nonzero((cx == xx) & (cy == yy))[0]))
        block = order(block)
        for w0 in range(0, len(block), 32):
            sp = [spans(*pts[i], x0) for i in block[w0:w0 + 32]]
            tops = [min(s) for s in sp]
            if mode == "rel":
                steps = max(max(s) - min(s) + 1 for s in sp)
                row = lambda li, t: tops[li] + t
            else:
                y_lo = min(tops)
                steps = max(max(s) for s in sp) - y_lo + 1
                row = lambda li, t: y_lo + t
            for t in range(steps):
                cur = [(row(li, t), s.get(row(li, t))) for li, s in enumerate(sp)]
                for j in range(max((c[1][1] if c[1] else 0) for c in cur)):
                    addrs = [(y - y0) * S + c[0] + j if c and j < c[1] else None for y, c in cur]
                    ins += 1
                    lanes_busy += sum(a is not None for a in addrs)
                    for p0 in range(0, 32, 8):
                        groups = {}
                        for a in addrs[p0:p0 + 8]:
                            if a is not None:
                                groups.setdefault(a % 8, set()).add(a)
                        if groups:
                            wf += max(len(v) for v in groups.values())
    return ins, lanes_busy / ins / 32, wf / ins


def by_start_row(block):
    return sorted(block, key=lambda i: (math.ceil(pts[i][1] - R - 0.01), pts[i][0]))


if __name__ == "__main__":
    ident = lambda b: b
    cases = [("rel", "product order", ident, lambda n: n),
             ("rel", "row stride padded to 3 mod 8", ident, lambda n: n + (3 - n) % 8),
             ("rel", "row stride padded to 0 mod 8", ident, lambda n: n + (-n) % 8),
             ("rel", "block sorted by start row", by_start_row, lambda n: n),
             ("abs", "product order", ident, lambda n: n),
             ("abs", "bands of 3 rows, then x",
              lambda b: sorted(b, key=lambda i: (math.floor(pts[i][1] / 3), pts[i][0])), lambda n: n)]
    for mode, name, order, stride in cases:
        ins, eff, wpi = run(mode, order, stride)
        print(f"{mode} {name:32s} warp-iterations {ins:6d}  lane efficiency {eff:.3f}  "
              f"wavefronts per LDS.128 {wpi:.2f}  shared cycles {2 * wpi * ins:8.0f}")
