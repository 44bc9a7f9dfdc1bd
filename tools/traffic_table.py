"""profiles/traffic_vgg16.json (tools/traffic.py) -> the per-layer measured / algorithmic table
(profiles/r2_traffic_vgg16.md).  Algorithmic bytes follow DESIGN.md section 5.
  python tools/traffic_table.py > profiles/r2_traffic_vgg16.md"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
VGG = [(3, 64, 0), (64, 64, 1), (64, 128, 0), (128, 128, 1), (128, 256, 0), (256, 256, 0), (256, 256, 1),
       (256, 512, 0), (512, 512, 0), (512, 512, 1), (512, 512, 0), (512, 512, 0), (512, 512, 0)]
N, P, m = 256, 64, 6


def main():
    rows = json.load(open(os.path.join(ROOT, "profiles", "traffic_vgg16.json")))["launches"]
    it = iter(rows)
    h = 224
    out, tot = [], {"x": [0, 0], "c": [0, 0], "o": [0, 0], "f": [0, 0]}
    for i, (C, K, pool) in enumerate(VGG):
        th = -(-h // m)
        T = N * th * th
        Cp = max(8, C) if C < 64 else C
        x_b = 4 * N * C * h * h + 4 * P * T * Cp + 4 * K * C * 9 + 4 * P * Cp * K
        act = N * K * (h // 2) ** 2 if pool else N * K * h * h
        k1 = next(it)
        assert k1["kernel"].startswith("wino_transforms"), k1
        nxt = next(it)
        if nxt["kernel"].startswith("wino_smallc"):
            f_b = 4 * P * T * C + 4 * P * C * K + 4 * act     # the C real channel rows of V, U, activation
            out.append(f"| {i + 1} | {C} | {K} | {h} | {k1['traffic'] / 1e6:.0f} / {x_b / 1e6:.0f} | "
                       f"fused K3+K4+act: {nxt['traffic'] / 1e6:.0f} / {f_b / 1e6:.0f} | |")
            tot["f"][0] += nxt["traffic"]; tot["f"][1] += f_b
        else:
            k4 = next(it)
            c_b = 4 * P * T * Cp + 4 * P * Cp * K + 4 * P * K * T
            o_b = 4 * P * K * T + 4 * act
            out.append(f"| {i + 1} | {C} | {K} | {h} | {k1['traffic'] / 1e6:.0f} / {x_b / 1e6:.0f} | "
                       f"{nxt['traffic'] / 1e6:.0f} / {c_b / 1e6:.0f} | {k4['traffic'] / 1e6:.0f} / {o_b / 1e6:.0f} |")
            tot["c"][0] += nxt["traffic"]; tot["c"][1] += c_b
            tot["o"][0] += k4["traffic"]; tot["o"][1] += o_b
        tot["x"][0] += k1["traffic"]; tot["x"][1] += x_b
        if pool:
            h //= 2
    r = lambda k: f"{tot[k][0] / 1e6:.0f} / {tot[k][1] / 1e6:.0f} ({tot[k][0] / max(tot[k][1], 1):.3f})"
    print("# DRAM traffic per kernel launch, VGG-16 batch 256 forward, deferred L2 write-back included\n")
    print("Capture: `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none\n"
          "--profile-from-start off python bench.py --traffic` (an L2 eviction kernel after every libwino kernel; its DRAM\n"
          "writes are the dirty lines the kernel left in L2) -> `tools/traffic.py` -> `profiles/traffic_vgg16.json` ->\n"
          "`tools/traffic_table.py`.  Algorithmic bytes: K1+K2 = x + V + w + U; K3 = U + V read + M written; K4 = M read +\n"
          "activation written; layer 1 (C = 3) runs K3 + K4 + ReLU as one kernel that reads the three real channel rows of V\n"
          "and writes the activation -- its 6.06 GB of M no longer exists (P = 64, channels padded to the 64- / 8-channel\n"
          "stage, fp32).  MB = 1e6 bytes.\n")
    print("| layer | C | K | H | K1+K2 measured / algorithmic MB | K3 measured / algorithmic MB | K4+act measured / algorithmic MB |")
    print("|---|---|---|---|---|---|---|")
    print("\n".join(out))
    print(f"| all | | | | {r('x')} | {r('c')}; fused layer 1: {r('f')} | {r('o')} |")
    print("\nEvery kernel moves its algorithmic bytes and no more (<= 9% over, from L2 write-allocate of partial lines\n"
          "and U re-reads): there are no wasted re-reads to remove; what remains is the V / M round trip itself (DESIGN.md 10.3).")


if __name__ == "__main__":
    main()
