"""Author the two model descriptions the reference does not ship, in the
reference's own model format (/root/reference/proj/docs/model-format.md):

  data/models/mobilenetv2_sim.json  - MobileNet-V2 @224: stem, 17 inverted-residual blocks, head
                                      (33 subgraphs after the loader's dedup; PAPER.md:142 says 34-38)
  data/models/bert_base_sim.json    - BERT-base (L=12, H=768, A=12, seq 512): 12 subgraphs
                                      (PAPER.md:143 says 11-13); dense / batch_matmul / softmax
                                      families each span >= 16,384 schedules.

Usage: python data/make_models.py   (deterministic; output committed)
"""
import json
import os

HERE = os.path.dirname(os.path.abspath(__file__))
P2 = [1, 2, 4, 8, 16, 32, 64, 128]


def op(kind, shape, **attrs):
    o = {"op_kind": kind, "input_shape": list(shape)}
    if attrs:
        o["attrs"] = attrs
    return o


def knob(name, values):
    return {"name": name, "values": list(values)}


def tiles_for(res):
    # spatial tile sizes that divide the feature map, plus a few non-divisors like the
    # reference's ResNet file uses (7, 14, 28 alongside powers of two)
    base = [1, 2, 4, 7, 8, 14, 28, 56]
    return [t for t in base if t <= max(res, 2)][:6] or [1, 2]


def mobilenetv2():
    subgraphs = []

    def sg(ops, core, knobs, weight=1):
        subgraphs.append({"ops": ops, "core_op": core, "weight": weight, "knobs": knobs})

    def conv_knobs(res, cout):
        t = tiles_for(res)
        return [knob("tile_h", t), knob("tile_w", t), knob("tile_c", [c for c in P2 if c <= cout] or [1]),
                knob("unroll", [1, 2, 4])]

    def dw_knobs(res, ch):
        t = tiles_for(res)
        return [knob("tile_h", t), knob("tile_w", t), knob("tile_c", [c for c in P2 if c <= ch] or [1]),
                knob("vector_width", [1, 2, 4, 8])]

    res = 224
    sg([op("conv2d", [1, 3, res, res], kernel=3, stride=2), op("relu", [1, 32, res // 2, res // 2])], "conv2d",
       conv_knobs(res // 2, 32))
    res //= 2
    cin = 32
    for t, c, n, s in [(1, 16, 1, 1), (6, 24, 2, 2), (6, 32, 3, 2), (6, 64, 4, 2), (6, 96, 3, 1), (6, 160, 3, 2),
                       (6, 320, 1, 1)]:
        for i in range(n):
            stride = s if i == 0 else 1
            hidden = cin * t
            if t != 1:
                sg([op("conv2d", [1, cin, res, res], kernel=1, stride=1), op("relu", [1, hidden, res, res])], "conv2d",
                   conv_knobs(res, hidden))
            out_res = res // stride
            sg([op("depthwise_conv2d", [1, hidden, res, res], kernel=3, stride=stride),
                op("relu", [1, hidden, out_res, out_res])], "depthwise_conv2d", dw_knobs(out_res, hidden))
            proj = [op("conv2d", [1, hidden, out_res, out_res], kernel=1, stride=1)]
            if stride == 1 and cin == c:
                proj.append(op("add", [1, c, out_res, out_res]))
            sg(proj, "conv2d", conv_knobs(out_res, c))
            cin, res = c, out_res
    sg([op("conv2d", [1, 320, res, res], kernel=1, stride=1), op("relu", [1, 1280, res, res])], "conv2d",
       conv_knobs(res, 1280))
    sg([op("pooling", [1, 1280, res, res])], "pooling",
       [knob("tile_c", [1, 2, 4, 8, 16, 32, 64, 128]), knob("vector_width", [1, 2, 4, 8]), knob("unroll", [1, 2, 4])])
    sg([op("dense", [1, 1280], units=1000)], "dense",
       [knob("tile_m", [1, 2, 4, 8]), knob("tile_n", [1, 2, 4, 8, 10, 20, 40]), knob("tile_k", P2),
        knob("unroll", [1, 2, 4])])
    sg([op("softmax", [1, 1000], axis=1)], "softmax",
       [knob("tile_rows", [1, 2, 5, 10]), knob("vector_width", [1, 2, 4, 8]), knob("unroll", [1, 2, 4])])
    return {"name": "mobilenetv2_sim", "subgraphs": subgraphs}


def bert_base(seq=512, hidden=768, heads=12, ffn=3072, layers=12):
    T = [1, 2, 4, 8, 16, 32, 64, 128, 256, 512]
    dense_knobs = [knob("tile_m", T), knob("tile_n", T), knob("tile_k", P2), knob("unroll", [1, 2, 4, 8]),
                   knob("vector_width", [1, 4])]
    bmm_knobs = [knob("tile_batch", [1, 2, 3, 4, 6, 12]), knob("tile_m", T), knob("tile_n", T),
                 knob("unroll", [1, 2, 4, 8]), knob("vector_width", [1, 2, 4, 8])]
    sm_knobs = [knob("tile_rows", P2), knob("vector_width", [1, 2, 4, 8]), knob("unroll", [1, 2, 4]),
                knob("threads", [32, 64, 128, 256, 512, 1024]), knob("tile_cols", P2), knob("split", [1, 2])]
    hd = hidden // heads
    s = [
        {"ops": [op("embedding", [1, seq], vocab=30522), op("add", [1, seq, hidden])], "core_op": "embedding",
         "weight": 1, "knobs": [knob("tile_rows", P2), knob("tile_cols", P2), knob("unroll", [1, 2, 4])]},
        {"ops": [op("layer_norm", [1, seq, hidden], axis=2)], "core_op": "layer_norm", "weight": 2 * layers + 1,
         "knobs": [knob("tile_rows", P2), knob("vector_width", [1, 2, 4, 8]), knob("unroll", [1, 2, 4])]},
        {"ops": [op("dense", [seq, hidden], units=3 * hidden)], "core_op": "dense", "weight": layers,
         "knobs": dense_knobs},
        {"ops": [op("dense", [seq, hidden], units=hidden), op("add", [1, seq, hidden])], "core_op": "dense",
         "weight": layers, "knobs": dense_knobs},
        {"ops": [op("dense", [seq, hidden], units=ffn), op("gelu", [1, seq, ffn])], "core_op": "dense",
         "weight": layers, "knobs": dense_knobs},
        {"ops": [op("dense", [seq, ffn], units=hidden), op("add", [1, seq, hidden])], "core_op": "dense",
         "weight": layers, "knobs": dense_knobs},
        {"ops": [op("dense", [1, hidden], units=hidden), op("tanh", [1, hidden])], "core_op": "dense", "weight": 1,
         "knobs": dense_knobs},
        {"ops": [op("batch_matmul", [heads, seq, hd], transpose_b=1)], "core_op": "batch_matmul", "weight": layers,
         "knobs": bmm_knobs},
        {"ops": [op("batch_matmul", [heads, seq, seq])], "core_op": "batch_matmul", "weight": layers,
         "knobs": bmm_knobs},
        {"ops": [op("softmax", [heads, seq, seq], axis=2)], "core_op": "softmax", "weight": layers, "knobs": sm_knobs},
        {"ops": [op("dense", [1, hidden], units=2), op("softmax", [1, 2])], "core_op": "softmax", "weight": 1,
         "knobs": sm_knobs},
        {"ops": [op("transpose", [1, seq, heads, hd]), op("reshape", [heads, seq, hd])], "core_op": "transpose",
         "weight": 3 * layers, "knobs": [knob("tile_rows", [1, 2, 4, 8, 16, 32]), knob("tile_cols", [1, 2, 4, 8, 16, 32])]},
    ]
    return {"name": "bert_base_sim", "subgraphs": s}


def main():
    out = os.path.join(HERE, "models")
    os.makedirs(out, exist_ok=True)
    for m in (mobilenetv2(), bert_base()):
        with open(os.path.join(out, m["name"] + ".json"), "w") as f:
            json.dump(m, f, indent=1)
            f.write("\n")
        print(m["name"], len(m["subgraphs"]), "subgraph entries")


if __name__ == "__main__":
    main()
