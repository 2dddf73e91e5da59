"""Writes the graph-description corpus (examples/*.json).

The paper's Section 6 applications (Gauss, Laplacian, FChain, SobelX,
EdgFig1, Sobel, Unsharp, Harris "4 local + 9 point", Tomasi "4 local + 10
point"; SPEC.md:494 names them but the reference ships no files) plus the
five BASELINE configurations, in the reference's graph-file schema
(ref: src/graph_io.cpp:237-374).  Every intermediate image declares its
width/height/format so a test can flip "virtual" off for the reference,
whose expand() rejects virtual images.  Default size 256x256.
Run: python examples/make_corpus.py
"""
import json
import pathlib

W = H = 256
OUT = pathlib.Path(__file__).resolve().parent


# ---- expression helpers (ExprOp names of expr.cpp to_string) -------------
def ci(v): return {"op": "const_i", "value": v}
def cf(v): return {"op": "const_f", "value": float(v)}
def inp(k): return {"op": "in", "index": k}
def win(dx=0, dy=0, k=0): return {"op": "win", "index": k, "dx": dx, "dy": dy}
def mask(dx=0, dy=0): return {"op": "mask", "dx": dx, "dy": dy}
def b(op, l, r): return {"op": op, "lhs": l, "rhs": r}
def u(op, a): return {"op": op, "arg": a}
def sel(c, t, e): return {"op": "select", "cond": c, "then": t, "else": e}
def cast(to, a, policy="saturate"): return {"op": "cast", "to": to, "policy": policy, "arg": a}


def img(name, fmt, virtual=False, w=W, h=H):
    d = {"name": name, "width": w, "height": h, "format": fmt}
    if virtual:
        d["virtual"] = True
    return d


def node(kernel, *params, **attrs):
    n = {"kernel": kernel, "params": list(params)}
    if attrs:
        n["attrs"] = attrs
    return n


def sig(*params):
    out = []
    for p in params:
        direction, kind, fmt, name = p
        out.append({"direction": direction, "kind": kind, "format": fmt, "name": name})
    return out


def doc(name, images, nodes, outputs, **extra):
    d = {"name": name, "images": images, "nodes": nodes, "outputs": outputs}
    d.update(extra)
    return d


BIN5 = [1, 4, 6, 4, 1]
BINOMIAL5 = [a * c for a in BIN5 for c in BIN5]

corpus = {}

# Gauss: one 5x5 local node (Convolve, binomial / 256 -> U8)
corpus["gauss"] = doc(
    "gauss", [img("in", "U8"), img("out", "U8")],
    [node("Convolve", "in", "g5", "out", scale=256, out="U8")], ["out"],
    matrices=[{"name": "g5", "format": "S32", "rows": 5, "cols": 5, "values": BINOMIAL5}])

# Laplacian: custom convolution 3x3 -> S16
corpus["laplacian"] = doc(
    "laplacian", [img("in", "U8"), img("out", "S16")],
    [node("Convolve", "in", "lap", "out")], ["out"],
    matrices=[{"name": "lap", "format": "S32", "rows": 3, "cols": 3, "values": [0, 1, 0, 1, -4, 1, 0, 1, 0]}])

# FChain: three convolution (local) nodes
corpus["fchain"] = doc(
    "fchain",
    [img("in", "U8"), img("c1", "U8", True), img("c2", "U8", True), img("out", "U8")],
    [node("Convolve", "in", "gauss3", "c1", scale=16, out="U8"),
     node("Convolve", "c1", "box3", "c2", scale=9, out="U8"),
     node("Convolve", "c2", "sharpen3", "out", out="U8")], ["out"],
    matrices=[{"name": "gauss3", "format": "S32", "rows": 3, "cols": 3, "values": [1, 2, 1, 2, 4, 2, 1, 2, 1]},
              {"name": "box3", "format": "S32", "rows": 3, "cols": 3, "values": [1] * 9},
              {"name": "sharpen3", "format": "S32", "rows": 3, "cols": 3,
               "values": [0, -1, 0, -1, 5, -1, 0, -1, 0]}])

# SobelX: horizontal derivative only (gy unbound -> its expansion is dead)
corpus["sobelx"] = doc(
    "sobelx", [img("in", "U8"), img("gx", "S16")],
    [node("Sobel3x3", "in", "gx", None)], ["gx"])

# EdgFig1 (Listing 1 / Fig. 1): ChannelExtract -> Gaussian3x3 -> Sobel3x3 ->
# Magnitude(gy, gy) -> Threshold; gx is computed but never used
corpus["edge_fig1"] = doc(
    "edge_fig1",
    [img("yuv", "UYVY"), img("y", "U8", True), img("g", "U8", True), img("gx", "S16", True),
     img("gy", "S16", True), img("mag", "S16", True), img("edges", "U8")],
    [node("ChannelExtract", "yuv", "y", channel="Y"), node("Gaussian3x3", "y", "g"),
     node("Sobel3x3", "g", "gx", "gy"), node("Magnitude", "gy", "gy", "mag"),
     node("Threshold", "mag", "thresh", None, "edges")], ["edges"],
    scalars=[{"name": "thresh", "format": "S16", "value": 100}])

# Sobel: both derivatives through three CV nodes
corpus["sobel"] = doc(
    "sobel",
    [img("in", "U8"), img("gx", "S16", True), img("gy", "S16", True), img("mag", "S16", True), img("out", "U8")],
    [node("Sobel3x3", "in", "gx", "gy"), node("Magnitude", "gx", "gy", "mag"),
     node("ConvertDepth", "mag", "out", shift=2)], ["out"])

# Unsharp: one Gauss node and three point nodes
corpus["unsharp"] = doc(
    "unsharp",
    [img("in", "U8"), img("blur", "U8", True), img("diff", "S16", True), img("sum", "S16", True),
     img("out", "U8")],
    [node("Gaussian3x3", "in", "blur"), node("Subtract", "in", "blur", "diff"),
     node("Add", "in", "diff", "sum"), node("ConvertDepth", "sum", "out")], ["out"])


# Harris (4 local + 9 point): Sobel, 3 products, 3 box filters, det / trace
# point nodes, and a user point for the response decision
def corner_images(extra):
    base = [img("in", "U8"), img("gx", "S16", True), img("gy", "S16", True),
            img("ixx", "S32", True), img("iyy", "S32", True), img("ixy", "S32", True),
            img("sxx", "S32", True), img("syy", "S32", True), img("sxy", "S32", True)]
    return base + extra


corner_front = [node("Sobel3x3", "in", "gx", "gy"),
                node("Multiply", "gx", "gx", "ixx"), node("Multiply", "gy", "gy", "iyy"),
                node("Multiply", "gx", "gy", "ixy"),
                node("Box3x3", "ixx", "sxx"), node("Box3x3", "iyy", "syy"), node("Box3x3", "ixy", "sxy")]

harris_decide = {
    "name": "HarrisDecide", "kind": "point",
    "signature": sig(("input", "image", "S32", "det"), ("input", "image", "S32", "trace"),
                     ("output", "image", "U8", "corners")),
    "body": cast("U8", sel(b("gt", b("sub", inp(0), b("mul", cf(0.04), b("mul", inp(1), inp(1)))), cf(1.0e7)),
                           ci(255), ci(0)))}
corpus["harris"] = doc(
    "harris",
    corner_images([img("pxy", "S32", True), img("pxx_yy", "S32", True), img("det", "S32", True),
                   img("trace", "S32", True), img("mask", "U8", True), img("corners", "U8")]),
    corner_front + [node("Multiply", "sxx", "syy", "pxx_yy"), node("Multiply", "sxy", "sxy", "pxy"),
                    node("Subtract", "pxx_yy", "pxy", "det"), node("Add", "sxx", "syy", "trace"),
                    node("HarrisDecide", "det", "trace", "mask"), node("Copy", "mask", "corners")], ["corners"],
    custom_kernels=[harris_decide])

# Tomasi (4 local + 10 point): min eigenvalue of the structure tensor
tomasi_lambda = {
    "name": "MinEigen", "kind": "point",
    "signature": sig(("input", "image", "S32", "trace"), ("input", "image", "S32", "d2"),
                     ("input", "image", "S32", "sxy2"), ("output", "image", "F32", "lambda")),
    "body": cast("F32", b("mul", cf(0.5), b("sub", inp(0), u("sqrt", b("add", inp(1), b("mul", ci(4), inp(2)))))))}
tomasi_decide = {
    "name": "EigenThreshold", "kind": "point",
    "signature": sig(("input", "image", "F32", "lambda"), ("output", "image", "U8", "mask")),
    "body": cast("U8", sel(b("gt", inp(0), cf(2000.0)), ci(255), ci(0)))}
corpus["tomasi"] = doc(
    "tomasi",
    corner_images([img("trace", "S32", True), img("d", "S32", True), img("d2", "S32", True),
                   img("sxy2", "S32", True), img("lambda", "F32", True), img("mask", "U8", True),
                   img("corners", "U8")]),
    corner_front + [node("Add", "sxx", "syy", "trace"), node("Subtract", "sxx", "syy", "d"),
                    node("Multiply", "d", "d", "d2"), node("Multiply", "sxy", "sxy", "sxy2"),
                    node("MinEigen", "trace", "d2", "sxy2", "lambda"),
                    node("EigenThreshold", "lambda", "mask"), node("Copy", "mask", "corners")], ["corners"],
    custom_kernels=[tomasi_lambda, tomasi_decide])

# ---- the BASELINE configurations as graph files ----------------------------
corpus["cfg1_edge"] = doc(
    "cfg1_edge",
    [img("in", "U8", w=1920, h=1080), img("g", "U8", True, 1920, 1080), img("gx", "S16", True, 1920, 1080),
     img("gy", "S16", True, 1920, 1080), img("mag", "S16", w=1920, h=1080)],
    [node("Gaussian3x3", "in", "g"), node("Sobel3x3", "g", "gx", "gy"), node("Magnitude", "gx", "gy", "mag")],
    ["mag"])

harris_response = {
    "name": "HarrisResponse", "kind": "point",
    "signature": sig(("input", "image", "S32", "sxx"), ("input", "image", "S32", "syy"),
                     ("input", "image", "S32", "sxy"), ("output", "image", "F32", "resp")),
    "body": cast("F32", b("sub", b("sub", b("mul", inp(0), inp(1)), b("mul", inp(2), inp(2))),
                          b("mul", cf(0.04), b("mul", b("add", inp(0), inp(1)), b("add", inp(0), inp(1))))))}
threshold_f32 = {
    "name": "ThresholdF32", "kind": "point",
    "signature": sig(("input", "image", "F32", "resp"), ("output", "image", "U8", "mask")),
    "body": cast("U8", sel(b("gt", inp(0), cf(1.0e9)), ci(255), ci(0)))}
corpus["cfg2_harris"] = doc(
    "cfg2_harris",
    corner_images([img("resp", "F32", True), img("mask", "U8")]),
    corner_front + [node("HarrisResponse", "sxx", "syy", "sxy", "resp"), node("ThresholdF32", "resp", "mask")],
    ["mask"], custom_kernels=[harris_response, threshold_f32])

blur5 = {
    "name": "Blur5x5", "kind": "local", "window": [5, 5], "boundary": "clamp", "combine": "sum",
    "signature": sig(("input", "image", "U8", "in"), ("output", "image", "U8", "out")),
    "mask": BINOMIAL5, "tap_body": b("mul", mask(), win()),
    "post_body": cast("U8", b("mul", inp(0), cf(1.0 / 256.0)))}
corpus["cfg3_unsharp"] = doc(
    "cfg3_unsharp",
    [img("in", "U8"), img("blur", "U8", True), img("diff", "S16", True), img("sum", "S16", True),
     img("sharp", "U8")],
    [node("Blur5x5", "in", "blur"), node("Subtract", "in", "blur", "diff"), node("Add", "in", "diff", "sum"),
     node("ConvertDepth", "sum", "sharp")], ["sharp"], custom_kernels=[blur5])

corpus["cfg4_stats"] = doc(
    "cfg4_stats",
    [img("in", "U8"), img("conv", "S16", True), img("u8", "U8", True)],
    [node("Convolve", "in", "binomial5", "conv", scale=256), node("ConvertDepth", "conv", "u8"),
     node("Histogram", "u8", "dist"), node("MeanStdDev", "u8", "mean", "stddev")],
    ["dist", "mean", "stddev"],
    matrices=[{"name": "binomial5", "format": "S32", "rows": 5, "cols": 5, "values": BINOMIAL5}],
    arrays=[{"name": "dist", "format": "S32", "capacity": 256}],
    scalars=[{"name": "mean", "format": "F32"}, {"name": "stddev", "format": "F32"}])

for name, d in corpus.items():
    (OUT / f"{name}.json").write_text(json.dumps(d, indent=2) + "\n")
print(f"wrote {len(corpus)} graph files to {OUT}")
