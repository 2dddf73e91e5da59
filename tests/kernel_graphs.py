"""Single-kernel graph files covering every built-in kernel of the registry
(28 kernels; ref: src/registry.cpp) with several formats, attributes and
border-heavy sizes.  Shared by tests/golden/make_kernel_golden.py (which runs
them on the unmodified reference engine) and tests/test_gpu_kernel_files.py
(which runs them on the B200, fused and unfused).  Inputs are the
reference's random_buffer(desc, seed + object id) for every source image."""
import json

SIZES = [(37, 23), (64, 5), (1, 1)]


def img(name, fmt, w, h):
    return {"name": name, "width": w, "height": h, "format": fmt}


def graph(name, images, nodes, outputs, **extra):
    d = {"name": name, "images": images, "nodes": nodes, "outputs": outputs}
    d.update(extra)
    return d


def node(kernel, *params, **attrs):
    n = {"kernel": kernel, "params": list(params)}
    if attrs:
        n["attrs"] = attrs
    return n


def specs(w, h):
    """(name, graph dict) for one image size."""
    out = []

    def unary(kernel, fin, fout, tag="", **attrs):
        out.append((f"{kernel}{tag}", graph(kernel, [img("in", fin, w, h), img("out", fout, w, h)],
                                             [node(kernel, "in", "out", **attrs)], ["out"])))

    def binary(kernel, fin, fout, tag="", **attrs):
        out.append((f"{kernel}{tag}", graph(kernel, [img("a", fin, w, h), img("b", fin, w, h),
                                                      img("out", fout, w, h)],
                                             [node(kernel, "a", "b", "out", **attrs)], ["out"])))

    unary("ChannelExtract", "UYVY", "U8", "_uyvy_Y", channel="Y")
    unary("ChannelExtract", "RGB", "U8", "_rgb_G", channel="G")
    out.append(("ChannelCombine", graph("ChannelCombine", [img("r", "U8", w, h), img("g", "U8", w, h),
                                                           img("b", "U8", w, h), img("out", "RGB", w, h)],
                                        [node("ChannelCombine", "r", "g", "b", "out")], ["out"])))
    binary("Add", "U8", "S16")
    binary("Add", "S16", "S16", "_s16")
    binary("Add", "S16", "S32", "_u16", out="S32")
    binary("Add", "U8", "U8", "_sat_u8", out="U8")
    binary("Subtract", "U8", "S16")
    binary("Subtract", "S16", "S16", "_s16")
    binary("Multiply", "S16", "S32")
    binary("Multiply", "U8", "U8", "_scaled", out="U8", scale=0.37)
    binary("AbsDiff", "U8", "U8")
    binary("AbsDiff", "S16", "S16", "_s16")
    for k in ("And", "Or", "Xor"):
        binary(k, "U8", "U8")
    binary("Xor", "S16", "S16", "_s16")
    unary("Not", "U8", "U8")
    binary("Magnitude", "S16", "S16")
    binary("Phase", "S16", "U8")
    out.append(("Threshold_binary", graph(
        "Threshold", [img("in", "U8", w, h), img("out", "U8", w, h)],
        [node("Threshold", "in", "t", None, "out")], ["out"],
        scalars=[{"name": "t", "format": "U8", "value": 100}])))
    out.append(("Threshold_range", graph(
        "Threshold", [img("in", "S16", w, h), img("out", "U8", w, h)],
        [node("Threshold", "in", "lo", "hi", "out", mode="range")], ["out"],
        scalars=[{"name": "lo", "format": "S16", "value": -1000}, {"name": "hi", "format": "S16", "value": 2500}])))
    unary("ConvertDepth", "S16", "U8", "_shr2_sat", shift=2)
    unary("ConvertDepth", "S16", "U8", "_wrap", policy="wrap")
    unary("ConvertDepth", "U8", "S16", "_shl3", to="S16", shift=3)
    unary("Copy", "S32", "S32")
    unary("Box3x3", "U8", "U8")
    unary("Box3x3", "S16", "S16", "_s16")
    unary("Gaussian3x3", "U8", "U8")
    unary("Gaussian3x3", "F32", "F32", "_f32")
    out.append(("Sobel3x3", graph("Sobel3x3", [img("in", "U8", w, h), img("gx", "S16", w, h), img("gy", "S16", w, h)],
                                  [node("Sobel3x3", "in", "gx", "gy")], ["gx", "gy"])))
    for k in ("Dilate3x3", "Erode3x3", "Median3x3"):
        unary(k, "U8", "U8")
    out.append(("Convolve_3x3_s16", graph(
        "Convolve", [img("in", "U8", w, h), img("out", "S16", w, h)],
        [node("Convolve", "in", "m", "out", scale=4)], ["out"],
        matrices=[{"name": "m", "format": "S32", "rows": 3, "cols": 3, "values": [1, -2, 3, -4, 9, 4, -3, 2, -1]}])))
    out.append(("Convolve_5x3_f32", graph(
        "Convolve", [img("in", "U8", w, h), img("out", "F32", w, h)],
        [node("Convolve", "in", "m", "out")], ["out"],
        matrices=[{"name": "m", "format": "F32", "rows": 3, "cols": 5,
                   "values": [0.1, 0.25, -0.5, 0.25, 0.1, 0.05, 1.5, 0.0, -1.5, 0.05, 0.1, 0.2, 0.3, 0.2, 0.1]}])))
    out.append(("Histogram", graph(
        "Histogram", [img("in", "U8", w, h)], [node("Histogram", "in", "dist", bins=16, offset=10, range=200)],
        ["dist"], arrays=[{"name": "dist", "format": "S32", "capacity": 16}])))
    out.append(("MinMaxLoc", graph(
        "MinMaxLoc", [img("in", "U8", w, h)], [node("MinMaxLoc", "in", "mn", "mx", "mnl", "mxl")],
        ["mn", "mx", "mnl", "mxl"],
        scalars=[{"name": "mn", "format": "U8"}, {"name": "mx", "format": "U8"}],
        arrays=[{"name": "mnl", "format": "S32", "capacity": 2}, {"name": "mxl", "format": "S32", "capacity": 2}])))
    out.append(("MeanStdDev", graph(
        "MeanStdDev", [img("in", "U8", w, h)], [node("MeanStdDev", "in", "mean", "sd")], ["mean", "sd"],
        scalars=[{"name": "mean", "format": "F32"}, {"name": "sd", "format": "F32"}])))
    unary("IntegralImage", "U8", "S32")
    for interp in ("nearest", "bilinear"):
        for (ow, oh) in ((2 * w + 1, h + 3), (max(1, w // 2), max(1, h // 3))):
            for fmt in ("U8", "S16", "F32"):
                out.append((f"ScaleImage_{interp}_{fmt}_{ow}x{oh}", graph(
                    "ScaleImage", [img("in", fmt, w, h), img("out", fmt, ow, oh)],
                    [node("ScaleImage", "in", "out", interp=interp)], ["out"])))
    unary("EqualizeHist", "U8", "U8")
    return out


def all_cases():
    """[(case id, json text)] over all sizes."""
    cases = []
    for (w, h) in SIZES:
        for name, g in specs(w, h):
            cases.append((f"{name}_{w}x{h}", json.dumps(g)))
    return cases


KERNELS = ["ChannelExtract", "ChannelCombine", "Add", "Subtract", "Multiply", "AbsDiff", "And", "Or", "Xor", "Not",
           "Magnitude", "Phase", "Threshold", "ConvertDepth", "Copy", "Box3x3", "Gaussian3x3", "Sobel3x3",
           "Dilate3x3", "Erode3x3", "Median3x3", "Convolve", "Histogram", "MinMaxLoc", "MeanStdDev",
           "IntegralImage", "ScaleImage", "EqualizeHist"]
