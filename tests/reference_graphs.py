"""Graph files for reference-pinned parity beyond the registry one-node
cases (tests/kernel_graphs.py): user-defined local kernels with Constant /
Undefined borders, Min / Max combines, real masks and extra pointwise
inputs (ref:src/execute.cpp:193-267, 504-622; ref:src/graph_io.cpp:166-222),
chains of them through virtual intermediates (the fusion refusals of
DESIGN.md §1), U16 images (ref:src/execute.cpp:41-44, ref:src/registry.cpp:119-128),
the cfg4 fused Convolve -> ConvertDepth -> Histogram + MeanStdDev shape with
identity bins, and random DAGs over the registry.  tests/test_gpu_reference_graphs.py
runs each on the B200 (run_plan and run_naive) and on the UNMODIFIED
reference (oracle/_ref, non-virtual intermediates) and compares bytes."""
import json
import random


def img(name, fmt, w, h, virtual=False):
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
    return [{"direction": d, "kind": "image", "format": f, "name": n} for d, f, n in params]


# ---- expression helpers (ref:src/expr.cpp:78-104 op names)
def ci(v):
    return {"op": "const_i", "value": v}


def cf(v):
    return {"op": "const_f", "value": v}


def inp(i):
    return {"op": "in", "index": i}


def win(dx=0, dy=0, index=0):
    return {"op": "win", "index": index, "dx": dx, "dy": dy}


def mask(dx=0, dy=0):
    return {"op": "mask", "dx": dx, "dy": dy}


def op(name, a, b=None):
    if b is None:
        return {"op": name, "arg": a}
    return {"op": name, "lhs": a, "rhs": b}


def cast(to, a, policy="saturate"):
    return {"op": "cast", "to": to, "policy": policy, "arg": a}


def local(name, window, boundary, combine, tap, post, signature, mask_vals=None, boundary_value=None):
    k = {"name": name, "kind": "local", "window": list(window), "boundary": boundary, "combine": combine,
         "signature": signature, "tap_body": tap, "post_body": post}
    if mask_vals is not None:
        k["mask"] = mask_vals
    if boundary_value is not None:
        k["boundary_value"] = boundary_value
    return k


def point(name, body, signature):
    return {"name": name, "kind": "point", "signature": signature, "body": body}


GAUSS = [1, 2, 1, 2, 4, 2, 1, 2, 1]


def custom_local_cases(w, h):
    """(name, graph dict)."""
    out = []
    u8io = sig(("input", "U8", "in"), ("output", "U8", "out"))

    def one(name, k, fout="U8"):
        k = dict(k)
        k["signature"] = sig(("input", "U8", "in"), ("output", fout, "out"))
        out.append((name, {"name": name, "images": [img("in", "U8", w, h), img("out", fout, w, h)],
                           "custom_kernels": [k], "nodes": [node(k["name"], "in", "out")], "outputs": ["out"]}))

    one("const7_gauss_sum", local("CGauss", (3, 3), "constant", "sum", op("mul", mask(), win()),
                                  cast("U8", op("mul", inp(0), cf(1 / 16))), u8io, GAUSS, boundary_value=7))
    one("const200_max5x3", local("CMax", (5, 3), "constant", "max", win(),
                                 cast("U8", inp(0)), u8io, boundary_value=200))
    one("const0_min3x5_s16", local("CMin", (3, 5), "constant", "min", op("sub", op("mul", win(), ci(2)), mask()),
                                   cast("S16", inp(0)), u8io, list(range(15)), boundary_value=0), "S16")
    one("undef_sum3x3_s16", local("USum", (3, 3), "undefined", "sum", op("mul", mask(), win()),
                                  cast("S16", inp(0)), u8io, [-1, 0, 1, -2, 0, 2, -1, 0, 1]), "S16")
    one("undef_min5x5", local("UMin", (5, 5), "undefined", "min", win(), cast("U8", inp(0)), u8io))
    one("undef_max3x1", local("UMax", (3, 1), "undefined", "max", op("add", win(), mask()),
                              cast("U8", inp(0)), u8io, [5, 0, 9]))
    one("clamp_min3x3", local("KMin", (3, 3), "clamp", "min", win(), cast("U8", inp(0)), u8io))
    one("clamp_max5x5", local("KMax", (5, 5), "clamp", "max", op("mul", win(), mask()),
                              cast("U8", op("shr", inp(0), ci(3))), u8io, [(i * 7) % 9 for i in range(25)]))
    one("clamp_realmask3x3_s16", local("KReal", (3, 3), "clamp", "sum", op("mul", mask(), win()),
                                       cast("S16", inp(0)), u8io, [0.1, -0.25, 0.5, 1.5, -2.75, 0.3, 0.05, 0.2, -0.125]),
        "S16")
    one("const3_realmask5x3_f32", local("CReal", (5, 3), "constant", "sum", op("mul", mask(), win()),
                                        cast("F32", op("mul", inp(0), cf(0.37))), u8io,
                                        [0.5, 0.25, 0.125, 0.25, 0.5, 1.0, 2.0, -3.0, 2.0, 1.0, 0.1, 0.2, 0.3, 0.2,
                                         0.1], boundary_value=3), "F32")
    one("undef_realmask3x3_u8", local("UReal", (3, 3), "undefined", "sum", op("mul", mask(), win()),
                                      cast("U8", inp(0)), u8io, [0.0625, 0.125, 0.0625, 0.125, 0.25, 0.125, 0.0625,
                                                                 0.125, 0.0625]))
    # post body with an extra pointwise input (slot 1 = aux at the output pixel)
    k = local("PostAux", (3, 3), "constant", "sum", win(), cast("S16", op("sub", inp(0), op("mul", inp(1), ci(9)))),
              sig(("input", "U8", "in"), ("input", "U8", "aux"), ("output", "S16", "out")), boundary_value=11)
    out.append(("const11_post_extra_input", {
        "name": "post_extra", "images": [img("in", "U8", w, h), img("aux", "U8", w, h), img("out", "S16", w, h)],
        "custom_kernels": [k], "nodes": [node("PostAux", "in", "aux", "out")], "outputs": ["out"]}))
    # chains through virtual intermediates: constant -> undefined locals,
    # point -> constant local (fusion refused), undefined local -> point
    kc = local("CBox", (3, 3), "constant", "sum", win(), cast("U8", op("div", inp(0), ci(9))), u8io, boundary_value=40)
    ku = local("UMax3", (3, 3), "undefined", "max", win(), cast("U8", inp(0)), u8io)
    kp = point("Inv", cast("U8", op("sub", ci(255), inp(0))), u8io)
    out.append(("chain_const_undef", {
        "name": "chain1", "images": [img("in", "U8", w, h), img("m", "U8", w, h, True), img("out", "U8", w, h)],
        "custom_kernels": [kc, ku], "nodes": [node("CBox", "in", "m"), node("UMax3", "m", "out")], "outputs": ["out"]}))
    out.append(("chain_point_const", {
        "name": "chain2", "images": [img("in", "U8", w, h), img("m", "U8", w, h, True), img("out", "U8", w, h)],
        "custom_kernels": [kp, kc], "nodes": [node("Inv", "in", "m"), node("CBox", "m", "out")], "outputs": ["out"]}))
    out.append(("chain_undef_point", {
        "name": "chain3", "images": [img("in", "U8", w, h), img("m", "U8", w, h, True), img("out", "U8", w, h)],
        "custom_kernels": [ku, kp], "nodes": [node("UMax3", "in", "m"), node("Inv", "m", "out")], "outputs": ["out"]}))
    out.append(("chain_gauss_const_sobel", {
        "name": "chain4", "images": [img("in", "U8", w, h), img("m", "U8", w, h, True), img("gx", "S16", w, h),
                                     img("gy", "S16", w, h)],
        "custom_kernels": [kc], "nodes": [node("CBox", "in", "m"), node("Sobel3x3", "m", "gx", "gy")],
        "outputs": ["gx", "gy"]}))
    return out


def u16_cases(w, h):
    out = []

    def g(name, images, nodes, outputs, **extra):
        d = {"name": name, "images": images, "nodes": nodes, "outputs": outputs}
        d.update(extra)
        out.append((name, d))

    A, B = img("a", "U16", w, h), img("b", "U16", w, h)
    g("u16_add_s32", [A, B, img("o", "S32", w, h)], [node("Add", "a", "b", "o")], ["o"])
    g("u16_sub_u8_s32", [A, img("b", "U8", w, h), img("o", "S32", w, h)], [node("Subtract", "a", "b", "o")], ["o"])
    g("u16_mul_s32", [A, B, img("o", "S32", w, h)], [node("Multiply", "a", "b", "o")], ["o"])
    g("u16_absdiff", [A, B, img("o", "U16", w, h)], [node("AbsDiff", "a", "b", "o")], ["o"])
    g("u16_box3x3", [A, img("o", "U16", w, h)], [node("Box3x3", "a", "o")], ["o"])
    g("u16_gauss3x3", [A, img("o", "U16", w, h)], [node("Gaussian3x3", "a", "o")], ["o"])
    g("u16_median", [A, img("o", "U16", w, h)], [node("Median3x3", "a", "o")], ["o"])
    g("u16_to_u8_shr8", [A, img("o", "U8", w, h)], [node("ConvertDepth", "a", "o", shift=8)], ["o"])
    g("u16_to_u8_wrap", [A, img("o", "U8", w, h)], [node("ConvertDepth", "a", "o", policy="wrap")], ["o"])
    g("u16_copy", [A, img("o", "U16", w, h)], [node("Copy", "a", "o")], ["o"])
    g("u16_not", [A, img("o", "U16", w, h)], [node("Not", "a", "o")], ["o"])
    g("u16_threshold", [A, img("o", "U8", w, h)], [node("Threshold", "a", "t", None, "o")], ["o"],
      scalars=[{"name": "t", "format": "U16", "value": 30000}])
    g("u16_minmaxloc", [A], [node("MinMaxLoc", "a", "mn", "mx", "mnl", "mxl")], ["mn", "mx", "mnl", "mxl"],
      scalars=[{"name": "mn", "format": "U16"}, {"name": "mx", "format": "U16"}],
      arrays=[{"name": "mnl", "format": "S32", "capacity": 2}, {"name": "mxl", "format": "S32", "capacity": 2}])
    g("u16_meanstddev", [A], [node("MeanStdDev", "a", "mean", "sd")], ["mean", "sd"],
      scalars=[{"name": "mean", "format": "F32"}, {"name": "sd", "format": "F32"}])
    g("u16_histogram", [A], [node("Histogram", "a", "dist", bins=32, offset=1000, range=60000)], ["dist"],
      arrays=[{"name": "dist", "format": "S32", "capacity": 32}])
    g("u16_integral", [A, img("o", "S32", w, h)], [node("IntegralImage", "a", "o")], ["o"])
    k = local("Lap16", (3, 3), "clamp", "sum", op("mul", mask(), win()), cast("S32", inp(0)),
              sig(("input", "U16", "in"), ("output", "S32", "out")), [0, -1, 0, -1, 4, -1, 0, -1, 0])
    g("u16_custom_local", [A, img("o", "S32", w, h)], [node("Lap16", "a", "o")], ["o"], custom_kernels=[k])
    return out


def stats_cases(w, h):
    """cfg4's fused shape (Convolve -> ConvertDepth -> Histogram + MeanStdDev)
    with bin layouts the device merge treats specially (identity bins)."""
    out = []
    binom = [1, 4, 6, 4, 1]
    m = [a * b for a in binom for b in binom]
    for bins, offset, rng in ((16, 0, 16), (256, 0, 256), (64, 0, 64), (16, 100, 16), (7, 3, 250)):
        name = f"conv_stats_bins{bins}_off{offset}_range{rng}"
        out.append((name, {
            "name": name,
            "images": [img("in", "U8", w, h), img("c", "S16", w, h, True), img("u", "U8", w, h, True)],
            "matrices": [{"name": "m", "format": "S32", "rows": 5, "cols": 5, "values": m}],
            "nodes": [node("Convolve", "in", "m", "c", scale=256), node("ConvertDepth", "c", "u"),
                      node("Histogram", "u", "dist", bins=bins, offset=offset, range=rng),
                      node("MeanStdDev", "u", "mean", "sd")],
            "arrays": [{"name": "dist", "format": "S32", "capacity": bins}],
            "scalars": [{"name": "mean", "format": "F32"}, {"name": "sd", "format": "F32"}],
            "outputs": ["dist", "mean", "sd"]}))
    return out


def random_dag(seed, w, h):
    """A random DAG over registry kernels (the C++ soundness suite's mix,
    tests/cpp/test_graphvx.cpp RandomGraph), virtual intermediates, every
    sink declared as output."""
    rng = random.Random(seed)
    images, nodes, scalars = [], [], []
    u8, s16, consumed = [], [], set()
    for i in range(2):
        images.append(img(f"in{i}", "U8", w, h))
        u8.append(f"in{i}")
    n = 0

    def fresh(fmt, pool):
        nonlocal n
        name = f"t{n}"
        n += 1
        images.append(img(name, fmt, w, h, True))
        pool.append(name)
        return name

    def pick(pool):
        x = rng.choice(pool)
        consumed.add(x)
        return x

    for _ in range(rng.randint(3, 8)):
        k = rng.randrange(11)
        if k == 0:
            nodes.append(node("Gaussian3x3", pick(u8), fresh("U8", u8)))
        elif k == 1:
            nodes.append(node("Box3x3", pick(u8), fresh("U8", u8)))
        elif k == 2:
            src = pick(u8)
            nodes.append(node("Sobel3x3", src, fresh("S16", s16), fresh("S16", s16)))
        elif k == 3:
            nodes.append(node("Dilate3x3", pick(u8), fresh("U8", u8)))
        elif k == 4:
            nodes.append(node("Median3x3", pick(u8), fresh("U8", u8)))
        elif k == 5:
            a, b = pick(u8), pick(u8)
            nodes.append(node("Subtract", a, b, fresh("S16", s16)))
        elif k == 6 and len(s16) >= 2:
            a, b = pick(s16), pick(s16)
            nodes.append(node("Magnitude", a, b, fresh("S16", s16)))
        elif k == 7 and s16:
            nodes.append(node("ConvertDepth", pick(s16), fresh("U8", u8)))
        elif k == 8:
            a, b = pick(u8), pick(u8)
            nodes.append(node("AbsDiff", a, b, fresh("U8", u8)))
        elif k == 9:
            t = f"s{len(scalars)}"
            scalars.append({"name": t, "format": "U8", "value": rng.randrange(256)})
            nodes.append(node("Threshold", pick(u8), t, None, fresh("U8", u8)))
        else:
            nodes.append(node("Not", pick(u8), fresh("U8", u8)))
    sinks = [im["name"] for im in images if im.get("virtual") and im["name"] not in consumed]
    for im in images:
        if im["name"] in sinks:
            im.pop("virtual")
    d = {"name": f"dag{seed}", "images": images, "nodes": nodes, "outputs": sinks}
    if scalars:
        d["scalars"] = scalars
    return d


def reference_form(doc):
    """The same graph for the reference: no virtual images (its expand()
    rejects them, SURVEY.md §0 finding 1); declared outputs unchanged."""
    d = json.loads(json.dumps(doc))
    for im in d["images"]:
        im.pop("virtual", None)
    return d


def all_cases():
    cases = []
    for (w, h) in ((37, 23), (64, 5), (1, 1), (130, 7)):
        for name, g in custom_local_cases(w, h) + u16_cases(w, h) + stats_cases(w, h):
            cases.append((f"{name}_{w}x{h}", g))
    return cases
