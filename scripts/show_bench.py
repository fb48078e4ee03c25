import json, sys
for f in sys.argv[1:]:
    d = json.load(open(f))
    r = d["roofline"]
    print(f.split("/")[-1], "value %.1f attn %.1f TF/s (frac %.3f) speedup %.2f / bound %.2f = %.2f stages %s perm %.0f unperm %.0f GB/s dense %.1f mma %.1f e2e %.1f clk %s" % (
        d["value"], r["achieved"], r["frac"], d["speedup_vs_dense"], d["bound"], d["speedup_frac_of_bound"],
        {k: round(v, 3) for k, v in d["stages_ms"].items()}, d["permute_gbs"], d["unpermute_gbs"],
        d["dense_effective_tflops"], d["mma_issued_tflops"], d["e2e"]["value"], d["clocks"]))
