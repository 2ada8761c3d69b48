"""Copy the on-box ncu summaries (gpurun_out/ncu_<name>.json, scripts/ncu_r02.py) into
profiles/ under the names bench.py's PROFILE_OF reads, plus the launch list if present.
usage: python scripts/install_profiles.py [name ...]"""
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NAMES = {"xm_cfg2": "r02_xm_cfg2_ncu.json", "xm_cfg1": "r02_xm_cfg1_ncu.json", "xmi_cfg4": "r02_xmi_cfg4_ncu.json",
         "var_cfg3": "r02_term_var_cfg3_ncu.json", "varx_cfg3k": "r02_term_varx_cfg3k_ncu.json",
         "tma_cfg5": "r02_term_tma_cfg5_ncu.json", "xs_cfg5": "r02_term_xs_cfg5_ncu.json", "xs2_cfg5": "r02_term_xs2_cfg5_ncu.json", "varx_cfg5var": "r02_term_varx_cfg5var_ncu.json",
         "tma_hybrid256": "r02_term_tma_hybrid256_ncu.json", "xs_hybrid256": "r02_term_xs_hybrid256_ncu.json",
         "xs_hybrid512": "r02_term_xs_hybrid512_ncu.json", "tma_hybrid512": "r02_term_tma_hybrid512_ncu.json",
         "em_cfg2": "r02_em_cluster_ip_cfg2_ncu.json", "em_cfg5": "r02_em_tb_cfg5_ncu.json"}
for name in sys.argv[1:] or NAMES:
    src = os.path.join(ROOT, "gpurun_out", f"ncu_{name}.json")
    if not os.path.exists(src):
        print("missing", src)
        continue
    d = json.load(open(src))
    dst = os.path.join(ROOT, "profiles", NAMES[name])
    with open(dst, "w") as fh:
        json.dump(d, fh, indent=1)
    print(name, "->", NAMES[name], d["kernel_mangled"][:80])
