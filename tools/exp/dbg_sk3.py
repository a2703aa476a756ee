import os, sys
sys.path.insert(0, os.getcwd())
exec(open("tools/exp/dbg_sk4.py").read().split("run(3, 14")[0])
for env in [{"DG_NO_SPLITK": "1"}, {}]:
    for k in ("DG_NO_SPLITK", "DG_SK", "DG_SK_NORED"):
        os.environ.pop(k, None)
    os.environ.update(env); print(env)
    run(1, 28, 128, 128, 3, 1)
    run(1, 7, 512, 512, 3, 1)
