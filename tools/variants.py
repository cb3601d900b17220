"""Build experiment variants of libsaloba.so with extra -D flags (kernel A/B on one GPU call).

    python tools/variants.py name1="-DFOO=1" name2="-DBAR"     # -> build/variants/<name>/libsaloba.so
Run a variant with SALOBA_LIB=build/variants/<name>/libsaloba.so python bench.py ...
"""
import os
import shlex
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import build_native as bn  # noqa: E402

for arg in sys.argv[1:]:
    name, _, flags = arg.partition("=")
    d = os.path.join(bn.ROOT, "build", "variants", name)
    if os.environ.get("VARIANTS_PREBUILT") and os.path.exists(os.path.join(d, "libsaloba.so")):
        print(name, "prebuilt")  # built here before the GPU call: never rebuilt from newer sources there
        continue
    bn.build_saloba(force=False, out=os.path.join(d, "libsaloba.so"), defines=shlex.split(flags), objdir=d)
    print(name, "->", os.path.join(d, "libsaloba.so"))
