import sys, faulthandler
faulthandler.enable()
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from golden_io import GoldenScene
from paper_1604_01093_b200.runtime import runtime
sc = GoldenScene(sys.argv[1] if len(sys.argv) > 1 else "cfg3")
rt = runtime(0)
print("uploading", len(sc.caches), flush=True)
rt.slots_for([sc.caches[f] for f in sc.ids])
print("ok", flush=True)
