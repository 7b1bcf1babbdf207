import sys, time, cProfile, pstats, io
sys.path.insert(0,'/root/repo'); sys.argv=['x']
sys.path.insert(0,'/root/repo/tools')
import importlib.util
spec=importlib.util.spec_from_file_location('tsm','/root/repo/tools/time_species_meshes.py'); m=importlib.util.module_from_spec(spec); spec.loader.exec_module(m)
import paper_1702_08880_b200 as pkg
orig=pkg.assemble_species_meshes
calls=[0]
def wrapped(*a,**k):
    calls[0]+=1
    if calls[0]==3:
        pr=cProfile.Profile(); pr.enable(); r=orig(*a,**k); pr.disable()
        s=io.StringIO(); pstats.Stats(pr,stream=s).sort_stats('cumulative').print_stats(22); print(s.getvalue()[:4000])
        return r
    return orig(*a,**k)
pkg.assemble_species_meshes=wrapped
m.main()
