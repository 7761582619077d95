import sys, json
sys.path.insert(0,'/root/repo')
from paper_2308_06152_b200 import helm
from workloads import config_problem
p = config_problem("c4_weak_2049")
for cm, cp in [(1<<20,1),(1000000,1),(1000000,3),(1000000,4),(1000000,5),(1000000,14),(200000,4),(200000,5),(200000,3)]:
    H = helm.helm_setup(p, {"vectors":"high_order","inner_maxit":10,"coarsest_n":512,"col_min_n":cm,"col_pipe":cp})
    print(json.dumps({"col_min_n":cm,"col_pipe":cp,"vc1":round(H.helm_bench_graph("vcycle",1,20),2),"vc0":round(H.helm_bench_graph("vcycle",0,5),2),"vc2":round(H.helm_bench_graph("vcycle",2,20),2)}),flush=True)
    H.close()
