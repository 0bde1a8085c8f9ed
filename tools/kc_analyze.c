/* Design-study tool (not product, not oracle): replays the Jacobi rounds with
 * the snapshot rule and tallies, per iteration, work by degree class, the size
 * of each drop (cap - t) weighted by degree, and how many scanned entries hit
 * the top-K vertices by degree.  Drives the kernel design in DESIGN.md. */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>
#define NDB 24   /* log2 degree buckets */
#define NDROP 10 /* drop buckets: 0,1,2-3,4-7,...,128-255,>=256 */
#define NK 6     /* top-K thresholds */
typedef struct {
  uint64_t evals[NDB], entries[NDB];
  uint64_t drop_w[NDB][NDROP];   /* entries weighted by degree, per drop bucket */
  uint64_t topk[NK];             /* scanned entries whose target rank < K */
  uint64_t dropper_entries;      /* entries of vertices that dropped */
} itstat;
static int lg(uint64_t d){int b=0; while(d>1){d>>=1;b++;} return b;}
static int dropb(uint32_t d){ if(d==0) return 0; int b=1+lg(d); return b<NDROP-1?b:NDROP-1; }
static uint32_t hidx(const uint64_t* off,const uint32_t* nbr,const uint32_t* est,uint32_t u,uint32_t cap,uint32_t* sc){
  if(!cap) return 0; uint64_t b=off[u],e=off[u+1]; uint64_t deg=e-b; uint32_t m=deg<cap?(uint32_t)deg:cap; if(!m) return 0;
  memset(sc,0,4*((size_t)m+1)); for(uint64_t i=b;i<e;i++){uint32_t x=est[nbr[i]]; sc[x<m?x:m]++;}
  uint32_t s=0; for(uint32_t t=m;t>0;t--){s+=sc[t]; if(s>=t) return t;} return 0;}
int kc_analyze(uint32_t n,const uint64_t* off,const uint32_t* nbr,const uint32_t* rank,const uint32_t* ks,
               uint32_t H, itstat* out, int maxit){
  uint32_t* est=malloc(4ull*n); uint32_t* list=malloc(4ull*n); uint32_t* nv=malloc(4ull*n); uint8_t* fl=calloc(n,1);
  uint32_t maxd=0; for(uint32_t u=0;u<n;u++){uint32_t d=off[u+1]-off[u]; est[u]=d<H?d:H; if(d>maxd)maxd=d; list[u]=u;}
  uint64_t na=n; int it=0; int nth=omp_get_max_threads(); uint32_t** sc=malloc(sizeof(void*)*nth);
  for(int t=0;t<nth;t++) sc[t]=malloc(4ull*(maxd+2));
  memset(out,0,sizeof(itstat)*maxit);
  for(;;){
    itstat S; memset(&S,0,sizeof S); int any=0;
    #pragma omp parallel
    { itstat L; memset(&L,0,sizeof L); uint32_t* s=sc[omp_get_thread_num()];
      #pragma omp for schedule(dynamic,64) reduction(|:any)
      for(int64_t i=0;i<(int64_t)na;i++){ uint32_t u=list[i]; uint32_t cap=est[u]; uint64_t d=off[u+1]-off[u];
        uint32_t t=hidx(off,nbr,est,u,cap,s); nv[i]=t; int db=lg(d?d:1); L.evals[db]++; L.entries[db]+=d;
        L.drop_w[db][dropb(cap-t)]+=d;
        for(uint64_t j=off[u];j<off[u+1];j++){uint32_t r=rank[nbr[j]]; for(int k=0;k<NK;k++) if(r<ks[k]) L.topk[k]++;}
        if(t<cap){ any=1; L.dropper_entries+=d; __atomic_store_n(&fl[u],1,0);
          for(uint64_t j=off[u];j<off[u+1];j++){uint32_t v=nbr[j]; uint32_t ev=est[v]; if(t<ev&&cap>=ev) __atomic_store_n(&fl[v],1,0);} } }
      #pragma omp critical
      { for(int a=0;a<NDB;a++){S.evals[a]+=L.evals[a];S.entries[a]+=L.entries[a]; for(int b=0;b<NDROP;b++) S.drop_w[a][b]+=L.drop_w[a][b];}
        for(int k=0;k<NK;k++) S.topk[k]+=L.topk[k]; S.dropper_entries+=L.dropper_entries; } }
    for(int64_t i=0;i<(int64_t)na;i++) est[list[i]]=nv[i];
    if(it<maxit) out[it]=S;
    uint64_t k=0; for(uint32_t u=0;u<n;u++) if(fl[u]){fl[u]=0; list[k++]=u;} na=k; it++;
    if(!any) break;
  }
  return it;
}
